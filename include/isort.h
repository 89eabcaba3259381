/*
 * isort.h -- C ABI of the B200-native integer-sort engine (libisort.so).
 *
 * Drop-in boundary for the reference's sort path (arxiv 1206.3511,
 * /root/reference/proj).  The reference's public entry points live in
 * proj/core/include/intsort/sort.hpp and are bound to the harness through
 * SortFn / make_sort_fn (proj/core/include/intsort/bench.hpp:44-49).  Each
 * group below names the reference interface it replaces.  A C++ adapter with
 * the unchanged signatures (paper_1206_3511_b200/dropin/sort_b200.cpp) sits on
 * top; INTEGRATION.md shows how a maintainer swaps it in for sort.cpp.
 *
 * Conventions
 *  - All functions return ISORT_OK (0) or an ISORT_E* code; the message is in
 *    isort_last_error() (thread-local).  Argument errors that the reference
 *    reports with std::invalid_argument return ISORT_EINVAL with the
 *    reference's wording.
 *  - "Device" entry points take device pointers, a caller-provided temp
 *    buffer (size from the matching *_temp_bytes) and a cudaStream_t passed
 *    as void*.  They are asynchronous: no host synchronisation, except where
 *    noted (bucket sort reads back one small status word).
 *  - "Host" entry points take host pointers, own their device memory and
 *    synchronise before returning (the reference is synchronous).
 *  - There is no CPU fallback: without a usable CUDA device every call
 *    returns ISORT_ECUDA.
 */
#ifndef ISORT_H
#define ISORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISORT_OK 0
#define ISORT_ENOMEM 12
#define ISORT_EINVAL 22  /* reference: std::invalid_argument */
#define ISORT_ERANGE 34  /* n beyond the engine's per-call limit (2^32 - 1 keys, isort_max_keys()) */
#define ISORT_EIO 5      /* reference: intsort::SequenceIoError (sequence files) */
#define ISORT_ECUDA 1001
#define ISORT_ENCCL 1002

#define ISORT_ABI_VERSION 1

/* Layout-compatible with intsort::Record {Key key; uint64_t tag;}
 * (proj/core/include/intsort/record.hpp:20-25). */
typedef struct isort_record {
    uint64_t key;
    uint64_t tag;
} isort_record;

/* Payload handling for the device sorts. */
enum isort_vals_mode {
    ISORT_VALS_NONE = 0, /* keys only */
    ISORT_VALS_LOAD = 1, /* vals_in[] carried along (u32 payload) */
    ISORT_VALS_IOTA = 2  /* payload = original position, generated on device */
};

const char* isort_last_error(void);
int isort_abi_version(void);
/* Largest n one device call accepts. */
uint64_t isort_max_keys(void);
/* Bad input index of the last ISORT_EINVAL range failure (UINT64_MAX if none). */
uint64_t isort_last_bad_index(void);

/* Observability (used by bench.py).  isort_launch_count: kernels this library
 * has launched so far in the process.  isort_profile_begin/end: record a CUDA
 * event on the launching stream after every phase (memset, upfront, plan,
 * pass0..7, copy, windows, resolve, fallback) of the calls made in between on
 * this thread; end() synchronises, writes per-phase milliseconds and
 * NUL-terminated phase names (names_stride bytes each), the number of phases,
 * and the number of digit passes the last pipeline actually executed. */
uint64_t isort_launch_count(void);
/* Rank primitive of the one-sweep passes on the current device: 1 = shared
 * atomics (lane order verified by the load-time self-test), 0 = the
 * __match_any_sync fallback (self-test failed), -1 = no device. */
int isort_rank_mode(void);
/* Select `device`, create the library's state on it and run the lane-order
 * self-test the fast rank relies on.  Optional: the first sort does it lazily
 * (on a private stream, with the thread's capture mode relaxed, so even a first
 * call inside a CUDA-graph capture is safe); an explicit call keeps that
 * one-time cost out of timed or captured regions. */
int isort_init(int device);
/* Host entry points take their device workspace from a library-owned,
 * stream-ordered pool that keeps up to ISORT_POOL_KEEP_BYTES (env, default
 * 4 GiB) of freed memory mapped between calls, so repeated calls do not remap
 * pages.  isort_pool_trim releases all of it on `device` (the library also trims
 * and retries once when an allocation fails). */
int isort_pool_trim(int device);
int isort_profile_begin(void);
int isort_profile_end(float* ms, char* names, int names_stride, int max_phases, int* count,
                      int* n_active);

/* ------------------------------------------------------------------------
 * LSD radix sort, device-resident.
 * Replaces: intsort::radix_sort_lsd(const RecordSeq&, uint64_t base)
 *           (sort.hpp:37-40, sort.cpp:112-119) and the build_radix_plan /
 *           counting_sort_by_digit chain it runs (sort.cpp:57-110).
 * Stable; output identical for every base >= 2 (test_sort.cpp:136-149), so
 * the device sorts with 8-bit digits and skips digit passes that are the
 * identity.  keys_in is not modified; keys_out receives the sorted keys.
 * ---------------------------------------------------------------------- */
size_t isort_radix_temp_bytes(uint64_t n, int key_bytes, int vals_mode);
int isort_radix_sort_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                         uint32_t* vals_out, uint64_t n, int vals_mode, void* temp,
                         size_t temp_bytes, void* stream);
int isort_radix_sort_u64(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in,
                         uint32_t* vals_out, uint64_t n, int vals_mode, void* temp,
                         size_t temp_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Bucket sort, device-resident.
 * Replaces: intsort::bucket_sort(const RecordSeq&, Key range_bound)
 *           (sort.hpp:50-53, sort.cpp:136-152) with bucket_index
 *           (sort.cpp:121-134): n buckets, b = floor(n*key/(M+1)).
 * A key > range_bound returns ISORT_EINVAL with the reference's message for
 * the first offending input position (isort_last_bad_index()).  This call
 * synchronises `stream` once to read that status.
 * ---------------------------------------------------------------------- */
size_t isort_bucket_temp_bytes(uint64_t n, int key_bytes, int vals_mode);
int isort_bucket_sort_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                          uint32_t* vals_out, uint64_t n, uint64_t range_bound, int vals_mode,
                          void* temp, size_t temp_bytes, void* stream);
int isort_bucket_sort_u64(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in,
                          uint32_t* vals_out, uint64_t n, uint64_t range_bound, int vals_mode,
                          void* temp, size_t temp_bytes, void* stream);

/* Bucket sort over the key span [range_lo, range_hi]: n buckets,
 * b = floor(n * (key - range_lo) / (range_hi - range_lo + 1)).  Not a reference
 * entry point (its ranges start at 0, where this equals isort_bucket_sort_u32);
 * the multi-GPU sort's local step, where each rank holds one key range.  Keys
 * outside the span fail with ISORT_EINVAL like a key above range_bound. */
int isort_bucket_sort_span_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                               uint32_t* vals_out, uint64_t n, uint64_t range_lo, uint64_t range_hi,
                               int vals_mode, void* temp, size_t temp_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Key-range partition (multi-GPU sort).  Not in the
 * reference (single-threaded); the engine's scale-out step.
 * Stable partition of keys_in into `parts` destination ranges: destination of
 * a key = number of `splitters` (host array, parts - 1 ascending values) that
 * are <= key.  keys_out holds destination 0's keys, then 1's, ... each in input
 * order; counts (device, `parts` u64) receives the per-destination counts.
 * ---------------------------------------------------------------------- */
size_t isort_partition_temp_bytes(uint64_t n, int key_bytes, int vals_mode);
int isort_partition_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                        uint32_t* vals_out, uint64_t n, const uint32_t* splitters, int parts,
                        int vals_mode, uint64_t* counts, void* temp, size_t temp_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Host-memory entry points: the drop-in path (H2D, sort, D2H inside).
 * ---------------------------------------------------------------------- */
/* radix_sort_lsd(input, base): sort.hpp:40. */
int isort_radix_sort_records(const isort_record* in, isort_record* out, uint64_t n,
                             uint64_t base, int device);
/* bucket_sort(input, range_bound): sort.hpp:53. */
int isort_bucket_sort_records(const isort_record* in, isort_record* out, uint64_t n,
                              uint64_t range_bound, int device);
/* counting_sort_by_digit(input, RadixPlan{base, digits}, digit_index): sort.hpp:30-35. */
int isort_counting_sort_by_digit_records(const isort_record* in, isort_record* out, uint64_t n,
                                         uint64_t base, uint32_t digits, uint32_t digit_index,
                                         int device);
/* build_radix_plan(input, base).digits: sort.hpp:28. */
int isort_build_radix_plan_records(const isort_record* in, uint64_t n, uint64_t base,
                                   uint32_t* digits, int device);
/* Keys-only u32 through host buffers (the end-to-end benchmark call). */
int isort_radix_sort_host_u32(const uint32_t* in, uint32_t* out, uint64_t n, int device);
int isort_bucket_sort_host_u32(const uint32_t* in, uint32_t* out, uint64_t n,
                               uint64_t range_bound, int device);

/* Asynchronous bucket sort: the same pipeline with no host synchronisation (so
 * it can be captured in a CUDA graph).  The device writes the call's status to
 * `status`, which must be host-pinned (cudaHostAlloc); after the stream passes
 * that point, isort_bucket_finish_* reports a range error exactly as the
 * synchronous call does, or re-sorts a span of oversized super-buckets (rare).
 * `done` is set to 1 by the device when the other fields are final. */
typedef struct isort_bucket_status {
    uint64_t first_bad_not; /* ~index of the first key > range_bound; 0 if none */
    uint64_t span_lo_not;   /* ~start of the oversized span (radix fallback) */
    uint64_t span_hi;
    uint32_t oversized;     /* non-constant oversized super-buckets */
    uint32_t done;
} isort_bucket_status;
int isort_bucket_sort_u32_async(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                                uint32_t* vals_out, uint64_t n, uint64_t range_bound, int vals_mode, void* temp,
                                size_t temp_bytes, isort_bucket_status* status, void* stream);
int isort_bucket_finish_u32(const uint32_t* keys_in, uint32_t* keys_out, uint32_t* vals_out, uint64_t n,
                            uint64_t range_bound, int vals_mode, void* temp, size_t temp_bytes,
                            const isort_bucket_status* status, void* stream);

/* Device batch of bucket_index (sort.hpp:42-48, sort.cpp:121-134): out[i] =
 * floor(bucket_count * keys[i] / (range_bound + 1)) with the exact 128-bit
 * semantics, or UINT64_MAX where keys[i] > range_bound.  ISORT_EINVAL when
 * bucket_count == 0.  Device pointers; asynchronous on `stream`. */
int isort_bucket_index_u64(const uint64_t* keys, uint64_t* out, uint64_t m, uint64_t bucket_count,
                           uint64_t range_bound, void* stream);

/* One stable counting pass on device u32 keys by the general-base digit
 * (key / base^digit_index) mod base.
 * Replaces: intsort::counting_sort_by_digit(input, RadixPlan{base, digits},
 *           digit_index) (sort.hpp:30-35, sort.cpp:77-110), with its errors:
 *           base < 2, digit_index >= digits (ISORT_EINVAL, the reference's text).
 * vals_mode as for the sorts (ISORT_VALS_IOTA: the source position of each key).
 * Asynchronous on `stream`; temp from isort_counting_pass_temp_bytes(n). */
size_t isort_counting_pass_temp_bytes(uint64_t n);
int isort_counting_pass_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                            uint32_t* vals_out, uint64_t n, uint64_t base, uint32_t digits,
                            uint32_t digit_index, int vals_mode, void* temp, size_t temp_bytes,
                            void* stream);

/* Device-side is_sorted (verify.hpp:12-13) over u32 keys: *result = 1/0. */
int isort_is_sorted_u32(const uint32_t* keys, uint64_t n, int* result, void* stream);

/* ---- fused partition + exchange (multi-GPU, SURVEY 8e "fused variant") -------
 * Step 1: per-destination counts of the key-range partition of keys_in (the
 * destination-digit histogram); leaves its state in temp for step 2.
 * counts: device u64[parts]; splitters: host, parts-1 ascending.  temp:
 * isort_partition_temp_bytes(n, 4, ISORT_VALS_LOAD). */
int isort_partition_counts_u32(const uint32_t* keys_in, uint64_t n, const uint32_t* splitters, int parts,
                               uint64_t* counts, void* temp, size_t temp_bytes, void* stream);
/* Step 2: the stable partition pass, storing destination p's keys (payload)
 * contiguously from key_dst[p] (val_dst[p]) instead of a local send buffer --
 * typically a slot in rank p's receive buffer opened with isort_ipc_open, so the
 * partition writes straight over NVLink.  Same keys, splitters and temp as step
 * 1; key_dst / val_dst are host arrays of `parts` device pointers.  The kernel
 * ends with a system-scope fence; order the consumer after it (e.g. an NCCL
 * all-reduce on the same stream). */
int isort_partition_scatter_u32(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n,
                                const uint32_t* splitters, int parts, int vals_mode, void* const* key_dst,
                                void* const* val_dst, void* temp, size_t temp_bytes, void* stream);
/* Step 2 with a DEVICE-resident destination table (no host read of the count
 * matrix before the launch): dst_table[d] = device address where this rank's run
 * for destination d starts, dst_table[parts + d] = the same for the payload
 * (ignored for ISORT_VALS_NONE).  The multi-GPU sort computes the table on the
 * device from the all-gathered count matrix (paper_1206_3511_b200/partition.py). */
int isort_partition_scatter_table_u32(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n,
                                      const uint32_t* splitters, int parts, int vals_mode,
                                      const uint64_t* dst_table, void* temp, size_t temp_bytes, void* stream);
/* CUDA IPC for receive buffers: allocate + export a 64-byte handle, open a
 * peer's handle (peer access enabled lazily), close, free. */
int isort_ipc_alloc(size_t bytes, int device, void** ptr, unsigned char* handle);
int isort_ipc_open(const unsigned char* handle, int device, void** ptr);
int isort_ipc_close(void* ptr);
int isort_ipc_free(void* ptr);

/* ---- ISRT sequence files ----------------------------------
 * Format (sequence_io.hpp:12-16): "ISRT", version 0x01, u64 LE case_id, n,
 * range_bound, seed, then n u64 LE keys.  Errors are ISORT_EIO with the
 * messages intsort::read_sequence throws (sequence_io.cpp:72-119). */
typedef struct isort_sequence_header {
    uint64_t case_id;
    uint64_t n;
    uint64_t range_bound;
    uint64_t seed;
} isort_sequence_header;

/* Parse and validate the header (magic, version, truncation).  Host only. */
int isort_sequence_read_header(const char* path, isort_sequence_header* out);

/* Stream the keys of `path` into device memory `d_keys` (capacity keys of
 * key_bytes = 4 or 8): chunks are read into pinned staging buffers, copied
 * asynchronously and checked on the device (key > range_bound), replacing the
 * reference's read-and-check loop (sequence_io.cpp:93-119).  The first bad key
 * and truncation are reported exactly as the reference's 65,536-key chunked
 * reader reports them.  key_bytes = 4 also requires every key < 2^32 (ISORT_ERANGE
 * otherwise).  Synchronous; `*out` receives the header. */
int isort_sequence_load(const char* path, void* d_keys, uint64_t capacity, int key_bytes,
                        isort_sequence_header* out, int device);

#ifdef __cplusplus
}
#endif

#endif /* ISORT_H */
