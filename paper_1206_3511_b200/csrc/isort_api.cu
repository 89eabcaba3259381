// isort_api.cu -- extern "C" boundary of libisort.so (declared in include/isort.h);
// the ISRT sequence loader is in sequence_io.cu.
//
// Device entry points launch the sm_100a kernels of radix_onesweep.cuh /
// bucket_sort.cuh on the caller's stream.  Host entry points are the drop-in
// path behind intsort::radix_sort_lsd / bucket_sort (proj/core/src/sort.cpp):
// H2D of the 16-byte records, pack to SoA keys + u32 position payload, device
// sort, gather of whole records by position, D2H.  No CPU fallback exists.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <utility>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "../../include/isort.h"
#include "bucket_sort.cuh"
#include "isort_common.cuh"
#include "isort_internal.h"
#include "radix_onesweep.cuh"
#include "isort_launch.cuh"

namespace isort {

// ------------------------------------------------------------------ errors
thread_local std::string g_last_error;
thread_local uint64_t g_last_bad_index = ~0ull;

int set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}


// ------------------------------------------------------------ observability
// Kernel launches issued by this library (bench.py reports them as
// gpu_launches) and an optional per-phase event trail on the launching stream
// (bench.py turns it into the dominant kernel's live duration).
std::atomic<uint64_t> g_launches{0};

struct ProfSink {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<std::string> names;
    const RadixState* st = nullptr;
};
thread_local ProfSink g_prof;


void prof_mark(cudaStream_t s, const char* name) {
    if (!g_prof.on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    g_prof.ev.push_back(e);
    g_prof.names.emplace_back(name);
}


// ------------------------------------------------------- rank self-test
// The fast one-sweep rank relies on same-address shared atomics of one warp
// instruction being granted in ascending lane order (measured on B200, not a
// documented guarantee).  Verify it once per device before first use; if it
// ever fails, every pass uses the __match_any_sync rank instead (correct, ~5x
// slower) and isort_rank_mode() reports it.
std::mutex g_rank_mu;
int g_rank_ok[64] = {0};  // 0 unknown, 1 verified, -1 failed

// One run of the self-test on a private stream: 1 = lane order held, 0 = violations
// counted, -1 = the test could not run (an API error; nothing is cached then).  The
// thread's capture mode is relaxed for the duration, and every call is
// stream-ordered on the private stream, so a first library call made while the
// caller's stream is being captured into a CUDA graph neither fails nor
// invalidates that capture.
int run_rank_selftest() {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    cudaStream_t ts = nullptr;
    uint32_t* d = nullptr;
    uint32_t bad = ~0u;
    int result = -1;
    if (cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking) == cudaSuccess &&
        cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(uint32_t), ts) == cudaSuccess &&
        cudaMemsetAsync(d, 0, sizeof(uint32_t), ts) == cudaSuccess) {
        k_selftest_atomic_order<<<2 * sm_count(), 1024, 0, ts>>>(d, 0x5eedu);
        if (cudaGetLastError() == cudaSuccess &&
            cudaMemcpyAsync(&bad, d, sizeof(uint32_t), cudaMemcpyDeviceToHost, ts) == cudaSuccess &&
            cudaStreamSynchronize(ts) == cudaSuccess)
            result = bad == 0 ? 1 : 0;
    }
    if (d) cudaFreeAsync(d, ts);
    if (ts) {
        cudaStreamSynchronize(ts);
        cudaStreamDestroy(ts);
    }
    cudaGetLastError();  // a failed attempt leaves no sticky error for the caller's next check
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (result == 0)
        std::fprintf(stderr, "isort: shared-atomic lane-order self-test failed (%u violations); "
                             "using the __match_any_sync rank\n", bad);
    return result;
}

// 1 verified, 0 failed (cached), -1 unknown (the test could not run; retried next call).
int rank_state() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_rank_mu);
    int& c = g_rank_ok[dev & 63];
    if (c != 0) return c > 0 ? 1 : 0;
    if (const char* f = std::getenv("ISORT_FORCE_SAFE_RANK"); f && f[0] == '1') {  // tests of the fallback
        c = -1;
        return 0;
    }
    const int r = run_rank_selftest();
    if (r >= 0) c = r ? 1 : -1;
    return r;
}
bool rank_fast_path_ok() { return rank_state() == 1; }
void prof_state(const RadixState* st) { g_prof.st = st; }

std::atomic<int> g_sm_count[64];

}  // namespace isort

int isort::sm_count() {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = g_sm_count[dev & 63].load(std::memory_order_relaxed);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        g_sm_count[dev & 63].store(v, std::memory_order_relaxed);
    }
    return v;
}

namespace isort {


struct RadixLayout {
    size_t state = 0, lookback = 0, keys_alt = 0, vals_alt = 0, total = 0;
    uint32_t tiles = 0;
};

template <typename K>
RadixLayout radix_layout(uint64_t n, bool vals) {
    RadixLayout L;
    const int tile = vals ? pass_tile<K, true>(n) : pass_tile<K, false>(n);
    L.tiles = static_cast<uint32_t>((n + tile - 1) / tile);
    // Look-back rows for the worst tile count of any span m <= n (the bucket
    // sort's oversized fallback sorts a sub-span with the small-n tile).
    const uint64_t small = n < kSmallN ? n : kSmallN - 1;
    const int stile = vals ? pass_tile<K, true>(small) : pass_tile<K, false>(small);
    const uint64_t stiles = (small + stile - 1) / stile;
    const uint64_t lb_tiles = stiles > L.tiles ? stiles : L.tiles;
    size_t off = 0;
    L.state = off;
    off += align_up(sizeof(RadixState));
    off += align_up(sizeof(CountState));  // count_state(): zeroed with the state
    L.lookback = off;
    off += align_up(static_cast<size_t>(KeyTraits<K>::kDigits) * lb_tiles * kRadix * lb_word_bytes(n));
    L.keys_alt = off;
    off += align_up(n * sizeof(K));
    L.vals_alt = off;
    if (vals) off += align_up(n * sizeof(uint32_t));
    L.total = off;
    return L;
}

// Opt a kernel into >48 KB of dynamic shared memory, once per (kernel, device).
// Keyed by the kernel's address: distinct instantiations can share one type.
std::mutex g_smem_mu;
std::set<std::pair<const void*, int>> g_smem_done;

void set_max_smem_once_raw(const void* kernel, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(kernel, dev);
    std::lock_guard<std::mutex> g(g_smem_mu);
    if (g_smem_done.count(key)) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    g_smem_done.insert(key);
}

// CTAs of `kernel` resident per SM (occupancy API), once per (kernel, device).
std::map<std::pair<const void*, int>, int> g_occ;

int resident_per_sm_raw(const void* kernel, int block, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(kernel, dev);
    std::lock_guard<std::mutex> g(g_smem_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    if (per_sm < 1) per_sm = 1;
    g_occ[key] = per_sm;
    return per_sm;
}


template <typename K>
int radix_sort_device(const K* kin, K* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, int vmode,
                      void* temp, size_t temp_bytes, cudaStream_t s) {
    if (vmode < ISORT_VALS_NONE || vmode > ISORT_VALS_IOTA)
        return set_error(ISORT_EINVAL, "isort_radix_sort: bad vals_mode %d", vmode);
    if (n == 0) return ISORT_OK;
    if (n > kMaxLookbackN)
        return set_error(ISORT_ERANGE, "isort_radix_sort: n=%llu exceeds the per-call limit %llu",
                         (unsigned long long)n, (unsigned long long)kMaxLookbackN);
    const bool vals = vmode != ISORT_VALS_NONE;
    if (!kin || !kout || (vals && !vout) || (vmode == ISORT_VALS_LOAD && !vin))
        return set_error(ISORT_EINVAL, "isort_radix_sort: null buffer");
    const RadixLayout L = radix_layout<K>(n, vals);
    if (!temp || temp_bytes < L.total)
        return set_error(ISORT_EINVAL, "isort_radix_sort: temp buffer too small (%zu < %zu)", temp_bytes, L.total);
    char* t = static_cast<char*>(temp);
    auto* st = reinterpret_cast<RadixState*>(t + L.state);
    auto* lb = (t + L.lookback);
    auto* kalt = reinterpret_cast<K*>(t + L.keys_alt);
    auto* valt = vals ? reinterpret_cast<uint32_t*>(t + L.vals_alt) : nullptr;
    RadixDigitizer<K> dz;
    if (vals)
        return launch_radix_pipeline<K, true>(kin, kout, kalt, vin, vout, valt, vmode == ISORT_VALS_IOTA, n, st, lb,
                                              L.tiles, dz, true, true, s);
    // the counting pass needs two extra launches (K6); below kSmallN keys, where a sort is a
    // few launch latencies, the digit passes cost about the same
    return launch_radix_pipeline<K, false>(kin, kout, kalt, nullptr, nullptr, nullptr, false, n, st, lb, L.tiles, dz,
                                           kPlanSkipSorted | (n >= kSmallN ? kPlanCounting : 0), true, s);
}

// ------------------------------------------------------- host-side helpers
struct DeviceCtx {
    cudaStream_t stream = nullptr;
};

std::mutex g_ctx_mu;
DeviceCtx g_ctx[64];

int use_device(int device, cudaStream_t* out) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return set_error(ISORT_ECUDA, "no CUDA device available (%s); the engine has no CPU fallback",
                         cudaGetErrorString(e));
    if (device < 0 || device >= count || device >= 64)
        return set_error(ISORT_EINVAL, "device %d out of range (have %d)", device, count);
    ISORT_CUDA_TRY(cudaSetDevice(device));
    std::lock_guard<std::mutex> g(g_ctx_mu);
    if (!g_ctx[device].stream) ISORT_CUDA_TRY(cudaStreamCreateWithFlags(&g_ctx[device].stream, cudaStreamNonBlocking));
    *out = g_ctx[device].stream;
    return ISORT_OK;
}

// The library's stream-ordered memory pool, one per device.  Its release
// threshold keeps up to ISORT_POOL_KEEP_BYTES (default 4 GiB) of freed
// workspace mapped between calls: with the default pool (threshold 0) every
// synchronising call hands the pages back and the next one maps them again,
// which cost 5-45 ms per call for a 50 MB oversized-span fallback.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};

int lib_pool(cudaMemPool_t* out) {
    int dev = 0;
    ISORT_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return set_error(ISORT_EINVAL, "device %d out of range", dev);
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        ISORT_CUDA_TRY(cudaMemPoolCreate(&pool, &props));
        uint64_t keep = 4ull << 30;
        if (const char* e = std::getenv("ISORT_POOL_KEEP_BYTES")) keep = std::strtoull(e, nullptr, 10);
        ISORT_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        g_pools[dev] = pool;
    }
    *out = g_pools[dev];
    return ISORT_OK;
}

// RAII device allocation on the library's stream-ordered pool.
struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    int alloc(size_t bytes, cudaStream_t stream) {
        s = stream;
        cudaMemPool_t pool;
        if (int rc = lib_pool(&pool)) return rc;
        if (cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, stream) != cudaSuccess) {
            // out of memory with freed workspace still mapped: hand it back, retry once
            cudaGetLastError();
            p = nullptr;
            cudaStreamSynchronize(stream);
            cudaMemPoolTrimTo(pool, 0);
            ISORT_CUDA_TRY(cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, stream));
        }
        return ISORT_OK;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Packs records [lo, lo + m) into SoA u32 keys (low 32 bits) and folds the max key.
__global__ void k_pack_records_u32(const isort_record* __restrict__ rec, uint32_t* __restrict__ keys, uint64_t m,
                                   unsigned long long* __restrict__ max_key) {
    unsigned long long mx = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
        const uint64_t k = rec[i].key;
        keys[i] = static_cast<uint32_t>(k);
        mx = k > mx ? k : mx;
    }
    mx = warp_max<unsigned long long>(mx);
    if (lane_id() == 0 && mx) atomicMax(max_key, mx);
}

__global__ void k_pack_records_u64(const isort_record* __restrict__ rec, uint64_t* __restrict__ keys, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        keys[i] = rec[i].key;
}

__global__ void k_gather_records(const isort_record* __restrict__ in, const uint32_t* __restrict__ idx,
                                 isort_record* __restrict__ out, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = in[idx[i]];
}

// ------------------------------------------------ staged host <-> device transfers
// The drop-in's records live in pageable host memory (std::vector, record.hpp:27-30).
// A plain cudaMemcpy from pageable memory runs at a fraction of PCIe speed and
// cannot overlap anything.  Instead T worker threads each take every T-th chunk,
// copy it into one of their two pinned staging slots (library-owned, reused
// across calls) and issue its DMA on their own stream, so host copies, PCIe
// transfers in both directions and per-chunk device work (the key pack) overlap.
constexpr size_t kStageChunk = 16u << 20;  // bytes per chunk (a multiple of 16 B records)

// Host copy for the staging path with non-temporal (streaming) stores: the
// destination lines are not read first (no read-for-ownership) and do not
// displace the cache, which matters when every core copies at once and the
// host's memory bandwidth is the limit (the DMA uses it too).
inline void stream_copy(void* dst, const void* src, size_t bytes) {
#if defined(__SSE2__)
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15u)) & 15u;
    if (bytes < head + 64) {
        std::memcpy(d, s, bytes);
        return;
    }
    std::memcpy(d, s, head);
    d += head, s += head, bytes -= head;
    const size_t body = bytes & ~static_cast<size_t>(63);
    for (size_t i = 0; i < body; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
    }
    _mm_sfence();
    std::memcpy(d + body, s + body, bytes - body);
#else
    std::memcpy(dst, src, bytes);
#endif
}
constexpr int kStageSlots = 2;             // per worker

struct Staging {
    std::mutex mu;  // one transfer per device at a time
    int workers = 0;
    std::vector<cudaStream_t> streams;
    std::vector<void*> slots;           // workers * kStageSlots pinned buffers
    std::vector<cudaEvent_t> slot_done;  // the slot's last DMA finished
    std::vector<cudaEvent_t> done;       // per worker: all its work queued so far
};
Staging g_staging[64];

int staging_for(int dev, Staging** out) {
    Staging& st = g_staging[dev & 63];
    if (st.workers == 0) {
        int w = static_cast<int>(std::thread::hardware_concurrency());
        w = w >= 32 ? 32 : (w >= 2 ? w : 1);  // every core (measured: 16 threads 120 ms vs 8 threads 135-365 ms for 1e8 records)
        if (const char* e = std::getenv("ISORT_STAGING_THREADS")) w = std::max(1, std::atoi(e));
        for (int i = 0; i < w; ++i) {
            cudaStream_t sw;
            cudaEvent_t ev;
            ISORT_CUDA_TRY(cudaStreamCreateWithFlags(&sw, cudaStreamNonBlocking));
            ISORT_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            st.streams.push_back(sw);
            st.done.push_back(ev);
            for (int k = 0; k < kStageSlots; ++k) {
                void* p = nullptr;
                ISORT_CUDA_TRY(cudaHostAlloc(&p, kStageChunk, cudaHostAllocPortable));
                cudaEvent_t se;
                ISORT_CUDA_TRY(cudaEventCreateWithFlags(&se, cudaEventDisableTiming));
                st.slots.push_back(p);
                st.slot_done.push_back(se);
            }
        }
        st.workers = w;
    }
    *out = &st;
    return ISORT_OK;
}

// Runs fn(worker) on every worker thread (worker 0 on the calling thread); the
// first non-zero return code wins.
template <typename Fn>
int run_workers(int workers, Fn&& fn) {
    std::vector<int> rcs(workers, ISORT_OK);
    std::vector<std::thread> th;
    for (int w = 1; w < workers; ++w) th.emplace_back([&, w] { rcs[w] = fn(w); });
    rcs[0] = fn(0);
    for (auto& t : th) t.join();
    for (int rc : rcs)
        if (rc) return rc;
    return ISORT_OK;
}

// Pageable host -> device.  after(w_stream, offset, len) queues per-chunk device
// work behind the chunk's DMA.  The main stream `s` is made to wait for all of it.
template <typename After>
int upload_staged(void* dst, const void* src, size_t bytes, cudaStream_t s, Staging& st, After&& after) {
    const size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
    cudaEvent_t start;
    ISORT_CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    cudaEventRecord(start, s);  // dst was allocated stream-ordered on s
    const int dev = [] { int d = 0; cudaGetDevice(&d); return d; }();
    int rc = run_workers(st.workers, [&](int w) -> int {
        cudaSetDevice(dev);
        cudaStream_t ws = st.streams[w];
        ISORT_CUDA_TRY(cudaStreamWaitEvent(ws, start, 0));
        int k = 0;
        for (size_t c = static_cast<size_t>(w); c < chunks; c += static_cast<size_t>(st.workers), k ^= 1) {
            const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
            const int slot = w * kStageSlots + k;
            ISORT_CUDA_TRY(cudaEventSynchronize(st.slot_done[slot]));  // its previous DMA has read it
            stream_copy(st.slots[slot], static_cast<const char*>(src) + off, len);
            ISORT_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + off, st.slots[slot], len,
                                           cudaMemcpyHostToDevice, ws));
            ISORT_CUDA_TRY(cudaEventRecord(st.slot_done[slot], ws));
            if (int r = after(ws, off, len)) return r;
        }
        ISORT_CUDA_TRY(cudaEventRecord(st.done[w], ws));
        return ISORT_OK;
    });
    cudaEventDestroy(start);
    if (rc) return rc;
    for (int w = 0; w < st.workers; ++w) ISORT_CUDA_TRY(cudaStreamWaitEvent(s, st.done[w], 0));
    return ISORT_OK;
}

// Device -> pageable host, after everything queued on `s` so far.  Synchronous.
int download_staged(void* dst, const void* src, size_t bytes, cudaStream_t s, Staging& st) {
    const size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
    cudaEvent_t ready;
    ISORT_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    ISORT_CUDA_TRY(cudaEventRecord(ready, s));
    const int dev = [] { int d = 0; cudaGetDevice(&d); return d; }();
    int rc = run_workers(st.workers, [&](int w) -> int {
        cudaSetDevice(dev);
        cudaStream_t ws = st.streams[w];
        ISORT_CUDA_TRY(cudaStreamWaitEvent(ws, ready, 0));
        // two slots in flight: chunk j's DMA overlaps the host copy-out of chunk j - 1
        size_t prev_off = 0, prev_len = 0;
        int prev_slot = -1, k = 0;
        for (size_t c = static_cast<size_t>(w);; c += static_cast<size_t>(st.workers), k ^= 1) {
            const bool more = c < chunks;
            int slot = -1;
            size_t off = 0, len = 0;
            if (more) {
                off = c * kStageChunk;
                len = std::min(kStageChunk, bytes - off);
                slot = w * kStageSlots + k;
                ISORT_CUDA_TRY(cudaMemcpyAsync(st.slots[slot], static_cast<const char*>(src) + off, len,
                                               cudaMemcpyDeviceToHost, ws));
                ISORT_CUDA_TRY(cudaEventRecord(st.slot_done[slot], ws));
            }
            if (prev_slot >= 0) {
                ISORT_CUDA_TRY(cudaEventSynchronize(st.slot_done[prev_slot]));
                stream_copy(static_cast<char*>(dst) + prev_off, st.slots[prev_slot], prev_len);
            }
            if (!more) break;
            prev_slot = slot;
            prev_off = off;
            prev_len = len;
        }
        return ISORT_OK;
    });
    cudaEventDestroy(ready);
    return rc;
}

// Sort records by key through the device: staged H2D with the key pack per chunk
// -> (key, position) sort -> gather -> staged D2H.  `sort32/sort64(keys_in,
// keys_out, idx_out, n, s)` run the u32 / u64 pipelines.  One host read per call:
// the max key after the upload decides u32 or u64 keys (the sort cannot start
// before the last chunk has arrived anyway).
template <typename Sort32, typename Sort64, typename Temp32, typename Temp64>
int sort_records_via_device(const isort_record* in, isort_record* out, uint64_t n, int device, Sort32&& sort32,
                            Sort64&& sort64, Temp32&& temp32, Temp64&& temp64) {
    cudaStream_t s;
    int rc = use_device(device, &s);
    if (rc) return rc;
    if (n > kMaxLookbackN)
        return set_error(ISORT_ERANGE, "n=%llu exceeds the per-call limit %llu", (unsigned long long)n,
                         (unsigned long long)kMaxLookbackN);
    Staging* stg = nullptr;
    {
        std::lock_guard<std::mutex> g(g_pool_mu);  // creation of the per-device staging
        if ((rc = staging_for(device, &stg))) return rc;
    }
    std::lock_guard<std::mutex> g(stg->mu);
    // Device memory: the records (16n), the positions (4n) and one scratch region that
    // holds keys, sorted keys and the sort's temp, and then -- once only the positions
    // are needed -- the gathered output records (16n).  Peak ~36n bytes for u32 keys
    // (3.6 GB at 10^8), inside the pool's kept memory, so repeated calls map nothing.
    const size_t rec_bytes = n * sizeof(isort_record);
    const size_t k32_bytes = align_up(n * sizeof(uint32_t));
    const size_t scratch32 = std::max(rec_bytes, 2 * k32_bytes + temp32(n));
    DevBuf rec_in, scratch, idx, maxw;
    if ((rc = rec_in.alloc(rec_bytes, s)) || (rc = scratch.alloc(scratch32, s)) ||
        (rc = idx.alloc(n * sizeof(uint32_t), s)) || (rc = maxw.alloc(sizeof(unsigned long long), s)))
        return rc;
    ISORT_CUDA_TRY(cudaMemsetAsync(maxw.p, 0, sizeof(unsigned long long), s));
    auto* rin = rec_in.as<isort_record>();
    auto* k32 = scratch.as<uint32_t>();
    auto* mxp = maxw.as<unsigned long long>();
    // ISORT_HOST_TRACE=1: wall-clock split of the call on stderr (upload, sort, download)
    static const bool trace = [] { const char* e = std::getenv("ISORT_HOST_TRACE"); return e && e[0] == '1'; }();
    const auto now = [] { return std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t0 = trace ? now() : 0.0;
    rc = upload_staged(rin, in, n * sizeof(isort_record), s, *stg, [&](cudaStream_t ws, size_t off, size_t len) {
        const uint64_t lo = off / sizeof(isort_record), m = len / sizeof(isort_record);
        k_pack_records_u32<<<grid_for(m), 256, 0, ws>>>(rin + lo, k32 + lo, m, mxp);
        launched();
        return cudaGetLastError() == cudaSuccess ? ISORT_OK : set_error(ISORT_ECUDA, "k_pack_records_u32 launch");
    });
    if (rc) return rc;
    unsigned long long mx = 0;
    ISORT_CUDA_TRY(cudaMemcpyAsync(&mx, maxw.p, sizeof mx, cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    const double t1 = trace ? now() : 0.0;
    char* sc = scratch.as<char>();
    DevBuf scratch64;  // 40-bit keys (the generator's 2^40 bound): a larger scratch
    if (mx <= 0xffffffffull) {
        rc = sort32(k32, reinterpret_cast<uint32_t*>(sc + k32_bytes), idx.as<uint32_t>(), n, sc + 2 * k32_bytes, s);
    } else {
        const size_t k64_bytes = align_up(n * sizeof(uint64_t));
        if ((rc = scratch64.alloc(std::max(rec_bytes, 2 * k64_bytes + temp64(n)), s))) return rc;
        sc = scratch64.as<char>();
        auto* k64 = reinterpret_cast<uint64_t*>(sc);
        k_pack_records_u64<<<grid_for(n), 256, 0, s>>>(rin, k64, n);
        launched();
        rc = sort64(k64, reinterpret_cast<uint64_t*>(sc + k64_bytes), idx.as<uint32_t>(), n, sc + 2 * k64_bytes, s);
    }
    if (rc) {
        cudaStreamSynchronize(s);
        return rc;
    }
    auto* rec_out = reinterpret_cast<isort_record*>(sc);  // the keys and temp are dead now
    k_gather_records<<<grid_for(n), 256, 0, s>>>(rin, idx.as<uint32_t>(), rec_out, n);
    launched();
    ISORT_CUDA_TRY(cudaGetLastError());
    double t2 = 0.0;
    if (trace) {
        cudaStreamSynchronize(s);
        t2 = now();
    }
    rc = download_staged(out, rec_out, rec_bytes, s, *stg);
    if (trace)
        std::fprintf(stderr, "isort records n=%llu workers=%d: upload+pack %.1f ms, sort+gather %.1f ms, download %.1f ms\n",
                     (unsigned long long)n, stg->workers, t1 - t0, t2 - t1, now() - t2);
    return rc;
}

// (key, position) sort for the records path; `temp` (pairs_temp_bytes) comes from the caller.
template <typename K>
size_t radix_pairs_temp_bytes(uint64_t n) { return radix_layout<K>(n, true).total; }
template <typename K>
int radix_pairs(const K* keys, K* keys_out, uint32_t* idx, uint64_t n, void* temp, cudaStream_t s) {
    return radix_sort_device<K>(keys, keys_out, nullptr, idx, n, ISORT_VALS_IOTA, temp, radix_pairs_temp_bytes<K>(n),
                                s);
}

__global__ void k_max_records(const isort_record* __restrict__ rec, uint64_t n, unsigned long long* __restrict__ out) {
    unsigned long long m = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        m = rec[i].key > m ? rec[i].key : m;
    m = warp_max<unsigned long long>(m);
    if (lane_id() == 0 && m) atomicMax(out, m);
}

// digit_i(key) = floor(key / divisor) mod base  (sort.cpp:87-92)
__global__ void k_digit_keys(const isort_record* __restrict__ rec, uint64_t* __restrict__ d, uint64_t n,
                             uint64_t divisor, uint64_t base) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        d[i] = (rec[i].key / divisor) % base;
}

// Digit (key / divisor) mod base of u32 keys (counting_sort_by_digit, sort.cpp:95-97).
__global__ void k_digit_u32(const uint32_t* __restrict__ keys, uint32_t* __restrict__ d, uint64_t n,
                            uint64_t divisor, uint64_t base) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool pow2 = ((base & (base - 1)) == 0) && ((divisor & (divisor - 1)) == 0);
    const uint32_t dsh = pow2 ? static_cast<uint32_t>(__ffsll(static_cast<long long>(divisor)) - 1) : 0u;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t k = keys[i];
        d[i] = pow2 ? static_cast<uint32_t>(dsh < 64 ? (k >> dsh) & (base - 1) : 0)
                    : static_cast<uint32_t>((k / divisor) % base);  // < 2^32: the quotient is <= k
    }
}

// keys_out[i] = keys_in[idx[i]], and the payload (loaded, or the source position).
__global__ void k_gather_pass_u32(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                  const uint32_t* __restrict__ idx, uint32_t* __restrict__ kout,
                                  uint32_t* __restrict__ vout, uint64_t n, int vals_mode) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t j = idx[i];
        kout[i] = kin[j];
        if (vals_mode == ISORT_VALS_LOAD) vout[i] = vin[j];
        else if (vals_mode == ISORT_VALS_IOTA) vout[i] = j;
    }
}

__global__ void k_bucket_index(const uint64_t* __restrict__ keys, uint64_t* __restrict__ out, uint64_t m,
                               BucketIndexer bi) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride)
        out[i] = keys[i] > bi.bound ? ~0ull : bi.bucket(keys[i]);
}

__global__ void k_is_sorted_u32(const uint32_t* __restrict__ keys, uint64_t n, unsigned int* __restrict__ bad) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned int b = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i + 1 < n; i += stride)
        b |= keys[i] > keys[i + 1];
    if (__any_sync(ISORT_FULL_MASK, b) && lane_id() == 0) atomicOr(bad, 1u);
}



struct BucketLayout {
    RadixLayout r;
    size_t bstate = 0, total = 0;
};

template <typename K>
BucketLayout bucket_layout(uint64_t n, bool vals) {
    BucketLayout L;
    L.r = radix_layout<K>(n, vals);  // state, lookback (>= 3 digit slots), alt buffers
    size_t off = L.r.total;
    L.bstate = off;
    off += align_up(sizeof(BucketState));
    L.total = off;
    return L;
}


// After the pipeline: report a range error like the reference, or re-sort the
// span of non-constant oversized super-buckets with the radix pipeline.
template <typename K>
int bucket_finish_impl(const K* kin, K* kout, uint32_t* vout, uint64_t n, uint64_t bound, bool vals, void* temp,
                       size_t temp_bytes, const isort_bucket_status* hs, cudaStream_t s, uint64_t base = 0) {
    g_last_bad_index = ~0ull;
    if (n == 0) return ISORT_OK;
    if (!hs || !hs->done) return set_error(ISORT_EINVAL, "isort_bucket_finish: status not written by the device");
    const BucketLayout L = bucket_layout<K>(n, vals);
    if (!temp || temp_bytes < L.total)
        return set_error(ISORT_EINVAL, "isort_bucket_sort: temp buffer too small (%zu < %zu)", temp_bytes, L.total);
    char* t = static_cast<char*>(temp);
    auto* st = reinterpret_cast<RadixState*>(t + L.r.state);
    auto* lb = (t + L.r.lookback);
    auto* kalt = reinterpret_cast<K*>(t + L.r.keys_alt);
    auto* valt = vals ? reinterpret_cast<uint32_t*>(t + L.r.vals_alt) : nullptr;
    if (hs->first_bad_not != 0) {
        const uint64_t idx = ~hs->first_bad_not;
        K bad = 0;
        ISORT_CUDA_TRY(cudaMemcpy(&bad, kin + idx, sizeof(K), cudaMemcpyDeviceToHost));
        g_last_bad_index = idx;
        if (static_cast<uint64_t>(bad) < base)
            return set_error(ISORT_EINVAL, "bucket_sort: key %llu below range base %llu",
                             (unsigned long long)bad, (unsigned long long)base);
        return set_error(ISORT_EINVAL, "bucket_index: key %llu exceeds range bound %llu (sequence/spec mismatch)",
                         (unsigned long long)bad, (unsigned long long)bound);
    }
    if (hs->oversized) {
        const uint64_t lo = ~hs->span_lo_not, hi = hs->span_hi, m = hi - lo;
        DevBuf tk, tv;
        int rc;
        if ((rc = tk.alloc(m * sizeof(K), s)) || (vals && (rc = tv.alloc(m * 4, s)))) return rc;
        RadixDigitizer<K> rdz;
        const uint32_t tiles_m = radix_layout<K>(m, vals).tiles;  // grid for the span, not for n
        rc = vals ? launch_radix_pipeline<K, true>(kout + lo, tk.as<K>(), kalt + lo, vout + lo, tv.as<uint32_t>(),
                                                   valt + lo, false, m, st, lb, tiles_m, rdz, true, true, s)
                  : launch_radix_pipeline<K, false>(kout + lo, tk.as<K>(), kalt + lo, nullptr, nullptr, nullptr, false,
                                                    m, st, lb, tiles_m, rdz, true, true, s);
        if (rc) return rc;
        k_copy_range<K><<<grid_for(m), 256, 0, s>>>(tk.as<K>(), kout + lo, vals ? tv.as<uint32_t>() : nullptr,
                                                    vals ? vout + lo : nullptr, m);
        launched();
        prof_mark(s, "fallback");
        ISORT_CUDA_TRY(cudaGetLastError());
    }
    return ISORT_OK;
}

// The status of an asynchronous bucket sort, written to host-pinned memory.
__global__ void k_bucket_status(const RadixState* __restrict__ st, const BucketState* __restrict__ bst,
                                isort_bucket_status* status) {
    if (threadIdx.x == 0) {
        status->first_bad_not = st->first_bad;
        status->span_lo_not = bst->span_lo_not;
        status->span_hi = bst->span_hi;
        status->oversized = bst->oversized;
        __threadfence_system();
        status->done = 1;
    }
}

template <typename K, int MODE>
int bucket_sort_impl(const K* kin, K* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, uint64_t bound,
                     int vmode, void* temp, size_t temp_bytes, cudaStream_t s, isort_bucket_status* async_status,
                     uint64_t base);

template <typename K>
int bucket_sort_device(const K* kin, K* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, uint64_t bound,
                       int vmode, void* temp, size_t temp_bytes, cudaStream_t s,
                       isort_bucket_status* async_status = nullptr, uint64_t base = 0) {
    if (base > bound)
        return set_error(ISORT_EINVAL, "isort_bucket_sort: range base %llu above range bound %llu",
                         (unsigned long long)base, (unsigned long long)bound);
    if constexpr (sizeof(K) == 4) {  // u32 keys: always the power-of-two grid (choose_bucket_mode)
        return bucket_sort_impl<K, kPow2Narrow>(kin, kout, vin, vout, n, bound, vmode, temp, temp_bytes, s,
                                                async_status, base);
    } else {
        switch (choose_bucket_mode(n, bound, static_cast<uint64_t>(~static_cast<K>(0)), base)) {
            case kPow2Narrow:
                return bucket_sort_impl<K, kPow2Narrow>(kin, kout, vin, vout, n, bound, vmode, temp, temp_bytes, s,
                                                        async_status, base);
            case kMagicNarrow:
                return bucket_sort_impl<K, kMagicNarrow>(kin, kout, vin, vout, n, bound, vmode, temp, temp_bytes, s,
                                                         async_status, base);
            default:
                return bucket_sort_impl<K, kWide>(kin, kout, vin, vout, n, bound, vmode, temp, temp_bytes, s,
                                                  async_status, base);
        }
    }
}

template <typename K, int MODE>
int bucket_sort_impl(const K* kin, K* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, uint64_t bound,
                     int vmode, void* temp, size_t temp_bytes, cudaStream_t s, isort_bucket_status* async_status,
                     uint64_t base) {
    static_assert(KeyTraits<K>::kDigits >= kBucketMaxDigits, "look-back sized for the bucket digit slots");
    g_last_bad_index = ~0ull;
    if (vmode < ISORT_VALS_NONE || vmode > ISORT_VALS_IOTA)
        return set_error(ISORT_EINVAL, "isort_bucket_sort: bad vals_mode %d", vmode);
    if (n == 0) return ISORT_OK;  // sort.cpp:139-141
    if (n > kMaxLookbackN)
        return set_error(ISORT_ERANGE, "isort_bucket_sort: n=%llu exceeds the per-call limit %llu",
                         (unsigned long long)n, (unsigned long long)kMaxLookbackN);
    const bool vals = vmode != ISORT_VALS_NONE;
    if (!kin || !kout || (vals && !vout) || (vmode == ISORT_VALS_LOAD && !vin))
        return set_error(ISORT_EINVAL, "isort_bucket_sort: null buffer");
    const BucketLayout L = bucket_layout<K>(n, vals);
    if (!temp || temp_bytes < L.total)
        return set_error(ISORT_EINVAL, "isort_bucket_sort: temp buffer too small (%zu < %zu)", temp_bytes, L.total);
    char* t = static_cast<char*>(temp);
    auto* st = reinterpret_cast<RadixState*>(t + L.r.state);
    auto* lb = (t + L.r.lookback);
    auto* kalt = reinterpret_cast<K*>(t + L.r.keys_alt);
    auto* valt = vals ? reinterpret_cast<uint32_t*>(t + L.r.vals_alt) : nullptr;
    auto* bst = reinterpret_cast<BucketState*>(t + L.bstate);
    const BucketDigitizer<K, MODE> dz = BucketDigitizer<K, MODE>::make(n, bound, base);
    const bool iota = vmode == ISORT_VALS_IOTA;

    // M < kCountBins <= n: every bucket holds one key value, so a keys-only bucket
    // sort is the counting pass (K6) -- bucket b's contents are cnt copies of its value
    const int flags = kPlanSkipSorted | (base == 0 && bound < static_cast<uint64_t>(kCountBins) && n > bound &&
                                                 n >= kSmallN
                                             ? kPlanCounting : 0);
    int rc = vals ? launch_radix_pipeline<K, true>(kin, kout, kalt, vin, vout, valt, iota, n, st, lb, L.r.tiles, dz,
                                                   flags, true, s)
                  : launch_radix_pipeline<K, false>(kin, kout, kalt, nullptr, nullptr, nullptr, false, n, st, lb,
                                                    L.r.tiles, dz, flags, true, s);
    if (rc) return rc;
    ISORT_CUDA_TRY(cudaMemsetAsync(bst, 0, sizeof(BucketState), s));
    const int rank_ok = rank_state();
    if (rank_ok < 0) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs != cudaStreamCaptureStatusNone)
            return set_error(ISORT_ECUDA, "isort_bucket_sort: the lane-order self-test could not run; "
                                          "call isort_init() outside stream capture first");
    }
    if (rank_ok == 1) {
        if (vals)
            launch_segments<K, BucketDigitizer<K, MODE>, true>(kout, vout, n, st, bst, dz, s);
        else
            launch_segments<K, BucketDigitizer<K, MODE>, false>(kout, nullptr, n, st, bst, dz, s);
        prof_mark(s, "segments");
        launched(1);
        ISORT_CUDA_TRY(cudaGetLastError());
    } else {
        // The segment sort ranks with lane-ordered shared atomics; without them, finish
        // with the (match-based, stable) radix pipeline over the bucket-grouped keys --
        // a stable sort of the whole array is the same result.  Runs only when the range
        // check passed (the radix pipeline reuses the state).  Synchronises: not capturable.
        unsigned long long not_bad = 0;
        ISORT_CUDA_TRY(cudaMemcpyAsync(&not_bad, &st->first_bad, sizeof not_bad, cudaMemcpyDeviceToHost, s));
        ISORT_CUDA_TRY(cudaStreamSynchronize(s));
        if (not_bad == 0) {
            DevBuf tk, tv;
            if ((rc = tk.alloc(n * sizeof(K), s)) || (vals && (rc = tv.alloc(n * 4, s)))) return rc;
            RadixDigitizer<K> rdz;
            rc = vals ? launch_radix_pipeline<K, true>(kout, tk.as<K>(), kalt, vout, tv.as<uint32_t>(), valt, false, n,
                                                       st, lb, L.r.tiles, rdz, true, true, s)
                      : launch_radix_pipeline<K, false>(kout, tk.as<K>(), kalt, nullptr, nullptr, nullptr, false, n, st,
                                                        lb, L.r.tiles, rdz, true, true, s);
            if (rc) return rc;
            k_copy_range<K><<<grid_for(n), 256, 0, s>>>(tk.as<K>(), kout, vals ? tv.as<uint32_t>() : nullptr,
                                                        vals ? vout : nullptr, n);
            launched();
            ISORT_CUDA_TRY(cudaGetLastError());
        }  // else: the range error is still recorded in st and reported below
    }

    if (async_status) {  // status to host memory from the device: no host sync, capturable
        if (n == 0) return ISORT_OK;
        k_bucket_status<<<1, 32, 0, s>>>(st, bst, async_status);
        launched();
        ISORT_CUDA_TRY(cudaGetLastError());
        return ISORT_OK;
    }
    // one small read-back: range error and oversized span
    isort_bucket_status hs{};
    BucketState hb{};
    ISORT_CUDA_TRY(cudaMemcpyAsync(&hs.first_bad_not, &st->first_bad, sizeof hs.first_bad_not,
                                   cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaMemcpyAsync(&hb, bst, sizeof hb, cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    hs.span_lo_not = hb.span_lo_not;
    hs.span_hi = hb.span_hi;
    hs.oversized = hb.oversized;
    hs.done = 1;
    return bucket_finish_impl<K>(kin, kout, vout, n, bound, vals, temp, temp_bytes, &hs, s, base);
}

template <typename K>
size_t bucket_pairs_temp_bytes(uint64_t n) { return bucket_layout<K>(n, true).total; }
template <typename K>
int bucket_pairs(const K* keys, K* keys_out, uint32_t* idx, uint64_t n, uint64_t bound, void* temp, cudaStream_t s) {
    return bucket_sort_device<K>(keys, keys_out, nullptr, idx, n, bound, ISORT_VALS_IOTA, temp,
                                 bucket_pairs_temp_bytes<K>(n), s);
}

template <typename K>
int partition_device(const K* kin, K* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, const K* splitters,
                     int parts, int vmode, uint64_t* counts, void* temp, size_t temp_bytes, cudaStream_t s) {
    if (parts < 1 || parts > kMaxParts)
        return set_error(ISORT_EINVAL, "isort_partition: parts=%d outside [1, %d]", parts, kMaxParts);
    if (vmode < ISORT_VALS_NONE || vmode > ISORT_VALS_IOTA)
        return set_error(ISORT_EINVAL, "isort_partition: bad vals_mode %d", vmode);
    if (!counts) return set_error(ISORT_EINVAL, "isort_partition: null counts");
    DestDigitizer<K> dz{};
    dz.nsplit = parts - 1;
    for (int i = 0; i + 1 < parts; ++i) {
        dz.split[i] = splitters[i];
        if (i && splitters[i] < splitters[i - 1]) return set_error(ISORT_EINVAL, "isort_partition: splitters not ascending");
    }
    if (n == 0) {
        ISORT_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * parts, s));
        return ISORT_OK;
    }
    if (n > kMaxLookbackN)
        return set_error(ISORT_ERANGE, "isort_partition: n=%llu exceeds the per-call limit", (unsigned long long)n);
    const bool vals = vmode != ISORT_VALS_NONE;
    if (!kin || !kout || (vals && !vout) || (vmode == ISORT_VALS_LOAD && !vin))
        return set_error(ISORT_EINVAL, "isort_partition: null buffer");
    const RadixLayout L = radix_layout<K>(n, vals);
    if (!temp || temp_bytes < L.total)
        return set_error(ISORT_EINVAL, "isort_partition: temp buffer too small (%zu < %zu)", temp_bytes, L.total);
    char* t = static_cast<char*>(temp);
    auto* st = reinterpret_cast<RadixState*>(t + L.state);
    auto* lb = (t + L.lookback);
    auto* kalt = reinterpret_cast<K*>(t + L.keys_alt);
    auto* valt = vals ? reinterpret_cast<uint32_t*>(t + L.vals_alt) : nullptr;
    int rc = vals ? launch_radix_pipeline<K, true>(kin, kout, kalt, vin, vout, valt, vmode == ISORT_VALS_IOTA, n, st,
                                                   lb, L.tiles, dz, true, true, s)
                  : launch_radix_pipeline<K, false>(kin, kout, kalt, nullptr, nullptr, nullptr, false, n, st, lb,
                                                    L.tiles, dz, true, true, s);
    if (rc) return rc;
    k_copy_part_counts<<<1, kMaxParts, 0, s>>>(st, counts, parts);
    launched();
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

// Fused partition + exchange (multi-GPU step 3 + 5 in one kernel): counts first,
// then one stable pass that stores each destination's run at its own base.
template <typename K>
int make_dest_digitizer(const K* splitters, int parts, DestDigitizer<K>* dz) {
    if (parts < 1 || parts > kMaxParts)
        return set_error(ISORT_EINVAL, "isort_partition: parts=%d outside [1, %d]", parts, kMaxParts);
    *dz = DestDigitizer<K>{};
    dz->nsplit = parts - 1;
    for (int i = 0; i + 1 < parts; ++i) {
        if (!splitters) return set_error(ISORT_EINVAL, "isort_partition: null splitters");
        dz->split[i] = splitters[i];
        if (i && splitters[i] < splitters[i - 1])
            return set_error(ISORT_EINVAL, "isort_partition: splitters not ascending");
    }
    return ISORT_OK;
}

template <typename K>
int partition_counts_device(const K* kin, uint64_t n, const K* splitters, int parts, uint64_t* counts, void* temp,
                            size_t temp_bytes, cudaStream_t s) {
    DestDigitizer<K> dz;
    int rc = make_dest_digitizer(splitters, parts, &dz);
    if (rc) return rc;
    if (!counts) return set_error(ISORT_EINVAL, "isort_partition: null counts");
    if (n == 0) {
        ISORT_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * parts, s));
        return ISORT_OK;
    }
    if (n > kMaxLookbackN)
        return set_error(ISORT_ERANGE, "isort_partition: n=%llu exceeds the per-call limit", (unsigned long long)n);
    if (!kin) return set_error(ISORT_EINVAL, "isort_partition: null buffer");
    const RadixLayout L = radix_layout<K>(n, true);
    if (!temp || temp_bytes < L.total)
        return set_error(ISORT_EINVAL, "isort_partition: temp buffer too small (%zu < %zu)", temp_bytes, L.total);
    char* t = static_cast<char*>(temp);
    auto* st = reinterpret_cast<RadixState*>(t + L.state);
    rc = launch_histogram<K>(kin, n, st, (t + L.lookback), L.tiles, dz, kPlanKeepTrivial,
                             true, s);
    if (rc) return rc;
    k_copy_part_counts<<<1, kMaxParts, 0, s>>>(st, counts, parts);
    launched();
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

template <typename K>
int partition_scatter_device(const K* kin, const uint32_t* vin, uint64_t n, const K* splitters, int parts, int vmode,
                             void* const* key_dst, void* const* val_dst, const unsigned long long* dst_table,
                             void* temp, size_t temp_bytes, cudaStream_t s) {
    DestDigitizer<K> dz;
    int rc = make_dest_digitizer(splitters, parts, &dz);
    if (rc) return rc;
    if (vmode < ISORT_VALS_NONE || vmode > ISORT_VALS_IOTA)
        return set_error(ISORT_EINVAL, "isort_partition: bad vals_mode %d", vmode);
    if (n == 0) return ISORT_OK;
    const bool vals = vmode != ISORT_VALS_NONE;
    if (!kin || (!dst_table && (!key_dst || (vals && !val_dst))) || (vmode == ISORT_VALS_LOAD && !vin))
        return set_error(ISORT_EINVAL, "isort_partition: null buffer");
    const RadixLayout L = radix_layout<K>(n, true);
    if (!temp || temp_bytes < L.total)
        return set_error(ISORT_EINVAL, "isort_partition: temp buffer too small (%zu < %zu)", temp_bytes, L.total);
    ScatterTable tbl{};
    tbl.dev = dst_table;
    tbl.parts = parts;
    for (int p = 0; p < parts && !dst_table; ++p) {
        tbl.key[p] = reinterpret_cast<unsigned long long>(key_dst[p]);
        tbl.val[p] = vals ? reinterpret_cast<unsigned long long>(val_dst[p]) : 0ull;
    }
    char* t = static_cast<char*>(temp);
    auto* st = reinterpret_cast<RadixState*>(t + L.state);
    const ScatterTable& scat = tbl;  // a kernel argument (by value): no copy, no host sync
    // the look-back words and the ticket of the (single) pass slot start from zero
    ISORT_CUDA_TRY(cudaMemsetAsync(t + L.lookback, 0, static_cast<size_t>(L.tiles) * kRadix * lb_word_bytes(n), s));
    ISORT_CUDA_TRY(cudaMemsetAsync(&st->tile_ticket[0], 0, sizeof(st->tile_ticket), s));
    auto* lb = (t + L.lookback);
    const bool iota = vmode == ISORT_VALS_IOTA;
    // the layout is the payload one (it covers both); the tile count must match the
    // pass configuration actually launched (keys-only tiles are twice as long)
    const int stile = vals ? scatter_tile<K, true>(n) : scatter_tile<K, false>(n);
    const uint32_t tiles = static_cast<uint32_t>((n + stile - 1) / stile);
    if (n < kSmallN) {
        if (vals)
            launch_passes<K, true, DestDigitizer<K>, PassCfg<K, true, 1>, true>(kin, nullptr, nullptr, vin, nullptr,
                                                                              nullptr, iota, n, st, lb, tiles, dz, s,
                                                                              scat);
        else
            launch_passes<K, false, DestDigitizer<K>, PassCfg<K, false, 1>, true>(
                kin, nullptr, nullptr, nullptr, nullptr, nullptr, false, n, st, lb, tiles, dz, s, scat);
    } else {
        if (vals)
            launch_passes<K, true, DestDigitizer<K>, PassCfg<K, true, ISORT_PASS_CHUNKS>, true>(kin, nullptr, nullptr, vin, nullptr,
                                                                              nullptr, iota, n, st, lb, tiles, dz, s,
                                                                              scat);
        else
            launch_passes<K, false, DestDigitizer<K>, PassCfg<K, false, ISORT_PASS_CHUNKS>, true>(
                kin, nullptr, nullptr, nullptr, nullptr, nullptr, false, n, st, lb, tiles, dz, s, scat);
    }
    launched(1);
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

}  // namespace isort

using namespace isort;

extern "C" {

const char* isort_last_error(void) { return g_last_error.c_str(); }

uint64_t isort_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int isort_rank_mode(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return -1;
    return rank_fast_path_ok() ? 1 : 0;
}

int isort_pool_trim(int device) {
    cudaStream_t s;
    int rc = use_device(device, &s);
    if (rc) return rc;
    cudaMemPool_t pool;
    if ((rc = lib_pool(&pool))) return rc;
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    ISORT_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
    return ISORT_OK;
}

int isort_init(int device) {
    cudaStream_t s;
    int rc = use_device(device, &s);
    if (rc) return rc;
    if (rank_state() < 0) return set_error(ISORT_ECUDA, "isort_init: the lane-order self-test could not run");
    return ISORT_OK;
}

int isort_profile_begin(void) {
    for (cudaEvent_t e : g_prof.ev) cudaEventDestroy(e);
    g_prof.ev.clear();
    g_prof.names.clear();
    g_prof.st = nullptr;
    g_prof.on = true;
    return ISORT_OK;
}

int isort_profile_end(float* ms, char* names, int names_stride, int max_phases, int* count, int* n_active) {
    g_prof.on = false;
    const int m = static_cast<int>(g_prof.ev.size());
    int rc = ISORT_OK;
    if (m > 0) {
        cudaError_t e = cudaEventSynchronize(g_prof.ev.back());
        if (e != cudaSuccess) rc = set_error(ISORT_ECUDA, "isort_profile_end: %s", cudaGetErrorString(e));
    }
    int k = 0;
    for (int i = 1; i < m && k < max_phases && rc == ISORT_OK; ++i, ++k) {
        float t = 0.f;
        cudaEventElapsedTime(&t, g_prof.ev[i - 1], g_prof.ev[i]);
        if (ms) ms[k] = t;
        if (names && names_stride > 0) {
            std::snprintf(names + static_cast<size_t>(k) * names_stride, names_stride, "%s", g_prof.names[i].c_str());
        }
    }
    if (count) *count = k;
    if (n_active) {
        uint32_t na = 0;
        if (g_prof.st && rc == ISORT_OK) cudaMemcpy(&na, &g_prof.st->n_active, 4, cudaMemcpyDeviceToHost);
        *n_active = static_cast<int>(na);
    }
    for (cudaEvent_t e : g_prof.ev) cudaEventDestroy(e);
    g_prof.ev.clear();
    g_prof.names.clear();
    return rc;
}
int isort_abi_version(void) { return ISORT_ABI_VERSION; }
uint64_t isort_max_keys(void) { return kMaxLookbackN; }
uint64_t isort_last_bad_index(void) { return g_last_bad_index; }

size_t isort_radix_temp_bytes(uint64_t n, int key_bytes, int vals_mode) {
    const bool vals = vals_mode != ISORT_VALS_NONE;
    return key_bytes == 8 ? radix_layout<uint64_t>(n, vals).total : radix_layout<uint32_t>(n, vals).total;
}

int isort_radix_sort_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                         uint64_t n, int vals_mode, void* temp, size_t temp_bytes, void* stream) {
    return radix_sort_device<uint32_t>(keys_in, keys_out, vals_in, vals_out, n, vals_mode, temp, temp_bytes,
                                       static_cast<cudaStream_t>(stream));
}

int isort_radix_sort_u64(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                         uint64_t n, int vals_mode, void* temp, size_t temp_bytes, void* stream) {
    return radix_sort_device<uint64_t>(keys_in, keys_out, vals_in, vals_out, n, vals_mode, temp, temp_bytes,
                                       static_cast<cudaStream_t>(stream));
}

size_t isort_bucket_temp_bytes(uint64_t n, int key_bytes, int vals_mode) {
    const bool vals = vals_mode != ISORT_VALS_NONE;
    return key_bytes == 8 ? bucket_layout<uint64_t>(n, vals).total : bucket_layout<uint32_t>(n, vals).total;
}

int isort_bucket_sort_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                          uint64_t n, uint64_t range_bound, int vals_mode, void* temp, size_t temp_bytes,
                          void* stream) {
    return bucket_sort_device<uint32_t>(keys_in, keys_out, vals_in, vals_out, n, range_bound, vals_mode, temp,
                                        temp_bytes, static_cast<cudaStream_t>(stream));
}

int isort_bucket_sort_u64(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                          uint64_t n, uint64_t range_bound, int vals_mode, void* temp, size_t temp_bytes,
                          void* stream) {
    return bucket_sort_device<uint64_t>(keys_in, keys_out, vals_in, vals_out, n, range_bound, vals_mode, temp,
                                        temp_bytes, static_cast<cudaStream_t>(stream));
}

int isort_bucket_sort_span_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                               uint32_t* vals_out, uint64_t n, uint64_t range_lo, uint64_t range_hi, int vals_mode,
                               void* temp, size_t temp_bytes, void* stream) {
    return bucket_sort_device<uint32_t>(keys_in, keys_out, vals_in, vals_out, n, range_hi, vals_mode, temp,
                                        temp_bytes, static_cast<cudaStream_t>(stream), nullptr, range_lo);
}

int isort_bucket_sort_u32_async(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                                uint32_t* vals_out, uint64_t n, uint64_t range_bound, int vals_mode, void* temp,
                                size_t temp_bytes, isort_bucket_status* status, void* stream) {
    if (!status) return set_error(ISORT_EINVAL, "isort_bucket_sort_async: null status");
    status->done = 0;
    return bucket_sort_device<uint32_t>(keys_in, keys_out, vals_in, vals_out, n, range_bound, vals_mode, temp,
                                        temp_bytes, static_cast<cudaStream_t>(stream), status);
}

int isort_bucket_finish_u32(const uint32_t* keys_in, uint32_t* keys_out, uint32_t* vals_out, uint64_t n,
                            uint64_t range_bound, int vals_mode, void* temp, size_t temp_bytes,
                            const isort_bucket_status* status, void* stream) {
    return bucket_finish_impl<uint32_t>(keys_in, keys_out, vals_out, n, range_bound, vals_mode != ISORT_VALS_NONE,
                                        temp, temp_bytes, status, static_cast<cudaStream_t>(stream));
}

size_t isort_partition_temp_bytes(uint64_t n, int key_bytes, int vals_mode) {
    return isort_radix_temp_bytes(n, key_bytes, vals_mode);
}

int isort_partition_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                        uint64_t n, const uint32_t* splitters, int parts, int vals_mode, uint64_t* counts, void* temp,
                        size_t temp_bytes, void* stream) {
    return partition_device<uint32_t>(keys_in, keys_out, vals_in, vals_out, n, splitters, parts, vals_mode, counts,
                                      temp, temp_bytes, static_cast<cudaStream_t>(stream));
}

int isort_radix_sort_records(const isort_record* in, isort_record* out, uint64_t n, uint64_t base, int device) {
    g_last_bad_index = ~0ull;
    if (base < 2) return set_error(ISORT_EINVAL, "build_radix_plan: base must be >= 2");
    if (n == 0) return ISORT_OK;
    if (!in || !out) return set_error(ISORT_EINVAL, "isort_radix_sort_records: null buffer");
    return sort_records_via_device(
        in, out, n, device,
        [](const uint32_t* k, uint32_t* ko, uint32_t* idx, uint64_t m, void* t, cudaStream_t s) {
            return radix_pairs<uint32_t>(k, ko, idx, m, t, s);
        },
        [](const uint64_t* k, uint64_t* ko, uint32_t* idx, uint64_t m, void* t, cudaStream_t s) {
            return radix_pairs<uint64_t>(k, ko, idx, m, t, s);
        },
        radix_pairs_temp_bytes<uint32_t>, radix_pairs_temp_bytes<uint64_t>);
}

int isort_bucket_sort_records(const isort_record* in, isort_record* out, uint64_t n, uint64_t range_bound,
                              int device) {
    g_last_bad_index = ~0ull;
    if (n == 0) return ISORT_OK;  // sort.cpp:139-141: empty input, no range check
    if (!in || !out) return set_error(ISORT_EINVAL, "isort_bucket_sort_records: null buffer");
    return sort_records_via_device(
        in, out, n, device,
        [range_bound](const uint32_t* k, uint32_t* ko, uint32_t* idx, uint64_t m, void* t, cudaStream_t s) {
            return bucket_pairs<uint32_t>(k, ko, idx, m, range_bound, t, s);
        },
        [range_bound](const uint64_t* k, uint64_t* ko, uint32_t* idx, uint64_t m, void* t, cudaStream_t s) {
            return bucket_pairs<uint64_t>(k, ko, idx, m, range_bound, t, s);
        },
        bucket_pairs_temp_bytes<uint32_t>, bucket_pairs_temp_bytes<uint64_t>);
}

int isort_counting_sort_by_digit_records(const isort_record* in, isort_record* out, uint64_t n, uint64_t base,
                                         uint32_t digits, uint32_t digit_index, int device) {
    if (base < 2) return set_error(ISORT_EINVAL, "counting_sort_by_digit: base must be >= 2");
    if (digit_index >= digits)
        return set_error(ISORT_EINVAL, "counting_sort_by_digit: digit_index %u out of range for a %u-digit plan",
                         digit_index, digits);
    if (n == 0) return ISORT_OK;
    if (!in || !out) return set_error(ISORT_EINVAL, "isort_counting_sort_by_digit_records: null buffer");
    uint64_t divisor = 1;  // pow_u64 (sort.cpp:28-34), same wrap-around arithmetic
    for (uint32_t i = 0; i < digit_index; ++i) divisor *= base;
    if (divisor == 0)
        return set_error(ISORT_EINVAL, "counting_sort_by_digit: base^%u overflows 64 bits", digit_index);
    cudaStream_t s;
    int rc = use_device(device, &s);
    if (rc) return rc;
    if (n > kMaxLookbackN) return set_error(ISORT_ERANGE, "n exceeds the per-call limit");
    // The pass is a stable sort by the digit value: compute digits on the device,
    // then sort (digit, position) pairs and gather the records.
    DevBuf rec_in, rec_out, dig, dig_out, idx, temp;
    const size_t tb = radix_layout<uint64_t>(n, true).total;
    if ((rc = rec_in.alloc(n * sizeof(isort_record), s)) || (rc = rec_out.alloc(n * sizeof(isort_record), s)) ||
        (rc = dig.alloc(n * 8, s)) || (rc = dig_out.alloc(n * 8, s)) || (rc = idx.alloc(n * 4, s)) ||
        (rc = temp.alloc(tb, s)))
        return rc;
    ISORT_CUDA_TRY(cudaMemcpyAsync(rec_in.p, in, n * sizeof(isort_record), cudaMemcpyHostToDevice, s));
    k_digit_keys<<<grid_for(n), 256, 0, s>>>(rec_in.as<isort_record>(), dig.as<uint64_t>(), n, divisor, base);
    rc = radix_sort_device<uint64_t>(dig.as<uint64_t>(), dig_out.as<uint64_t>(), nullptr, idx.as<uint32_t>(), n,
                                     ISORT_VALS_IOTA, temp.p, tb, s);
    if (rc) return rc;
    k_gather_records<<<grid_for(n), 256, 0, s>>>(rec_in.as<isort_record>(), idx.as<uint32_t>(),
                                                rec_out.as<isort_record>(), n);
    ISORT_CUDA_TRY(cudaGetLastError());
    ISORT_CUDA_TRY(cudaMemcpyAsync(out, rec_out.p, n * sizeof(isort_record), cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    return ISORT_OK;
}

int isort_build_radix_plan_records(const isort_record* in, uint64_t n, uint64_t base, uint32_t* digits, int device) {
    if (base < 2) return set_error(ISORT_EINVAL, "build_radix_plan: base must be >= 2");
    if (!digits) return set_error(ISORT_EINVAL, "isort_build_radix_plan_records: null output");
    unsigned long long mx = 0;
    if (n > 0) {
        if (!in) return set_error(ISORT_EINVAL, "isort_build_radix_plan_records: null buffer");
        cudaStream_t s;
        int rc = use_device(device, &s);
        if (rc) return rc;
        DevBuf rec, m;
        if ((rc = rec.alloc(n * sizeof(isort_record), s)) || (rc = m.alloc(8, s))) return rc;
        ISORT_CUDA_TRY(cudaMemcpyAsync(rec.p, in, n * sizeof(isort_record), cudaMemcpyHostToDevice, s));
        ISORT_CUDA_TRY(cudaMemsetAsync(m.p, 0, 8, s));
        k_max_records<<<grid_for(n), 256, 0, s>>>(rec.as<isort_record>(), n, m.as<unsigned long long>());
        ISORT_CUDA_TRY(cudaMemcpyAsync(&mx, m.p, 8, cudaMemcpyDeviceToHost, s));
        ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    }
    // minimal digits with base^digits > max (sort.cpp:67-74)
    uint32_t d = 0;
    uint64_t v = mx;
    do {
        v /= base;
        ++d;
    } while (v != 0);
    *digits = d;
    return ISORT_OK;
}

static int host_keys_u32(const uint32_t* in, uint32_t* out, uint64_t n, int device, bool bucket, uint64_t range_bound) {
    g_last_bad_index = ~0ull;
    if (n == 0) return ISORT_OK;
    if (!in || !out) return set_error(ISORT_EINVAL, "null host buffer");
    cudaStream_t s;
    int rc = use_device(device, &s);
    if (rc) return rc;
    const size_t tb = bucket ? bucket_layout<uint32_t>(n, false).total : radix_layout<uint32_t>(n, false).total;
    DevBuf din, dout, temp;
    if ((rc = din.alloc(n * 4, s)) || (rc = dout.alloc(n * 4, s)) || (rc = temp.alloc(tb, s))) return rc;
    ISORT_CUDA_TRY(cudaMemcpyAsync(din.p, in, n * 4, cudaMemcpyHostToDevice, s));
    rc = bucket ? bucket_sort_device<uint32_t>(din.as<uint32_t>(), dout.as<uint32_t>(), nullptr, nullptr, n,
                                               range_bound, ISORT_VALS_NONE, temp.p, tb, s)
                : radix_sort_device<uint32_t>(din.as<uint32_t>(), dout.as<uint32_t>(), nullptr, nullptr, n,
                                              ISORT_VALS_NONE, temp.p, tb, s);
    if (rc) {
        cudaStreamSynchronize(s);
        return rc;
    }
    ISORT_CUDA_TRY(cudaMemcpyAsync(out, dout.p, n * 4, cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    return ISORT_OK;
}

int isort_radix_sort_host_u32(const uint32_t* in, uint32_t* out, uint64_t n, int device) {
    return host_keys_u32(in, out, n, device, false, 0);
}

int isort_bucket_sort_host_u32(const uint32_t* in, uint32_t* out, uint64_t n, uint64_t range_bound, int device) {
    return host_keys_u32(in, out, n, device, true, range_bound);
}

int isort_bucket_index_u64(const uint64_t* keys, uint64_t* out, uint64_t m, uint64_t bucket_count,
                           uint64_t range_bound, void* stream) {
    if (bucket_count == 0) return set_error(ISORT_EINVAL, "bucket_index: bucket_count must be >= 1");
    if (m == 0) return ISORT_OK;
    if (!keys || !out) return set_error(ISORT_EINVAL, "isort_bucket_index_u64: null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_bucket_index<<<grid_for(m), 256, 0, s>>>(keys, out, m, BucketIndexer::make(bucket_count, range_bound));
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

int isort_is_sorted_u32(const uint32_t* keys, uint64_t n, int* result, void* stream) {
    if (!result) return set_error(ISORT_EINVAL, "isort_is_sorted_u32: null result");
    if (n < 2) {
        *result = 1;
        return ISORT_OK;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevBuf flag;
    int rc = flag.alloc(4, s);
    if (rc) return rc;
    ISORT_CUDA_TRY(cudaMemsetAsync(flag.p, 0, 4, s));
    k_is_sorted_u32<<<grid_for(n), 256, 0, s>>>(keys, n, flag.as<unsigned int>());
    unsigned int bad = 0;
    ISORT_CUDA_TRY(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    *result = bad ? 0 : 1;
    return ISORT_OK;
}

size_t isort_counting_pass_temp_bytes(uint64_t n) {
    return 3 * align_up(n * 4) + radix_layout<uint32_t>(n, true).total;
}

int isort_counting_pass_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                            uint64_t n, uint64_t base, uint32_t digits, uint32_t digit_index, int vals_mode,
                            void* temp, size_t temp_bytes, void* stream) {
    g_last_bad_index = ~0ull;
    if (base < 2) return set_error(ISORT_EINVAL, "counting_sort_by_digit: base must be >= 2");
    if (digit_index >= digits)
        return set_error(ISORT_EINVAL, "counting_sort_by_digit: digit_index %u out of range for a %u-digit plan",
                         digit_index, digits);
    if (vals_mode < ISORT_VALS_NONE || vals_mode > ISORT_VALS_IOTA)
        return set_error(ISORT_EINVAL, "isort_counting_pass: bad vals_mode %d", vals_mode);
    if (n == 0) return ISORT_OK;
    if (n > kMaxLookbackN) return set_error(ISORT_ERANGE, "isort_counting_pass: n exceeds the per-call limit");
    const bool vals = vals_mode != ISORT_VALS_NONE;
    if (!keys_in || !keys_out || (vals && !vals_out) || (vals_mode == ISORT_VALS_LOAD && !vals_in))
        return set_error(ISORT_EINVAL, "isort_counting_pass: null buffer");
    const size_t need = isort_counting_pass_temp_bytes(n);
    if (!temp || temp_bytes < need)
        return set_error(ISORT_EINVAL, "isort_counting_pass: temp buffer too small (%zu < %zu)", temp_bytes, need);
    uint64_t divisor = 1;  // pow_u64 (sort.cpp:28-34): the same wrap-around product
    for (uint32_t i = 0; i < digit_index; ++i) divisor *= base;
    if (divisor == 0)
        return set_error(ISORT_EINVAL, "counting_sort_by_digit: base^%u overflows 64 bits", digit_index);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* t = static_cast<char*>(temp);
    auto* dig = reinterpret_cast<uint32_t*>(t);
    auto* dig_sorted = reinterpret_cast<uint32_t*>(t + align_up(n * 4));
    auto* idx = reinterpret_cast<uint32_t*>(t + 2 * align_up(n * 4));
    void* rtemp = t + 3 * align_up(n * 4);
    // A counting pass is the stable sort by the digit: (digit, position) pairs
    // through the radix pipeline (digits < 256 take one one-sweep pass), then a gather.
    k_digit_u32<<<grid_for(n), 256, 0, s>>>(keys_in, dig, n, divisor, base);
    launched();
    int rc = radix_sort_device<uint32_t>(dig, dig_sorted, nullptr, idx, n, ISORT_VALS_IOTA, rtemp,
                                         radix_layout<uint32_t>(n, true).total, s);
    if (rc) return rc;
    k_gather_pass_u32<<<grid_for(n), 256, 0, s>>>(keys_in, vals_in, idx, keys_out, vals_out, n, vals_mode);
    launched();
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

int isort_partition_counts_u32(const uint32_t* keys_in, uint64_t n, const uint32_t* splitters, int parts,
                               uint64_t* counts, void* temp, size_t temp_bytes, void* stream) {
    return partition_counts_device<uint32_t>(keys_in, n, splitters, parts, counts, temp, temp_bytes,
                                             static_cast<cudaStream_t>(stream));
}

int isort_partition_scatter_u32(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n,
                                const uint32_t* splitters, int parts, int vals_mode, void* const* key_dst,
                                void* const* val_dst, void* temp, size_t temp_bytes, void* stream) {
    return partition_scatter_device<uint32_t>(keys_in, vals_in, n, splitters, parts, vals_mode, key_dst, val_dst,
                                              nullptr, temp, temp_bytes, static_cast<cudaStream_t>(stream));
}

int isort_partition_scatter_table_u32(const uint32_t* keys_in, const uint32_t* vals_in, uint64_t n,
                                      const uint32_t* splitters, int parts, int vals_mode,
                                      const uint64_t* dst_table, void* temp, size_t temp_bytes, void* stream) {
    if (!dst_table) return set_error(ISORT_EINVAL, "isort_partition: null destination table");
    return partition_scatter_device<uint32_t>(keys_in, vals_in, n, splitters, parts, vals_mode, nullptr, nullptr,
                                              reinterpret_cast<const unsigned long long*>(dst_table), temp,
                                              temp_bytes, static_cast<cudaStream_t>(stream));
}

int isort_ipc_alloc(size_t bytes, int device, void** ptr, unsigned char* handle) {
    if (!ptr || !handle) return set_error(ISORT_EINVAL, "isort_ipc_alloc: null argument");
    ISORT_CUDA_TRY(cudaSetDevice(device));
    ISORT_CUDA_TRY(cudaMalloc(ptr, bytes ? bytes : 16));
    cudaIpcMemHandle_t h;
    ISORT_CUDA_TRY(cudaIpcGetMemHandle(&h, *ptr));
    static_assert(sizeof(h) == 64, "64-byte IPC handle");
    memcpy(handle, &h, sizeof h);
    return ISORT_OK;
}

int isort_ipc_open(const unsigned char* handle, int device, void** ptr) {
    if (!ptr || !handle) return set_error(ISORT_EINVAL, "isort_ipc_open: null argument");
    ISORT_CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    ISORT_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return ISORT_OK;
}

int isort_ipc_close(void* ptr) {
    ISORT_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return ISORT_OK;
}

int isort_ipc_free(void* ptr) {
    ISORT_CUDA_TRY(cudaFree(ptr));
    return ISORT_OK;
}

}  // extern "C"


