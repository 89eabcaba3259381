// sequence_io.cu -- ISRT sequence files straight into device memory
// (isort_sequence_read_header / isort_sequence_load in
// include/isort.h).  Format and messages: proj/core/include/intsort/
// sequence_io.hpp:12-16, proj/core/src/sequence_io.cpp:72-128.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/isort.h"
#include "isort_internal.h"

namespace isort {

// ------------------------------------------------------- ISRT sequence files
// sequence_io.hpp:12-16 / sequence_io.cpp:72-119.  The reference reads 65,536
// keys at a time and checks each chunk before reading the next, so a key > M in
// a complete chunk is reported before a truncation found later.
constexpr uint64_t kSeqHeaderBytes = 5 + 4 * 8;
constexpr uint64_t kSeqRefChunk = 1ull << 16;        // sequence_io.cpp:14
constexpr uint64_t kSeqStageKeys = 4ull << 20;       // keys per pinned staging buffer

template <typename... A>
int seq_error(const char* fmt, A... a) {
    return set_error(ISORT_EIO, fmt, a...);
}

inline uint64_t le64(const unsigned char* b) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    return v;
}

struct SeqFile {
    FILE* f = nullptr;
    ~SeqFile() {
        if (f) fclose(f);
    }
};

int seq_open(const char* path, SeqFile& sf, isort_sequence_header* h) {
    if (!path || !h) return set_error(ISORT_EINVAL, "isort_sequence: null argument");
    sf.f = fopen(path, "rb");
    if (!sf.f) return seq_error("cannot open %s for reading", path);
    unsigned char pre[5];
    if (fread(pre, 1, 5, sf.f) != 5) return seq_error("sequence file truncated in preamble");
    static const unsigned char kMagic[4] = {0x49, 0x53, 0x52, 0x54};
    if (memcmp(pre, kMagic, 4) != 0) return seq_error("bad magic: not a sequence file");
    if (pre[4] != 0x01) return seq_error("unsupported sequence file version %d", static_cast<int>(pre[4]));
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) {
        unsigned char b[8];
        if (fread(b, 1, 8, sf.f) != 8) return seq_error("sequence file truncated in header");
        v[i] = le64(b);
    }
    h->case_id = v[0];
    h->n = v[1];
    h->range_bound = v[2];
    h->seed = v[3];
    return ISORT_OK;
}

// Device check + narrowing of one staged chunk: keys > M and (u32 output) keys
// >= 2^32 record their position (first = max of complements).
template <typename K>
__global__ void k_seq_keys(const uint64_t* __restrict__ src, K* __restrict__ dst, uint64_t count, uint64_t pos0,
                           uint64_t bound, unsigned long long* __restrict__ first_bad,
                           unsigned long long* __restrict__ first_wide) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t v = src[i];
        if (v > bound) atomicMax(first_bad, ~(pos0 + i));
        if (sizeof(K) == 4 && (v >> 32) != 0) atomicMax(first_wide, ~(pos0 + i));
        dst[i] = static_cast<K>(v);
    }
}

struct SeqStaging {  // per device, kept for the process: pinned host + device chunks
    void* host[2] = {nullptr, nullptr};
    uint64_t* dev[2] = {nullptr, nullptr};
    unsigned long long* flags = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr};
};
std::mutex g_seq_mu;
SeqStaging g_seq[64];

int seq_staging(int device, SeqStaging** out) {
    SeqStaging& sg = g_seq[device];
    if (!sg.flags) {
        for (int b = 0; b < 2; ++b) {
            ISORT_CUDA_TRY(cudaHostAlloc(&sg.host[b], kSeqStageKeys * 8, cudaHostAllocDefault));
            ISORT_CUDA_TRY(cudaMalloc(&sg.dev[b], kSeqStageKeys * 8));
            ISORT_CUDA_TRY(cudaEventCreateWithFlags(&sg.copied[b], cudaEventDisableTiming));
        }
        ISORT_CUDA_TRY(cudaMalloc(&sg.flags, 2 * sizeof(unsigned long long)));
    }
    *out = &sg;
    return ISORT_OK;
}

// Read `bytes` at `offset` with several threads (page-cache reads are bound by
// one core's copy rate, well below PCIe).
bool pread_parallel(int fd, void* dst, uint64_t bytes, uint64_t offset) {
    const unsigned hw = std::thread::hardware_concurrency();
    const uint64_t parts = bytes < (8ull << 20) ? 1 : (hw >= 8 ? 8 : (hw ? hw : 1));
    std::atomic<bool> ok{true};
    auto work = [&](uint64_t i) {
        const uint64_t lo = bytes * i / parts, hi = bytes * (i + 1) / parts;
        char* p = static_cast<char*>(dst) + lo;
        uint64_t done = 0;
        while (done < hi - lo) {
            const ssize_t r = pread(fd, p + done, hi - lo - done, static_cast<off_t>(offset + lo + done));
            if (r <= 0) {
                ok = false;
                return;
            }
            done += static_cast<uint64_t>(r);
        }
    };
    std::vector<std::thread> th;
    for (uint64_t i = 1; i < parts; ++i) th.emplace_back(work, i);
    work(0);
    for (auto& t : th) t.join();
    return ok;
}

template <typename K>
int seq_load(SeqFile& sf, const char* path, const isort_sequence_header& h, K* d_keys, int device) {
    // keys the reference checks before it meets a short chunk
    if (fseeko(sf.f, 0, SEEK_END) != 0) return seq_error("cannot seek %s", path);
    const uint64_t size = static_cast<uint64_t>(ftello(sf.f));
    const uint64_t avail = size >= kSeqHeaderBytes ? (size - kSeqHeaderBytes) / 8 : 0;
    const bool truncated = avail < h.n;
    const uint64_t checked = truncated ? (avail / kSeqRefChunk) * kSeqRefChunk : h.n;
    if (fseeko(sf.f, static_cast<off_t>(kSeqHeaderBytes), SEEK_SET) != 0) return seq_error("cannot seek %s", path);

    cudaStream_t s;
    int rc = use_device(device, &s);
    if (rc) return rc;
    std::lock_guard<std::mutex> g(g_seq_mu);
    SeqStaging* sg = nullptr;
    if ((rc = seq_staging(device, &sg))) return rc;
    ISORT_CUDA_TRY(cudaMemsetAsync(sg->flags, 0, 2 * sizeof(unsigned long long), s));
    for (uint64_t off = 0, c = 0; off < checked; off += kSeqStageKeys, ++c) {
        const int b = static_cast<int>(c & 1);
        const uint64_t cnt = checked - off < kSeqStageKeys ? checked - off : kSeqStageKeys;
        if (c >= 2) ISORT_CUDA_TRY(cudaEventSynchronize(sg->copied[b]));  // staging buffer b is free again
        if (!pread_parallel(fileno(sf.f), sg->host[b], cnt * 8, kSeqHeaderBytes + off * 8))
            return seq_error("sequence file truncated in payload");
        ISORT_CUDA_TRY(cudaMemcpyAsync(sg->dev[b], sg->host[b], cnt * 8, cudaMemcpyHostToDevice, s));
        ISORT_CUDA_TRY(cudaEventRecord(sg->copied[b], s));
        k_seq_keys<K><<<grid_for(cnt), 256, 0, s>>>(sg->dev[b], d_keys + off, cnt, off, h.range_bound, sg->flags,
                                                    sg->flags + 1);
        launched();
        ISORT_CUDA_TRY(cudaGetLastError());
    }
    unsigned long long fl[2] = {0, 0};
    ISORT_CUDA_TRY(cudaMemcpyAsync(fl, sg->flags, sizeof fl, cudaMemcpyDeviceToHost, s));
    ISORT_CUDA_TRY(cudaStreamSynchronize(s));
    if (fl[0] != 0) {  // first key > M, named with its value as the reference does
        const uint64_t pos = ~fl[0];
        unsigned char kb[8];
        if (fseeko(sf.f, static_cast<off_t>(kSeqHeaderBytes + 8 * pos), SEEK_SET) != 0 || fread(kb, 1, 8, sf.f) != 8)
            return seq_error("cannot re-read %s", path);
        g_last_bad_index = pos;
        return seq_error("key %llu at position %llu exceeds declared range bound %llu", (unsigned long long)le64(kb),
                         (unsigned long long)pos, (unsigned long long)h.range_bound);
    }
    if (truncated) return seq_error("sequence file truncated in payload");
    if (fl[1] != 0) {
        g_last_bad_index = ~fl[1];
        return set_error(ISORT_ERANGE, "key at position %llu does not fit 32 bits: load with key_bytes = 8",
                         (unsigned long long)~fl[1]);
    }
    return ISORT_OK;
}

}  // namespace isort

using namespace isort;

extern "C" {

int isort_sequence_read_header(const char* path, isort_sequence_header* out) {
    SeqFile sf;
    isort_sequence_header h{};
    const int rc = seq_open(path, sf, &h);
    if (rc) return rc;
    *out = h;
    return ISORT_OK;
}

int isort_sequence_load(const char* path, void* d_keys, uint64_t capacity, int key_bytes, isort_sequence_header* out,
                        int device) {
    g_last_bad_index = ~0ull;
    if (key_bytes != 4 && key_bytes != 8) return set_error(ISORT_EINVAL, "isort_sequence_load: key_bytes must be 4 or 8");
    SeqFile sf;
    isort_sequence_header h{};
    int rc = seq_open(path, sf, &h);
    if (rc) return rc;
    if (out) *out = h;
    if (h.n > capacity)
        return set_error(ISORT_EINVAL, "isort_sequence_load: %llu keys exceed the buffer capacity %llu",
                         (unsigned long long)h.n, (unsigned long long)capacity);
    if (h.n > 0 && !d_keys) return set_error(ISORT_EINVAL, "isort_sequence_load: null buffer");
    return key_bytes == 4 ? seq_load<uint32_t>(sf, path, h, static_cast<uint32_t*>(d_keys), device)
                          : seq_load<uint64_t>(sf, path, h, static_cast<uint64_t*>(d_keys), device);
}

}  // extern "C"
