// isort_internal.h -- what the translation units of libisort.so share (not part
// of the ABI): error recording, the launch counter, device contexts, helpers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>

#include "../../include/isort.h"
#include "isort_common.cuh"

namespace isort {

// Records the message for isort_last_error() and returns `code`.
int set_error(int code, const char* fmt, ...);
extern thread_local uint64_t g_last_bad_index;  // isort_last_bad_index()
extern std::atomic<uint64_t> g_launches;        // isort_launch_count()

// Selects `device` and returns the library's stream on it (host entry points).
int use_device(int device, cudaStream_t* out);

inline void launched(int k = 1) { g_launches.fetch_add(static_cast<uint64_t>(k), std::memory_order_relaxed); }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Grid for a grid-stride kernel over n items: enough CTAs, at most per_sm per SM.
inline unsigned grid_for(uint64_t n, int block = 256, int per_sm = 8) {
    const uint64_t want = (n + block - 1) / block;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * sm_count();
    return static_cast<unsigned>(want < cap ? (want ? want : 1) : cap);
}

}  // namespace isort

#define ISORT_CUDA_TRY(expr)                                                                     \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return ::isort::set_error(ISORT_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                      __FILE__, __LINE__);                                       \
    } while (0)
