// isort_common.cuh -- shared device helpers for the B200 integer-sort engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#define ISORT_FULL_MASK 0xffffffffu

namespace isort {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;  // bins per digit pass
constexpr int kMaxDigits = 8;            // u64 keys: 8 x 8-bit digits

// Number of SMs of the current device (cudaDevAttrMultiProcessorCount, cached per
// device; 148 on B200).  Persistent grids are sized in multiples of it.
int sm_count();

template <typename K>
struct KeyTraits;
template <>
struct KeyTraits<uint32_t> {
    static constexpr int kDigits = 4;
};
template <>
struct KeyTraits<uint64_t> {
    static constexpr int kDigits = 8;
};

// ---------------------------------------------------------------- memory ops
// Decoupled look-back status words live in L2; relaxed gpu-scope atomics are
// sufficient because the flag and the count share one 32-bit word.
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Streaming read-only load (input keys are read exactly once per pass).
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ldg_stream(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldg_stream_v4(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, uint32_t shift) {
    return static_cast<uint32_t>(key >> shift) & (kRadix - 1);
}

// Inclusive warp scan (Kogge-Stone over shuffles).
__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(ISORT_FULL_MASK, v, o);
        if (lane_id() >= static_cast<uint32_t>(o)) v += t;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T t = __shfl_xor_sync(ISORT_FULL_MASK, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// Block-wide max of a 64-bit value (BLOCK threads, all participating); the
// result is valid in every thread.  Two barriers.
template <int BLOCK>
__device__ __forceinline__ long long block_reduce_max_ll(long long v) {
    __shared__ long long s_red[BLOCK / 32];
    v = warp_max<long long>(v);
    __syncthreads();
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    long long r = s_red[0];
#pragma unroll
    for (int w = 1; w < BLOCK / 32; ++w) r = r > s_red[w] ? r : s_red[w];
    return r;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(ISORT_FULL_MASK, v, o);
    return v;
}

// ---- bulk (TMA) shared -> global stores
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Bulk shared -> global copy (TMA store), tracked by the issuing thread's bulk group.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until this thread's bulk stores have read their shared-memory source (.read)
// or have fully completed.
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Orders this thread's generic-proxy shared accesses before later async-proxy ones.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace isort
