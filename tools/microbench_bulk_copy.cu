// Microbenchmark: rate of small cp.async.bulk shared->global copies issued by many threads per CTA
// (the bulk write-out experiment).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(s))), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

template <int COPIERS>
__global__ void __launch_bounds__(512, 2) k(uint32_t* out, uint64_t n_words, int iters, int bytes) {
    extern __shared__ __align__(128) uint32_t sm[];
    for (int i = threadIdx.x; i < 12288; i += 512) sm[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int words = bytes / 4;
    uint64_t base = (uint64_t)blockIdx.x * 12288ull * iters;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x < COPIERS) {
            const int t = threadIdx.x;
            const uint64_t goff = (base + (uint64_t)it * 12288 + (uint64_t)t * words) % (n_words - words);
            bulk_s2g(out + (goff & ~3ull), sm + ((t * words) % (12288 - words) & ~3), bytes);
            bulk_commit();
            bulk_wait_read0();
        }
        __syncthreads();
    }
}
int main() {
    const uint64_t n_words = 100000000ull;
    uint32_t* out; cudaMalloc(&out, n_words * 4);
    cudaFuncSetAttribute(k<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * 4);
    cudaFuncSetAttribute(k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int grid = 296, iters = 200;
    for (int bytes : {64, 192, 384, 1024}) {
        for (int c = 0; c < 2; ++c) {
            auto kern = c ? k<32> : k<256>;
            int copiers = c ? 32 : 256;
            kern<<<grid, 512, 12288 * 4>>>(out, n_words, iters, bytes);
            cudaEventRecord(a);
            kern<<<grid, 512, 12288 * 4>>>(out, n_words, iters, bytes);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double copies = (double)grid * iters * copiers;
            printf("bytes=%4d copiers=%3d: %.3f ms, %.2f Gcopies/s chip, %.1f cycles/copy/SM @1.965GHz, %.0f GB/s\n", bytes,
                   copiers, ms, copies / ms / 1e6, 148 * 1.965e6 * ms / copies, copies * bytes / ms / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
