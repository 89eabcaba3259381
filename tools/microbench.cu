// microbench.cu -- throughput of the warp primitives a stable radix rank can be
// built from, measured on the B200 (results go to profiles/microbench_*.txt).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_match(uint32_t* out, uint32_t seed) {
    uint32_t v0 = (threadIdx.x * 2654435761u + seed) & 255, v1 = v0 ^ 17, v2 = v0 ^ 33, v3 = v0 ^ 71;
    uint32_t acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        acc += __match_any_sync(0xffffffff, v0) + __match_any_sync(0xffffffff, v1) +
               __match_any_sync(0xffffffff, v2) + __match_any_sync(0xffffffff, v3);
        v0 = (v0 + acc) & 255; v1 = (v1 + 3) & 255; v2 = (v2 + 5) & 255; v3 = (v3 + 7) & 255;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// 8-bit peer mask from ballots (CUB MatchAny style)
__device__ __forceinline__ uint32_t match8_ballot(uint32_t d) {
    uint32_t peers = 0xffffffff;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const uint32_t m = __ballot_sync(0xffffffff, (d >> b) & 1);
        peers &= ((d >> b) & 1) ? m : ~m;
    }
    return peers;
}

__global__ void k_ballot8(uint32_t* out, uint32_t seed) {
    uint32_t v0 = (threadIdx.x * 2654435761u + seed) & 255, v1 = v0 ^ 17;
    uint32_t acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        acc += match8_ballot(v0) + match8_ballot(v1);
        v0 = (v0 + acc) & 255; v1 = (v1 + 3) & 255;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_atoms_ret(uint32_t* out, uint32_t seed) {
    __shared__ uint32_t h[16][257];
    for (int i = threadIdx.x; i < 16 * 257; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t* wh = h[threadIdx.x >> 5];
    uint32_t v = (threadIdx.x * 2654435761u + seed), acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        v = v * 1664525u + 1013904223u;
        acc += atomicAdd(&wh[(v >> 24)], 1u);
        acc += atomicAdd(&wh[(v >> 16) & 255], 1u);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_atoms_noret(uint32_t* out, uint32_t seed) {
    __shared__ uint32_t h[16][257];
    for (int i = threadIdx.x; i < 16 * 257; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t* wh = h[threadIdx.x >> 5];
    uint32_t v = (threadIdx.x * 2654435761u + seed);
    for (int i = 0; i < ITERS; ++i) {
        v = v * 1664525u + 1013904223u;
        atomicAdd(&wh[(v >> 24)], 1u);
        atomicAdd(&wh[(v >> 16) & 255], 1u);
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = wh[threadIdx.x & 255];
}

__global__ void k_lds_rand(uint32_t* out, uint32_t seed) {
    __shared__ uint32_t h[16][257];
    for (int i = threadIdx.x; i < 16 * 257; i += blockDim.x) (&h[0][0])[i] = i;
    __syncthreads();
    const uint32_t* wh = h[threadIdx.x >> 5];
    uint32_t v = (threadIdx.x * 2654435761u + seed), acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        v = v * 1664525u + 1013904223u;
        acc += wh[(v >> 24)] + wh[(v >> 16) & 255];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Lane order of same-address shared atomics: record, per trial, whether the
// returned old values are increasing with lane index among colliding lanes.
__global__ void k_atoms_order(uint32_t* violations, uint32_t seed) {
    __shared__ uint32_t h[16][257];
    uint32_t* wh = h[threadIdx.x >> 5];
    uint32_t v = seed ^ (blockIdx.x * 7919u);
    uint32_t bad = 0;
    for (int t = 0; t < 2048; ++t) {
        for (int i = threadIdx.x & 31; i < 257; i += 32) wh[i] = 0;
        __syncwarp();
        v = v * 1664525u + 1013904223u;
        const uint32_t mod = 1u + ((v >> 8) & 15u);           // 1..16 distinct bins
        const uint32_t bin = ((threadIdx.x & 31) * 2654435761u + v) % mod;
        const uint32_t old = atomicAdd(&wh[bin], 1u);
        const uint32_t peers = __match_any_sync(0xffffffff, bin);
        const uint32_t below = __popc(peers & ((1u << (threadIdx.x & 31)) - 1));
        bad += (old != below);
        __syncwarp();
    }
    atomicAdd(violations, bad);
}

template <typename K>
float time_kernel(K kern, uint32_t* buf, int blocks, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, threads>>>(buf, 1);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(buf, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* buf;
    CK(cudaMalloc(&buf, 64 << 20));
    const int blocks = sms * 4, threads = 512;
    const double warps = static_cast<double>(blocks) * threads / 32;
    const double ghz = clk / 1e6;
    struct { const char* name; float ms; double ops_per_warp_iter; } r[] = {
        {"match.any (per warp instr)", time_kernel(k_match, buf, blocks, threads), 4},
        {"ballot x8 match (per 8-bit peer mask)", time_kernel(k_ballot8, buf, blocks, threads), 2},
        {"atoms.add with return, 256 bins/warp (per warp instr)", time_kernel(k_atoms_ret, buf, blocks, threads), 2},
        {"red.shared.add (no return), 256 bins/warp", time_kernel(k_atoms_noret, buf, blocks, threads), 2},
        {"lds random bins (per warp instr)", time_kernel(k_lds_rand, buf, blocks, threads), 2},
    };
    printf("SMs=%d clock=%.3f GHz blocks=%d threads=%d\n", sms, ghz, blocks, threads);
    for (auto& x : r) {
        const double total = warps * ITERS * x.ops_per_warp_iter;
        const double per_sm_cycle = total / (x.ms * 1e-3 * ghz * 1e9) / sms;
        printf("%-58s %8.3f ms  %7.3f warp-ops/cycle/SM  (%6.2f cycles/op/SM)\n", x.name, x.ms, per_sm_cycle,
               1.0 / per_sm_cycle);
    }
    CK(cudaMemset(buf, 0, 4));
    k_atoms_order<<<sms * 4, 512>>>(buf, 12345);
    uint32_t bad = 0;
    CK(cudaMemcpy(&bad, buf, 4, cudaMemcpyDeviceToHost));
    printf("same-address atoms lane-order violations: %u of %llu lane-trials\n", bad,
           static_cast<unsigned long long>(sms) * 4 * 512 * 2048);
    return 0;
}
