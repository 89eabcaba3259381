// cub_yardstick.cu -- bench-only calibration: CUB DeviceRadixSort (CUDA 12.9's
// onesweep implementation) on the BASELINE C2 shape, same box.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cub_yardstick tools/cub_yardstick.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <cstdint>

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 100000000ull;
    std::vector<uint32_t> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = (uint32_t)mix64(42 + (i + 1) * 0x9e3779b97f4a7c15ULL);
    uint32_t *k, *k2, *v, *v2;
    cudaMalloc(&k, n * 4); cudaMalloc(&k2, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&v2, n * 4);
    cudaMemcpy(k, h.data(), n * 4, cudaMemcpyHostToDevice);
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb1, k, k2, (int)n);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, k, k2, v, v2, (int)n);
    void* tmp; cudaMalloc(&tmp, tb1 > tb2 ? tb1 : tb2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        for (int w = 0; w < 3; ++w) {
            if (mode == 0) cub::DeviceRadixSort::SortKeys(tmp, tb1, k, k2, (int)n);
            else cub::DeviceRadixSort::SortPairs(tmp, tb2, k, k2, v, v2, (int)n);
        }
        const int reps = 10;
        cudaEventRecord(a);
        for (int r = 0; r < reps; ++r) {
            if (mode == 0) cub::DeviceRadixSort::SortKeys(tmp, tb1, k, k2, (int)n);
            else cub::DeviceRadixSort::SortPairs(tmp, tb2, k, k2, v, v2, (int)n);
        }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
        printf("CUB %s n=%zu: %.3f ms  %.2f Gkeys/s\n", mode == 0 ? "SortKeys " : "SortPairs", n, ms, n / ms / 1e6);
    }
    return 0;
}
