// exp_pass.cu -- A/B harness for the one-sweep digit pass (never linked into the product).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/exp_pass tools/exp_pass.cu
//   tools/exp_pass [n] [vals: 0|2] [reps]
//
// Sorts n SplitMix64 u32 keys (seed 42: the reference generate() keys) with the
// v10 pipeline (K1 + K2 + 4 x k_onesweep) and the v2 pass (K1 + K2 + 4 x k_pass),
// checks both outputs are identical (keys and, with vals=2, stable positions) and
// sorted, and prints per-pass CUDA-event times.  Tile shape of k_pass:
// -DEXP_BLOCK, -DEXP_IPT.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "exp_onesweep_pass.cuh"

using namespace isort;

#ifndef OLD_BLOCK
#define OLD_BLOCK 512
#endif
#ifndef OLD_IPT
#define OLD_IPT 24
#endif
#ifndef OLD_IPTV
#define OLD_IPTV 12
#endif
#ifndef EXP_BLOCK
#define EXP_BLOCK 512
#endif
#ifndef EXP_IPT
#define EXP_IPT 24
#endif
#ifndef EXP_IPTV
#define EXP_IPTV 12
#endif
#ifndef EXP_IPT2
#define EXP_IPT2 22
#endif
#ifndef EXP_IPT2V
#define EXP_IPT2V 10
#endif

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__global__ void k_gen(uint32_t* k, uint64_t n, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        k[i] = (uint32_t)(z ^ (z >> 31));
    }
}
__global__ void k_diff(const uint32_t* a, const uint32_t* b, uint64_t n, unsigned long long* bad) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        c += a[i] != b[i];
    if (c) atomicAdd(bad, c);
}
__global__ void k_unsorted(const uint32_t* a, uint64_t n, unsigned long long* bad) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
        c += a[i] > a[i + 1];
    if (c) atomicAdd(bad, c);
}

// keys sorted; with positions: kin[pos[i]] == kout[i] and positions ascending inside runs
__global__ void k_check(const uint32_t* kin, const uint32_t* kout, const uint32_t* pos, uint64_t n,
                        unsigned long long* bad) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (i + 1 < n && kout[i] > kout[i + 1]) ++c;
        if (pos) {
            if (kin[pos[i]] != kout[i]) ++c;
            if (i + 1 < n && kout[i] == kout[i + 1] && pos[i] >= pos[i + 1]) ++c;
        }
    }
    if (c) atomicAdd(bad, c);
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000000ull;
    const int vmode = argc > 2 ? std::atoi(argv[2]) : 0;
    const int reps = argc > 3 ? std::atoi(argv[3]) : 10;
    const bool vals = vmode != 0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t *kin, *kout_a, *kout_b, *kalt, *vout_a, *vout_b, *valt;
    CK(cudaMalloc(&kin, n * 4));
    CK(cudaMalloc(&kout_a, n * 4));
    CK(cudaMalloc(&kout_b, n * 4));
    CK(cudaMalloc(&kalt, n * 4));
    CK(cudaMalloc(&vout_a, n * 4));
    CK(cudaMalloc(&vout_b, n * 4));
    CK(cudaMalloc(&valt, n * 4));
    k_gen<<<1024, 256>>>(kin, n, 42);
    RadixState* st;
    CK(cudaMalloc(&st, sizeof(RadixState)));
    const uint64_t max_tiles = n / 4096 + 2;
    void* lbv;
    const size_t lb_bytes = 4 * max_tiles * kRadix * sizeof(unsigned long long);
    CK(cudaMalloc(&lbv, lb_bytes));
    unsigned long long* dbad;
    CK(cudaMalloc(&dbad, 8));
    cudaStream_t s = 0;
    RadixDigitizer<uint32_t> dz;

    constexpr int kUfRep = 32, kUfBlock = 1024;
    const size_t uf_smem = 4 * kRadix * kUfRep * 4;
    auto* k1 = k_upfront<uint32_t, RadixDigitizer<uint32_t>, kUfBlock, kUfRep, true>;
    CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)uf_smem));

    // v10 pass
    constexpr int kOldIpt = OLD_IPT, kOldIptV = OLD_IPTV;
    using OldSm = OnesweepSmem<uint32_t, OLD_BLOCK, kOldIpt, 2, false, false>;
    using OldSmV = OnesweepSmem<uint32_t, OLD_BLOCK, kOldIptV, 2, true, false>;
    auto* kold = k_onesweep<uint32_t, RadixDigitizer<uint32_t>, OLD_BLOCK, kOldIpt, 2, false, false, false>;
    auto* koldv = k_onesweep<uint32_t, RadixDigitizer<uint32_t>, OLD_BLOCK, kOldIptV, 2, true, false, false>;
    CK(cudaFuncSetAttribute(kold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OldSm)));
    CK(cudaFuncSetAttribute(koldv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OldSmV)));
    // v2 pass
    using NewSm = PassSmem<uint32_t, EXP_BLOCK, EXP_IPT, false, false>;
    using NewSmV = PassSmem<uint32_t, EXP_BLOCK, EXP_IPTV, true, false>;
    auto* knew = k_pass<uint32_t, RadixDigitizer<uint32_t>, EXP_BLOCK, EXP_IPT, false, false, false>;
    auto* knewv = k_pass<uint32_t, RadixDigitizer<uint32_t>, EXP_BLOCK, EXP_IPTV, true, false, false>;
    CK(cudaFuncSetAttribute(knew, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NewSm)));
    CK(cudaFuncSetAttribute(knewv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NewSmV)));
    using P2Sm = Pass2Smem<uint32_t, EXP_BLOCK, EXP_IPT2, false, false>;
    using P2SmV = Pass2Smem<uint32_t, EXP_BLOCK, EXP_IPT2V, true, false>;
    auto* kp2 = k_pass2<uint32_t, RadixDigitizer<uint32_t>, EXP_BLOCK, EXP_IPT2, false, false, false>;
    auto* kp2v = k_pass2<uint32_t, RadixDigitizer<uint32_t>, EXP_BLOCK, EXP_IPT2V, true, false, false>;
    CK(cudaFuncSetAttribute(kp2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(P2Sm)));
    CK(cudaFuncSetAttribute(kp2v, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(P2SmV)));
    int occ_p2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p2, vals ? kp2v : kp2, EXP_BLOCK,
                                                     vals ? sizeof(P2SmV) : sizeof(P2Sm)));
    std::printf("v2b: ipt %d smem %zu occ %d\n", vals ? EXP_IPT2V : EXP_IPT2, vals ? sizeof(P2SmV) : sizeof(P2Sm), occ_p2);
    int occ_old = 0, occ_new = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_old, vals ? koldv : kold, OLD_BLOCK,
                                                     vals ? sizeof(OldSmV) : sizeof(OldSm)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_new, vals ? knewv : knew, EXP_BLOCK,
                                                     vals ? sizeof(NewSmV) : sizeof(NewSm)));
    std::printf("n=%llu vals=%d sms=%d  old: smem %zu occ %d  new: block %d ipt %d smem %zu occ %d\n",
                (unsigned long long)n, vmode, sms, vals ? sizeof(OldSmV) : sizeof(OldSm), occ_old, EXP_BLOCK,
                vals ? EXP_IPTV : EXP_IPT, vals ? sizeof(NewSmV) : sizeof(NewSm), occ_new);

    std::vector<cudaEvent_t> ev(8);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    auto run = [&](int variant, uint32_t* kout, uint32_t* vout, float* pass_ms) {
        const bool use_new = variant != 0;
        const int tile = variant == 2 ? EXP_BLOCK * (vals ? EXP_IPT2V : EXP_IPT2)
                         : use_new    ? EXP_BLOCK * (vals ? EXP_IPTV : EXP_IPT)
                                      : OLD_BLOCK * (vals ? kOldIptV : kOldIpt) * 2;
        const uint32_t tiles = (uint32_t)((n + tile - 1) / tile);
        CK(cudaMemsetAsync(st, 0, sizeof(RadixState), s));
        CK(cudaMemsetAsync(lbv, 0, (size_t)4 * tiles * kRadix * (use_new ? 8 : 4), s));
        const uint64_t want = (n + 4ull * kUfBlock - 1) / (4ull * kUfBlock);
        const unsigned g1 = (unsigned)(want < 2ull * sms ? want : 2ull * sms);
        k1<<<g1, kUfBlock, uf_smem, s>>>(kin, n, st, dz);
        k_plan<4><<<1, kRadix, 0, s>>>(st, n, kPlanSkipSorted);
        CK(cudaEventRecord(ev[0], s));
        const int occ = variant == 2 ? occ_p2 : (use_new ? occ_new : occ_old);
        const unsigned grid = tiles < (uint32_t)(occ * sms) ? tiles : occ * sms;
        for (int p = 0; p < 4; ++p) {
            if (variant == 2) {
                if (vals)
                    kp2v<<<grid, EXP_BLOCK, sizeof(P2SmV), s>>>(kin, kout, kalt, nullptr, vout, valt, 1, n, st,
                                                                (unsigned long long*)lbv, tiles, p, dz, NoScatter{});
                else
                    kp2<<<grid, EXP_BLOCK, sizeof(P2Sm), s>>>(kin, kout, kalt, nullptr, nullptr, nullptr, 0, n, st,
                                                              (unsigned long long*)lbv, tiles, p, dz, NoScatter{});
            } else if (use_new) {
                if (vals)
                    knewv<<<grid, EXP_BLOCK, sizeof(NewSmV), s>>>(kin, kout, kalt, nullptr, vout, valt, 1, n, st,
                                                                  (unsigned long long*)lbv, tiles, p, dz, NoScatter{});
                else
                    knew<<<grid, EXP_BLOCK, sizeof(NewSm), s>>>(kin, kout, kalt, nullptr, nullptr, nullptr, 0, n, st,
                                                                (unsigned long long*)lbv, tiles, p, dz, NoScatter{});
            } else {
                if (vals)
                    koldv<<<grid, OLD_BLOCK, sizeof(OldSmV), s>>>(kin, kout, kalt, nullptr, vout, valt, 1, n, st,
                                                            (uint32_t*)lbv, tiles, p, dz, NoScatter{});
                else
                    kold<<<grid, OLD_BLOCK, sizeof(OldSm), s>>>(kin, kout, kalt, nullptr, nullptr, nullptr, 0, n, st,
                                                          (uint32_t*)lbv, tiles, p, dz, NoScatter{});
            }
            CK(cudaEventRecord(ev[p + 1], s));
        }
        CK(cudaGetLastError());
        CK(cudaEventSynchronize(ev[4]));
        for (int p = 0; p < 4; ++p) {
            float t;
            CK(cudaEventElapsedTime(&t, ev[p], ev[p + 1]));
            pass_ms[p] += t;
        }
    };
    uint32_t *kout_c, *vout_c;
    CK(cudaMalloc(&kout_c, n * 4));
    CK(cudaMalloc(&vout_c, n * 4));
#ifdef EXP_ONLY_OLD
    constexpr int kVariants = 1;
#else
    constexpr int kVariants = 3;
#endif
    for (int which = 0; which < kVariants; ++which) {
        const bool use_new = which != 0;
        uint32_t* ko = which == 0 ? kout_a : (which == 1 ? kout_b : kout_c);
        uint32_t* vo = which == 0 ? vout_a : (which == 1 ? vout_b : vout_c);
        float pm[4] = {0, 0, 0, 0}, dummy[4] = {0, 0, 0, 0};
        for (int r = 0; r < 3; ++r) run(which, ko, vo, dummy);
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float tot = 0;
        for (int r = 0; r < reps; ++r) {
            CK(cudaEventRecord(a, s));
            run(which, ko, vo, pm);
            CK(cudaEventRecord(b, s));
            CK(cudaEventSynchronize(b));
            float t;
            CK(cudaEventElapsedTime(&t, a, b));
            tot += t;
        }
        std::printf("%s: sort %.4f ms (%.1f Gkeys/s)  passes %.4f %.4f %.4f %.4f ms  (pass frac of 6453.7 GB/s: %.3f)\n",
                    which == 2 ? "v2b k_pass2" : (use_new ? "v2 k_pass  " : "v10 onesweep"), tot / reps, n / (tot / reps) / 1e6, pm[0] / reps,
                    pm[1] / reps, pm[2] / reps, pm[3] / reps,
                    8.0 * n / ((pm[1] + pm[2] + pm[3]) / 3 / reps * 1e-3) / 1e9 / 6453.7);
    }
    unsigned long long bad = 0;
    CK(cudaMemset(dbad, 0, 8));
    k_check<<<1024, 256>>>(kin, kout_a, vals ? vout_a : nullptr, n, dbad);
    CK(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
    std::printf("v10 check (sorted, stable positions) violations: %llu\n", bad);
    if (kVariants == 1) return 0;
    CK(cudaMemset(dbad, 0, 8));
    k_diff<<<1024, 256>>>(kout_a, kout_b, n, dbad);
    CK(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
    std::printf("keys differ: %llu\n", bad);
    if (vals) {
        CK(cudaMemset(dbad, 0, 8));
        k_diff<<<1024, 256>>>(vout_a, vout_b, n, dbad);
        CK(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
        std::printf("positions differ: %llu\n", bad);
    }
    CK(cudaMemset(dbad, 0, 8));
    k_unsorted<<<1024, 256>>>(kout_b, n, dbad);
    CK(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
    std::printf("v2 unsorted pairs: %llu\n", bad);
    CK(cudaMemset(dbad, 0, 8));
    k_diff<<<1024, 256>>>(kout_a, kout_c, n, dbad);
    CK(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
    std::printf("v2b keys differ: %llu\n", bad);
    if (vals) {
        CK(cudaMemset(dbad, 0, 8));
        k_diff<<<1024, 256>>>(vout_a, vout_c, n, dbad);
        CK(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
        std::printf("v2b positions differ: %llu\n", bad);
    }
    return 0;
}
