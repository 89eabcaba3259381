// isort_launch.cuh -- kernel configuration and the launch templates of the
// sort pipelines, shared by the translation units of libisort.so.
//
// isort_api.cu (the C ABI) sees only declarations of the launch templates; their
// definitions -- and with them every kernel instantiation -- are compiled in the
// inst_*.cu units (ISORT_LAUNCH_DEFINITIONS), one per key type / digitizer
// family, so nvcc/ptxas build the ~200 kernels in parallel.  Every kernel is
// compiled exactly as before (whole-kernel templates; no cross-unit code).
#pragma once

#include <cuda_runtime.h>

#include "bucket_sort.cuh"
#include "isort_common.cuh"
#include "isort_internal.h"
#include "radix_onesweep.cuh"
#include "radix_onesweep_tma.cuh"

namespace isort {

// Host helpers defined in isort_api.cu.
void prof_mark(cudaStream_t s, const char* name);  // per-phase event trail (isort_profile_*)
void prof_state(const RadixState* st);             // the state the trail reads n_active from
bool rank_fast_path_ok();                          // lane-ordered shared atomics verified
int rank_state();
void set_max_smem_once_raw(const void* kernel, size_t bytes);
int resident_per_sm_raw(const void* kernel, int block, size_t smem);
template <typename F>
inline void set_max_smem_once(F* kernel, size_t bytes) {
    set_max_smem_once_raw(reinterpret_cast<const void*>(kernel), bytes);
}
template <typename F>
inline int resident_per_sm(F* kernel, int block, size_t smem) {
    return resident_per_sm_raw(reinterpret_cast<const void*>(kernel), block, smem);
}

// ----------------------------------------------------- kernel configuration
// Tile shapes per (key width, payload).  Tile = BLOCK * IPT keys.
#ifndef ISORT_PASS_BLOCK
#define ISORT_PASS_BLOCK 512
#endif
// One-sweep tile shape: BLOCK threads x IPT keys per chunk, CHUNKS chunks per
// tile.  Large inputs use 2 chunks of 24 keys per thread (DESIGN.md 3.1 has the
// sweep); inputs below kSmallN use one 8,192-key chunk per tile so a few million
// keys still fill all SMs (raising the threshold to 16M or 32M measured no gain).
#ifndef ISORT_SMALL_N
#define ISORT_SMALL_N (4ull << 20)
#endif
constexpr uint64_t kSmallN = ISORT_SMALL_N;

#ifndef ISORT_PASS_CHUNKS
#define ISORT_PASS_CHUNKS 2
#endif
template <typename K, bool VALS, int CHUNKS = ISORT_PASS_CHUNKS>
struct PassCfg {
    static constexpr int kBlock = ISORT_PASS_BLOCK;
#ifndef ISORT_PASS_IPT32
#define ISORT_PASS_IPT32 24
#endif
#ifndef ISORT_PASS_IPT32V
#define ISORT_PASS_IPT32V 12
#endif
#ifndef ISORT_PASS_IPT64
#define ISORT_PASS_IPT64 12
#endif
    // keys per thread per chunk; the 1-chunk small-n tile: 16 (1M keys: 51 us vs 57 with 12, 53 with 24)
#ifndef ISORT_PASS_IPT_SMALL
#define ISORT_PASS_IPT_SMALL 16
#endif
    static constexpr int kIpt = sizeof(K) == 4 ? (VALS ? ISORT_PASS_IPT32V : (CHUNKS == 1 ? ISORT_PASS_IPT_SMALL : ISORT_PASS_IPT32))
                                               : (VALS ? 6 : ISORT_PASS_IPT64);
    static constexpr int kChunks = CHUNKS;
    static constexpr int kTile = kBlock * kIpt * kChunks;
    static constexpr int kCtasPerSm = ISORT_PASS_MINB_OF(kBlock);
};

// Keys-only u32 passes over large inputs take the bulk-copy write-out kernel
// (k_onesweep_t, radix_onesweep_tma.cuh): one chunk of kIpt keys per thread.
#ifndef ISORT_PASS_TMA
#define ISORT_PASS_TMA 1
#endif
#ifndef ISORT_PASS_IPT_T
#define ISORT_PASS_IPT_T 32
#endif
#ifndef ISORT_PASS_BLOCK_T
#define ISORT_PASS_BLOCK_T 512
#endif
#ifndef ISORT_PASS_IPT_TV
#define ISORT_PASS_IPT_TV 16  // with a payload: 8,192-pair tiles (two staged arrays)
#endif
#ifndef ISORT_PASS_TMA_VALS
#define ISORT_PASS_TMA_VALS 1
#endif
#ifndef ISORT_PASS_IPT_T64
#define ISORT_PASS_IPT_T64 16  // u64 keys (keys only): 8,192-key tiles
#endif
#ifndef ISORT_PASS_IPT_T64V
#define ISORT_PASS_IPT_T64V 12  // u64 keys with a payload: 6,144-pair tiles
#endif
#ifndef ISORT_PASS_TMA_U64
#define ISORT_PASS_TMA_U64 1
#endif
#ifndef ISORT_PASS_TMA_U64V
#define ISORT_PASS_TMA_U64V 1
#endif
// With a payload the bulk-copy pass wins up to ~2 x 10^8 pairs and then loses to k_onesweep
// (uniform keys, ms per 10^8 pairs at n = 1e8 / 2.5e8 / 5e8 / 1e9: 0.507 / 0.525 / 0.560 / 0.591
// against 0.527 / 0.514 / 0.518 / 0.520; the keys-only pass does not degrade: 0.228 at 1e9), so
// larger sorts with a payload keep k_onesweep.
#ifndef ISORT_PASS_TMA_VALS_MAX_N
#define ISORT_PASS_TMA_VALS_MAX_N 150000000ull
#endif
constexpr uint64_t kTmaValsMaxN = ISORT_PASS_TMA_VALS_MAX_N;
template <typename K, bool VALS = false>
struct PassCfgT {
    static constexpr int kBlock = ISORT_PASS_BLOCK_T;
    static constexpr int kIpt = sizeof(K) == 8 ? (VALS ? ISORT_PASS_IPT_T64V : ISORT_PASS_IPT_T64)
                                               : (VALS ? ISORT_PASS_IPT_TV : ISORT_PASS_IPT_T);
    static constexpr int kTile = kBlock * kIpt;
    static constexpr int kCtasPerSm = ISORT_PASS_CTAS_T_OF(kBlock);
};
// Which digitizers take it: the radix digit (one PRMT; 0.242 against 0.279 ms per pass at
// 10^8) and the u32 bucket-index digit (a 64-bit multiply and shift: computed once, in the count,
// and kept packed in registers for the rank -- 0.260 / 0.254 against 0.282 / 0.275 ms in k_onesweep;
// 0.279 / 0.276 when the digit is computed twice).
template <typename Dz>
struct TmaPassDigitizer : std::false_type {};
template <typename K>
struct TmaPassDigitizer<RadixDigitizer<K>> : std::true_type {};
#ifndef ISORT_PASS_TMA_BUCKET
#define ISORT_PASS_TMA_BUCKET 1
#endif
#if ISORT_PASS_TMA_BUCKET
template <typename K, int MODE>
struct TmaPassDigitizer<BucketDigitizer<K, MODE>> : std::integral_constant<bool, sizeof(K) == 4> {};
#endif
template <typename K, int MODE>
struct CachesDigit<BucketDigitizer<K, MODE>> : std::true_type {};
template <typename K, bool VALS, typename Dz>
constexpr bool pass_uses_tma() {
    return ISORT_PASS_TMA && TmaPassDigitizer<Dz>::value &&
           (sizeof(K) == 4 ? (!VALS || ISORT_PASS_TMA_VALS) : (VALS ? ISORT_PASS_TMA_U64V : ISORT_PASS_TMA_U64));
}

// Smallest tile any digit pass of a pipeline over n keys may use: it sizes the
// look-back rows of a temp layout (radix_layout).  Each launch computes its own
// tile count from the configuration it runs (launch_radix_pipeline).
template <typename K, bool VALS>
inline int pass_tile(uint64_t n) {
    if (n < kSmallN) return PassCfg<K, VALS, 1>::kTile;
    const int t = PassCfg<K, VALS, ISORT_PASS_CHUNKS>::kTile;
    if (ISORT_PASS_TMA && (sizeof(K) == 4 ? (!VALS || ISORT_PASS_TMA_VALS) : (VALS ? ISORT_PASS_TMA_U64V : ISORT_PASS_TMA_U64)))
        return PassCfgT<K, VALS>::kTile < t ? PassCfgT<K, VALS>::kTile : t;
    return t;
}
// Tile of the partition (scatter) pass, which keeps the k_onesweep shapes.
template <typename K, bool VALS>
inline int scatter_tile(uint64_t n) {
    return n < kSmallN ? PassCfg<K, VALS, 1>::kTile : PassCfg<K, VALS, ISORT_PASS_CHUNKS>::kTile;
}

// Upfront histogram replication (lane copies per bin): 64 KB of counters.
template <int D>
#ifndef ISORT_UF_REP
#define ISORT_UF_REP 32
#endif
#ifndef ISORT_UF_BLOCK
#define ISORT_UF_BLOCK 1024
#endif
struct UpfrontCfg {
    static constexpr int kRep = D <= 4 ? ISORT_UF_REP : 8;
    static constexpr size_t kSmem = static_cast<size_t>(D) * kRadix * kRep * sizeof(uint32_t);
};

constexpr int kUpfrontBlock = ISORT_UF_BLOCK;

// The counting pass's state sits right after RadixState in every temp layout
// (radix_layout), inside the region the pipeline zeroes.
inline CountState* count_state(RadixState* st) {
    return reinterpret_cast<CountState*>(reinterpret_cast<char*>(st) + align_up(sizeof(RadixState)));
}

// Bytes per look-back status word for a call over n keys (radix_onesweep.cuh).
inline size_t lb_word_bytes(uint64_t n) { return n <= kNarrowLbMaxN ? 4 : 8; }

// ------------------------------------------------------------- bucket sort
#ifndef ISORT_SEG_BLOCK
#define ISORT_SEG_BLOCK 512
#endif
#ifndef ISORT_SEG_IPT
#define ISORT_SEG_IPT 32
#endif
constexpr int kSegBlock = ISORT_SEG_BLOCK;
// keys per thread of a segment-sort stage (the stage lives in registers between
// a pass's count and scatter): 32 for u32 keys (a 16,384-key stage; bigger
// stages amortise the per-stage barriers -- 8,192 / 10,240 / 16,384 / 18,432 keys
// measured 73.5 / 77.4 / 83.5 / 83.8 Gkeys/s), fewer with a payload or u64 keys
template <typename K, bool VALS>
constexpr int seg_ipt() {
    return sizeof(K) == 4 ? (VALS ? 20 : ISORT_SEG_IPT) : (VALS ? 12 : 16);
}

// ---------------------------------------------------------- launch templates
template <typename K, bool VALS, typename Dz, typename Cfg, bool SCATTER = false>
void launch_passes(const K* kin, K* kout, K* kalt, const uint32_t* vin, uint32_t* vout, uint32_t* valt, bool iota,
                   uint64_t n, RadixState* st, void* lookback, uint32_t tiles, const Dz& dz, cudaStream_t s,
                   const ScatterArg<SCATTER> scat = ScatterArg<SCATTER>{});
template <typename K, bool VALS, typename Dz>
void launch_passes_t(const K* kin, K* kout, K* kalt, const uint32_t* vin, uint32_t* vout, uint32_t* valt, bool iota,
                     uint64_t n, RadixState* st, void* lookback, uint32_t tiles, const Dz& dz, cudaStream_t s);
template <typename K, typename Dz>
int launch_histogram(const K* kin, uint64_t n, RadixState* st, void* lookback, uint32_t tiles, const Dz& dz,
                     int plan_flags, bool zero_state, cudaStream_t s);
template <typename K, bool VALS, typename Dz>
int launch_radix_pipeline(const K* kin, K* kout, K* kalt, const uint32_t* vin, uint32_t* vout,
                          uint32_t* valt, bool iota, uint64_t n, RadixState* st, void* lookback,
                          uint32_t tiles, const Dz& dz, int plan_flags, bool zero_state,
                          cudaStream_t s);
template <typename K, typename Dz, bool VALS>
void launch_segments(K* keys, uint32_t* vals, uint64_t n, const RadixState* st, BucketState* bst, const Dz& dz,
                     cudaStream_t s);

#ifdef ISORT_LAUNCH_DEFINITIONS
template <typename K, bool VALS, typename Dz, typename Cfg, bool SCATTER>
void launch_passes(const K* kin, K* kout, K* kalt, const uint32_t* vin, uint32_t* vout, uint32_t* valt, bool iota,
                   uint64_t n, RadixState* st, void* lookback, uint32_t tiles, const Dz& dz, cudaStream_t s,
                   const ScatterArg<SCATTER> scat) {
    constexpr int D = Dz::kDigits;
    using Smem = OnesweepSmem<K, Cfg::kBlock, Cfg::kIpt, Cfg::kChunks, VALS, !Dz::kCheapDigit>;
    using Narrow = uint32_t;            // look-back status words: n < 2^30
    using Wide = unsigned long long;    // n up to 2^32 - 1
    const bool fast = rank_fast_path_ok();
    const bool narrow = lb_word_bytes(n) == 4;
    auto* kern = fast ? (narrow ? k_onesweep<K, Dz, Cfg::kBlock, Cfg::kIpt, Cfg::kChunks, VALS, false, SCATTER, Narrow>
                                : k_onesweep<K, Dz, Cfg::kBlock, Cfg::kIpt, Cfg::kChunks, VALS, false, SCATTER, Wide>)
                      : (narrow ? k_onesweep<K, Dz, Cfg::kBlock, Cfg::kIpt, Cfg::kChunks, VALS, true, SCATTER, Narrow>
                                : k_onesweep<K, Dz, Cfg::kBlock, Cfg::kIpt, Cfg::kChunks, VALS, true, SCATTER, Wide>);
    set_max_smem_once(kern, sizeof(Smem));
    const unsigned grid3 = tiles < static_cast<uint32_t>(Cfg::kCtasPerSm * sm_count()) ? tiles
                                                                                     : Cfg::kCtasPerSm * sm_count();
    for (int slot = 0; slot < D; ++slot) {
        kern<<<grid3, Cfg::kBlock, sizeof(Smem), s>>>(kin, kout, kalt, vin, vout, valt, iota ? 1 : 0, n, st, lookback,
                                                        tiles, slot, dz, scat);
        static const char* kPassNames[kMaxDigits] = {"pass0", "pass1", "pass2", "pass3",
                                                     "pass4", "pass5", "pass6", "pass7"};
        prof_mark(s, kPassNames[slot]);
    }
}

// Passes with the bulk-copy write-out (k_onesweep_t), one launch per digit slot.
template <typename K, bool VALS, typename Dz>
void launch_passes_t(const K* kin, K* kout, K* kalt, const uint32_t* vin, uint32_t* vout, uint32_t* valt, bool iota,
                     uint64_t n, RadixState* st, void* lookback, uint32_t tiles, const Dz& dz, cudaStream_t s) {
    constexpr int D = Dz::kDigits;
    using Cfg = PassCfgT<K, VALS>;
    using Smem = OnesweepTSmem<K, Cfg::kBlock, Cfg::kIpt, VALS>;
    const bool fast = rank_fast_path_ok();
    const bool narrow = lb_word_bytes(n) == 4;
    auto* kern = fast ? (narrow ? k_onesweep_t<K, Dz, Cfg::kBlock, Cfg::kIpt, VALS, false, uint32_t>
                                : k_onesweep_t<K, Dz, Cfg::kBlock, Cfg::kIpt, VALS, false, unsigned long long>)
                      : (narrow ? k_onesweep_t<K, Dz, Cfg::kBlock, Cfg::kIpt, VALS, true, uint32_t>
                                : k_onesweep_t<K, Dz, Cfg::kBlock, Cfg::kIpt, VALS, true, unsigned long long>);
    set_max_smem_once(kern, sizeof(Smem));
    const unsigned cap = static_cast<unsigned>(Cfg::kCtasPerSm * sm_count());
    const unsigned grid3 = tiles < cap ? tiles : cap;
    for (int slot = 0; slot < D; ++slot) {
        kern<<<grid3, Cfg::kBlock, sizeof(Smem), s>>>(kin, kout, kalt, vin, vout, valt, iota ? 1 : 0, n, st, lookback,
                                                        tiles, slot, dz);
        static const char* kPassNames[kMaxDigits] = {"pass0", "pass1", "pass2", "pass3",
                                                     "pass4", "pass5", "pass6", "pass7"};
        prof_mark(s, kPassNames[slot]);
    }
}

// Histogram step of a pipeline: zero the state, K1 (all digit histograms, max,
// sortedness, range check), K2 (scans + pass plan).
template <typename K, typename Dz>
int launch_histogram(const K* kin, uint64_t n, RadixState* st, void* lookback, uint32_t tiles, const Dz& dz,
                     int plan_flags, bool zero_state, cudaStream_t s) {
    constexpr int D = Dz::kDigits;
    prof_mark(s, "start");
    prof_state(st);
    if (zero_state) {
        const size_t bytes = reinterpret_cast<char*>(lookback) - reinterpret_cast<char*>(st) +
                             static_cast<size_t>(D) * tiles * kRadix * lb_word_bytes(n);
        ISORT_CUDA_TRY(cudaMemsetAsync(st, 0, bytes, s));
        prof_mark(s, "memset");
    }
    const bool vec = (reinterpret_cast<uintptr_t>(kin) & 15u) == 0;
    using UCfg = UpfrontCfg<D>;
    const uint64_t want = (n + 4ull * kUpfrontBlock - 1) / (4ull * kUpfrontBlock);
    auto* k1 = vec ? k_upfront<K, Dz, kUpfrontBlock, UCfg::kRep, true> : k_upfront<K, Dz, kUpfrontBlock, UCfg::kRep, false>;
    set_max_smem_once(k1, UCfg::kSmem);
    const uint64_t cap1 = static_cast<uint64_t>(resident_per_sm(k1, kUpfrontBlock, UCfg::kSmem)) * sm_count();
    const unsigned grid1 = static_cast<unsigned>(want < cap1 ? (want ? want : 1) : cap1);
    k1<<<grid1, kUpfrontBlock, UCfg::kSmem, s>>>(kin, n, st, dz);
    prof_mark(s, "upfront");
    int top = 0;
    uint32_t top_bins = kRadix, sb_fine = 0, sb_coarse = 0;
    dz.plan_args(&plan_flags, &top, &top_bins, &sb_fine, &sb_coarse);
    k_plan<D><<<1, kRadix, 0, s>>>(st, n, plan_flags, top, top_bins, sb_fine, sb_coarse);
    prof_mark(s, "plan");
    launched(2);
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

// Launch the whole radix pipeline for digitizer `dz` (radix digits, or the
// bucket sort's bucket-index digits).  Buffers: kin (const) -> kout, with kalt
// as ping-pong; the plan decides which passes run.
template <typename K, bool VALS, typename Dz>
int launch_radix_pipeline(const K* kin, K* kout, K* kalt, const uint32_t* vin, uint32_t* vout,
                          uint32_t* valt, bool iota, uint64_t n, RadixState* st, void* lookback,
                          uint32_t tiles, const Dz& dz, int plan_flags, bool zero_state,
                          cudaStream_t s) {
    constexpr int D = Dz::kDigits;
    if (VALS) plan_flags &= ~kPlanCounting;  // a payload needs the scatter
    int rc = launch_histogram<K, Dz>(kin, n, st, lookback, tiles, dz, plan_flags, zero_state, s);
    if (rc) return rc;

    // `tiles` is the layout's row capacity (the smallest tile); each shape counts its own tiles
    auto tiles_of = [&](int tile) { return static_cast<uint32_t>((n + tile - 1) / tile); };
    if (n < kSmallN) {
        using Cfg = PassCfg<K, VALS, 1>;
        launch_passes<K, VALS, Dz, Cfg>(kin, kout, kalt, vin, vout, valt, iota, n, st, lookback, tiles_of(Cfg::kTile),
                                        dz, s);
    } else if (pass_uses_tma<K, VALS, Dz>() && (!VALS || n <= kTmaValsMaxN)) {
        if constexpr (pass_uses_tma<K, VALS, Dz>())
            launch_passes_t<K, VALS, Dz>(kin, kout, kalt, vin, vout, valt, iota, n, st, lookback,
                                         tiles_of(PassCfgT<K, VALS>::kTile), dz, s);
    } else {
        using Cfg = PassCfg<K, VALS, ISORT_PASS_CHUNKS>;
        launch_passes<K, VALS, Dz, Cfg>(kin, kout, kalt, vin, vout, valt, iota, n, st, lookback, tiles_of(Cfg::kTile),
                                        dz, s);
    }
    launched(D);
    // the plan's early-out shapes (radix_onesweep.cuh, k_finish_a / k_finish_b): sorted
    // copy, run-wise reversal, counting pass -- each kernel returns at once unless chosen
    const uint64_t cblocks = (n + 4095) / 4096;
    const unsigned fgrid = static_cast<unsigned>(cblocks < 2ull * sm_count() ? (cblocks ? cblocks : 1) : 2ull * sm_count());
    CountState* cs = count_state(st);
    // the look-back rows are unused on the early-out paths: they hold the reversal's
    // long-run list (at most n / (kRevShortRun + 1) runs of 16 bytes, inside the rows)
    auto* long_runs = static_cast<unsigned long long*>(lookback);
    const bool counting = !VALS && (plan_flags & kPlanCounting);
    constexpr size_t kHistSmem = static_cast<size_t>(kCountBins) * kCountRep * sizeof(uint32_t);
    auto* fa = k_finish_a<K, VALS>;
    if (counting) set_max_smem_once(fa, kHistSmem);
    fa<<<fgrid, kCountBlock, counting ? kHistSmem : 0, s>>>(kin, kout, vin, vout, iota ? 1 : 0, n, st, cs);
    prof_mark(s, "finish_a");
    launched(1);
    if (counting || VALS) {
        k_finish_b<K, VALS><<<fgrid, kCountBlock, 0, s>>>(kout, vout, n, st, cs, long_runs);
        prof_mark(s, "finish_b");
        launched(1);
    }
    if (VALS) {
        k_rev_long_runs<<<fgrid, 512, 0, s>>>(vout, st, long_runs);
        prof_mark(s, "rev_long");
        launched(1);
    }
    ISORT_CUDA_TRY(cudaGetLastError());
    return ISORT_OK;
}

// K5 launch: persistent, as many CTAs as fit (at most one per ~4K keys).
template <typename K, typename Dz, bool VALS>
void launch_segments(K* keys, uint32_t* vals, uint64_t n, const RadixState* st, BucketState* bst, const Dz& dz,
                     cudaStream_t s) {
    constexpr int kSegIpt = seg_ipt<K, VALS>();
    using Smem = SegSmem<K, kSegBlock, kSegIpt, VALS>;
    static_assert(sizeof(Smem) <= 232448, "segment stage exceeds shared memory");
    auto* kern = k_bucket_segments<K, Dz, kSegBlock, kSegIpt, VALS>;
    set_max_smem_once(kern, sizeof(Smem));
    const int per_sm = resident_per_sm(kern, kSegBlock, sizeof(Smem));
    const uint64_t want = (n + kSegBlock * kSegIpt / 2 - 1) / (kSegBlock * kSegIpt / 2);
    const uint64_t cap = static_cast<uint64_t>(per_sm) * sm_count();
    kern<<<static_cast<unsigned>(want < cap ? want : cap), kSegBlock, sizeof(Smem), s>>>(keys, vals, n, st, bst, dz);
}

// Explicit instantiation helpers for the inst_*.cu units.
#define ISORT_INST_PIPELINE(K, V, DZ)                                                                       \
    template int launch_radix_pipeline<K, V, DZ>(const K*, K*, K*, const uint32_t*, uint32_t*, uint32_t*, bool, \
                                                 uint64_t, RadixState*, void*, uint32_t, const DZ&, int, bool,   \
                                                 cudaStream_t);
#define ISORT_INST_HISTOGRAM(K, DZ) \
    template int launch_histogram<K, DZ>(const K*, uint64_t, RadixState*, void*, uint32_t, const DZ&, int, bool, cudaStream_t);
#define ISORT_INST_PASSES(K, V, DZ, CFG, SC)                                                                    \
    template void launch_passes<K, V, DZ, CFG, SC>(const K*, K*, K*, const uint32_t*, uint32_t*, uint32_t*, bool, \
                                                   uint64_t, RadixState*, void*, uint32_t, const DZ&, cudaStream_t, \
                                                   const ScatterArg<SC>);
#define ISORT_INST_SEGMENTS(K, DZ, V) \
    template void launch_segments<K, DZ, V>(K*, uint32_t*, uint64_t, const RadixState*, BucketState*, const DZ&, cudaStream_t);
#endif  // ISORT_LAUNCH_DEFINITIONS

}  // namespace isort
