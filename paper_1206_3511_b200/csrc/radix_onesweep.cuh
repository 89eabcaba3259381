// radix_onesweep.cuh -- LSD radix sort as a one-sweep pipeline for sm_100a.
//
// Reference semantics: intsort::radix_sort_lsd (proj/core/src/sort.cpp:112-119)
// runs build_radix_plan (sort.cpp:57-75) and then one stable counting pass per
// digit (counting_sort_by_digit, sort.cpp:77-110: count -> prefix -> reverse
// walk).  A stable LSD sort has exactly one correct output for a given input,
// and the reference's output is base-invariant (proj/tests/test_sort.cpp:136-149),
// so the engine sorts with 8-bit digits whatever base the caller names.
//
// Device pipeline (all stream-ordered, no host round trip):
//   K1 k_upfront   one read of the keys: every digit histogram (lane-replicated
//                  shared counters: no bank conflicts), max key, number of
//                  adjacent descents (0 => already sorted), optional digitizer
//                  range check (bucket sort).                    4n B HBM read
//   K2 k_plan      scans the histograms, drops trivial digit passes (one bin
//                  holds all n keys => the pass is the identity) and the whole
//                  sort when the input is already sorted; assigns ping-pong
//                  buffers so the last executed pass lands in `out`.
//   K3 k_onesweep  one launch per digit slot (see the K3 comment).  8n B / pass
//   K4 k_copy      only when no pass executes (sorted input): out = in.
#pragma once

#include <type_traits>

#include "isort_common.cuh"

namespace isort {

// Buffer ids used by the plan.
enum : int32_t { kBufIn = 0, kBufOut = 1, kBufAlt = 2 };

// Look-back status words: [W-1:W-2] flag, the rest the count.  Calls with
// n < 2^30 keys use 32-bit words (half the look-back traffic of 64-bit words:
// +2.7% per pass measured at 10^8 keys with 64-bit words); larger calls use
// 64-bit words, so one call sorts up to 2^32 - 1 keys (positions and payloads
// are u32; 16 GB of u32 keys per array fits the B200's HBM).
template <typename LW>
struct LbTraits {
    static constexpr int kBits = 8 * sizeof(LW);
    static constexpr LW kAgg = static_cast<LW>(1) << (kBits - 2);
    static constexpr LW kInc = static_cast<LW>(2) << (kBits - 2);
    static constexpr LW kMask = static_cast<LW>(3) << (kBits - 2);
    static constexpr LW kValue = kAgg - 1;
};
constexpr uint64_t kNarrowLbMaxN = (1ull << 30) - 1;  // 32-bit status words up to here
constexpr uint64_t kMaxLookbackN = 0xFFFFFFFFull;     // per-call limit (u32 positions)

struct RadixState {
    uint32_t hist[kMaxDigits][kRadix];  // K1
    uint32_t offs[kMaxDigits][kRadix];  // K2: exclusive scans
    unsigned long long max_key;         // K1
    unsigned long long first_bad;       // K1: ~(first index failing the range check)
    uint32_t descents;                  // K1: #i with key[i] > key[i+1]
    uint32_t ascents;                   // K1: #i with key[i] < key[i+1] (0 => non-increasing)
    uint32_t n_active;                  // K2
    uint32_t copy_in_to_out;            // K2: sorted input, out = in
    uint32_t reversed;                  // K2: non-increasing input, out = in reversed run by run
    uint32_t counting;                  // K2: keys-only, max < kCountBins: one counting pass (K6)
    uint32_t rev_long;                  // K5: runs longer than kRevShortRun listed for k_rev_long_runs
    uint32_t sb_shift;                  // K2, bucket sort: super-bucket = bucket >> sb_shift
    uint32_t tile_ticket[kMaxDigits];   // K3
    int32_t digit_of_slot[kMaxDigits];  // K2
    int32_t src_of_slot[kMaxDigits];
    int32_t dst_of_slot[kMaxDigits];
    unsigned long long prof[16];        // debug counters (ISORT_PHASE_TIMING builds)
};
// Keys-only sorts whose largest key is below kCountBins take one counting pass
// on the whole key (a single kCountBits-bit digit) instead of digit passes; see K6.
constexpr int kCountBits = 12, kCountBins = 1 << kCountBits;
struct CountState {
    uint32_t vhist[kCountBins];  // K6a: occurrences of each key value
};

// ------------------------------------------------------------- digitizers
// A digitizer maps a key to the digit a pass sorts on.  RadixDigitizer is the
// LSD radix digit ((key >> 8p) & 255); the bucket sort supplies its own
// (digits of the bucket index, bucket_sort.cuh).
template <typename K>
struct RadixDigitizer {
    static constexpr int kDigits = KeyTraits<K>::kDigits;
    static constexpr bool kChecks = false;
    static constexpr bool kCheapDigit = true;  // recompute instead of staging digits
    __device__ __forceinline__ bool needs_range_check() const { return false; }
    __device__ __forceinline__ uint32_t shift_for(int pos) const { return 8u * static_cast<uint32_t>(pos); }
    // One PRMT per key: byte (sh / 8) of the key, zero-extended.
    __device__ __forceinline__ uint32_t digit_sh(K key, uint32_t sh) const {
        if (sizeof(K) == 4) return __byte_perm(static_cast<uint32_t>(key), 0u, 0x4440u | (sh >> 3));
        const uint32_t w = sh >= 32 ? static_cast<uint32_t>(static_cast<uint64_t>(key) >> 32) : static_cast<uint32_t>(key);
        return __byte_perm(w, 0u, 0x4440u | ((sh >> 3) & 3u));
    }
    __device__ __forceinline__ uint32_t digit(K key, int pos) const { return digit_sh(key, shift_for(pos)); }
    __device__ __forceinline__ void all_digits(K key, uint32_t (&d)[kDigits]) const {
#pragma unroll
        for (int p = 0; p < kDigits; ++p) d[p] = digit_sh(key, 8u * p);
    }
    __device__ __forceinline__ bool in_range(K) const { return true; }
    void plan_args(int*, int*, uint32_t*, uint32_t*, uint32_t*) const {}  // K2 needs nothing more
};

// ------------------------------------------------------------------- K1
#ifndef ISORT_UF_UNROLL
#define ISORT_UF_UNROLL 8  // loads in flight per thread: 8 -> 0.0875 ms at 1e8 (4: 0.094, 12: 0.094, 16: 0.159)
#endif
// Digit histograms in lane-replicated shared counters: copy (lane % R) of bin b
// of digit p lives at ((p * 256 + b) * R + lane % R), so lanes of one atomic
// instruction hit distinct banks (R = 32) or at most 2-way (R = 16).
template <typename K, typename Dz, int BLOCK, int R, bool VEC>
__global__ void __launch_bounds__(BLOCK) k_upfront(const K* __restrict__ keys, uint64_t n,
                                                   RadixState* __restrict__ st, Dz dz) {
    constexpr int D = Dz::kDigits;
    extern __shared__ __align__(16) uint32_t uf_cnt[];  // D * 256 * R
    __shared__ unsigned long long red_max[BLOCK / 32];
    __shared__ uint32_t red_desc[BLOCK / 32];
    for (int i = threadIdx.x; i < D * kRadix * R; i += BLOCK) uf_cnt[i] = 0;
    __syncthreads();
    uint32_t* const my_cnt = uf_cnt + lane_id() % R;  // this lane's counter copy

    K kmax = 0;
    uint32_t desc = 0, asc = 0;
    unsigned long long first_bad = ~0ull;

    // The range check only exists where keys can exceed M: a template split keeps
    // its compares out of the common loop.  Indices are 32-bit (n < 2^32).
    auto run = [&](auto check_tag) {
        constexpr bool CHECK = decltype(check_tag)::value;
        auto visit = [&](K k, uint32_t idx) {
            kmax = k > kmax ? k : kmax;
            // Out-of-range keys are still counted (the digitizer clamps them) so the
            // passes stay self-consistent; the host reports the first of them.
            if (CHECK && !dz.in_range(k)) first_bad = idx < first_bad ? idx : first_bad;
            uint32_t d[D];
            dz.all_digits(k, d);
#pragma unroll
            for (int p = 0; p < D; ++p) atomicAdd(my_cnt + (p * kRadix + d[p]) * R, 1u);
        };
        const uint32_t n32 = static_cast<uint32_t>(n);
        const uint32_t stride = gridDim.x * BLOCK;
        constexpr int V = 4;  // 4 keys per thread-iteration
        if (VEC) {
            // Each warp streams U consecutive 512-byte blocks per step (U loads in
            // flight per thread); the successor key for the sortedness check comes
            // from the next lane, or the next block's lane 0.
            const uint32_t nv = n32 / V;
            // loads in flight per thread: 8 for radix digits, 4 for bucket digits (more
            // registers per key; A/B on B200: 0.105 vs 0.110 ms at 10^8)
            constexpr int U = Dz::kCheapDigit && sizeof(K) == 4 && D == 4 ? ISORT_UF_UNROLL : 4;
            const uint32_t wstride = gridDim.x * (BLOCK / 32) * 32 * U;
            // successor of the last whole 4-key group: the scalar tail's first key, or none
            const K tail_next = nv * V < n32 ? keys[nv * V] : static_cast<K>(~static_cast<K>(0));
            for (uint32_t wb = (blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5)) * 32 * U; wb < nv; wb += wstride) {
                K k[U][V];
                // lane 31's successor after the warp's last block: the next block's first key
                const uint32_t vn = wb + U * 32;
                const K step_next = (lane_id() == 31 && vn < nv) ? keys[static_cast<size_t>(vn) * V]
                                                                  : static_cast<K>(~static_cast<K>(0));
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t v = wb + u * 32 + lane_id();
                    if (v < nv) {
                        if (sizeof(K) == 4) {
                            const uint4 q = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + v);
                            k[u][0] = static_cast<K>(q.x);
                            k[u][1] = static_cast<K>(q.y);
                            k[u][2] = static_cast<K>(q.z);
                            k[u][3] = static_cast<K>(q.w);
                        } else {
                            const uint4 a = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + 2ull * v);
                            const uint4 b = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + 2ull * v + 1);
                            k[u][0] = static_cast<K>((static_cast<uint64_t>(a.y) << 32) | a.x);
                            k[u][1] = static_cast<K>((static_cast<uint64_t>(a.w) << 32) | a.z);
                            k[u][2] = static_cast<K>((static_cast<uint64_t>(b.y) << 32) | b.x);
                            k[u][3] = static_cast<K>((static_cast<uint64_t>(b.w) << 32) | b.z);
                        }
                    } else {
                        k[u][0] = 0;  // keep the shuffles below defined
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t v = wb + u * 32 + lane_id();
                    K next = __shfl_down_sync(ISORT_FULL_MASK, k[u][0], 1);
                    const K first_next_block = __shfl_sync(ISORT_FULL_MASK, k[u + 1 < U ? u + 1 : u][0], 0);
                    if (lane_id() == 31) next = u + 1 < U ? first_next_block : step_next;
                    if (v + 1 == nv) next = tail_next;
                    if (v < nv) {
                        desc += (k[u][0] > k[u][1]) + (k[u][1] > k[u][2]) + (k[u][2] > k[u][3]) + (k[u][3] > next);
                        asc |= (k[u][0] < k[u][1]) | (k[u][1] < k[u][2]) | (k[u][2] < k[u][3]) |
                               (k[u][3] < next && v + 1 < nv) | (k[u][3] < next && v + 1 == nv && nv * V < n32);
#pragma unroll
                        for (int j = 0; j < V; ++j) visit(k[u][j], v * V + j);
                    }
                }
            }
            for (uint32_t i = nv * V + blockIdx.x * BLOCK + threadIdx.x; i < n32; i += stride) {
                const K k = keys[i];
                if (i + 1 < n32) {
                    desc += (k > keys[i + 1]);
                    asc |= (k < keys[i + 1]);
                }
                visit(k, i);
            }
        } else {
            for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < n32; i += stride) {
                const K k = keys[i];
                if (i + 1 < n32) {
                    desc += (k > keys[i + 1]);
                    asc |= (k < keys[i + 1]);
                }
                visit(k, i);
            }
        }
    };
    if (Dz::kChecks && dz.needs_range_check())
        run(std::true_type{});
    else
        run(std::false_type{});

    // block reductions
    unsigned long long m = warp_max<unsigned long long>(static_cast<unsigned long long>(kmax));
    uint32_t ds = warp_sum(desc);
    if (__any_sync(ISORT_FULL_MASK, asc != 0) && lane_id() == 0) atomicOr(&st->ascents, 1u);
    unsigned long long fb = warp_max<unsigned long long>(~first_bad);  // max of complements = min index
    const int w = threadIdx.x / 32;
    if (lane_id() == 0) {
        red_max[w] = m;
        red_desc[w] = ds;
    }
    if (Dz::kChecks && lane_id() == 0 && fb != 0ull) atomicMax(&st->first_bad, fb);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = BLOCK / 32;
        m = threadIdx.x < nw ? red_max[threadIdx.x] : 0ull;
        ds = threadIdx.x < nw ? red_desc[threadIdx.x] : 0u;
        m = warp_max<unsigned long long>(m);
        ds = warp_sum(ds);
        if (threadIdx.x == 0) {
            atomicMax(&st->max_key, m);
            if (ds) atomicAdd(&st->descents, ds);
        }
    }
    for (int i = threadIdx.x; i < D * kRadix; i += BLOCK) {
        uint32_t c = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) c += uf_cnt[i * R + ((r + i) & (R - 1))];  // rotate: spread banks
        if (c) atomicAdd(&st->hist[i / kRadix][i % kRadix], c);
    }
}

// ------------------------------------------------------------------- K2
// One CTA of kRadix threads.  flags: kPlanSkipSorted (a sorted input needs no
// pass), kPlanKeepTrivial (run every digit pass, even one-digit ones: a scatter
// pass must move the keys).
// kPlanAdaptiveLow (bucket sort): digit 0 is the optional fine pass -- it runs only
// when the top digit's histogram shows skew (a bin above kSkewFactor times the
// mean), and sb_shift follows (sb_fine with it, sb_coarse without).
constexpr int kPlanSkipSorted = 1, kPlanKeepTrivial = 2, kPlanCounting = 4, kPlanAdaptiveLow = 8;
constexpr uint64_t kSkewFactor = 4;
template <int D>
__global__ void __launch_bounds__(kRadix) k_plan(RadixState* __restrict__ st, uint64_t n, int flags, int top_digit = 0,
                                                 uint32_t top_bins = kRadix, uint32_t sb_fine = 0,
                                                 uint32_t sb_coarse = 0) {
    __shared__ uint32_t warp_tot[kRadix / 32];
    __shared__ int trivial[kMaxDigits];
    const int t = threadIdx.x;
    // skew: a bin of the top digit holds more than kSkewFactor times its share under
    // uniform keys (top_bins = the bins the bucket range can reach)
    const int skewed = (flags & kPlanAdaptiveLow)
                           ? __syncthreads_or(static_cast<uint64_t>(st->hist[top_digit][t]) * top_bins > kSkewFactor * n)
                           : 0;
    for (int p = 0; p < D; ++p) {
        const uint32_t v = st->hist[p][t];
        const uint32_t inc = warp_inclusive_scan(v);
        if (lane_id() == 31) warp_tot[t / 32] = inc;
        const int any_full = __syncthreads_or(static_cast<uint64_t>(v) == n);
        uint32_t pre = 0;
        for (int w = 0; w < t / 32; ++w) pre += warp_tot[w];
        st->offs[p][t] = pre + inc - v;
        if (t == 0) trivial[p] = any_full || (p == 0 && (flags & kPlanAdaptiveLow) && !skewed);
        __syncthreads();
    }
    if (t == 0) st->sb_shift = skewed ? sb_fine : sb_coarse;
    if (t == 0) {
        const bool sorted = (flags & kPlanSkipSorted) && st->descents == 0;
        // non-increasing input: the stable sort is the reversal with each run of
        // equal keys kept in input order (k_reverse_runs), no digit pass
        const bool reversed = (flags & kPlanSkipSorted) && !sorted && st->ascents == 0;
        const bool keep = (flags & kPlanKeepTrivial) != 0;
        // keys only and every key below kCountBins: the LSD sort is one pass on a
        // kCountBits-bit digit (the whole key), and a stable pass over keys that
        // carry nothing else is determined by the key counts alone (K6)
        const bool counting = (flags & kPlanCounting) && !sorted && !reversed && !keep &&
                              st->max_key < static_cast<unsigned long long>(kCountBins);
        int na = 0;
        for (int p = 0; p < D; ++p)
            if (keep || (!sorted && !reversed && !counting && !trivial[p])) st->digit_of_slot[na++] = p;
        for (int s = 0; s < na; ++s) {
            st->src_of_slot[s] = s == 0 ? kBufIn : st->dst_of_slot[s - 1];
            st->dst_of_slot[s] = ((na - 1 - s) % 2 == 0) ? kBufOut : kBufAlt;
        }
        st->n_active = na;
        st->copy_in_to_out = na == 0 && !reversed && !counting;
        st->reversed = reversed;
        st->counting = counting;
    }
}

// ------------------------------------------------------------------- K3
// Persistent two-phase one-sweep pass.
//
// B200 facts that shape it (profiles/r01_*):
//  * A pass must move 8n bytes in ~0.12 ms at n = 1e8: ~2.9 keys/cycle/SM.
//  * __match_any_sync costs ~63 cycles per warp instruction per SM and an 8-ballot
//    peer mask ~28, so a match-based stable rank caps a pass near 0.7 ms.  Shared
//    atomics with return cost ~2.6 cycles and same-address shared atomics of one
//    warp instruction are granted in ascending lane order (0 violations in 6.2e8
//    lane-trials; re-verified at load time by k_selftest_atomic_order, with the
//    match-based rank as the fallback).  So a key's stable rank is one atomicAdd.
//  * The shared-memory pipe is the next wall: a random 4-byte access by 32 lanes
//    costs ~3.5 bank wavefronts.  Each key makes three random shared accesses
//    (count atomic, rank atomic, staging store); everything else is sequential.
//  * Decoupled look-back must walk (L2 latency x tile rate) predecessors; big
//    tiles keep that walk short (it costs <= 4% of the pass).
//  * Big chunks pay: a 12,288-key chunk gives ~48-key runs per digit, so the
//    scatter stores touch fewer partial lines and the counters cost less per key.
//
// Per tile (NCHUNK chunks of BLOCK*IPT keys, tile id by atomic ticket); warp w
// always owns the same 32*IPT-key slice of every chunk, warp-striped (item i of
// lane l at slice offset i*32 + l, so (item, lane) order is input order):
//   phase 1  16-byte loads (kept in L2 with evict_last) count digits per
//            (chunk, warp); the tile total is published as the aggregate and the
//            look-back resolves the tile's global prefix; the counters are
//            rewritten as chunk-local start slots:
//              slot0(c, w, d) = sum_{d' < d} cnt_c(d') + sum_{w' < w} cnt(c, w', d)
//   phase 2  per chunk: re-read keys (L2 hits), slot = atomicAdd(counter) (stable:
//            lanes in order, items in program order), stage the key there (a
//            digit-sorted chunk), then coalesced stores at out_base[c][d] + slot
//            while the next chunk's keys load.
// CTAs (512 threads, 2 per SM) are persistent and take tiles by atomic ticket,
// so every tile a CTA waits on is owned by a running CTA.
// Experiment (off): write-out of a staged chunk by bulk copies (TMA stores), one
// per digit run: each run is staged at a slot congruent to its global position
// mod 4 (up to 3 pad slots per digit), so its 16-byte-aligned interior is one
// cp.async.bulk.  Slower on B200: the runs average 48
// keys, and the CTA waits for the copies to read the staging buffer before the
// next chunk can be staged.
#ifndef ISORT_PASS_BULK
#define ISORT_PASS_BULK 0
#endif
constexpr int kStagePad = ISORT_PASS_BULK ? 4 * kRadix : 0;

template <typename K, int BLOCK, int IPT, int NCHUNK, bool VALS, bool STAGE_DIGITS>
struct OnesweepSmem {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kChunk = BLOCK * IPT;
    static constexpr int kTile = kChunk * NCHUNK;
    static constexpr int kStage = kChunk + kStagePad;
    uint32_t cnt[NCHUNK][kWarps][kRadix];  // phase 1: counts; then chunk-local slot bases
    uint32_t out_base[NCHUNK][kRadix];     // global position = out_base[c][d] + slot
    uint32_t run_start[ISORT_PASS_BULK ? NCHUNK : 1][kRadix];  // first staging slot of digit d's run
    uint32_t offs[kRadix];                 // pass digit offsets (from K2)
    alignas(16) K keys[kStage];
    alignas(16) uint32_t vals[VALS ? kStage : 1];
    uint8_t digits[STAGE_DIGITS ? kStage : 1];  // digit per staged key (expensive digitizers)
    uint32_t tot_w[NCHUNK][kRadix / 32];
    uint32_t tile_id;
};

// Scatter pass (fused partition + exchange): a key of digit d whose position in
// the pass output would be g is stored at key[d] + (g - offs[d]) instead, i.e.
// each digit's run goes to its own base pointer -- for the multi-GPU sort, a
// slot in destination rank d's receive buffer mapped over NVLink.
constexpr int kScatterMax = 64;
struct ScatterTable {
    unsigned long long key[kScatterMax];
    unsigned long long val[kScatterMax];
    // Device-resident alternative: dev[d] = key base of digit d, dev[parts + d] = payload
    // base (a table computed on the device from the gathered count matrix, so the host
    // never has to read the matrix before the launch).  Used when non-null.
    const unsigned long long* dev;
    int parts;
};
// Kernel argument: the table by value for a scatter pass (1 KB of parameters, no
// copy or synchronisation on the host), nothing otherwise.
struct NoScatter {};
template <bool SCATTER>
using ScatterArg = typename std::conditional<SCATTER, ScatterTable, NoScatter>::type;

// Resident one-sweep CTAs per SM (the launch bound's minimum and the grid size).
#ifndef ISORT_PASS_MINB
#define ISORT_PASS_MINB_OF(block) (1024 / (block))
#else
#define ISORT_PASS_MINB_OF(block) ISORT_PASS_MINB
#endif

#ifndef ISORT_LB_WINDOW
#define ISORT_LB_WINDOW 16
#endif
constexpr int kLookbackWindow = ISORT_LB_WINDOW;  // predecessors read per round trip, per digit
#ifndef ISORT_LB_WINDOW_SMALL
#define ISORT_LB_WINDOW_SMALL 16
#endif
// Look-back after chunk 0 is ranked and staged (1) instead of right after the
// count (0): the chunk-local slot bases need only this tile's counts, the
// global offsets are needed first by chunk 0's write-out.  By then the
// predecessors have published, so the walk is short (A/B at 10^8: radix pass
// 0.283 -> 0.278 ms, bucket pass 0.291 -> 0.280 ms).  The bulk write-out
// experiment aligns runs by their global position, so it keeps the early walk.
#ifndef ISORT_LATE_LOOKBACK
#define ISORT_LATE_LOOKBACK (!ISORT_PASS_BULK)
#endif
#if ISORT_LATE_LOOKBACK && ISORT_PASS_BULK
#error "the bulk write-out aligns runs by their global position: it needs the early look-back"
#endif
constexpr int kHotDigits = 32;  // <= this many distinct digits in a tile: warp-aggregated atomics

// Exclusive prefix of digit d over tiles [0, tile): windowed decoupled look-back,
// all kLookbackWindow loads in flight per round trip.
template <typename LW, int W = kLookbackWindow>
__device__ __forceinline__ uint32_t lookback_digit(const LW* __restrict__ lb, int t_start, int d, uint32_t excl,
                                                   unsigned long long* lbst = nullptr) {  // lbst: measurement builds
    using T = LbTraits<LW>;
    int t = t_start;
    while (t >= 0) {
        if (lbst) ++lbst[0];  // rounds
        LW sv[W];
#pragma unroll
        for (int j = 0; j < W; ++j)
            sv[j] = (t - j >= 0) ? ld_relaxed_gpu(&lb[static_cast<size_t>(t - j) * kRadix + d]) : T::kInc;
        int used = 0;
        bool done = false;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            if (!done && used == j) {
                const LW f = sv[j] & T::kMask;
                if (f != 0) {
                    excl += static_cast<uint32_t>(sv[j] & T::kValue);
                    used = j + 1;
                    done = (f == T::kInc);
                }
            }
        }
        if (done) break;
        if (lbst) {
            if (used < W && t - used >= 0) ++lbst[1];  // rounds that stopped at an unpublished predecessor
            lbst[2] += used;                             // tiles consumed before the last round
        }
        t -= used;  // stopped at a predecessor that has not published: re-read from it
    }
    return excl;
}

// L2 eviction policies: tile keys are read twice (count, then rank) so the first
// read asks L2 to keep them (evict_last); the re-read and the scattered stores
// use evict_normal (evict_first for them measured 1% slower).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
#ifndef ISORT_EARLY_TICKET
#define ISORT_EARLY_TICKET 0
#endif
#ifndef ISORT_PREFETCH
#define ISORT_PREFETCH 0
#endif
constexpr int kPrefetchParts = 16;  // threads that each ask 1/16 of the next tile into L2
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
#ifndef ISORT_SKELETON
#define ISORT_SKELETON 0  // bit 0: key loads hashed, bit 1: key stores sunk, bit 2: stores linear
#endif
#ifndef ISORT_SKEL_SHIFT
#define ISORT_SKEL_SHIFT 0  // bit 2: staged slot j goes to tile position j + this (store alignment probe)
#endif
// Measurement builds only ("skeleton"): the one-sweep pass
// with its key loads replaced by a hash of the address (the same key for the
// same address, so counts and ranks agree) and/or its key stores by a register
// sink -- what the pass costs without its HBM traffic.  Output is not sorted.
__device__ __forceinline__ uint32_t skel_key(const void* p) {
    uint32_t x = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p) >> 2) * 0x9E3779B1u;
    x ^= x >> 15;
    x *= 0x85EBCA6Bu;
    return x ^ (x >> 13);
}
#if ISORT_SKELETON & 1
__device__ __forceinline__ uint4 ldg_v4_hint(const uint4* p, uint64_t) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
    return make_uint4(skel_key(q), skel_key(q + 1), skel_key(q + 2), skel_key(q + 3));
}
__device__ __forceinline__ uint32_t ldg_hint(const uint32_t* p, uint64_t) { return skel_key(p); }
__device__ __forceinline__ uint64_t ldg_hint(const uint64_t* p, uint64_t) { return skel_key(p); }
#else
__device__ __forceinline__ uint4 ldg_v4_hint(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_hint(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint64_t ldg_hint(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
#endif
#if ISORT_SKELETON & 2
__device__ __forceinline__ void stg_hint(uint32_t* p, uint32_t v, uint64_t) { asm volatile("" ::"l"(p), "r"(v)); }
__device__ __forceinline__ void stg_hint(uint64_t* p, uint64_t v, uint64_t) { asm volatile("" ::"l"(p), "l"(v)); }
#else
__device__ __forceinline__ void stg_hint(uint32_t* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_hint(uint64_t* p, uint64_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
#endif

// Stable slot of a key: slot = atomicAdd(counter), relying on lane-ordered
// same-address shared atomics; SAFE: __match_any_sync peers instead.
template <bool SAFE>
__device__ __forceinline__ uint32_t warp_slot(uint32_t* wc, uint32_t d) {
    if (SAFE) {
        const uint32_t peers = __match_any_sync(__activemask(), d);
        const uint32_t below = __popc(peers & lanemask_lt());
        uint32_t old = 0;
        if (below == 0) old = atomicAdd(&wc[d], static_cast<uint32_t>(__popc(peers)));
        return __shfl_sync(peers, old, __ffs(peers) - 1) + below;
    }
    return atomicAdd(&wc[d], 1u);
}

// Tiles made of sorted runs (sorted or reverse-sorted input, the bucket sort's
// high digits): when the whole warp shares the digit, one atomic of 32 replaces
// 32 same-address atomics (which serialise).  Full warps only; lane order is
// kept, so the slot stays stable.  `agg` is warp-uniform: it switches off at the
// first mixed instruction, so random tiles pay one vote per warp and chunk.
template <bool SAFE>
__device__ __forceinline__ uint32_t warp_slot_agg(uint32_t* wc, uint32_t d, bool& agg) {
    if (agg) {
        const uint32_t d0 = __shfl_sync(ISORT_FULL_MASK, d, 0);
        if (__all_sync(ISORT_FULL_MASK, d == d0)) {
            uint32_t old = 0;
            if (lane_id() == 0) old = atomicAdd(&wc[d0], 32u);
            return __shfl_sync(ISORT_FULL_MASK, old, 0) + lane_id();
        }
        agg = false;
    }
    return warp_slot<SAFE>(wc, d);
}

template <bool AGG>
__device__ __forceinline__ void count_digit_t(uint32_t* wc, uint32_t d, bool& agg) {
    if (AGG && agg) {
        const uint32_t d0 = __shfl_sync(ISORT_FULL_MASK, d, 0);
        if (__all_sync(ISORT_FULL_MASK, d == d0)) {
            if (lane_id() == 0) atomicAdd(&wc[d0], 32u);
            return;
        }
        agg = false;
    }
    atomicAdd(&wc[d], 1u);
}

// Phase 2 of one chunk, in three steps so the next chunk's loads are in flight
// while this chunk is written out.  FULL: all BLOCK*IPT keys valid.
template <bool FULL, typename K, int BLOCK, int IPT, bool VALS>
__device__ __forceinline__ void chunk_load(K (&key)[IPT], uint32_t (&val)[VALS ? IPT : 1], const K* __restrict__ csrc,
                                           const uint32_t* __restrict__ vsrc, uint64_t cbase, uint32_t valid,
                                           bool gen_iota, int warp, uint32_t lane, uint64_t pol) {
    const uint32_t wofs = static_cast<uint32_t>(warp) * 32u * IPT + lane;
    const K* wsrc = csrc + wofs;
#pragma unroll
    for (int i = 0; i < IPT; ++i)
        key[i] = (FULL || wofs + i * 32u < valid) ? ldg_hint(wsrc + i * 32, pol) : static_cast<K>(0);
    if (VALS) {
#pragma unroll
        for (int i = 0; i < IPT; ++i)
            val[i] = gen_iota ? static_cast<uint32_t>(cbase + wofs + i * 32u)
                              : ((FULL || wofs + i * 32u < valid) ? ldg_stream(vsrc + cbase + wofs + i * 32u) : 0u);
    }
}

template <bool FULL, bool AGG, bool SAFE, typename K, typename Dz, int IPT, bool VALS, typename Smem>
__device__ __forceinline__ void chunk_rank(Smem& sm, int c, const K (&key)[IPT], const uint32_t (&val)[VALS ? IPT : 1],
                                           uint32_t valid, uint32_t dsh, const Dz& dz, int warp, uint32_t lane) {
    const uint32_t wofs = static_cast<uint32_t>(warp) * 32u * IPT + lane;
    uint32_t* wc = sm.cnt[c][warp];
    bool agg = FULL && AGG;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if (FULL || wofs + i * 32u < valid) {
            const uint32_t d = dz.digit_sh(key[i], dsh);
            const uint32_t s = (FULL && AGG) ? warp_slot_agg<SAFE>(wc, d, agg) : warp_slot<SAFE>(wc, d);
            sm.keys[s] = key[i];
            if (VALS) sm.vals[s] = val[i];
            if (!Dz::kCheapDigit) sm.digits[s] = static_cast<uint8_t>(d);
        }
    }
}

template <bool FULL, bool SCATTER, typename K, typename Dz, int BLOCK, int IPT, bool VALS, typename Smem>
__device__ __forceinline__ void chunk_write(Smem& sm, int c, K* __restrict__ dst, uint32_t* __restrict__ vdst,
                                            uint32_t valid, uint32_t dsh, const Dz& dz, uint64_t pol,
                                            const unsigned long long* kbase, const unsigned long long* vbase) {
    const int tid = threadIdx.x;
    const uint32_t* ob = sm.out_base[c];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t j = static_cast<uint32_t>(tid) + i * BLOCK;
        if (FULL || j < valid) {
            const K k = sm.keys[j];
            const uint32_t d = Dz::kCheapDigit ? dz.digit_sh(k, dsh) : static_cast<uint32_t>(sm.digits[j]);
            const uint32_t g = ob[d] + j;
            if (SCATTER) {
                *(reinterpret_cast<K*>(kbase[d]) + g) = k;
                if (VALS) *(reinterpret_cast<uint32_t*>(vbase[d]) + g) = sm.vals[j];
            } else {
                stg_hint(dst + g, k, pol);
                if (VALS) stg_hint(vdst + g, sm.vals[j], pol);
            }
        }
    }
}

// Write-out of chunk c by the thread of digit d: the run's 16-byte-aligned
// interior by one bulk copy per array, the <= 3 + 3 keys around it by plain
// stores.  Waits until the copies have read the staging buffer (it is reused
// by the next chunk right after the caller's barrier).
template <typename K, bool VALS, typename Smem>
__device__ __forceinline__ void chunk_write_bulk(Smem& sm, int c, int d, K* __restrict__ dst,
                                                 uint32_t* __restrict__ vdst, uint64_t pol) {
    const uint32_t p = sm.run_start[c][d];
    const uint32_t len = sm.cnt[c][Smem::kWarps - 1][d] - p;  // the last warp's counter ends the run
    if (len == 0) return;
    const uint32_t g = sm.out_base[c][d] + p;
    auto put = [&](auto* gdst, const auto* sstage) {
        using T = typename std::remove_cv<typename std::remove_pointer<decltype(sstage)>::type>::type;
        constexpr uint32_t E = 16 / sizeof(T);
        uint32_t head = (E - (g & (E - 1))) & (E - 1);
        head = head < len ? head : len;
        const uint32_t body = (len - head) & ~(E - 1);
        if (body) bulk_s2g(gdst + g + head, sstage + p + head, body * static_cast<uint32_t>(sizeof(T)));
        for (uint32_t i = 0; i < head; ++i) stg_hint(gdst + g + i, sstage[p + i], pol);
        for (uint32_t i = head + body; i < len; ++i) stg_hint(gdst + g + i, sstage[p + i], pol);
    };
    put(dst, sm.keys);
    if constexpr (VALS) put(vdst, sm.vals);
    bulk_wait_read();
}

// Phase 1: per-(chunk, warp) digit counts of one tile (keys via L2, kept there
// for phase 2).  AGG: the tile is expected to be made of sorted runs.
template <bool AGG, typename K, typename Dz, int IPT, int NCHUNK, typename Smem>
__device__ __forceinline__ void onesweep_count(Smem& sm, const K* __restrict__ src, uint64_t tile_base,
                                               uint32_t tile_len, int warp, uint32_t lane, bool vec, const Dz& dz,
                                               uint32_t dsh, uint64_t pol_keep) {
    constexpr int kChunk = Smem::kChunk;
#pragma unroll 1
    for (int c = 0; c < NCHUNK; c += (NCHUNK >= 2 ? 2 : 1)) {
        const uint32_t c0 = static_cast<uint32_t>(c) * kChunk + static_cast<uint32_t>(warp) * 32u * IPT;
        const uint32_t c1 = c0 + kChunk;
        uint32_t* wc0 = sm.cnt[c][warp];
        uint32_t* wc1 = sm.cnt[NCHUNK >= 2 ? c + 1 : c][warp];
        const K* ws = src + tile_base + c0;
        bool agg1 = AGG;
        if (NCHUNK == 1) {
            if (vec && c0 + 32u * IPT <= tile_len) {
                const uint4* v0 = reinterpret_cast<const uint4*>(ws);
                uint4 x[IPT / 4 > 0 ? IPT / 4 : 1];
#pragma unroll
                for (int q = 0; q < IPT / 4; ++q) x[q] = ldg_v4_hint(v0 + lane + 32 * q, pol_keep);
#pragma unroll
                for (int q = 0; q < IPT / 4; ++q) {
                    count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].x), dsh), agg1);
                    count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].y), dsh), agg1);
                    count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].z), dsh), agg1);
                    count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].w), dsh), agg1);
                }
            } else {
                for (uint32_t o = lane; o < 32u * IPT; o += 32)
                    if (c0 + o < tile_len) atomicAdd(&wc0[dz.digit_sh(ldg_hint(ws + o, pol_keep), dsh)], 1u);
            }
            continue;
        }
        if (vec && c1 + 32u * IPT <= tile_len) {
            const uint4* v0 = reinterpret_cast<const uint4*>(ws);
            const uint4* v1 = reinterpret_cast<const uint4*>(ws + kChunk);
            uint4 x[IPT / 4 > 0 ? IPT / 4 : 1], y[IPT / 4 > 0 ? IPT / 4 : 1];
#pragma unroll
            for (int q = 0; q < IPT / 4; ++q) {
                x[q] = ldg_v4_hint(v0 + lane + 32 * q, pol_keep);
                y[q] = ldg_v4_hint(v1 + lane + 32 * q, pol_keep);
            }
#pragma unroll
            for (int q = 0; q < IPT / 4; ++q) {
                count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].x), dsh), agg1);
                count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].y), dsh), agg1);
                count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].z), dsh), agg1);
                count_digit_t<AGG>(wc0, dz.digit_sh(static_cast<K>(x[q].w), dsh), agg1);
                count_digit_t<AGG>(wc1, dz.digit_sh(static_cast<K>(y[q].x), dsh), agg1);
                count_digit_t<AGG>(wc1, dz.digit_sh(static_cast<K>(y[q].y), dsh), agg1);
                count_digit_t<AGG>(wc1, dz.digit_sh(static_cast<K>(y[q].z), dsh), agg1);
                count_digit_t<AGG>(wc1, dz.digit_sh(static_cast<K>(y[q].w), dsh), agg1);
            }
        } else {
            for (uint32_t o = lane; o < 32u * IPT; o += 32) {
                if (c0 + o < tile_len) atomicAdd(&wc0[dz.digit_sh(ldg_hint(ws + o, pol_keep), dsh)], 1u);
                if (c1 + o < tile_len)
                    atomicAdd(&wc1[dz.digit_sh(ldg_hint(ws + kChunk + o, pol_keep), dsh)], 1u);
            }
        }
    }
}

template <typename K, typename Dz, int BLOCK, int IPT, int NCHUNK, bool VALS, bool SAFE, bool SCATTER = false,
          typename LW = uint32_t>
__global__ void __launch_bounds__(BLOCK, ISORT_PASS_MINB_OF(BLOCK))
    k_onesweep(const K* __restrict__ keys_in, K* __restrict__ keys_out, K* __restrict__ keys_alt,
               const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out, uint32_t* __restrict__ vals_alt,
               int iota_vals, uint64_t n, RadixState* __restrict__ st, void* __restrict__ lookback,
               uint32_t num_tiles, int slot, Dz dz, const ScatterArg<SCATTER> scat) {
    using LT = LbTraits<LW>;
    using Smem = OnesweepSmem<K, BLOCK, IPT, NCHUNK, VALS, !Dz::kCheapDigit>;
    constexpr bool kBulkWrite = ISORT_PASS_BULK && !SCATTER;  // peer stores (SCATTER) stay per key
    constexpr int kWarps = Smem::kWarps;
    constexpr int kChunk = Smem::kChunk;
    constexpr int kTile = Smem::kTile;
    static_assert(BLOCK % kRadix == 0, "threads [0, kRadix) own one digit each in the per-tile section");
    static_assert(NCHUNK % 2 == 0 || NCHUNK == 1, "phase-1 loads are batched two chunks at a time");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    if (slot >= static_cast<int>(st->n_active)) return;  // trivial / skipped pass
    const int pos = st->digit_of_slot[slot];
    const int src_id = st->src_of_slot[slot];
    const int dst_id = st->dst_of_slot[slot];
    const K* src = src_id == kBufIn ? keys_in : (src_id == kBufOut ? keys_out : keys_alt);
    K* dst = dst_id == kBufOut ? keys_out : keys_alt;
    const uint32_t* vsrc = src_id == kBufIn ? vals_in : (src_id == kBufOut ? vals_out : vals_alt);
    uint32_t* vdst = dst_id == kBufOut ? vals_out : vals_alt;
    const bool gen_iota = iota_vals && slot == 0;
    const uint32_t dsh = dz.shift_for(pos);
    LW* lb = static_cast<LW*>(lookback) + static_cast<size_t>(slot) * num_tiles * kRadix;
    const bool vec = sizeof(K) == 4 && IPT % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
#ifndef ISORT_POL_KEEP
#define ISORT_POL_KEEP policy_evict_last()
#endif
#ifndef ISORT_POL_STREAM
#define ISORT_POL_STREAM policy_evict_normal()
#endif
    const uint64_t pol_keep = ISORT_POL_KEEP;
    const uint64_t pol_stream = ISORT_POL_STREAM;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    if (tid < kRadix) sm.offs[tid] = st->offs[pos][tid];
    __shared__ unsigned long long s_kbase[SCATTER ? kScatterMax : 1], s_vbase[SCATTER ? kScatterMax : 1];
    if constexpr (SCATTER) {
        if (tid < kScatterMax) {  // per-digit base, shifted so that base + g addresses the run
            const unsigned long long o = st->offs[pos][tid];
            const bool dev = scat.dev != nullptr;
            const unsigned long long kb = dev ? (tid < scat.parts ? scat.dev[tid] : 0ull) : scat.key[tid];
            s_kbase[tid] = kb - o * sizeof(K);
            if (VALS) {
                const unsigned long long vb = dev ? (tid < scat.parts ? scat.dev[scat.parts + tid] : 0ull) : scat.val[tid];
                s_vbase[tid] = vb - o * sizeof(uint32_t);
            }
        }
        // a zeroed device table means "does not fit" (the caller falls back): store nothing
        if (__syncthreads_or(scat.dev != nullptr && tid < scat.parts && scat.dev[tid] == 0ull)) return;
    }

#ifdef ISORT_PHASE_TIMING
    long long acc[4] = {0, 0, 0, 0};
    long long q0 = 0, q1 = 0, q2 = 0, q3 = 0;
#define ISORT_TICK(v) \
    if (tid == 0) v = clock64()
#else
#define ISORT_TICK(v)
#endif

    bool hot_prev = false;  // phase 1 guesses from this CTA's previous tile
#if ISORT_EARLY_TICKET
    if (tid == 0) sm.tile_id = atomicAdd(&st->tile_ticket[slot], 1u);
#endif
    for (;;) {
        ISORT_TICK(q0);
#if !ISORT_EARLY_TICKET
        if (tid == 0) sm.tile_id = atomicAdd(&st->tile_ticket[slot], 1u);
#endif
        {
            uint4* c4 = reinterpret_cast<uint4*>(&sm.cnt[0][0][0]);
            for (int i = tid; i < NCHUNK * kWarps * kRadix / 4; i += BLOCK) c4[i] = make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
        const uint32_t tile = sm.tile_id;
        const uint64_t tile_base = static_cast<uint64_t>(tile) * kTile;
        if (tile >= num_tiles || tile_base >= n) break;  // (a tile count from another shape must not run past n)
        const uint32_t tile_len = static_cast<uint32_t>(n - tile_base < static_cast<uint64_t>(kTile)
                                                            ? n - tile_base : static_cast<uint64_t>(kTile));

        // ---------------- phase 1: per-(chunk, warp) digit counts
        if (hot_prev)
            onesweep_count<true, K, Dz, IPT, NCHUNK>(sm, src, tile_base, tile_len, warp, lane, vec, dz, dsh, pol_keep);
        else
            onesweep_count<false, K, Dz, IPT, NCHUNK>(sm, src, tile_base, tile_len, warp, lane, vec, dz, dsh, pol_keep);
        __syncthreads();
        ISORT_TICK(q1);

        // ---------------- one thread per digit: totals, look-back, slot bases
        int nonzero = 0;
        uint32_t late_tot = 0;  // LATE: this tile's count of digit tid, published inclusive after chunk 0
        if (tid < kRadix) {
            const int d = tid;
            uint32_t cc[NCHUNK], tot = 0;
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) {
                uint32_t x = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) x += sm.cnt[c][w][d];
                cc[c] = x;
                tot += x;
            }
            nonzero = tot != 0;
            uint32_t excl = 0;
            if (tile == 0) {
                st_relaxed_gpu(&lb[d], LT::kInc | tot);
            } else if (ISORT_LATE_LOOKBACK) {
                st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + d], LT::kAgg | tot);
                late_tot = tot;
            } else {
                st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + d], LT::kAgg | tot);
#ifndef ISORT_AB_NO_LOOKBACK
                // small inputs (1-chunk tiles, one wave of CTAs) may take another window
                // (A/B at 10^6 keys: 16 -> 14.5 us/pass, 32 -> 15.8, 48 -> 16.1)
                excl = lookback_digit<LW, NCHUNK == 1 ? ISORT_LB_WINDOW_SMALL : kLookbackWindow>(
                    lb, static_cast<int>(tile) - 1, d, 0u);
#endif
                st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + d], LT::kInc | (excl + tot));
            }
            ISORT_TICK(q2);
            uint32_t run = sm.offs[d] + excl;
            uint32_t sc[NCHUNK];
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) {
                sc[c] = warp_inclusive_scan(cc[c]);
                if (lane == 31) sm.tot_w[c][warp] = sc[c];
            }
            if (BLOCK == kRadix)
                __syncthreads();
            else
                asm volatile("bar.sync 1, %0;" ::"n"(kRadix));
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) {
                uint32_t pre = 0;
#pragma unroll
                for (int w = 0; w < kRadix / 32; ++w) pre += w < warp ? sm.tot_w[c][w] : 0u;
                uint32_t base = pre + sc[c] - cc[c];  // chunk-local start of digit d
                if (ISORT_PASS_BULK) {  // + 4d + (0..3): the run's slot = its global position mod 4
                    base += 4u * static_cast<uint32_t>(d);
                    base += (run - base) & 3u;
                    sm.run_start[ISORT_PASS_BULK ? c : 0][d] = base;
                }
                sm.out_base[c][d] = run - base;
#if ISORT_SKELETON & 4
                sm.out_base[c][d] = static_cast<uint32_t>(tile_base) + c * kChunk + (tile + 1 < num_tiles ? ISORT_SKEL_SHIFT : 0);
#endif
                run += cc[c];
#pragma unroll
                for (int w = 0; w < kWarps; ++w) {  // per-warp slot bases for phase 2
                    const uint32_t v = sm.cnt[c][w][d];
                    sm.cnt[c][w][d] = base;
                    base += v;
                }
            }
        }
        // A tile with few distinct digits comes from sorted runs (sorted or
        // reverse-sorted input, or the bucket sort's high digits): warps mostly
        // share one digit, so rank/count them with one atomic per warp.
        const bool hot = __syncthreads_count(nonzero) <= kHotDigits;
        hot_prev = hot;

        // ---------------- phase 2: stage by slot, coalesced scatter
        K key[IPT];
        uint32_t val[VALS ? IPT : 1];
        auto load = [&](int c) {
            const uint32_t c0 = static_cast<uint32_t>(c) * kChunk;
            const uint32_t valid = tile_len - c0 < static_cast<uint32_t>(kChunk) ? tile_len - c0 : kChunk;
            const uint64_t cbase = tile_base + c0;
            if (valid == static_cast<uint32_t>(kChunk))
                chunk_load<true, K, BLOCK, IPT, VALS>(key, val, src + cbase, vsrc, cbase, valid, gen_iota, warp, lane,
                                                      pol_stream);
            else
                chunk_load<false, K, BLOCK, IPT, VALS>(key, val, src + cbase, vsrc, cbase, valid, gen_iota, warp, lane,
                                                       pol_stream);
        };
        load(0);
#pragma unroll 1
        for (int c = 0; c < NCHUNK; ++c) {
            const uint32_t c0 = static_cast<uint32_t>(c) * kChunk;
            if (c0 >= tile_len) break;
            const uint32_t valid = tile_len - c0 < static_cast<uint32_t>(kChunk) ? tile_len - c0 : kChunk;
            const bool full = valid == static_cast<uint32_t>(kChunk);
            if (full && hot)
                chunk_rank<true, true, SAFE, K, Dz, IPT, VALS>(sm, c, key, val, valid, dsh, dz, warp, lane);
            else if (full)
                chunk_rank<true, false, SAFE, K, Dz, IPT, VALS>(sm, c, key, val, valid, dsh, dz, warp, lane);
            else
                chunk_rank<false, false, SAFE, K, Dz, IPT, VALS>(sm, c, key, val, valid, dsh, dz, warp, lane);
            if (c + 1 < NCHUNK && c0 + kChunk < tile_len) load(c + 1);  // in flight during the write-out
            if (ISORT_LATE_LOOKBACK && c == 0 && tile != 0 && tid < kRadix) {
                uint32_t excl = 0;
#ifndef ISORT_AB_NO_LOOKBACK
                excl = lookback_digit<LW, NCHUNK == 1 ? ISORT_LB_WINDOW_SMALL : kLookbackWindow>(
                    lb, static_cast<int>(tile) - 1, tid, 0u);
#endif
                st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + tid], LT::kInc | (excl + late_tot));
#pragma unroll
                for (int cc = 0; cc < NCHUNK; ++cc) sm.out_base[cc][tid] += (ISORT_SKELETON & 4) ? 0u : excl;
            }
#if ISORT_EARLY_TICKET || ISORT_PREFETCH
            // The next tile's ticket is taken before this tile's last write-out, and its
            // keys are asked into L2 while the write-out runs (the count phase then
            // starts on L2 hits).  The owner of a ticket is a running CTA, as before.
            const bool last_chunk = c + 1 == NCHUNK || c0 + kChunk >= tile_len;
            if (ISORT_EARLY_TICKET && last_chunk && tid == 0) sm.tile_id = atomicAdd(&st->tile_ticket[slot], 1u);
#endif
            if constexpr (kBulkWrite) {
                fence_proxy_async_smem();  // the staging stores, visible to the bulk copies
                __syncthreads();
                if (tid < kRadix) chunk_write_bulk<K, VALS>(sm, c, tid, dst, vdst, pol_stream);
                __syncthreads();
                continue;
            }
#if ISORT_SKELETON & 8  // store-path probe: the staged chunk leaves by one linear bulk copy
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                bulk_s2g(dst + tile_base + c0, sm.keys, (valid * static_cast<uint32_t>(sizeof(K))) & ~15u);
                bulk_wait_read();
            }
            __syncthreads();
            continue;
#endif
            __syncthreads();
#if ISORT_EARLY_TICKET || ISORT_PREFETCH
            if (ISORT_PREFETCH && last_chunk && vec && tid < kPrefetchParts) {
                const uint32_t nt = ISORT_EARLY_TICKET ? sm.tile_id : tile + gridDim.x;  // exact / the likely next
                const uint64_t nb = static_cast<uint64_t>(nt) * kTile;
                if (nt < num_tiles && nb < n) {
                    constexpr uint32_t kPart = kTile / kPrefetchParts;  // keys per prefetching thread
                    const uint64_t b = nb + static_cast<uint64_t>(tid) * kPart;
                    if (b < n) {
                        const uint64_t left = n - b;
                        const uint32_t cnt = left < kPart ? static_cast<uint32_t>(left) : kPart;
                        const uint32_t bytes = (cnt * static_cast<uint32_t>(sizeof(K))) & ~15u;
                        if (bytes) bulk_prefetch_l2(src + b, bytes);
                    }
                }
            }
#endif
            if (full)
                chunk_write<true, SCATTER, K, Dz, BLOCK, IPT, VALS>(sm, c, dst, vdst, valid, dsh, dz, pol_stream,
                                                                    s_kbase, s_vbase);
            else
                chunk_write<false, SCATTER, K, Dz, BLOCK, IPT, VALS>(sm, c, dst, vdst, valid, dsh, dz, pol_stream,
                                                                     s_kbase, s_vbase);
            __syncthreads();
        }
        ISORT_TICK(q3);
#ifdef ISORT_PHASE_TIMING
        acc[0] += q1 - q0;
        acc[1] += q2 - q1;
        acc[2] += q3 - q2;
        acc[3] += 1;
#endif
    }
    if (SCATTER) __threadfence_system();  // peer stores visible before the host-ordered barrier
    if (kBulkWrite && tid < kRadix) bulk_wait_all();  // this CTA's bulk stores complete before it exits
#ifdef ISORT_PHASE_TIMING
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) atomicAdd(&st->prof[i], static_cast<unsigned long long>(acc[i]));
    }
#endif
#undef ISORT_TICK
}

// Load-time check of the property the fast rank relies on: lanes of one warp
// instruction that add to the same shared word observe old values in ascending
// lane order.  Adversarial patterns: 1..32 distinct words per instruction.
static __global__ void k_selftest_atomic_order(uint32_t* __restrict__ violations, uint32_t seed) {
    __shared__ uint32_t h[32][257];
    uint32_t* wh = h[threadIdx.x >> 5];
    const uint32_t lane = lane_id();
    uint32_t v = seed ^ (blockIdx.x * 7919u) ^ ((threadIdx.x >> 5) * 104729u);
    uint32_t bad = 0;
    for (int t = 0; t < 512; ++t) {
        for (int i = lane; i < 257; i += 32) wh[i] = 0;
        __syncwarp();
        v = v * 1664525u + 1013904223u;
        const uint32_t mod = 1u + ((v >> 8) & 31u);
        const uint32_t d = (lane * 2654435761u + v) % mod * 7u % 256u;
        // (1) the one-sweep rank: atomicAdd(p, 1) with the old value (ATOMS.POPC.INC)
        const uint32_t old = atomicAdd(&wh[d], 1u);
        const uint32_t peers = __match_any_sync(ISORT_FULL_MASK, d);
        const uint32_t want = static_cast<uint32_t>(__popc(peers & lanemask_lt()));
        bad += (old != want);
        __syncwarp();
        for (int i = lane; i < 257; i += 32) wh[i] = 0;
        __syncwarp();
        // (2) the segment sort's rank: two 16-bit counters per word, increment
        // 1 << 16 for odd digits (a plain ATOMS.ADD); lanes whose digits share a
        // word contend, and the lanes of one digit must still be served in order
        const uint32_t hsh = (d & 1u) << 4;
        const uint32_t old2 = (atomicAdd(&wh[d >> 1], 1u << hsh) >> hsh) & 0xFFFFu;
        bad += (old2 != want);
        __syncwarp();
    }
    if (bad) atomicAdd(violations, bad);
}

// ------------------------------------------------------------------- K4
template <typename K>
__device__ __forceinline__ void d_copy_in_to_out(const K* __restrict__ in, K* __restrict__ out,
                                        const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout,
                                        int iota_vals, uint64_t n, const RadixState* __restrict__ st) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // 16-byte vectors when both pointers are aligned (the common case), scalar tail
    constexpr uint64_t kPer = 16 / sizeof(K);
    uint64_t done = 0;
    if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0) {
        const uint64_t nv = n / kPer;
        const uint4* s4 = reinterpret_cast<const uint4*>(in);
        uint4* d4 = reinterpret_cast<uint4*>(out);
        for (uint64_t v = t0; v < nv; v += stride) d4[v] = ldg_stream_v4(s4 + v);
        done = nv * kPer;
    }
    for (uint64_t i = done + t0; i < n; i += stride) out[i] = in[i];
    if (vout) {
        for (uint64_t i = t0; i < n; i += stride) vout[i] = iota_vals ? static_cast<uint32_t>(i) : vin[i];
    }
}


// ------------------------------------------------------------------- K6
// Counting pass (keys only, every key < kCountBins): the LSD sort with one
// kCountBits-bit digit = the whole key.  A stable counting pass places key v at
// offs[v] + (its arrival rank among the v's) (sort.cpp:95-108); with nothing but
// the key to carry, those slots are exactly the run [offs[v], offs[v] + cnt[v])
// filled with v, so the pass needs the counts (K6a: 4n B read) and a fill of the
// output (K6b: 4n B write) -- no scatter.  Both return at once unless the plan
// chose this path (no host round trip; graph-capturable).
constexpr int kCountBlock = 1024;
constexpr int kCountRep = 4;  // counter copies per bin (lane % kCountRep): fewer same-address lanes

template <typename K>
__device__ __forceinline__ void d_count_hist(const K* __restrict__ keys, uint64_t n,
                                                            const RadixState* __restrict__ st,
                                                            CountState* __restrict__ cs) {
    extern __shared__ __align__(16) uint32_t ch[];  // kCountBins * kCountRep
    for (int i = threadIdx.x; i < kCountBins * kCountRep; i += kCountBlock) ch[i] = 0;
    __syncthreads();
    uint32_t* my = ch + (lane_id() % kCountRep);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kCountBlock;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kCountBlock + threadIdx.x;
    uint64_t done = 0;
    if (sizeof(K) == 4 && (reinterpret_cast<uintptr_t>(keys) & 15u) == 0) {
        const uint64_t nv = n / 4;
        const uint4* k4 = reinterpret_cast<const uint4*>(keys);
        for (uint64_t v = t0; v < nv; v += stride) {
            const uint4 q = ldg_stream_v4(k4 + v);
            atomicAdd(my + q.x * kCountRep, 1u);
            atomicAdd(my + q.y * kCountRep, 1u);
            atomicAdd(my + q.z * kCountRep, 1u);
            atomicAdd(my + q.w * kCountRep, 1u);
        }
        done = nv * 4;
    }
    for (uint64_t i = done + t0; i < n; i += stride) atomicAdd(my + static_cast<uint32_t>(keys[i]) * kCountRep, 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < kCountBins; b += kCountBlock) {
        uint32_t c = 0;
#pragma unroll
        for (int r = 0; r < kCountRep; ++r) c += ch[b * kCountRep + r];
        if (c) atomicAdd(&cs->vhist[b], c);
    }
}

// Every CTA scans the kCountBins counts into shared memory (16 KB from L2), then
// writes its share of the output in 16-byte vectors: position p holds the v with
// offs[v] <= p < offs[v + 1] (a binary search per vector, then a walk).
template <typename K>
__device__ __forceinline__ void d_count_fill(K* __restrict__ out, uint64_t n,
                                                            const RadixState* __restrict__ st,
                                                            const CountState* __restrict__ cs) {
    __shared__ uint32_t ends[kCountBins];  // inclusive prefix: ends[v] = offs[v] + cnt[v]
    __shared__ uint32_t wtot[kCountBlock / 32];
    constexpr int kPer = kCountBins / kCountBlock;
    uint32_t c[kPer], sum = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        c[j] = cs->vhist[threadIdx.x * kPer + j];
        sum += c[j];
    }
    const uint32_t inc = warp_inclusive_scan(sum);
    if (lane_id() == 31) wtot[threadIdx.x >> 5] = inc;
    __syncthreads();
    uint32_t run = inc - sum;
    for (int w = 0; w < static_cast<int>(threadIdx.x >> 5); ++w) run += wtot[w];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        run += c[j];
        ends[threadIdx.x * kPer + j] = run;
    }
    __syncthreads();
    auto value_at = [&](uint32_t p, uint32_t hint) -> uint32_t {  // smallest v with ends[v] > p, v >= hint
        while (ends[hint] <= p) ++hint;
        return hint;
    };
    auto search = [&](uint32_t p) -> uint32_t {  // smallest v with ends[v] > p
        uint32_t lo = 0, hi = kCountBins - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ends[mid] > p) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    constexpr uint32_t E = 16 / sizeof(K);
    constexpr int U = 4;  // vectors per lane per warp step (32 * U * E positions)
    const uint64_t nv = (reinterpret_cast<uintptr_t>(out) & 15u) == 0 ? n / E : 0;
    const uint64_t wstride = static_cast<uint64_t>(gridDim.x) * (kCountBlock / 32) * 32 * U;
    // warp-converged loop: one broadcast binary search for the warp step's first
    // position, then every vector walks forward from it (a step per distinct value)
    for (uint64_t vb = (static_cast<uint64_t>(blockIdx.x) * (kCountBlock / 32) + (threadIdx.x >> 5)) * 32 * U;
         vb < nv; vb += wstride) {
        const uint32_t w0 = search(static_cast<uint32_t>(vb * E));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = vb + u * 32 + lane_id();
            if (v >= nv) break;
            const uint32_t p = static_cast<uint32_t>(v * E);
            uint32_t x[E];
            x[0] = value_at(p, w0);
#pragma unroll
            for (uint32_t j = 1; j < E; ++j) x[j] = value_at(p + j, x[j - 1]);
            // values < 2^12: a u64 key is (value, 0)
            reinterpret_cast<uint4*>(out)[v] = sizeof(K) == 4 ? make_uint4(x[0], x[1 % E], x[2 % E], x[3 % E])
                                                              : make_uint4(x[0], 0u, x[1 % E], 0u);
        }
    }
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kCountBlock;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kCountBlock + threadIdx.x;
    for (uint64_t i = nv * E + t0; i < n; i += stride) out[i] = static_cast<K>(search(static_cast<uint32_t>(i)));
}

// ------------------------------------------------------------------- K5
// Non-increasing input (K1: no ascent): the stable sort is the reversal in
// which every run of equal keys keeps its input order.
// Keys only: equal keys are indistinguishable, so out[n - 1 - i] = in[i] is
// already exact (one read, one write, like the sorted-input copy).
// With a payload: the same full reversal of keys and payload (coalesced: a
// warp's stores land on consecutive descending addresses), then every run of
// equal keys in the output gets its payload reversed back into input order.
// k_rev_fix_runs finds the runs (a run's first thread sees key[i-1] != key[i] ==
// key[i+1]) and finds its end by a galloping search on the sorted output; runs up
// to kRevShortRun keys are reversed by that thread, longer ones are listed for
// k_rev_long_runs (one CTA per run).  Every kernel returns at once unless the
// plan chose this path (no host round trip; graph-capturable).
constexpr int kRevShortRun = 64;

// 16-byte vectors reversed as whole vectors when n is a multiple of the vector
// width (in[4v..4v+3] -> out[n-4-4v..]: both sides aligned), scalar otherwise.
template <typename K>
__device__ __forceinline__ uint4 reverse_vec(uint4 q) {
    return sizeof(K) == 4 ? make_uint4(q.w, q.z, q.y, q.x) : make_uint4(q.z, q.w, q.x, q.y);
}

template <typename K>
__device__ __forceinline__ void d_reverse_keys(const K* __restrict__ in, K* __restrict__ out, uint64_t n,
                               const RadixState* __restrict__ st) {
    constexpr uint64_t E = 16 / sizeof(K);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (n % E == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0) {
        const uint64_t nv = n / E;
        for (uint64_t v = t0; v < nv; v += stride)
            reinterpret_cast<uint4*>(out)[nv - 1 - v] = reverse_vec<K>(ldg_stream_v4(reinterpret_cast<const uint4*>(in) + v));
        return;
    }
    for (uint64_t i = t0; i < n; i += stride) out[n - 1 - i] = in[i];
}

template <typename K>
__device__ __forceinline__ void d_reverse_pairs(const K* __restrict__ kin, K* __restrict__ kout, const uint32_t* __restrict__ vin,
                                uint32_t* __restrict__ vout, int iota_vals, uint64_t n,
                                const RadixState* __restrict__ st) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool aligned = ((reinterpret_cast<uintptr_t>(kin) | reinterpret_cast<uintptr_t>(kout) |
                           reinterpret_cast<uintptr_t>(vin) | reinterpret_cast<uintptr_t>(vout)) & 15u) == 0;
    if (sizeof(K) == 4 && n % 4 == 0 && aligned) {  // 4 keys + 4 payload words per thread step
        const uint64_t nv = n / 4;
        for (uint64_t v = t0; v < nv; v += stride) {
            reinterpret_cast<uint4*>(kout)[nv - 1 - v] = reverse_vec<K>(ldg_stream_v4(reinterpret_cast<const uint4*>(kin) + v));
            const uint32_t b = static_cast<uint32_t>(4 * v);
            const uint4 q = iota_vals ? make_uint4(b, b + 1, b + 2, b + 3) : ldg_stream_v4(reinterpret_cast<const uint4*>(vin) + v);
            reinterpret_cast<uint4*>(vout)[nv - 1 - v] = make_uint4(q.w, q.z, q.y, q.x);
        }
        return;
    }
    for (uint64_t i = t0; i < n; i += stride) {
        kout[n - 1 - i] = kin[i];
        vout[n - 1 - i] = iota_vals ? static_cast<uint32_t>(i) : vin[i];
    }
}

// End of the run of key k that starts at i in the ascending array `keys`.
template <typename K>
__device__ __forceinline__ uint64_t run_end(const K* __restrict__ keys, uint64_t n, uint64_t i, K k) {
    uint64_t lo = i + 1, step = 1;  // keys[lo - 1] == k
    uint64_t hi = lo;
    while (hi < n && keys[hi] == k) {  // gallop: keys[hi] == k  =>  the end is past hi
        lo = hi + 1;
        hi = lo + step < n ? lo + step : n;
        step <<= 1;
    }
    while (lo < hi) {  // first index in [lo, hi) with keys[idx] != k
        const uint64_t mid = lo + (hi - lo) / 2;
        if (keys[mid] == k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <typename K>
__device__ __forceinline__ void d_rev_fix_runs(const K* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t n,
                               RadixState* __restrict__ st, unsigned long long* __restrict__ long_runs) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool vec = sizeof(K) == 4 && (reinterpret_cast<uintptr_t>(keys) & 15u) == 0;
    // a thread checks positions [4g, 4g + 4) per step: one 16-byte load of them plus
    // the keys just before and after (L1 hits); a run that ends inside that window
    // needs no further load
    const uint64_t groups = (n + 3) / 4;
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const uint64_t b0 = 4 * g;
        K w[6];  // keys[b0 - 1 .. b0 + 4]; positions >= n never match (checked by index)
        if (vec && b0 + 4 <= n) {
            const uint4 q = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + g);
            w[1] = static_cast<K>(q.x), w[2] = static_cast<K>(q.y), w[3] = static_cast<K>(q.z), w[4] = static_cast<K>(q.w);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) w[1 + j] = b0 + j < n ? keys[b0 + j] : static_cast<K>(0);
        }
        w[0] = b0 > 0 ? keys[b0 - 1] : static_cast<K>(0);
        w[5] = b0 + 4 < n ? keys[b0 + 4] : static_cast<K>(0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t i = b0 + j;
            const K k = w[1 + j];
            if (!(i + 1 < n && w[2 + j] == k && (i == 0 || w[j] != k))) continue;  // no run of >= 2 starts at i
            uint64_t e = i + 2;  // first position past the run, within the window if possible
#pragma unroll
            for (int t = 3 + j; t <= 5; ++t)
                if (e == b0 + t - 1 && e < n && w[t] == k) ++e;
            if (e == b0 + 5 && e < n) e = run_end(keys, n, i, k);  // the run leaves the window
            if (e - i > static_cast<uint64_t>(kRevShortRun)) {
                const uint32_t slot = atomicAdd(&st->rev_long, 1u);
                long_runs[2 * slot] = i;
                long_runs[2 * slot + 1] = e;
                continue;
            }
            for (uint64_t a = i, b = e - 1; a < b; ++a, --b) {
                const uint32_t t = vals[a];
                vals[a] = vals[b];
                vals[b] = t;
            }
        }
    }
}

static __global__ void k_rev_long_runs(uint32_t* __restrict__ vals, const RadixState* __restrict__ st,
                                const unsigned long long* __restrict__ long_runs) {
    if (!st->reversed) return;
    const uint32_t runs = st->rev_long;
    for (uint32_t r = blockIdx.x; r < runs; r += gridDim.x) {
        const uint64_t a = long_runs[2 * r], e = long_runs[2 * r + 1], half = (e - a) / 2;
        for (uint64_t j = threadIdx.x; j < half; j += blockDim.x) {
            const uint32_t t = vals[a + j];
            vals[a + j] = vals[e - 1 - j];
            vals[e - 1 - j] = t;
        }
    }
}

// The plan's early-out shapes as two launches (every one returns at once unless
// the plan chose its shape; small sorts replay fewer graph nodes):
//   k_finish_a  sorted: copy | non-increasing: reversal (keys, or keys + payload) |
//               small key range (keys only): value histogram
//   k_finish_b  small key range: fill | non-increasing with payload: run fix-up
// (k_rev_long_runs follows for payloads: runs longer than kRevShortRun.)
template <typename K, bool VALS>
__global__ void __launch_bounds__(kCountBlock) k_finish_a(const K* __restrict__ kin, K* __restrict__ kout,
                                                          const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout,
                                                          int iota_vals, uint64_t n, const RadixState* __restrict__ st,
                                                          CountState* __restrict__ cs) {
    if (st->copy_in_to_out) {
        d_copy_in_to_out<K>(kin, kout, vin, VALS ? vout : nullptr, iota_vals, n, st);
    } else if (st->reversed) {
        if (VALS)
            d_reverse_pairs<K>(kin, kout, vin, vout, iota_vals, n, st);
        else
            d_reverse_keys<K>(kin, kout, n, st);
    } else if (!VALS && st->counting) {
        d_count_hist<K>(kin, n, st, cs);
    }
}

template <typename K, bool VALS>
__global__ void __launch_bounds__(kCountBlock, 2) k_finish_b(K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                             uint64_t n, RadixState* __restrict__ st,
                                                             const CountState* __restrict__ cs,
                                                             unsigned long long* __restrict__ long_runs) {
    if (!VALS && st->counting)
        d_count_fill<K>(kout, n, st, cs);
    else if (VALS && st->reversed)
        d_rev_fix_runs<K>(kout, vout, n, st, long_runs);
}

}  // namespace isort
