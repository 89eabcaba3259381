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
//   K1 k_upfront   one read of the keys: every digit histogram, max key, number
//                  of adjacent descents (0 => already sorted), plus an optional
//                  digitizer range check (bucket sort).          4n B  HBM read
//   K2 k_plan      scans the histograms, drops trivial digit passes (one bin
//                  holds all n keys => the pass is the identity) and the whole
//                  sort when the input is already sorted; assigns ping-pong
//                  buffers so the last executed pass lands in `out`.
//   K3 k_onesweep  one launch per digit slot.  Tile = BLOCK*IPT keys, tile id by
//                  atomic ticket (forward progress for the look-back).  Warp-level
//                  __match_any_sync ranking into per-warp smem histograms,
//                  decoupled look-back over tiles for the global digit offsets,
//                  smem-staged digit-sorted tile, then coalesced stores.
//                                                                 8n B / pass
//   K4 k_copy      only when no pass executes (sorted input): out = in.
#pragma once

#include "isort_common.cuh"

namespace isort {

// Buffer ids used by the plan.
enum : int32_t { kBufIn = 0, kBufOut = 1, kBufAlt = 2 };

// Look-back status word: [31:30] flag, [29:0] count.
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kFlagMask = 3u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr uint64_t kMaxLookbackN = (1ull << 30) - 1;

struct RadixState {
    uint32_t hist[kMaxDigits][kRadix];  // K1
    uint32_t offs[kMaxDigits][kRadix];  // K2: exclusive scans
    unsigned long long max_key;         // K1
    unsigned long long not_min_key;     // K1: ~min (so a zeroed word is the identity)
    unsigned long long first_bad;       // K1: ~(first index failing the range check)
    uint32_t descents;                  // K1: #i with key[i] > key[i+1]
    uint32_t n_active;                  // K2
    uint32_t copy_in_to_out;            // K2
    uint32_t tile_ticket[kMaxDigits];   // K3
    int32_t digit_of_slot[kMaxDigits];  // K2
    int32_t src_of_slot[kMaxDigits];
    int32_t dst_of_slot[kMaxDigits];
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
    __device__ __forceinline__ uint32_t digit(K key, int pos) const {
        return digit_of<K>(key, 8u * static_cast<uint32_t>(pos));
    }
    __device__ __forceinline__ void all_digits(K key, uint32_t (&d)[kDigits]) const {
#pragma unroll
        for (int p = 0; p < kDigits; ++p) d[p] = digit(key, p);
    }
    __device__ __forceinline__ bool in_range(K) const { return true; }
};

// ------------------------------------------------------------------- K1
template <typename K, typename Dz, int BLOCK, bool VEC>
__global__ void __launch_bounds__(BLOCK) k_upfront(const K* __restrict__ keys, uint64_t n,
                                                   RadixState* __restrict__ st, Dz dz) {
    constexpr int D = Dz::kDigits;
    __shared__ uint32_t sh[D][kRadix];
    __shared__ unsigned long long red_max[BLOCK / 32];
    __shared__ unsigned long long red_nmin[BLOCK / 32];
    __shared__ uint32_t red_desc[BLOCK / 32];
    for (int i = threadIdx.x; i < D * kRadix; i += BLOCK) (&sh[0][0])[i] = 0;
    __syncthreads();

    K kmax = 0;
    K kmin = static_cast<K>(~static_cast<K>(0));
    uint32_t desc = 0;
    unsigned long long first_bad = ~0ull;

    auto visit = [&](K k, uint64_t idx) {
        kmax = k > kmax ? k : kmax;
        kmin = k < kmin ? k : kmin;
        // Out-of-range keys are still counted (the digitizer clamps them) so the
        // passes stay self-consistent; the host reports the first of them.
        if (Dz::kChecks && !dz.in_range(k)) first_bad = idx < first_bad ? idx : first_bad;
        uint32_t d[D];
        dz.all_digits(k, d);
#pragma unroll
        for (int p = 0; p < D; ++p) atomicAdd(&sh[p][d[p]], 1u);
    };

    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * BLOCK;
    constexpr int V = 16 / sizeof(K) >= 4 ? 4 : 4;  // 4 keys per thread-iteration
    if (VEC) {
        // 4 consecutive keys per iteration via 16-byte vector loads.
        const uint64_t nv = n / V;
        for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * BLOCK + threadIdx.x; v < nv; v += stride) {
            K k[V];
            if (sizeof(K) == 4) {
                const uint4 q = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + v);
                k[0] = static_cast<K>(q.x);
                k[1] = static_cast<K>(q.y);
                k[2] = static_cast<K>(q.z);
                k[3] = static_cast<K>(q.w);
            } else {
                const uint4 a = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + 2 * v);
                const uint4 b = ldg_stream_v4(reinterpret_cast<const uint4*>(keys) + 2 * v + 1);
                k[0] = static_cast<K>((static_cast<uint64_t>(a.y) << 32) | a.x);
                k[1] = static_cast<K>((static_cast<uint64_t>(a.w) << 32) | a.z);
                k[2] = static_cast<K>((static_cast<uint64_t>(b.y) << 32) | b.x);
                k[3] = static_cast<K>((static_cast<uint64_t>(b.w) << 32) | b.z);
            }
            const uint64_t i0 = v * V;
            const K next = (i0 + V < n) ? keys[i0 + V] : static_cast<K>(~static_cast<K>(0));
            desc += (k[0] > k[1]) + (k[1] > k[2]) + (k[2] > k[3]) + (k[3] > next);
#pragma unroll
            for (int j = 0; j < V; ++j) visit(k[j], i0 + j);
        }
        for (uint64_t i = nv * V + static_cast<uint64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n; i += stride) {
            const K k = keys[i];
            if (i + 1 < n) desc += (k > keys[i + 1]);
            visit(k, i);
        }
    } else {
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n; i += stride) {
            const K k = keys[i];
            if (i + 1 < n) desc += (k > keys[i + 1]);
            visit(k, i);
        }
    }

    // block reductions
    unsigned long long m = warp_max<unsigned long long>(static_cast<unsigned long long>(kmax));
    unsigned long long nm = warp_max<unsigned long long>(~static_cast<unsigned long long>(kmin));
    uint32_t ds = warp_sum(desc);
    unsigned long long fb = ~first_bad;  // max of complements = min index
    fb = warp_max<unsigned long long>(fb);
    const int w = threadIdx.x / 32;
    if (lane_id() == 0) {
        red_max[w] = m;
        red_nmin[w] = nm;
        red_desc[w] = ds;
    }
    if (Dz::kChecks && lane_id() == 0 && fb != 0ull) atomicMax(&st->first_bad, fb);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = BLOCK / 32;
        m = threadIdx.x < nw ? red_max[threadIdx.x] : 0ull;
        nm = threadIdx.x < nw ? red_nmin[threadIdx.x] : 0ull;
        ds = threadIdx.x < nw ? red_desc[threadIdx.x] : 0u;
        m = warp_max<unsigned long long>(m);
        nm = warp_max<unsigned long long>(nm);
        ds = warp_sum(ds);
        if (threadIdx.x == 0) {
            atomicMax(&st->max_key, m);
            atomicMax(&st->not_min_key, nm);
            if (ds) atomicAdd(&st->descents, ds);
        }
    }
    for (int i = threadIdx.x; i < D * kRadix; i += BLOCK) {
        const uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(&st->hist[i / kRadix][i % kRadix], c);
    }
}

// ------------------------------------------------------------------- K2
// One CTA of kRadix threads.  `allow_skip_sorted`: a sorted input needs no pass.
template <int D>
__global__ void __launch_bounds__(kRadix) k_plan(RadixState* __restrict__ st, uint64_t n,
                                                 int allow_skip_sorted) {
    __shared__ uint32_t warp_tot[kRadix / 32];
    __shared__ int trivial[kMaxDigits];
    const int t = threadIdx.x;
    for (int p = 0; p < D; ++p) {
        const uint32_t v = st->hist[p][t];
        const uint32_t inc = warp_inclusive_scan(v);
        if (lane_id() == 31) warp_tot[t / 32] = inc;
        const int any_full = __syncthreads_or(static_cast<uint64_t>(v) == n);
        uint32_t pre = 0;
        for (int w = 0; w < t / 32; ++w) pre += warp_tot[w];
        st->offs[p][t] = pre + inc - v;
        if (t == 0) trivial[p] = any_full;
        __syncthreads();
    }
    if (t == 0) {
        const bool sorted = allow_skip_sorted && st->descents == 0;
        int na = 0;
        for (int p = 0; p < D; ++p)
            if (!sorted && !trivial[p]) st->digit_of_slot[na++] = p;
        for (int s = 0; s < na; ++s) {
            st->src_of_slot[s] = s == 0 ? kBufIn : st->dst_of_slot[s - 1];
            st->dst_of_slot[s] = ((na - 1 - s) % 2 == 0) ? kBufOut : kBufAlt;
        }
        st->n_active = na;
        st->copy_in_to_out = na == 0;
    }
}

// ------------------------------------------------------------------- K3
template <typename K, int BLOCK, int IPT, bool VALS, bool STAGE_DIGITS>
struct OnesweepSmem {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * IPT;
    K keys[kTile];
    uint32_t vals[VALS ? kTile : 1];
    uint8_t digits[STAGE_DIGITS ? kTile : 1];  // digit per staged key (expensive digitizers)
    uint32_t warp_hist[kWarps][kRadix + 1];  // +1: bin kRadix absorbs out-of-range slots
    uint32_t tile_start[kRadix];
    uint32_t out_base[kRadix];
    uint32_t scan_tot[kRadix / 32];
    uint32_t tile_id;
};

template <typename K, typename Dz, int BLOCK, int IPT, bool VALS>
__global__ void __launch_bounds__(BLOCK) k_onesweep(const K* __restrict__ keys_in, K* __restrict__ keys_out,
                                                    K* __restrict__ keys_alt, const uint32_t* __restrict__ vals_in,
                                                    uint32_t* __restrict__ vals_out, uint32_t* __restrict__ vals_alt,
                                                    int iota_vals, uint64_t n, RadixState* __restrict__ st,
                                                    uint32_t* __restrict__ lookback, uint32_t num_tiles, int slot,
                                                    Dz dz) {
    using Smem = OnesweepSmem<K, BLOCK, IPT, VALS, !Dz::kCheapDigit>;
    constexpr int kWarps = Smem::kWarps;
    constexpr int kTile = Smem::kTile;
    static_assert(BLOCK >= kRadix, "one thread per digit bin");
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

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();

    if (tid == 0) sm.tile_id = atomicAdd(&st->tile_ticket[slot], 1u);
    for (int i = tid; i < kWarps * (kRadix + 1); i += BLOCK) (&sm.warp_hist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = sm.tile_id;
    const uint64_t tile_base = static_cast<uint64_t>(tile) * kTile;
    const uint32_t valid = static_cast<uint32_t>((n - tile_base < static_cast<uint64_t>(kTile) ? n - tile_base : static_cast<uint64_t>(kTile)));
    uint32_t* lb = lookback + static_cast<size_t>(slot) * num_tiles * kRadix;

    // ---- load (warp-striped: item i of lane l is tile offset warp*32*IPT + i*32 + l)
    K key[IPT];
    uint32_t val[IPT];
    const uint32_t wofs = static_cast<uint32_t>(warp) * 32u * IPT + lane;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t o = wofs + i * 32u;
        key[i] = o < valid ? ldg_stream(src + tile_base + o) : static_cast<K>(0);
    }
    if (VALS) {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const uint32_t o = wofs + i * 32u;
            if (gen_iota)
                val[i] = static_cast<uint32_t>(tile_base + o);
            else
                val[i] = o < valid ? ldg_stream(vsrc + tile_base + o) : 0u;
        }
    }

    // ---- warp-level stable ranking: items in (i, lane) order == input order
    uint32_t rank[IPT], dg[IPT];
    uint32_t* wh = sm.warp_hist[warp];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t o = wofs + i * 32u;
        const uint32_t d = o < valid ? dz.digit(key[i], pos) : static_cast<uint32_t>(kRadix);
        dg[i] = d;
        const uint32_t peers = __match_any_sync(ISORT_FULL_MASK, d);
        const int leader = 31 - __clz(peers);
        uint32_t b = 0;
        if (static_cast<int>(lane) == leader) {
            b = wh[d];
            wh[d] = b + __popc(peers);
        }
        b = __shfl_sync(ISORT_FULL_MASK, b, leader);
        rank[i] = b + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // ---- per-digit: exclusive prefix over warps (in place), tile count
    uint32_t count = 0;
    if (tid < kRadix) {
#pragma unroll 4
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = sm.warp_hist[w][tid];
            sm.warp_hist[w][tid] = count;
            count += c;
        }
        // publish this tile's aggregate as early as possible
        st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + tid], (tile == 0 ? kFlagInc : kFlagAgg) | count);
        const uint32_t inc = warp_inclusive_scan(count);
        if (lane == 31) sm.scan_tot[tid >> 5] = inc;
        sm.tile_start[tid] = inc - count;  // warp-local for now
    }
    __syncthreads();
    if (tid < kRadix) {
        uint32_t pre = 0;
        for (int w = 0; w < (tid >> 5); ++w) pre += sm.scan_tot[w];
        const uint32_t start = sm.tile_start[tid] + pre;
        sm.tile_start[tid] = start;
        for (int w = 0; w < kWarps; ++w) sm.warp_hist[w][tid] += start;

        // ---- decoupled look-back over preceding tiles
        uint32_t excl = 0;
        if (tile > 0) {
            int t = static_cast<int>(tile) - 1;
            for (;;) {
                const uint32_t s = ld_relaxed_gpu(&lb[static_cast<size_t>(t) * kRadix + tid]);
                if ((s & kFlagMask) == 0) continue;
                excl += s & kValueMask;
                if (s & kFlagInc) break;
                --t;
            }
            st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + tid], kFlagInc | (excl + count));
        }
        sm.out_base[tid] = st->offs[pos][tid] + excl - start;
    }
    __syncthreads();

    // ---- stage the tile in digit order
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t o = wofs + i * 32u;
        if (o < valid) {
            const uint32_t p = sm.warp_hist[warp][dg[i]] + rank[i];
            sm.keys[p] = key[i];
            if (VALS) sm.vals[p] = val[i];
            if (!Dz::kCheapDigit) sm.digits[p] = static_cast<uint8_t>(dg[i]);
        }
    }
    __syncthreads();

    // ---- coalesced scatter: consecutive j with equal digit -> consecutive addresses
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t j = static_cast<uint32_t>(tid) + i * BLOCK;
        if (j < valid) {
            const K k = sm.keys[j];
            const uint32_t d = Dz::kCheapDigit ? dz.digit(k, pos) : static_cast<uint32_t>(sm.digits[j]);
            const uint32_t g = sm.out_base[d] + j;
            dst[g] = k;
            if (VALS) vdst[g] = sm.vals[j];
        }
    }
}

// ------------------------------------------------------------------- K4
template <typename K>
__global__ void k_copy_if_unsorted_skip(const K* __restrict__ in, K* __restrict__ out,
                                        const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout,
                                        int iota_vals, uint64_t n, const RadixState* __restrict__ st) {
    if (!st->copy_in_to_out) return;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        out[i] = in[i];
        if (vout) vout[i] = iota_vals ? static_cast<uint32_t>(i) : vin[i];
    }
}

}  // namespace isort
