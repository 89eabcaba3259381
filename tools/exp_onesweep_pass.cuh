// onesweep_pass.cuh -- K3 v2: one stable digit pass of the LSD radix sort, one
// read of the keys, for sm_100a.
//
// Reference loop replaced: counting_sort_by_digit (proj/core/src/sort.cpp:95-108:
// count -> prefix -> reverse-walk place), one call per digit of the plan.
//
// Why this shape (profiles/r02/ncu_onesweep_v10_alone.txt): the v10 pass (count
// phase + L2 re-read + rank phase, radix_onesweep.cuh) kept the L1TEX data pipe
// 74% busy at ~19 wavefronts per 32 keys: two random shared atomics (count and
// rank, ~3.35 wavefronts each), a random staging store (~3.4), the staged read,
// and two global reads of every key.  Every random shared access costs the same
// ~3.4 wavefronts, so the pass is bounded by how many of them each key makes and
// by how busy the pipe stays.  This pass:
//   * reads each key ONCE, warp-striped into registers (item i of lane l of warp
//     w is key w*32*IPT + i*32 + l of the tile, so (item, lane) order is input
//     order), and prefetches the next tile's keys into the same registers while
//     the current tile is written out;
//   * ranks with ONE shared atomic per key on per-warp counters (lane-ordered
//     same-address atomics: the in-warp rank is stable), keeping the rank packed
//     two per register;
//   * turns the counters into slot bases (per digit: exclusive scan over warps +
//     the digit's start in the tile) and stages key i at base[warp][d] + rank;
//   * resolves the decoupled look-back AFTER its own staging stores, so the L2
//     round trips of the look-back overlap the other warps' staging, and writes
//     the staged (digit-sorted) tile out coalesced.
// Random shared accesses per key stay at three (rank atomic, base load, staging
// store); the second global read, the count loop and its barrier go away.
//
// Look-back status words are 64-bit ([63:62] flag, [61:0] count), so one call
// sorts up to 2^32 - 1 keys (positions and payloads are u32).
#pragma once

#include "../paper_1206_3511_b200/csrc/radix_onesweep.cuh"

namespace isort {

constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbInc = 2ull << 62;
constexpr unsigned long long kLbFlagMask = 3ull << 62;
constexpr unsigned long long kLbValueMask = kLbAgg - 1;

__device__ __forceinline__ unsigned long long ld_relaxed_gpu64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive prefix of digit d over tiles [0, t_start]: windowed decoupled
// look-back, kLookbackWindow64 loads in flight per round trip.
#ifndef ISORT_LB_WINDOW64
#define ISORT_LB_WINDOW64 8
#endif
constexpr int kLookbackWindow64 = ISORT_LB_WINDOW64;
__device__ __forceinline__ uint32_t lookback64(const unsigned long long* __restrict__ lb, int t_start, int d) {
    uint64_t excl = 0;
    int t = t_start;
    while (t >= 0) {
        unsigned long long sv[kLookbackWindow64];
#pragma unroll
        for (int j = 0; j < kLookbackWindow64; ++j)
            sv[j] = (t - j >= 0) ? ld_relaxed_gpu64(&lb[static_cast<size_t>(t - j) * kRadix + d]) : kLbInc;
        int used = 0;
        bool done = false;
#pragma unroll
        for (int j = 0; j < kLookbackWindow64; ++j) {
            if (!done && used == j) {
                const unsigned long long f = sv[j] & kLbFlagMask;
                if (f != 0) {
                    excl += sv[j] & kLbValueMask;
                    used = j + 1;
                    done = (f == kLbInc);
                }
            }
        }
        if (done) break;
        t -= used;  // stopped at a predecessor that has not published: re-read from it
    }
    return static_cast<uint32_t>(excl);
}

template <typename K, int BLOCK, int IPT, bool VALS, bool STAGE_DIGITS>
struct PassSmem {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * IPT;
    uint32_t cnt[kWarps][kRadix];  // rank counters, then slot bases (digit start + warp prefix)
    uint32_t out_base[kRadix];     // global position = out_base[d] + staging slot
    uint32_t offs[kRadix];         // the pass's digit offsets (K2)
    uint32_t tot_w[kRadix / 32];
    uint32_t next_tile;
    alignas(16) K keys[kTile];
    alignas(16) uint32_t vals[VALS ? kTile : 1];
    uint8_t digits[STAGE_DIGITS ? kTile : 1];  // digit per staged key (expensive digitizers)
};

// Ranks held between the atomic and the staging store: two 16-bit ranks per
// register for cheap digitizers (the digit is recomputed), (digit << 16 | rank)
// per key otherwise.
template <bool CHEAP, int IPT>
struct RankRegs {
    static constexpr int kRegs = CHEAP ? (IPT + 1) / 2 : IPT;
    uint32_t r[kRegs];
    __device__ __forceinline__ void put(int i, uint32_t rank, uint32_t d) {
        if (CHEAP) {
            if (i & 1)
                r[i >> 1] |= rank << 16;
            else
                r[i >> 1] = rank;
        } else {
            r[i] = (d << 16) | rank;
        }
    }
    __device__ __forceinline__ uint32_t rank(int i) const {
        return CHEAP ? ((i & 1) ? (r[i >> 1] >> 16) : (r[i >> 1] & 0xFFFFu)) : (r[i] & 0xFFFFu);
    }
    __device__ __forceinline__ uint32_t digit(int i) const { return r[i] >> 16; }
};

template <bool FULL, typename K, int IPT, bool VALS>
__device__ __forceinline__ void pass_load_t(K (&key)[IPT], uint32_t (&val)[VALS ? IPT : 1], const K* __restrict__ src,
                                            const uint32_t* __restrict__ vsrc, uint64_t tbase, uint32_t tlen,
                                            bool gen_iota, uint32_t wofs, uint64_t pol) {
    constexpr bool full = FULL;
    const K* s = src + tbase + wofs;
#pragma unroll
    for (int i = 0; i < IPT; ++i)
        key[i] = (full || wofs + i * 32u < tlen) ? ldg_hint(s + i * 32, pol) : static_cast<K>(0);
    if (VALS) {
#pragma unroll
        for (int i = 0; i < IPT; ++i)
            val[i] = gen_iota ? static_cast<uint32_t>(tbase + wofs + i * 32u)
                              : ((full || wofs + i * 32u < tlen) ? ldg_stream(vsrc + tbase + wofs + i * 32u) : 0u);
    }
}
template <typename K, int IPT, bool VALS>
__device__ __forceinline__ void pass_load(K (&key)[IPT], uint32_t (&val)[VALS ? IPT : 1], const K* __restrict__ src,
                                          const uint32_t* __restrict__ vsrc, uint64_t tbase, uint32_t tlen,
                                          bool gen_iota, uint32_t wofs, uint64_t pol) {
    if (wofs - (threadIdx.x & 31u) + 32u * IPT <= tlen)  // the whole warp's slice is in the tile (warp-uniform)
        pass_load_t<true, K, IPT, VALS>(key, val, src, vsrc, tbase, tlen, gen_iota, wofs, pol);
    else
        pass_load_t<false, K, IPT, VALS>(key, val, src, vsrc, tbase, tlen, gen_iota, wofs, pol);
}

// Rank step of one tile: one shared atomic per key on this warp's counters.
// FULL: every key of the tile is valid (no per-key bounds checks).  AGG: the
// tile is expected to be made of sorted runs (warp-aggregated atomics).
template <bool FULL, bool AGG, bool SAFE, typename K, typename Dz, int IPT, typename RR>
__device__ __forceinline__ void pass_rank(uint32_t* wc, const K (&key)[IPT], RR& rk, uint32_t wofs, uint32_t tile_len,
                                          uint32_t dsh, const Dz& dz) {
    bool agg = AGG;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if (FULL || wofs + i * 32u < tile_len) {
            const uint32_t d = dz.digit_sh(key[i], dsh);
            const uint32_t r = AGG ? warp_slot_agg<SAFE>(wc, d, agg) : warp_slot<SAFE>(wc, d);
            rk.put(i, r, d);
        }
    }
}

// Staging step: key i at base[warp][d] + rank (the tile becomes digit-sorted).
template <bool FULL, bool VALS, bool CHEAP, typename K, typename Dz, int IPT, typename RR>
__device__ __forceinline__ void pass_stage(K* skeys, uint32_t* svals, uint8_t* sdig, const uint32_t* wb,
                                           const K (&key)[IPT], const uint32_t (&val)[VALS ? IPT : 1], const RR& rk,
                                           uint32_t wofs, uint32_t tile_len, uint32_t dsh, const Dz& dz) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if (FULL || wofs + i * 32u < tile_len) {
            const uint32_t d = CHEAP ? dz.digit_sh(key[i], dsh) : rk.digit(i);
            const uint32_t s = wb[d] + rk.rank(i);
            skeys[s] = key[i];
            if (VALS) svals[s] = val[i];
            if (!CHEAP) sdig[s] = static_cast<uint8_t>(d);
        }
    }
}

// Write-out of the staged tile: slot j goes to out_base[digit] + j, coalesced
// along the digit runs.
template <bool FULL, bool SCATTER, bool VALS, bool CHEAP, int BLOCK, int IPT, typename K, typename Dz>
__device__ __forceinline__ void pass_write(const K* skeys, const uint32_t* svals, const uint8_t* sdig,
                                           const uint32_t* ob, K* __restrict__ dst, uint32_t* __restrict__ vdst,
                                           uint32_t tile_len, uint32_t dsh, const Dz& dz, uint64_t pol,
                                           const unsigned long long* kbase, const unsigned long long* vbase) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t j = static_cast<uint32_t>(threadIdx.x) + i * BLOCK;
        if (FULL || j < tile_len) {
            const K k = skeys[j];
            const uint32_t d = CHEAP ? dz.digit_sh(k, dsh) : static_cast<uint32_t>(sdig[j]);
            const uint32_t g = ob[d] + j;
            if (SCATTER) {
                *(reinterpret_cast<K*>(kbase[d]) + g) = k;
                if (VALS) *(reinterpret_cast<uint32_t*>(vbase[d]) + g) = svals[j];
            } else {
                stg_hint(dst + g, k, pol);
                if (VALS) stg_hint(vdst + g, svals[j], pol);
            }
        }
    }
}

// Per digit d (threads [0, kRadix)): the tile's count of d over the warps, its
// aggregate published to the look-back, the digit's start in the tile (block
// scan over digits) and the per-warp slot bases written over the counters.
template <int BLOCK, int kWarps>
__device__ __forceinline__ void pass_scan(uint32_t (*cnt)[kRadix], uint32_t* tot_w, unsigned long long* lb_tile,
                                          bool first_tile, uint32_t& tot, uint32_t& start) {
    const int d = threadIdx.x;
    const uint32_t lane = lane_id();
    static_assert(kWarps % 2 == 0, "warp counts packed in pairs");
    uint32_t c[kWarps / 2];  // two 16-bit per-warp counts per register (<= 32 * IPT each)
    tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; w += 2) {
        const uint32_t a = cnt[w][d], b = cnt[w + 1][d];
        c[w / 2] = a | (b << 16);
        tot += a + b;
    }
    st_relaxed_gpu64(&lb_tile[d], (first_tile ? kLbInc : kLbAgg) | static_cast<unsigned long long>(tot));
    const uint32_t inc = warp_inclusive_scan(tot);
    if (lane == 31) tot_w[d >> 5] = inc;
    if (BLOCK == kRadix)
        __syncthreads();
    else
        asm volatile("bar.sync 1, %0;" ::"n"(kRadix));
    uint32_t pre = 0;
#pragma unroll
    for (int w = 0; w < kRadix / 32; ++w) pre += w < (d >> 5) ? tot_w[w] : 0u;
    start = pre + inc - tot;
    uint32_t b = start;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        cnt[w][d] = b;
        b += (w & 1) ? (c[w / 2] >> 16) : (c[w / 2] & 0xFFFFu);
    }
}

template <typename K, typename Dz, int BLOCK, int IPT, bool VALS, bool SAFE, bool SCATTER = false>
__global__ void __launch_bounds__(BLOCK, ISORT_PASS_MINB_OF(BLOCK))
    k_pass(const K* __restrict__ keys_in, K* __restrict__ keys_out, K* __restrict__ keys_alt,
           const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out, uint32_t* __restrict__ vals_alt,
           int iota_vals, uint64_t n, RadixState* __restrict__ st, unsigned long long* __restrict__ lookback,
           uint32_t num_tiles, int slot, Dz dz, const ScatterArg<SCATTER> scat) {
    constexpr bool kCheap = Dz::kCheapDigit;
    using Smem = PassSmem<K, BLOCK, IPT, VALS, !kCheap>;
    constexpr int kWarps = Smem::kWarps;
    constexpr int kTile = Smem::kTile;
    static_assert(BLOCK >= kRadix && BLOCK % kRadix == 0, "threads [0, kRadix) own one digit each");
    static_assert(32 * IPT < 65536, "16-bit in-warp ranks");
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
    unsigned long long* lb = lookback + static_cast<size_t>(slot) * num_tiles * kRadix;
    const uint64_t pol_in = policy_evict_first();  // each key is read once
    const uint64_t pol_out = policy_evict_normal();

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint32_t wofs = static_cast<uint32_t>(warp) * 32u * IPT + lane;
    __shared__ unsigned long long s_kbase[SCATTER ? kScatterMax : 1], s_vbase[SCATTER ? kScatterMax : 1];
    if (tid < kRadix) sm.offs[tid] = st->offs[pos][tid];
    if constexpr (SCATTER) {
        if (tid < kScatterMax) {  // per-digit base, shifted so that base + g addresses the run
            const unsigned long long o = st->offs[pos][tid];
            s_kbase[tid] = scat.key[tid] - o * sizeof(K);
            if (VALS) s_vbase[tid] = scat.val[tid] - o * sizeof(uint32_t);
        }
    }
    {
        uint4* c4 = reinterpret_cast<uint4*>(&sm.cnt[0][0]);
        for (int i = tid; i < kWarps * kRadix / 4; i += BLOCK) c4[i] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) sm.next_tile = atomicAdd(&st->tile_ticket[slot], 1u);
    __syncthreads();
    uint32_t tile = sm.next_tile;

    K key[IPT];
    uint32_t val[VALS ? IPT : 1];
    auto tile_len_of = [&](uint32_t t) -> uint32_t {
        const uint64_t b = static_cast<uint64_t>(t) * kTile;
        return n - b < static_cast<uint64_t>(kTile) ? static_cast<uint32_t>(n - b) : static_cast<uint32_t>(kTile);
    };
    auto valid_tile = [&](uint32_t t) { return t < num_tiles && static_cast<uint64_t>(t) * kTile < n; };
    if (valid_tile(tile))
        pass_load<K, IPT, VALS>(key, val, src, vsrc, static_cast<uint64_t>(tile) * kTile, tile_len_of(tile), gen_iota,
                                wofs, pol_in);
    bool hot = false;  // the previous tile had few distinct digits: warp-aggregated ranks
    while (valid_tile(tile)) {
        const uint32_t tile_len = tile_len_of(tile);
        const bool full = tile_len == static_cast<uint32_t>(kTile);

        // ---------------- rank: one shared atomic per key on this warp's counters
        RankRegs<kCheap, IPT> rk;
        if (full && hot)
            pass_rank<true, true, SAFE>(sm.cnt[warp], key, rk, wofs, tile_len, dsh, dz);
        else if (full)
            pass_rank<true, false, SAFE>(sm.cnt[warp], key, rk, wofs, tile_len, dsh, dz);
        else
            pass_rank<false, false, SAFE>(sm.cnt[warp], key, rk, wofs, tile_len, dsh, dz);
        __syncthreads();

        // ---------------- per digit: tile total, aggregate, slot bases
        uint32_t tot = 0, start = 0;
        if (tid < kRadix) {
            const int d = tid;
            static_assert(kWarps % 2 == 0, "warp counts packed in pairs");
            uint32_t c[kWarps / 2];  // two 16-bit per-warp counts per register (<= 32 * IPT each)
#pragma unroll
            for (int w = 0; w < kWarps; w += 2) {
                const uint32_t a = sm.cnt[w][d], b = sm.cnt[w + 1][d];
                c[w / 2] = a | (b << 16);
                tot += a + b;
            }
            st_relaxed_gpu64(&lb[static_cast<size_t>(tile) * kRadix + d],
                             (tile == 0 ? kLbInc : kLbAgg) | static_cast<unsigned long long>(tot));
            const uint32_t inc = warp_inclusive_scan(tot);
            if (lane == 31) sm.tot_w[warp] = inc;
            if (BLOCK == kRadix)
                __syncthreads();
            else
                asm volatile("bar.sync 1, %0;" ::"n"(kRadix));
            uint32_t pre = 0;
#pragma unroll
            for (int w = 0; w < kRadix / 32; ++w) pre += w < warp ? sm.tot_w[w] : 0u;
            start = pre + inc - tot;
            uint32_t b = start;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                sm.cnt[w][d] = b;
                b += (w & 1) ? (c[w / 2] >> 16) : (c[w / 2] & 0xFFFFu);
            }
        }
        const bool hot_next = __syncthreads_count(tid < kRadix && tot != 0) <= kHotDigits;

        // ---------------- stage: key i at base[warp][d] + rank (a digit-sorted tile)
        if (full)
            pass_stage<true, VALS, kCheap>(sm.keys, sm.vals, sm.digits, sm.cnt[warp], key, val, rk, wofs, tile_len, dsh,
                                           dz);
        else
            pass_stage<false, VALS, kCheap>(sm.keys, sm.vals, sm.digits, sm.cnt[warp], key, val, rk, wofs, tile_len, dsh,
                                            dz);
        // ---------------- look-back (its L2 round trips overlap the other warps' staging)
        if (tid == 0) sm.next_tile = atomicAdd(&st->tile_ticket[slot], 1u);
        if (tid < kRadix) {
            const int d = tid;
            uint32_t excl = 0;
            if (tile != 0) {
                excl = lookback64(lb, static_cast<int>(tile) - 1, d);
                st_relaxed_gpu64(&lb[static_cast<size_t>(tile) * kRadix + d],
                                 kLbInc | static_cast<unsigned long long>(excl + tot));
            }
            sm.out_base[d] = sm.offs[d] + excl - start;
        }
        __syncthreads();
        const uint32_t next = sm.next_tile;

        // ---------------- next tile's keys load while this one is written out
        if (valid_tile(next))
            pass_load<K, IPT, VALS>(key, val, src, vsrc, static_cast<uint64_t>(next) * kTile, tile_len_of(next),
                                    gen_iota, wofs, pol_in);
        if (full)
            pass_write<true, SCATTER, VALS, kCheap, BLOCK, IPT>(sm.keys, sm.vals, sm.digits, sm.out_base, dst, vdst, tile_len, dsh, dz, pol_out, s_kbase,
                                                                s_vbase);
        else
            pass_write<false, SCATTER, VALS, kCheap, BLOCK, IPT>(sm.keys, sm.vals, sm.digits, sm.out_base, dst, vdst, tile_len, dsh, dz, pol_out, s_kbase,
                                                                 s_vbase);
        {  // counters of the next tile (the staging reads of the bases are done)
            uint4* c4 = reinterpret_cast<uint4*>(&sm.cnt[0][0]);
            for (int i = tid; i < kWarps * kRadix / 4; i += BLOCK) c4[i] = make_uint4(0, 0, 0, 0);
        }
        hot = hot_next;
        __syncthreads();
        tile = next;
    }
    if (SCATTER) __threadfence_system();  // peer stores visible before the host-ordered barrier
}


// ------------------------------------------------------------------ K3 v2b
// The same pass, software-pipelined across two staged tiles so the look-back
// never stalls the CTA: tile A waits in staging buffer A (its aggregate already
// published) while tile B is loaded, ranked and scanned; only then is A's
// look-back resolved (every predecessor has had a whole tile step to publish),
// and B is staged into buffer B while A is written out.  Per tile step:
//   rank(B) | bar | scan(B) + look-back(A) | bar | stage(B) + write-out(A) | bar
// Each warp zeroes its own counters after its staging reads (only warp w reads
// cnt[w] while staging), so no barrier separates staging from the next rank.
template <typename K, int BLOCK, int IPT, bool VALS, bool STAGE_DIGITS>
struct Pass2Smem {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * IPT;
    uint32_t cnt[kWarps][kRadix];
    uint32_t out_base[2][kRadix];
    uint32_t offs[kRadix];
    uint32_t tot_w[kRadix / 32];
    uint32_t next_tile;
    alignas(16) K keys[2][kTile];
    alignas(16) uint32_t vals[2][VALS ? kTile : 1];
    uint8_t digits[2][STAGE_DIGITS ? kTile : 1];
};

template <typename K, typename Dz, int BLOCK, int IPT, bool VALS, bool SAFE, bool SCATTER = false>
__global__ void __launch_bounds__(BLOCK, ISORT_PASS_MINB_OF(BLOCK))
    k_pass2(const K* __restrict__ keys_in, K* __restrict__ keys_out, K* __restrict__ keys_alt,
            const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out, uint32_t* __restrict__ vals_alt,
            int iota_vals, uint64_t n, RadixState* __restrict__ st, unsigned long long* __restrict__ lookback,
            uint32_t num_tiles, int slot, Dz dz, const ScatterArg<SCATTER> scat) {
    constexpr bool kCheap = Dz::kCheapDigit;
    using Smem = Pass2Smem<K, BLOCK, IPT, VALS, !kCheap>;
    constexpr int kWarps = Smem::kWarps;
    constexpr int kTile = Smem::kTile;
    static_assert(BLOCK >= kRadix && BLOCK % kRadix == 0, "threads [0, kRadix) own one digit each");
    static_assert(32 * IPT < 65536, "16-bit in-warp ranks");
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
    unsigned long long* lb = lookback + static_cast<size_t>(slot) * num_tiles * kRadix;
    const uint64_t pol_in = policy_evict_first();  // each key is read once
    const uint64_t pol_out = policy_evict_normal();

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint32_t wofs = static_cast<uint32_t>(warp) * 32u * IPT + lane;
    __shared__ unsigned long long s_kbase[SCATTER ? kScatterMax : 1], s_vbase[SCATTER ? kScatterMax : 1];
    if (tid < kRadix) sm.offs[tid] = st->offs[pos][tid];
    if constexpr (SCATTER) {
        if (tid < kScatterMax) {  // per-digit base, shifted so that base + g addresses the run
            const unsigned long long o = st->offs[pos][tid];
            s_kbase[tid] = scat.key[tid] - o * sizeof(K);
            if (VALS) s_vbase[tid] = scat.val[tid] - o * sizeof(uint32_t);
        }
    }
    {
        uint4* c4 = reinterpret_cast<uint4*>(&sm.cnt[0][0]);
        for (int i = tid; i < kWarps * kRadix / 4; i += BLOCK) c4[i] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) sm.next_tile = atomicAdd(&st->tile_ticket[slot], 1u);
    __syncthreads();

    auto tile_len_of = [&](uint32_t t) -> uint32_t {
        const uint64_t b = static_cast<uint64_t>(t) * kTile;
        return n - b < static_cast<uint64_t>(kTile) ? static_cast<uint32_t>(n - b) : static_cast<uint32_t>(kTile);
    };
    auto valid_tile = [&](uint32_t t) { return t < num_tiles && static_cast<uint64_t>(t) * kTile < n; };

    K key[IPT];
    uint32_t val[VALS ? IPT : 1];
    bool hot = false;
    uint32_t tile_a = sm.next_tile;
    if (!valid_tile(tile_a)) return;
    uint32_t tot_a = 0, start_a = 0;  // digit `tid`'s count and start in tile a
    int cur = 0;
    uint32_t tile_b;
    {  // prologue: tile a ranked, scanned (aggregate published) and staged; tile b loading
        const uint32_t len = tile_len_of(tile_a);
        pass_load<K, IPT, VALS>(key, val, src, vsrc, static_cast<uint64_t>(tile_a) * kTile, len, gen_iota, wofs,
                                pol_in);
        RankRegs<kCheap, IPT> rk;
        if (len == static_cast<uint32_t>(kTile))
            pass_rank<true, false, SAFE>(sm.cnt[warp], key, rk, wofs, len, dsh, dz);
        else
            pass_rank<false, false, SAFE>(sm.cnt[warp], key, rk, wofs, len, dsh, dz);
        __syncthreads();
        if (tid < kRadix)
            pass_scan<BLOCK, kWarps>(sm.cnt, sm.tot_w, lb + static_cast<size_t>(tile_a) * kRadix, tile_a == 0, tot_a,
                                     start_a);
        if (tid == 0) sm.next_tile = atomicAdd(&st->tile_ticket[slot], 1u);
        hot = __syncthreads_count(tid < kRadix && tot_a != 0) <= kHotDigits;
        tile_b = sm.next_tile;
        if (len == static_cast<uint32_t>(kTile))
            pass_stage<true, VALS, kCheap>(sm.keys[0], sm.vals[0], sm.digits[0], sm.cnt[warp], key, val, rk, wofs, len,
                                           dsh, dz);
        else
            pass_stage<false, VALS, kCheap>(sm.keys[0], sm.vals[0], sm.digits[0], sm.cnt[warp], key, val, rk, wofs,
                                            len, dsh, dz);
        __syncwarp();
        {
            uint4* c4 = reinterpret_cast<uint4*>(sm.cnt[warp]);
            for (int i = lane; i < kRadix / 4; i += 32) c4[i] = make_uint4(0, 0, 0, 0);
        }
        if (valid_tile(tile_b))
            pass_load<K, IPT, VALS>(key, val, src, vsrc, static_cast<uint64_t>(tile_b) * kTile, tile_len_of(tile_b),
                                    gen_iota, wofs, pol_in);
        __syncthreads();
    }
    for (;;) {
        // keys of tile b are in registers (or in flight)
        const bool have_b = valid_tile(tile_b);
        const uint32_t len_b = have_b ? tile_len_of(tile_b) : 0u;
        const bool full_b = len_b == static_cast<uint32_t>(kTile);
        RankRegs<kCheap, IPT> rk;
        if (have_b) {
            if (full_b && hot)
                pass_rank<true, true, SAFE>(sm.cnt[warp], key, rk, wofs, len_b, dsh, dz);
            else if (full_b)
                pass_rank<true, false, SAFE>(sm.cnt[warp], key, rk, wofs, len_b, dsh, dz);
            else
                pass_rank<false, false, SAFE>(sm.cnt[warp], key, rk, wofs, len_b, dsh, dz);
        }
        __syncthreads();
        uint32_t tot_b = 0, start_b = 0;
        if (tid < kRadix) {
            if (have_b)
                pass_scan<BLOCK, kWarps>(sm.cnt, sm.tot_w, lb + static_cast<size_t>(tile_b) * kRadix, tile_b == 0,
                                         tot_b, start_b);
            if (tid == 0 && have_b) sm.next_tile = atomicAdd(&st->tile_ticket[slot], 1u);
            // tile a: every predecessor published its aggregate at least one tile step ago
            const int d = tid;
            uint32_t excl = 0;
            if (tile_a != 0) {
                excl = lookback64(lb, static_cast<int>(tile_a) - 1, d);
                st_relaxed_gpu64(&lb[static_cast<size_t>(tile_a) * kRadix + d],
                                 kLbInc | static_cast<unsigned long long>(excl + tot_a));
            }
            sm.out_base[cur][d] = sm.offs[d] + excl - start_a;
        }
        const bool hot_b = __syncthreads_count(tid < kRadix && tot_b != 0) <= kHotDigits;
        const uint32_t tile_c = have_b ? sm.next_tile : 0xFFFFFFFFu;
        if (have_b) {
            if (full_b)
                pass_stage<true, VALS, kCheap>(sm.keys[cur ^ 1], sm.vals[cur ^ 1], sm.digits[cur ^ 1], sm.cnt[warp],
                                               key, val, rk, wofs, len_b, dsh, dz);
            else
                pass_stage<false, VALS, kCheap>(sm.keys[cur ^ 1], sm.vals[cur ^ 1], sm.digits[cur ^ 1], sm.cnt[warp],
                                                key, val, rk, wofs, len_b, dsh, dz);
            __syncwarp();
            uint4* c4 = reinterpret_cast<uint4*>(sm.cnt[warp]);
            for (int i = lane; i < kRadix / 4; i += 32) c4[i] = make_uint4(0, 0, 0, 0);
            if (valid_tile(tile_c))  // tile c's keys load during the write-out of tile a
                pass_load<K, IPT, VALS>(key, val, src, vsrc, static_cast<uint64_t>(tile_c) * kTile,
                                        tile_len_of(tile_c), gen_iota, wofs, pol_in);
        }
        {
            const uint32_t len_a = tile_len_of(tile_a);
            if (len_a == static_cast<uint32_t>(kTile))
                pass_write<true, SCATTER, VALS, kCheap, BLOCK, IPT>(sm.keys[cur], sm.vals[cur], sm.digits[cur],
                                                                    sm.out_base[cur], dst, vdst, len_a, dsh, dz,
                                                                    pol_out, s_kbase, s_vbase);
            else
                pass_write<false, SCATTER, VALS, kCheap, BLOCK, IPT>(sm.keys[cur], sm.vals[cur], sm.digits[cur],
                                                                     sm.out_base[cur], dst, vdst, len_a, dsh, dz,
                                                                     pol_out, s_kbase, s_vbase);
        }
        __syncthreads();
        if (!have_b) break;
        tile_a = tile_b;
        tile_b = tile_c;
        tot_a = tot_b;
        start_a = start_b;
        hot = hot_b;
        cur ^= 1;
    }
    if (SCATTER) __threadfence_system();  // peer stores visible before the host-ordered barrier
}

}  // namespace isort
