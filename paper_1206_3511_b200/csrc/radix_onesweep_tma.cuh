// radix_onesweep_tma.cuh -- the one-sweep digit pass with a bulk-copy (TMA)
// write-out: keys-only passes over large inputs (K3t).
//
// Same contract as k_onesweep (radix_onesweep.cuh): one stable counting pass of
// the LSD sort (sort.cpp:77-110) over tiles taken by atomic ticket, global
// offsets by decoupled look-back.  What differs is the shape of a tile:
//   * one chunk of BLOCK * IPT keys per tile, read ONCE: the keys stay in
//     registers between the count and the rank (warp-striped, so (item, lane)
//     order is input order);
//   * every digit's run is staged at a slot congruent to its global position
//     modulo one 16-byte block, so the run's aligned interior leaves shared memory
//     by one cp.async.bulk (TMA store) issued by the digit's thread; only the
//     <= 3 + 3 keys around it are plain stores.  The copy engine reads the staged
//     run while the CTA already counts its next tile: nothing waits for it until
//     the next tile's rank, a whole count phase and per-digit section later;
//   * the aligned slots need the run's global position, so the look-back comes
//     before the rank (k_onesweep walks after chunk 0 is staged).  A walk right
//     after the publication mostly waits for the nearest predecessors to publish;
//     so the PREVIOUS tile's write-out (the copies' issue and the edge stores) sits
//     between this tile's publication and its walk (ISORT_T_LATE_WRITE): walk
//     rounds that stop at an unpublished predecessor drop from 2.2 to 0.4 per tile;
//   * the next tile's ticket is taken after the rank and its keys are loaded
//     right after the barrier that ends the rank.
// Per 32 keys this removes the second key read (1 L1 wavefront), the staged-key
// load (1), the out_base lookup (~1.5) and most of the scattered STG (~2.5 ->
// 0.6): 14.5 L1 wavefronts against 19.0, 0.242 ms against 0.279 ms per pass at
// 10^8 keys (DESIGN.md section 3.1 has the phase split and what was tried).
#pragma once

#include "radix_onesweep.cuh"

namespace isort {

template <typename K, int BLOCK, int IPT, bool VALS = false>
struct OnesweepTSmem {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * IPT;
    static constexpr int kVec = 16 / static_cast<int>(sizeof(K));  // keys per 16-byte block
    static constexpr int kSlotVec = VALS ? 4 : kVec;               // slots follow the global index modulo this
    static constexpr int kStage = kTile + kSlotVec * kRadix;       // <= kSlotVec - 1 pad slots before each run (+ 1 spare)
    uint32_t cnt[kWarps][kRadix];  // counts; then per-warp slot bases
    uint32_t offs[kRadix];         // pass digit offsets (from K2)
    uint32_t tot_w[kWarps];
    uint32_t run_slot[2][kRadix];  // digit d's run (by tile parity): first staging slot,
    uint32_t run_len[2][kRadix];   // keys,
    uint32_t run_g[2][kRadix];     // and global index of its first key
    uint32_t tile_next;
    alignas(16) K keys[kStage];
    alignas(16) uint32_t vals[VALS ? kStage : 4];  // the payload, staged at the key's slot
};

// Look-back window (predecessors read per round trip and digit).  The walk is spent
// waiting for the nearest predecessors to publish, not reading: at 10^8 keys it
// takes ~8,400 of a tile's 27,400 cycles whatever the window (2 / 4 / 8 / 16 / 24:
// 0.2623 / 0.2632 / 0.2652 / 0.274 / 0.28 ms per pass), and every round reads
// window x 1 KB per tile from L2, so a narrow window is the cheaper one.
#ifndef ISORT_PASS_CTAS_T  // resident CTAs per SM (the launch bound's minimum and the grid size)
#define ISORT_PASS_CTAS_T_OF(block) (1024 / (block))
#else
#define ISORT_PASS_CTAS_T_OF(block) ISORT_PASS_CTAS_T
#endif
#ifndef ISORT_T_LATE_WRITE
#define ISORT_T_LATE_WRITE 1
#endif

// Digitizers whose digit costs more than one instruction (the bucket index: a 64-bit multiply, a
// 64-bit shift) compute it once, in the count, and keep it packed four to a register for the rank.
#ifndef ISORT_T_DIGIT_CACHE
#define ISORT_T_DIGIT_CACHE 1
#endif
template <typename Dz>
struct CachesDigit : std::false_type {};
#ifndef ISORT_T_LB_WINDOW
#define ISORT_T_LB_WINDOW 4
#endif
constexpr int kLookbackWindowT = ISORT_T_LB_WINDOW;

template <typename K, typename Dz, int BLOCK, int IPT, bool VALS, bool SAFE, typename LW>
__global__ void __launch_bounds__(BLOCK, ISORT_PASS_CTAS_T_OF(BLOCK))
    k_onesweep_t(const K* __restrict__ keys_in, K* __restrict__ keys_out, K* __restrict__ keys_alt,
                 const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out, uint32_t* __restrict__ vals_alt,
                 int iota_vals, uint64_t n, RadixState* __restrict__ st, void* __restrict__ lookback,
                 uint32_t num_tiles, int slot, Dz dz) {
    using LT = LbTraits<LW>;
    using Smem = OnesweepTSmem<K, BLOCK, IPT, VALS>;

    constexpr int kWarps = Smem::kWarps;
    constexpr int kTile = Smem::kTile;
    constexpr uint32_t kVec = Smem::kVec;
    static_assert(BLOCK >= kRadix && BLOCK % 32 == 0, "threads [0, kRadix) own a digit");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    if (slot >= static_cast<int>(st->n_active)) return;  // trivial / skipped pass
    const int pos = st->digit_of_slot[slot];
    const int src_id = st->src_of_slot[slot];
    const int dst_id = st->dst_of_slot[slot];
    const K* src = src_id == kBufIn ? keys_in : (src_id == kBufOut ? keys_out : keys_alt);
    K* dst = dst_id == kBufOut ? keys_out : keys_alt;
    const uint32_t dsh = dz.shift_for(pos);
    LW* lb = static_cast<LW*>(lookback) + static_cast<size_t>(slot) * num_tiles * kRadix;
    constexpr uint32_t kSlotVec = Smem::kSlotVec;
    // A staged slot follows the global index: slot == index + mis (mod kSlotVec), mis = the element index of
    // the output's first element within its 16-byte block.  Keys only: the key array's phase (2 or 4 keys per
    // block).  With a payload: u32 keys use the key array's phase, u64 keys the payload array's (4 per block);
    // the other array leaves by bulk copies too when its phase agrees, else by plain stores.
    const uint32_t mis_k = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) / sizeof(K)) & (kVec - 1);
    const uint64_t pol = ISORT_POL_STREAM;
#ifndef ISORT_T_POL_EDGE
#define ISORT_T_POL_EDGE pol
#endif
    const uint64_t pol_edge = ISORT_T_POL_EDGE;  // the run-edge stores (partial sectors their neighbours complete)
    const uint32_t* vsrc = src_id == kBufIn ? vals_in : (src_id == kBufOut ? vals_out : vals_alt);
    uint32_t* vdst = dst_id == kBufOut ? vals_out : vals_alt;
    const bool gen_iota = VALS && iota_vals && slot == 0;  // the first executed pass generates positions
    const uint32_t mis_v = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(vdst) / 4) & 3u;
    const uint32_t mis = (VALS && sizeof(K) == 8) ? mis_v : mis_k;
    const bool kbulk = !(VALS && sizeof(K) == 8) || ((mis_v ^ mis_k) & (kVec - 1)) == 0;
    const bool vbulk = VALS && (sizeof(K) == 8 || mis_v == mis_k);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint32_t wofs = static_cast<uint32_t>(warp) * 32u * IPT + lane;
    uint32_t* const wc = sm.cnt[warp];
    if (tid < kRadix) sm.offs[tid] = st->offs[pos][tid];
    if (tid == 0) sm.tile_next = atomicAdd(&st->tile_ticket[slot], 1u);
    {
        uint4* c4 = reinterpret_cast<uint4*>(&sm.cnt[0][0]);
        for (int i = tid; i < kWarps * kRadix / 4; i += BLOCK) c4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();

    auto len_of = [&](uint32_t t) -> uint32_t {
        if (t >= num_tiles) return 0u;
        const uint64_t b = static_cast<uint64_t>(t) * kTile;
        if (b >= n) return 0u;
        return n - b < static_cast<uint64_t>(kTile) ? static_cast<uint32_t>(n - b) : static_cast<uint32_t>(kTile);
    };
    uint32_t tile = sm.tile_next;
    uint32_t tile_len = len_of(tile);
    K key[IPT];
    uint32_t val[VALS ? IPT : 1];
    constexpr bool kCache = ISORT_T_DIGIT_CACHE && CachesDigit<Dz>::value && IPT % 4 == 0;
    uint32_t dpk[kCache ? IPT / 4 : 1] = {};  // the tile's digits, four per register
    auto put_digit = [&](int i, uint32_t d) {
        if constexpr (kCache) dpk[i / 4] = (i % 4 == 0) ? d : (dpk[i / 4] | (d << (8 * (i % 4))));
    };
    auto get_digit = [&](int i, K k) -> uint32_t {
        if constexpr (kCache) return (dpk[i / 4] >> (8 * (i % 4))) & 0xFFu;
        return dz.digit_sh(k, dsh);
    };
    auto load_tile = [&](uint32_t t, uint32_t len) {  // warp-striped: (item, lane) order = input order
        const uint64_t tb = static_cast<uint64_t>(t < num_tiles ? t : 0u) * kTile;
        const K* ws = src + tb + wofs;
        if (len == static_cast<uint32_t>(kTile)) {  // a whole tile: no per-key bounds
#pragma unroll
            for (int i = 0; i < IPT; ++i) key[i] = ldg_hint(ws + i * 32, pol);
            if constexpr (VALS) {
                if (gen_iota) {
#pragma unroll
                    for (int i = 0; i < IPT; ++i) val[i] = static_cast<uint32_t>(tb + wofs + i * 32u);
                } else {
#pragma unroll
                    for (int i = 0; i < IPT; ++i) val[i] = ldg_stream(vsrc + tb + wofs + i * 32u);
                }
            }
            return;
        }
#pragma unroll
        for (int i = 0; i < IPT; ++i) key[i] = wofs + i * 32u < len ? ldg_hint(ws + i * 32, pol) : static_cast<K>(0);
        if constexpr (VALS) {
#pragma unroll
            for (int i = 0; i < IPT; ++i)
                val[i] = gen_iota ? static_cast<uint32_t>(tb + wofs + i * 32u)
                                  : (wofs + i * 32u < len ? ldg_stream(vsrc + tb + wofs + i * 32u) : 0u);
        }
    };
    load_tile(tile, tile_len);

#ifdef ISORT_PHASE_TIMING
    long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long q0 = 0, q1 = 0, q2 = 0, q3 = 0, q4 = 0, qa = 0, qb = 0, qc = 0, qd = 0, qe = 0;
#define ISORT_TTICK(v) \
    if (tid == 0) v = clock64()
#else
#define ISORT_TTICK(v)
#endif
    // Write-out of digit d's run of the tile of parity p -> dst[run_g, run_g + run_len): thread d
    // issues the bulk copy of its aligned interior, thread kRadix + d stores the keys
    // around it (the same split inside every warp, or the write-out before the loads,
    // measured no faster).
    auto write_run = [&](int p, int d, bool copier, bool edges) {
        const uint32_t run_len = sm.run_len[p][d];
        if (run_len != 0) {
            const uint32_t run_g = sm.run_g[p][d];
            const K* sp = sm.keys + sm.run_slot[p][d];
            K* gp = dst + run_g;
            {  // keys: head up to the first 16-byte boundary, bulk-copied interior, tail
                uint32_t head = (kVec - ((run_g + mis_k) & (kVec - 1))) & (kVec - 1);
                head = head < run_len ? head : run_len;
                const uint32_t body = kbulk ? (run_len - head) & ~(kVec - 1) : 0u;
                if (!kbulk) head = 0;
                if (copier && body) bulk_s2g(gp + head, sp + head, body * static_cast<uint32_t>(sizeof(K)));
                if (edges) {
                    for (uint32_t i = 0; i < head; ++i) stg_hint(gp + i, sp[i], pol_edge);
                    for (uint32_t i = head + body; i < run_len; ++i) stg_hint(gp + i, sp[i], pol_edge);
                }
            }
            if constexpr (VALS) {
                const uint32_t* vp = sm.vals + sm.run_slot[p][d];
                uint32_t* vg = vdst + run_g;
                uint32_t head = (4u - ((run_g + mis_v) & 3u)) & 3u;
                head = head < run_len ? head : run_len;
                const uint32_t body = vbulk ? (run_len - head) & ~3u : 0u;
                if (!vbulk) head = 0;
                if (copier && body) bulk_s2g(vg + head, vp + head, body * 4u);
                if (edges) {
                    for (uint32_t i = 0; i < head; ++i) stg_hint(vg + i, vp[i], pol_edge);
                    for (uint32_t i = head + body; i < run_len; ++i) stg_hint(vg + i, vp[i], pol_edge);
                }
            }
        }
    };
    auto write_out = [&](int p) {
        constexpr bool kSplit = BLOCK >= 2 * kRadix;  // else thread d does both
        if (tid < (kSplit ? 2 * kRadix : kRadix)) write_run(p, tid & (kRadix - 1), tid < kRadix, tid >= kRadix || !kSplit);
    };
    int par = 0;             // parity of the tile being counted / ranked
    bool have_prev = false;  // LATE_WRITE: a staged tile (parity par ^ 1) still waits for its write-out
    bool hot_prev = false;  // the count guesses from this CTA's previous tile
    while (tile_len != 0) {
        ISORT_TTICK(q0);
        const bool full = tile_len == static_cast<uint32_t>(kTile);
        // ---------------- count: per-warp digit counts of the keys in registers
        if (full && hot_prev) {
            bool agg = true;
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const uint32_t d = dz.digit_sh(key[i], dsh);
                put_digit(i, d);
                count_digit_t<true>(wc, d, agg);
            }
        } else if (full) {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const uint32_t d = dz.digit_sh(key[i], dsh);
                put_digit(i, d);
                atomicAdd(&wc[d], 1u);
            }
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const uint32_t d = dz.digit_sh(key[i], dsh);
                put_digit(i, d);
                if (wofs + i * 32u < tile_len) atomicAdd(&wc[d], 1u);
            }
        }
        __syncthreads();
        ISORT_TTICK(q1);

        // ---------------- one thread per digit: total, look-back, aligned run start, slot bases
        int nonzero = 0;
#if ISORT_T_LATE_WRITE
        if (tid >= kRadix && have_prev) write_out(par ^ 1);  // the previous tile's run edges
#endif
        if (tid < kRadix) {
            ISORT_TTICK(qa);
#if !ISORT_T_LATE_WRITE
            bulk_wait_read();  // the previous tile's copies have read the staging buffer
#endif
            ISORT_TTICK(qb);
            const int d = tid;
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) tot += sm.cnt[w][d];
            nonzero = tot != 0;
            ISORT_TTICK(qd);
#if ISORT_T_LATE_WRITE
            // the previous tile leaves between this tile's publication and its walk: the
            // copies are issued while the predecessors this walk needs are still publishing
            if (tile == 0) st_relaxed_gpu(&lb[d], LT::kInc | tot);
            else st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + d], LT::kAgg | tot);
            if (have_prev) write_out(par ^ 1);
#endif
            uint32_t excl = 0;
            if (tile == 0) {
                if (!ISORT_T_LATE_WRITE) st_relaxed_gpu(&lb[d], LT::kInc | tot);
            } else {
                if (!ISORT_T_LATE_WRITE) st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + d], LT::kAgg | tot);
#ifdef ISORT_LB_STATS
                unsigned long long lbst[3] = {0, 0, 0};
                excl = lookback_digit<LW, kLookbackWindowT>(lb, static_cast<int>(tile) - 1, d, 0u, lbst);
                if (tid == 0) {
                    atomicAdd(&st->prof[8], lbst[0]);
                    atomicAdd(&st->prof[9], lbst[1]);
                    atomicAdd(&st->prof[10], lbst[2]);
                    atomicAdd(&st->prof[11], 1ull);
                }
#else
                excl = lookback_digit<LW, kLookbackWindowT>(lb, static_cast<int>(tile) - 1, d, 0u);
#endif
                st_relaxed_gpu(&lb[static_cast<size_t>(tile) * kRadix + d], LT::kInc | (excl + tot));
            }
            ISORT_TTICK(qc);
#if ISORT_T_LATE_WRITE
            bulk_wait_read();  // the previous tile's copies have read the staging buffer
#endif
            const uint32_t sc = warp_inclusive_scan(tot);
            if (lane == 31) sm.tot_w[warp] = sc;
            if (BLOCK == kRadix)
                __syncthreads();
            else
                asm volatile("bar.sync 1, %0;" ::"n"(kRadix));
            uint32_t pre = 0;
#pragma unroll
            for (int w = 0; w < kRadix / 32; ++w) pre += w < warp ? sm.tot_w[w] : 0u;
            const uint32_t run_g = sm.offs[d] + excl;
            uint32_t base = pre + sc - tot + kSlotVec * static_cast<uint32_t>(d);
            base += (run_g + mis - base) & (kSlotVec - 1);  // slot == global index + mis (mod kSlotVec)
            sm.run_slot[par][d] = base;
            sm.run_len[par][d] = tot;
            sm.run_g[par][d] = run_g;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {  // per-warp slot bases for the rank
                const uint32_t v = sm.cnt[w][d];
                sm.cnt[w][d] = base;
                base += v;
            }
        }
        const bool hot = __syncthreads_count(nonzero) <= kHotDigits;
        hot_prev = hot;
        ISORT_TTICK(q2);

        // ---------------- rank and stage
        if (full && hot) {
            bool agg = true;
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const uint32_t s = warp_slot_agg<SAFE>(wc, get_digit(i, key[i]), agg);
                sm.keys[s] = key[i];
                if constexpr (VALS) sm.vals[s] = val[i];
            }
        } else if (full) {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const uint32_t s = warp_slot<SAFE>(wc, get_digit(i, key[i]));
                sm.keys[s] = key[i];
                if constexpr (VALS) sm.vals[s] = val[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                if (wofs + i * 32u < tile_len) {
                    const uint32_t s = warp_slot<SAFE>(wc, get_digit(i, key[i]));
                    sm.keys[s] = key[i];
                    if constexpr (VALS) sm.vals[s] = val[i];
                }
            }
        }
        // the next ticket is taken late, as in K3: a tile's aggregate follows its ticket by
        // one count phase, so the look-back of the tiles behind it finds it published
        if (tid == 0) sm.tile_next = atomicAdd(&st->tile_ticket[slot], 1u);
        __syncwarp();
        {  // this warp's counters are done: zero them for its next count (no other warp reads them before)
            uint4* r = reinterpret_cast<uint4*>(wc);
#pragma unroll
            for (int q = 0; q < kRadix / 4 / 32; ++q) r[lane + 32 * q] = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();  // the staging stores, visible to the bulk copies
        __syncthreads();
        ISORT_TTICK(q3);
        const uint32_t next = sm.tile_next;
        const uint32_t next_len = len_of(next);
        load_tile(next, next_len);  // the next tile: in flight during the next count

#if !ISORT_T_LATE_WRITE
        write_out(par);
#endif
        par ^= 1;
        have_prev = true;
        tile = next;
        tile_len = next_len;
        ISORT_TTICK(q4);
#ifdef ISORT_PHASE_TIMING
        acc[0] += q1 - q0;  // count
        acc[1] += q2 - q1;  // per-digit section
        acc[2] += q3 - q2;  // rank + next loads
        acc[3] += 1;
        acc[4] += q4 - q3;  // write-out (thread 0's run)
        acc[5] += qb - qa;  // wait for the previous copies
        acc[6] += qc - qb;  // totals + look-back
        acc[7] += qd - qb;  // totals (the count's atomics drain first)
#endif
    }
#ifdef ISORT_PHASE_TIMING
    if (tid == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(&st->prof[i], static_cast<unsigned long long>(acc[i]));
#endif
#undef ISORT_TTICK
#if ISORT_T_LATE_WRITE
    if (have_prev) write_out(par ^ 1);  // the last tile (staged before the loop's final barrier)
#endif
    if (tid < kRadix) bulk_wait_all();  // this CTA's bulk stores complete before it exits
}

}  // namespace isort
