// bucket_sort.cuh -- bucket sort (n buckets over [0, M]) for sm_100a.
//
// Reference semantics: intsort::bucket_sort (proj/core/src/sort.cpp:136-152):
// n buckets, record r goes to bucket_index(r.key, n, M) = floor(n*key/(M+1))
// (sort.cpp:121-134, 128-bit product), arrival order kept inside a bucket,
// each bucket insertion-sorted (stable, sort.cpp:15-25), buckets concatenated.
// The result is the unique stable sort by key; a key > M throws
// std::invalid_argument naming that key (sort.cpp:125-129).
//
// Device pipeline:
//   K1  k_upfront (shared with radix) with BucketDigitizer: range check (first
//       offending position), sortedness, histograms of the top 8-bit digits of
//       the bucket index b.                                            4n B
//   K3  D_b stable one-sweep passes (low digit first) scatter the keys into
//       contiguous super-buckets: runs of 2^s_lo consecutive buckets (the top
//       8*D_b bits of b), bucket order, arrival order kept.    D_b x 8n B
//       D_b = ceil((L - 11) / 8) for L = bits(n - 1): a super-bucket covers
//       <= 2^11 buckets (~2K keys on average).
//   K5  k_bucket_windows: each CTA owns the super-buckets that START in its
//       window, stages them (plus up to kCap keys of overhang) in shared memory
//       and sorts them stably by key.  A stable sort of whole buckets laid out
//       in bucket order equals per-bucket insertion sort + concatenation,
//       because bucket_index is monotone in the key.                    8n B
//   K6  k_resolve_oversized: a super-bucket longer than a window's reach is
//       resolved from per-window summaries (boundary, min, max); one that
//       holds a single key value is already in arrival order, the others mark
//       a span that the radix pipeline re-sorts ("oversized buckets go to the
//       radix kernel").
#pragma once

#include "isort_common.cuh"
#include "radix_onesweep.cuh"

namespace isort {

// ------------------------------------------------------ bucket index
// b(key) = floor(count * key / (M + 1)) exactly as bucket_index computes it
// with unsigned __int128 (sort.cpp:131-133).
struct BucketIndexer {
    uint64_t count;       // number of buckets (= n)
    uint64_t bound;       // M (inclusive range bound)
    uint64_t div;         // M + 1 when it fits in 64 bits
    uint64_t magic;       // floor((2^64 - 1) / div), general path
    uint32_t pow2_shift;  // M + 1 == 2^pow2_shift (0..64), 255 otherwise

    static BucketIndexer make(uint64_t count, uint64_t bound) {
        BucketIndexer b{};
        b.count = count;
        b.bound = bound;
        if (bound == ~0ull) {
            b.pow2_shift = 64;
        } else {
            b.div = bound + 1;
            if ((b.div & (b.div - 1)) == 0) {
                b.pow2_shift = static_cast<uint32_t>(__builtin_ctzll(b.div));
            } else {
                b.pow2_shift = 255;
                b.magic = ~0ull / b.div;
            }
        }
        return b;
    }

    // Keys above M are clamped into the last bucket so the device passes stay
    // in bounds; k_upfront's range check reports them.
    __host__ __device__ __forceinline__ uint64_t bucket(uint64_t key) const {
        if (key > bound) return count - 1;
#ifdef __CUDA_ARCH__
        const uint64_t hi = __umul64hi(count, key);
#else
        const uint64_t hi = static_cast<uint64_t>((static_cast<unsigned __int128>(count) * key) >> 64);
#endif
        const uint64_t lo = count * key;
        if (pow2_shift != 255) {
            if (pow2_shift == 64) return hi;
            if (pow2_shift == 0) return lo;
            return (lo >> pow2_shift) | (hi << (64 - pow2_shift));
        }
        if (hi == 0) {
#ifdef __CUDA_ARCH__
            uint64_t q = __umul64hi(lo, magic);  // floor(lo/div) - 2 <= q <= floor(lo/div)
#else
            uint64_t q = static_cast<uint64_t>((static_cast<unsigned __int128>(lo) * magic) >> 64);
#endif
            uint64_t r = lo - q * div;
            while (r >= div) {
                ++q;
                r -= div;
            }
            return q;
        }
        // 128-by-64 division; the quotient is < count because key <= M.
        // Floating estimate, then exact integer correction.
        const double approx = (static_cast<double>(hi) * 18446744073709551616.0 + static_cast<double>(lo)) /
                              static_cast<double>(div);
        uint64_t q = approx <= 0.0 ? 0ull : (approx >= 1.8e19 ? count - 1 : static_cast<uint64_t>(approx));
        if (q >= count) q = count - 1;
        for (;;) {  // while q*div > p: --q
#ifdef __CUDA_ARCH__
            const uint64_t phi = __umul64hi(q, div);
#else
            const uint64_t phi = static_cast<uint64_t>((static_cast<unsigned __int128>(q) * div) >> 64);
#endif
            const uint64_t plo = q * div;
            if (phi > hi || (phi == hi && plo > lo)) {
                --q;
                continue;
            }
            break;
        }
        for (;;) {  // while (q+1)*div <= p: ++q
            const uint64_t q1 = q + 1;
#ifdef __CUDA_ARCH__
            const uint64_t phi = __umul64hi(q1, div);
#else
            const uint64_t phi = static_cast<uint64_t>((static_cast<unsigned __int128>(q1) * div) >> 64);
#endif
            const uint64_t plo = q1 * div;
            if (phi < hi || (phi == hi && plo <= lo)) {
                q = q1;
                continue;
            }
            break;
        }
        return q;
    }
};

// Divisor kinds, chosen on the host once per call (compile-time in the kernels):
//   kPow2Narrow   count * key < 2^64 and M + 1 = 2^s: one 64-bit multiply and a shift
//   kMagicNarrow  count * key < 2^64: 64-bit magic reciprocal + <= 2 corrections
//   kWide         general 128-by-64 division (BucketIndexer::bucket)
enum BucketMode : int { kPow2Narrow = 0, kMagicNarrow = 1, kWide = 2 };

template <int MODE>
__device__ __forceinline__ uint64_t bucket_of(const BucketIndexer& bi, uint64_t key) {
    if (MODE == kWide) return bi.bucket(key);
    if (key > bi.bound) return bi.count - 1;
    const uint64_t p = bi.count * key;  // exact: narrow modes guarantee < 2^64
    if (MODE == kPow2Narrow) return bi.pow2_shift >= 64 ? 0ull : p >> bi.pow2_shift;
    uint64_t q = __umul64hi(p, bi.magic);
    uint64_t r = p - q * bi.div;
    if (r >= bi.div) {
        ++q;
        r -= bi.div;
    }
    if (r >= bi.div) ++q;
    return q;
}

inline int choose_bucket_mode(uint64_t count, uint64_t bound, uint64_t key_max) {
    const uint64_t kmax = bound < key_max ? bound : key_max;
    const bool narrow = static_cast<unsigned __int128>(count) * kmax < (static_cast<unsigned __int128>(1) << 64);
    if (!narrow) return kWide;
    const bool pow2 = bound == ~0ull || ((bound + 1) & bound) == 0;
    return pow2 ? kPow2Narrow : kMagicNarrow;
}

constexpr int kBucketMaxDigits = 3;
constexpr uint32_t kSuperBucketBits = 11;  // super-bucket = up to 2^11 consecutive buckets

template <typename K, int MODE = kWide>
struct BucketDigitizer {
    static constexpr int kDigits = kBucketMaxDigits;
    static constexpr bool kChecks = true;
    static constexpr bool kCheapDigit = false;
    BucketIndexer bi;
    uint32_t shift[kBucketMaxDigits];  // digit p = (b >> shift[p]) & 255; unused: 63 (=> 0)
    uint32_t s_lo;                     // super-bucket = b >> s_lo
    uint32_t used;                     // number of digit passes that can be non-trivial

    static BucketDigitizer make(uint64_t n, uint64_t bound) {
        BucketDigitizer d{};
        d.bi = BucketIndexer::make(n, bound);
        const uint32_t L = n > 1 ? 64 - __builtin_clzll(n - 1) : 0;  // bits of the largest bucket index
        uint32_t db = L > kSuperBucketBits ? (L - kSuperBucketBits + 7) / 8 : 0;
        if (db > kBucketMaxDigits) db = kBucketMaxDigits;
        d.used = db;
        d.s_lo = L > 8 * db ? L - 8 * db : 0;
        for (uint32_t p = 0; p < kBucketMaxDigits; ++p) d.shift[p] = p < db ? d.s_lo + 8 * p : 63;
        return d;
    }
    __device__ __forceinline__ uint32_t digit_of_bucket(uint64_t b, int pos) const {
        return static_cast<uint32_t>(b >> shift_for(pos)) & (kRadix - 1);
    }
    __device__ __forceinline__ uint32_t shift_for(int pos) const {
        return pos == 0 ? shift[0] : (pos == 1 ? shift[1] : shift[2]);
    }
    __device__ __forceinline__ uint32_t digit_sh(K key, uint32_t sh) const {
        return static_cast<uint32_t>(bucket_of<MODE>(bi, static_cast<uint64_t>(key)) >> sh) & (kRadix - 1);
    }
    __device__ __forceinline__ uint32_t digit(K key, int pos) const { return digit_sh(key, shift_for(pos)); }
    __device__ __forceinline__ void all_digits(K key, uint32_t (&d)[kDigits]) const {
        const uint64_t b = bucket_of<MODE>(bi, static_cast<uint64_t>(key));
#pragma unroll
        for (int p = 0; p < kDigits; ++p) d[p] = static_cast<uint32_t>(b >> shift[p]) & (kRadix - 1);
    }
    __device__ __forceinline__ bool in_range(K key) const { return static_cast<uint64_t>(key) <= bi.bound; }
    __device__ __forceinline__ uint64_t bucket(K key) const { return bucket_of<MODE>(bi, static_cast<uint64_t>(key)); }
    __device__ __forceinline__ uint64_t super_bucket(K key) const {
        return bucket_of<MODE>(bi, static_cast<uint64_t>(key)) >> s_lo;
    }
};

// -------------------------------------------------------- bucket state
struct BucketState {
    unsigned long long span_lo_not;  // ~(min start) of non-constant oversized super-buckets
    unsigned long long span_hi;      // max end
    uint32_t oversized;              // non-constant oversized super-buckets
    uint32_t n_over;                 // oversized records written by K5
};

struct OverRec {
    unsigned long long start;  // absolute start of the trailing oversized super-bucket
    unsigned long long kmin, kmax;  // over the part the owner staged
    uint32_t window;
    uint32_t pad;
};

template <typename K>
struct WindowSummary {  // per window: first super-bucket start, min/max of the keys before it
    unsigned long long first;  // absolute, or ~0 if no super-bucket starts in the window
    unsigned long long hmin, hmax;
};

// ------------------------------------------------------------------ K5
template <int BLOCK, int IPT>
struct WindowCfg {
    static constexpr int kStage = BLOCK * IPT;  // keys staged per CTA
    static constexpr int kWindow = kStage / 2;  // owned range; reach = 1 window (super-buckets ~2K keys)
    static constexpr int kCap = kStage - kWindow;  // reach past the window
    static constexpr int kWarps = BLOCK / 32;
};

constexpr int kWinDigitBits = 9;  // window sort digit width (<= 9 bits: 512 bins)
constexpr int kWinBins = 1 << kWinDigitBits;
static_assert(kWinBins % 256 == 0 || kWinBins <= 256, "bins split evenly over the window CTA");

template <typename K, int BLOCK, int IPT, bool VALS>
struct WindowSmem {
    K keys[BLOCK * IPT];
    K keys2[BLOCK * IPT];  // ping-pong buffer of the in-smem sort
    uint32_t vals[VALS ? BLOCK * IPT : 1];
    uint32_t vals2[VALS ? BLOCK * IPT : 1];
    uint32_t cnt[BLOCK / 32][kWinBins];  // per-warp digit counters, then slot bases
    uint32_t scan_tot[BLOCK / 32];
    unsigned long long red_a[BLOCK / 32], red_b[BLOCK / 32];
    unsigned long long red6[6][BLOCK / 32];
    uint32_t prev_sb;
    int first, last, end;
};

template <typename T>
__device__ __forceinline__ T block_max_u64(T v, unsigned long long* red, int warps) {
    unsigned long long x = warp_max<unsigned long long>(static_cast<unsigned long long>(v));
    __syncthreads();
    if (lane_id() == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    x = 0;
    for (int w = 0; w < warps; ++w) x = red[w] > x ? red[w] : x;
    return static_cast<T>(x);
}

// Block-wide (min, max) of K values in one barrier pair.
template <typename K>
__device__ __forceinline__ void block_minmax(K lo, K hi, unsigned long long* ra, unsigned long long* rb, int warps,
                                             unsigned long long& out_lo, unsigned long long& out_hi) {
    const unsigned long long a = warp_max<unsigned long long>(~static_cast<unsigned long long>(lo));
    const unsigned long long b = warp_max<unsigned long long>(static_cast<unsigned long long>(hi));
    __syncthreads();
    if (lane_id() == 0) {
        ra[threadIdx.x >> 5] = a;
        rb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    unsigned long long x = 0, y = 0;
    for (int w = 0; w < warps; ++w) {
        x = ra[w] > x ? ra[w] : x;
        y = rb[w] > y ? rb[w] : y;
    }
    out_lo = ~x;
    out_hi = y;
}

// First index in [lo, hi) where the monotone predicate holds, or hi.  Called by a
// whole warp: 32 probes per round narrow the range 32x.
template <typename Pred>
__device__ __forceinline__ int warp_lower_bound(int lo, int hi, Pred pred) {
    // invariant: answer in [lo, hi]; pred(hi) is taken as true
    while (lo < hi) {
        const int step = (hi - lo + 31) / 32;
        const int idx = lo + static_cast<int>(lane_id()) * step;
        const bool p = idx >= hi || pred(idx);
        const uint32_t ball = __ballot_sync(ISORT_FULL_MASK, p);
        const int f = __ffs(ball) - 1;  // lane 31 probe may be < hi; ball can be 0
        if (ball == 0) {
            lo = lo + 31 * step + 1;
            continue;
        }
        if (f == 0) return lo;
        const int nlo = lo + (f - 1) * step + 1;
        const int nhi = min(lo + f * step, hi);
        if (step == 1) return nhi;
        lo = nlo;
        hi = nhi;
    }
    return hi;
}

template <typename K, typename Dz, int BLOCK, int IPT, bool VALS>
__global__ void __launch_bounds__(BLOCK, 1024 / BLOCK) k_bucket_windows(K* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t n,
                                                          const RadixState* __restrict__ rst,
                                                          BucketState* __restrict__ bst,
                                                          WindowSummary<K>* __restrict__ summ,
                                                          OverRec* __restrict__ over, Dz dz) {
    using Cfg = WindowCfg<BLOCK, IPT>;
    using Smem = WindowSmem<K, BLOCK, IPT, VALS>;
    constexpr int kStage = Cfg::kStage, kWindow = Cfg::kWindow, kWarps = Cfg::kWarps;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    if (rst->descents == 0 || rst->first_bad != 0) return;  // sorted input / range error: nothing to do

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kWindow;
    const int avail = static_cast<int>((n - w0 < static_cast<uint64_t>(kStage) ? n - w0 : static_cast<uint64_t>(kStage)));
    const int wlen = min(kWindow, avail);

#ifdef ISORT_PHASE_TIMING
    long long t0 = clock64(), t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    unsigned long long* prof = const_cast<unsigned long long*>(rst->prof);
#define WTICK(v) v = clock64()
#define WFLUSH(k)                                                                      \
    if (tid == 0) {                                                                    \
        const long long tn = clock64();                                                \
        atomicAdd(prof + 8, (unsigned long long)((t1 ? t1 : tn) - t0));               \
        if (t1) atomicAdd(prof + 9, (unsigned long long)((t2 ? t2 : tn) - t1));       \
        if (t2) atomicAdd(prof + 10, (unsigned long long)((t3 ? t3 : tn) - t2));      \
        if (t3) atomicAdd(prof + 11, (unsigned long long)((t4 ? t4 : tn) - t3));      \
        if (t4) atomicAdd(prof + 12, (unsigned long long)(tn - t4));                  \
        atomicAdd(prof + 13 + (k), 1ull);                                              \
    }
#else
#define WTICK(v)
#define WFLUSH(k)
#endif
    // ---- stage [w0, w0 + avail); super-bucket id (low 32 bits: adjacent ids differ
    // by far less than 2^32, so equality is exact) kept per position in sm.keys2
    uint32_t* sbuf = reinterpret_cast<uint32_t*>(sm.keys2);
    {
        K stage[IPT];
        uint32_t vstage[VALS ? IPT : 1];
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int j = tid + i * BLOCK;
            if (j < avail) {
                stage[i] = keys[w0 + j];
                if (VALS) vstage[i] = vals[w0 + j];
            }
        }
        if (tid == 0) sm.prev_sb = w0 ? static_cast<uint32_t>(dz.super_bucket(keys[w0 - 1])) : 0u;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int j = tid + i * BLOCK;
            if (j < avail) {
                sm.keys[j] = stage[i];
                sbuf[j] = static_cast<uint32_t>(dz.super_bucket(stage[i]));
                if (VALS) sm.vals[j] = vstage[i];
            }
        }
    }
    __syncthreads();
    WTICK(t1);
    // ---- super-bucket starts (all threads): first/last start in [0, wlen), first start in [wlen, avail)
    {
        int my_first = 0x7fffffff, my_last = -1, my_end = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int j = tid + i * BLOCK;
            if (j < avail) {
                const bool start = (w0 + j == 0) || sbuf[j] != (j ? sbuf[j - 1] : sm.prev_sb);
                if (start) {
                    if (j < wlen) {
                        my_first = min(my_first, j);
                        my_last = max(my_last, j);
                    } else {
                        my_end = min(my_end, j);
                    }
                }
            }
        }
        my_first = __reduce_min_sync(ISORT_FULL_MASK, my_first);
        my_last = __reduce_max_sync(ISORT_FULL_MASK, my_last);
        my_end = __reduce_min_sync(ISORT_FULL_MASK, my_end);
        if (tid == 0) {
            sm.first = 0x7fffffff;
            sm.last = -1;
            sm.end = 0x7fffffff;
        }
        __syncthreads();
        if (lane == 0) {
            if (my_first != 0x7fffffff) atomicMin(&sm.first, my_first);
            if (my_last >= 0) atomicMax(&sm.last, my_last);
            if (my_end != 0x7fffffff) atomicMin(&sm.end, my_end);
        }
        __syncthreads();
    }
    WTICK(t2);
    const int first = min(sm.first, wlen);
    int end = min(sm.end, avail);
    const bool oversized = first < wlen && end == avail && w0 + avail < n;
    const int ostart = sm.last;
    if (oversized) end = ostart;  // the trailing super-bucket is resolved by K6
    // ---- one block reduction: head (before `first`), sort range, oversized tail
    K hmin = static_cast<K>(~static_cast<K>(0)), hmax = 0, rmin = hmin, rmax = 0, omin = hmin, omax = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const int j = tid + i * BLOCK;
        if (j < avail) {
            const K k = sm.keys[j];
            if (j < first) {
                hmin = k < hmin ? k : hmin;
                hmax = k > hmax ? k : hmax;
            } else if (j < end) {
                rmin = k < rmin ? k : rmin;
                rmax = k > rmax ? k : rmax;
            } else if (oversized) {
                omin = k < omin ? k : omin;
                omax = k > omax ? k : omax;
            }
        }
    }
    {
        unsigned long long v[6] = {~static_cast<unsigned long long>(hmin), hmax, ~static_cast<unsigned long long>(rmin),
                                   rmax, ~static_cast<unsigned long long>(omin), omax};
#pragma unroll
        for (int q = 0; q < 6; ++q) v[q] = warp_max<unsigned long long>(v[q]);
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < 6; ++q) sm.red6[q][warp] = v[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            unsigned long long x = 0;
            for (int w = 0; w < kWarps; ++w) x = sm.red6[q][w] > x ? sm.red6[q][w] : x;
            v[q] = x;
        }
        hmin = static_cast<K>(~v[0]);
        hmax = static_cast<K>(v[1]);
        rmin = static_cast<K>(~v[2]);
        rmax = static_cast<K>(v[3]);
        omin = static_cast<K>(~v[4]);
        omax = static_cast<K>(v[5]);
    }
    if (tid == 0) {
        summ[blockIdx.x].first = first < wlen ? w0 + first : ~0ull;
        summ[blockIdx.x].hmin = first > 0 ? static_cast<unsigned long long>(hmin) : ~0ull;
        summ[blockIdx.x].hmax = first > 0 ? static_cast<unsigned long long>(hmax) : 0ull;
        if (oversized) {
            const uint32_t r = atomicAdd(&bst->n_over, 1u);
            over[r].start = w0 + ostart;
            over[r].kmin = omin;
            over[r].kmax = omax;
            over[r].window = blockIdx.x;
        }
    }
    WTICK(t3);
    if (first >= wlen) {  // no super-bucket starts here
        WFLUSH(0);
        return;
    }
    const int len = end - first;
    if (len <= 1) {
        WFLUSH(1);
        return;
    }

    // ---- stable in-smem LSD sort of sm.keys[first, end) by (key - min), r-bit digits
    // Same rank primitive as the one-sweep pass: per-warp counters pre-scanned into
    // slot bases, slot = atomicAdd (lane-ordered, program-ordered => stable).
    const K kmin = rmin, kmax = rmax;
    WTICK(t4);
    if (kmin == kmax) {  // one key value: arrival order is the answer
        WFLUSH(1);
        return;
    }
    const int bits = 64 - __clzll(static_cast<unsigned long long>(kmax - kmin));
    const int passes = (bits + kWinDigitBits - 1) / kWinDigitBits;
    const int r = (bits + passes - 1) / passes;
    const uint32_t nbins = 1u << r, mask = nbins - 1u;
    K* ka = sm.keys + first;
    K* kb = sm.keys2;
    uint32_t* va = sm.vals + first;
    uint32_t* vb = sm.vals2;
    // items per thread sized to this window's range, so every warp has work
    const int ipt = (len + BLOCK - 1) / BLOCK;
    const int wofs = warp * 32 * ipt + static_cast<int>(lane);
    for (int pass = 0; pass < passes; ++pass) {
        const uint32_t shift = static_cast<uint32_t>(pass * r);
        for (int i = tid; i < kWarps * static_cast<int>(nbins); i += BLOCK)
            sm.cnt[i / static_cast<int>(nbins)][i % static_cast<int>(nbins)] = 0;
        __syncthreads();
        uint32_t* wc = sm.cnt[warp];
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int o = wofs + i * 32;
            if (i < ipt && o < len)
                atomicAdd(&wc[static_cast<uint32_t>((ka[o] - kmin) >> shift) & mask], 1u);
        }
        __syncthreads();
        // bins [tid*BPT, tid*BPT + BPT): totals over warps, block scan over bins, per-warp bases
        constexpr int BPT = kWinBins / BLOCK > 0 ? kWinBins / BLOCK : 1;
        uint32_t btot[BPT], tsum = 0;
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            const uint32_t b = static_cast<uint32_t>(tid * BPT + q);
            uint32_t t = 0;
            if (b < nbins) {
#pragma unroll 4
                for (int w = 0; w < kWarps; ++w) t += sm.cnt[w][b];
            }
            btot[q] = t;
            tsum += t;
        }
        const uint32_t inc = warp_inclusive_scan(tsum);
        if (lane == 31) sm.scan_tot[warp] = inc;
        __syncthreads();
        {
            uint32_t base = inc - tsum;
            for (int w = 0; w < warp; ++w) base += sm.scan_tot[w];
#pragma unroll
            for (int q = 0; q < BPT; ++q) {
                const uint32_t b = static_cast<uint32_t>(tid * BPT + q);
                if (b < nbins) {
                    uint32_t bb = base;
#pragma unroll 4
                    for (int w = 0; w < kWarps; ++w) {
                        const uint32_t v = sm.cnt[w][b];
                        sm.cnt[w][b] = bb;
                        bb += v;
                    }
                }
                base += btot[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int o = wofs + i * 32;
            if (i < ipt && o < len) {
                const K k = ka[o];
                const uint32_t slot = atomicAdd(&wc[static_cast<uint32_t>((k - kmin) >> shift) & mask], 1u);
                kb[slot] = k;
                if (VALS) vb[slot] = va[o];
            }
        }
        __syncthreads();
        K* tk = ka;
        ka = kb;
        kb = tk;
        uint32_t* tv = va;
        va = vb;
        vb = tv;
    }
    for (int j = tid; j < len; j += BLOCK) {
        keys[w0 + first + j] = ka[j];
        if (VALS) vals[w0 + first + j] = va[j];
    }
    WFLUSH(2);
#undef WTICK
#undef WFLUSH
}

// ------------------------------------------------------------------ K6
// One CTA per oversized record: walk the following windows' summaries until a
// super-bucket start appears; combine min/max.  Non-constant => mark the span.
template <typename K, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_resolve_oversized(const WindowSummary<K>* __restrict__ summ,
                                                             uint32_t num_windows, const OverRec* __restrict__ over,
                                                             BucketState* __restrict__ bst, uint64_t n) {
    __shared__ unsigned long long red_a[BLOCK / 32], red_b[BLOCK / 32], red_c[BLOCK / 32];
    const uint32_t nrec = bst->n_over;
    for (uint32_t r = blockIdx.x; r < nrec; r += gridDim.x) {
        const OverRec rec = over[r];
        unsigned long long kmin = rec.kmin, kmax = rec.kmax;
        unsigned long long end = n;
        for (uint32_t base = rec.window + 1; base < num_windows; base += BLOCK) {
            const uint32_t w = base + threadIdx.x;
            unsigned long long f = ~0ull, hmin = ~0ull, hmax = 0;
            if (w < num_windows) {
                f = summ[w].first;
                hmin = summ[w].hmin;
                hmax = summ[w].hmax;
            }
            // first window (lowest index) with a start
            unsigned long long fw = f != ~0ull ? static_cast<unsigned long long>(w) : ~0ull;
            fw = ~block_max_u64(~fw, red_c, BLOCK / 32);
            const bool take = w < num_windows && static_cast<unsigned long long>(w) <= fw;
            const unsigned long long a = block_max_u64(take ? ~hmin : 0ull, red_a, BLOCK / 32);
            const unsigned long long b = block_max_u64(take ? hmax : 0ull, red_b, BLOCK / 32);
            kmin = (~a) < kmin ? ~a : kmin;
            kmax = b > kmax ? b : kmax;
            if (fw != ~0ull) {
                end = summ[fw].first;
                break;
            }
        }
        if (threadIdx.x == 0 && kmin != kmax) {
            atomicAdd(&bst->oversized, 1u);
            atomicMax(&bst->span_lo_not, ~rec.start);
            atomicMax(&bst->span_hi, end);
        }
        __syncthreads();
    }
}

template <typename K>
__global__ void k_copy_range(const K* __restrict__ src, K* __restrict__ dst, const uint32_t* __restrict__ vsrc,
                             uint32_t* __restrict__ vdst, uint64_t count) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        dst[i] = src[i];
        if (vdst) vdst[i] = vsrc[i];
    }
}

}  // namespace isort

namespace isort {

// ------------------------------------------------------- key-range partition
// Destination rank of a key for the multi-GPU sort: the number of splitters
// <= key (splitters ascending), so rank r receives keys in [s_{r-1}, s_r).
// One stable pass of the one-sweep pipeline with this digitizer partitions a
// shard by destination while keeping input order inside each destination.
constexpr int kMaxParts = 64;

template <typename K>
struct DestDigitizer {
    static constexpr int kDigits = 1;
    static constexpr bool kChecks = false;
    static constexpr bool kCheapDigit = false;
    K split[kMaxParts - 1];
    int nsplit;
    __device__ __forceinline__ uint32_t shift_for(int) const { return 0u; }
    __device__ __forceinline__ uint32_t digit_sh(K key, uint32_t) const {
        uint32_t d = 0;
#pragma unroll 8
        for (int i = 0; i < kMaxParts - 1; ++i) {
            if (i >= nsplit) break;
            d += key >= split[i];
        }
        return d;
    }
    __device__ __forceinline__ uint32_t digit(K key, int) const { return digit_sh(key, 0u); }
    __device__ __forceinline__ void all_digits(K key, uint32_t (&d)[kDigits]) const { d[0] = digit_sh(key, 0u); }
    __device__ __forceinline__ bool in_range(K) const { return true; }
};

__global__ void k_copy_part_counts(const RadixState* __restrict__ st, uint64_t* __restrict__ counts, int parts) {
    if (threadIdx.x < parts) counts[threadIdx.x] = st->hist[0][threadIdx.x];
}

}  // namespace isort
