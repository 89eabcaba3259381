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
//   K5  k_bucket_segments: persistent CTAs, each owning the super-buckets that
//       start in its share of the array, stage them in shared memory a few
//       thousand keys at a time and sort them stably by key, in place.  A
//       stable sort of whole buckets laid out in bucket order equals
//       per-bucket insertion sort + concatenation, because bucket_index is
//       monotone in the key.                                            8n B
//       A super-bucket longer than the stage is oversized: one that holds a
//       single key value is already in arrival order, the others mark a span
//       that the radix pipeline re-sorts ("oversized buckets go to the radix
//       kernel").
#pragma once

#include "isort_common.cuh"
#include "radix_onesweep.cuh"

namespace isort {

// ------------------------------------------------------ bucket index
// b(key) = floor(count * key / (M + 1)) exactly as bucket_index computes it
// with unsigned __int128 (sort.cpp:131-133).  `base` generalises the range to
// [base, M]: b = floor(count * (key - base) / (M - base + 1)).  The reference
// API always has base = 0; the multi-GPU local sort (one key range per rank)
// uses its range's lower end so the n buckets cover the keys it holds.
struct BucketIndexer {
    uint64_t count;       // number of buckets (= n)
    uint64_t bound;       // M (inclusive range bound)
    uint64_t base;        // lower end of the range (0 for the reference API)
    uint64_t span;        // M - base
    uint64_t div;         // M - base + 1 when it fits in 64 bits
    uint64_t magic;       // floor((2^64 - 1) / div), general path
    uint64_t qi, qf;      // count = qi * div + c', qf = ceil(2^64 * c' / div): b = k*qi + mulhi(k, qf)
    uint32_t pow2_shift;  // M - base + 1 == 2^pow2_shift (0..64), 255 otherwise
    uint32_t div32;       // count and div both < 2^32: the 32-bit reciprocal path applies

    static BucketIndexer make(uint64_t count, uint64_t bound, uint64_t base = 0) {
        BucketIndexer b{};
        b.count = count;
        b.bound = bound;
        b.base = base;
        const uint64_t span = bound - base;
        b.span = span;
        if (span == ~0ull) {
            b.pow2_shift = 64;
        } else {
            b.div = span + 1;
            b.magic = ~0ull / b.div;  // also for a power-of-two span: kMagicNarrow serves every base != 0
            b.qi = count / b.div;
            const unsigned __int128 num = static_cast<unsigned __int128>(count % b.div) << 64;
            b.qf = static_cast<uint64_t>(num / b.div) + (num % b.div != 0 ? 1u : 0u);  // < 2^64: c' < div
            b.div32 = b.div <= 0xFFFFFFFFull && count <= 0xFFFFFFFFull ? 1u : 0u;
            b.pow2_shift = (b.div & (b.div - 1)) == 0 ? static_cast<uint32_t>(__builtin_ctzll(b.div)) : 255u;
        }
        return b;
    }

    // Keys above M are clamped into the last bucket so the device passes stay
    // in bounds; k_upfront's range check reports them.
    __host__ __device__ __forceinline__ uint64_t bucket(uint64_t key) const {
        if (key > bound) return count - 1;
        if (key < base) return 0;
        key -= base;
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
        // 128-by-64 division; the quotient is < count because key - base <= M - base.
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
//   kPow2Narrow   count * key < 2^64, base 0 and M + 1 = 2^s: one 64-bit multiply and a shift
//   kMagicNarrow  count * (key - base) < 2^64: 64-bit magic reciprocal + <= 2 corrections
//   kWide         general 128-by-64 division (BucketIndexer::bucket)
enum BucketMode : int { kPow2Narrow = 0, kMagicNarrow = 1, kWide = 2 };

template <int MODE>
__device__ __forceinline__ uint64_t bucket_of(const BucketIndexer& bi, uint64_t key) {
    if (MODE == kWide) return bi.bucket(key);
    if (MODE == kPow2Narrow) {  // n * (key - base) < 2^64 (choose_bucket_mode)
        if (key - bi.base > bi.span) return key > bi.bound ? bi.count - 1 : 0;
        return bi.pow2_shift >= 64 ? 0ull : (bi.count * (key - bi.base)) >> bi.pow2_shift;
    }
    const uint64_t k = key - bi.base;
    if (k > bi.span) return key > bi.bound ? bi.count - 1 : 0;  // outside [base, M]: clamped
    const uint64_t p = bi.count * k;  // exact: narrow modes guarantee < 2^64
    uint64_t q = __umul64hi(p, bi.magic);
    uint64_t r = p - q * bi.div;
    if (r >= bi.div) {
        ++q;
        r -= bi.div;
    }
    if (r >= bi.div) ++q;
    return q;
}

// u32 keys always sort on a power-of-two bucket grid (kPow2Narrow, see
// BucketDigitizer::make): n < 2^32 and key - base < 2^32 keep n * (key - base)
// below 2^64 for every range [base, M].
inline int choose_bucket_mode(uint64_t count, uint64_t bound, uint64_t key_max, uint64_t base = 0) {
    if (key_max <= 0xFFFFFFFFull) return kPow2Narrow;
    const uint64_t kmax = (bound < key_max ? bound : key_max) - base;
    const bool narrow = static_cast<unsigned __int128>(count) * kmax < (static_cast<unsigned __int128>(1) << 64);
    if (!narrow) return kWide;
    const uint64_t span = bound - base;
    const bool pow2 = base == 0 && (span == ~0ull || ((span + 1) & span) == 0);  // kPow2Narrow: base 0
    return pow2 ? kPow2Narrow : kMagicNarrow;
}

constexpr int kBucketMaxDigits = 3;
constexpr uint32_t kSuperBucketBits = 11;  // super-bucket = up to 2^11 consecutive buckets

template <typename K, int MODE = kWide>
struct BucketDigitizer {
    static constexpr int kDigits = kBucketMaxDigits;
    static constexpr bool kChecks = true;
    // narrow modes recompute the digit in the scatter phase (a multiply and a
    // shift are cheaper than staging digits through shared memory)
    // narrow power-of-two bounds recompute the digit in the scatter phase; the
    // other modes stage it (A/B on the B200: 1.94 vs 2.18 ms at 10^8, kMagicNarrow)
    static constexpr bool kCheapDigit = MODE == kPow2Narrow;
    BucketIndexer bi;
    uint32_t shift[kBucketMaxDigits];  // digit p = (b >> shift[p]) & 255; unused: 63 (=> 0)
    uint32_t s_lo;                     // fine plan: super-bucket = b >> s_lo
    uint32_t s_lo_coarse;              // coarse plan (lowest digit pass skipped)
    uint32_t adaptive;                 // the lowest digit pass is optional (skew decides)
    uint32_t used;                     // number of digit passes that can be non-trivial

    uint32_t tsh[kBucketMaxDigits];    // kPow2Narrow: log2(M + 1) + shift[p], capped at 64 (=> 0)
    uint32_t tshc[kBucketMaxDigits];   // min(tsh, 63) with dmask = 0 when tsh == 64: branch-free digits
    uint32_t dmask[kBucketMaxDigits];
    uint32_t check_range;              // [base, M] narrower than the key type: keys can be out of range

    // The pipeline may group keys by ANY bucket function that is monotone in the
    // key: the final segment sort makes the output the unique stable sort by key
    // either way.  kPow2Narrow therefore rounds the range
    // [base, M] up to a power-of-two span 2^s and uses b = (n * (key - base)) >> s
    // -- one multiply and a shift for every bound M, against a 64-bit reciprocal
    // for the reference's exact floor(n * key / (M + 1)) (which only changes how
    // evenly the n buckets are filled: at most 2x fewer of them are used).  The
    // range check keeps the exact [base, M].  The exact reference bucket_index is
    // BucketIndexer::bucket (isort_bucket_index_u64, pinned by tests).
    static BucketDigitizer make(uint64_t n, uint64_t bound, uint64_t base = 0) {
        BucketDigitizer d{};
        uint64_t grid = bound;  // inclusive upper end of the bucket grid
        if (MODE == kPow2Narrow) {  // the grid need not reach past the key type's maximum
            const uint64_t kmax = static_cast<uint64_t>(static_cast<K>(~static_cast<K>(0)));
            const uint64_t span = (bound < kmax ? bound : kmax) - (base < kmax ? base : kmax);
            const uint32_t s = span ? 64 - __builtin_clzll(span) : 0;  // 2^s > span
            grid = s >= 64 ? ~0ull : base + ((1ull << s) - 1);
        }
        d.bi = BucketIndexer::make(n, grid, base);
        d.bi.bound = bound;  // exact range: clamping and the range check
        d.bi.span = bound - base;
        const uint32_t L = n > 1 ? 64 - __builtin_clzll(n - 1) : 0;  // bits of the largest bucket index
        uint32_t db = L > kSuperBucketBits ? (L - kSuperBucketBits + 7) / 8 : 0;
        if (db > kBucketMaxDigits) db = kBucketMaxDigits;
        // Skewed keys: one more, finer digit pass when a slot is free.  K1 counts the
        // fine digits; the coarse plan is the fine one without its lowest digit, so
        // K2 decides on the device (k_plan, kPlanAdaptiveLow) and tells the segment
        // kernel the super-bucket shift (RadixState::sb_shift).
        const uint32_t fine = db >= 1 && db < kBucketMaxDigits ? db + 1 : db;
        d.adaptive = fine > db ? 1u : 0u;
        db = fine;
        d.used = db;
        d.s_lo = L > 8 * db ? L - 8 * db : 0;
        d.s_lo_coarse = d.adaptive ? d.s_lo + 8 : d.s_lo;
        for (uint32_t p = 0; p < kBucketMaxDigits; ++p) {
            d.shift[p] = p < db ? d.s_lo + 8 * p : 63;
            const uint32_t t = (d.bi.pow2_shift < 64 ? d.bi.pow2_shift : 64) + d.shift[p];
            d.tsh[p] = t < 64 ? t : 64;
            d.tshc[p] = t < 64 ? t : 63;
            d.dmask[p] = t < 64 ? kRadix - 1 : 0;
        }
        d.check_range = (bound < static_cast<uint64_t>(~static_cast<K>(0)) || base != 0) ? 1u : 0u;
        return d;
    }
    // Bucket index.  u32 keys with a general divisor: floor(n*k/div) = k*qi +
    // floor(k*c'/div), and with qf = ceil(2^64 c'/div) = 2^64 c'/div + e (e < 1),
    // floor(k*qf / 2^64) is exact: k*e/2^64 < 2^-32 <= 1/div cannot carry k*c'/div
    // (whose fraction is <= (div-1)/div) past the next integer.  All in 32x32->64
    // multiplies (n, div < 2^32; k <= span < div); a divisor of 2^32 or more takes
    // the 64-bit reciprocal with corrections.
    __device__ __forceinline__ uint64_t bidx(K key) const {
        if constexpr (sizeof(K) == 4 && MODE == kMagicNarrow) {
            if (!bi.div32) return bucket_of<MODE>(bi, static_cast<uint64_t>(key));
            const uint64_t k64 = static_cast<uint64_t>(key) - bi.base;
            if (k64 > bi.span) return key > bi.bound ? bi.count - 1 : 0;
            const uint32_t k = static_cast<uint32_t>(k64);
            const uint64_t lo = static_cast<uint64_t>(k) * static_cast<uint32_t>(bi.qf);
            const uint64_t hi = static_cast<uint64_t>(k) * static_cast<uint32_t>(bi.qf >> 32);
            return k * static_cast<uint32_t>(bi.qi) + static_cast<uint32_t>((hi + (lo >> 32)) >> 32);
        } else {
            return bucket_of<MODE>(bi, static_cast<uint64_t>(key));
        }
    }
    // key - base: one 32-bit subtraction for u32 keys (base < 2^32 there; an
    // out-of-range key wraps, and its meaningless digit is never used)
    __device__ __forceinline__ uint64_t rel(K key) const {
        if constexpr (sizeof(K) == 4) return static_cast<uint32_t>(key) - static_cast<uint32_t>(bi.base);
        return static_cast<uint64_t>(key) - bi.base;
    }
    __device__ __forceinline__ uint32_t shift_for(int pos) const {
        const uint32_t* t = MODE == kPow2Narrow ? tsh : shift;
        return pos == 0 ? t[0] : (pos == 1 ? t[1] : t[2]);
    }
    // Digit of the bucket index.  Keys outside [base, M] only reach here when the
    // call is failing with a range error; their digits are then meaningless but < 256.
    __device__ __forceinline__ uint32_t digit_sh(K key, uint32_t sh) const {
        if (MODE == kPow2Narrow) {  // floor(n * k / 2^s) >> shift = (n * k) >> (s + shift); n, k < 2^32
            const uint64_t p = static_cast<uint64_t>(static_cast<uint32_t>(bi.count)) * rel(key);
            return sh < 64 ? static_cast<uint32_t>(p >> sh) & (kRadix - 1) : 0u;
        }
        return static_cast<uint32_t>(bidx(key) >> sh) & (kRadix - 1);
    }
    __device__ __forceinline__ uint32_t digit(K key, int pos) const { return digit_sh(key, shift_for(pos)); }
    __device__ __forceinline__ void all_digits(K key, uint32_t (&d)[kDigits]) const {
        if (MODE == kPow2Narrow) {
            const uint64_t p = static_cast<uint64_t>(static_cast<uint32_t>(bi.count)) * rel(key);
#pragma unroll
            for (int q = 0; q < kDigits; ++q) d[q] = static_cast<uint32_t>(p >> tshc[q]) & dmask[q];
            return;
        }
        const uint64_t b = bidx(key);
#pragma unroll
        for (int q = 0; q < kDigits; ++q) d[q] = static_cast<uint32_t>(b >> shift[q]) & (kRadix - 1);
    }
    __device__ __forceinline__ bool in_range(K key) const {
        return !check_range || static_cast<uint64_t>(key) - bi.base <= bi.span;
    }
    __device__ __forceinline__ bool needs_range_check() const { return check_range != 0; }
    __device__ __forceinline__ uint64_t bucket(K key) const { return bidx(key); }
    // K2's arguments: the optional fine pass and the two super-bucket shifts
    void plan_args(int* flags, int* top, uint32_t* top_bins, uint32_t* sb_fine, uint32_t* sb_coarse) const {
        if (adaptive) *flags |= kPlanAdaptiveLow;
        *top = used ? static_cast<int>(used) - 1 : 0;
        // bins of the top digit that bucket indices < n can reach
        const uint32_t L = bi.count > 1 ? 64 - __builtin_clzll(bi.count - 1) : 0;
        const uint32_t hi = used ? shift[used - 1] : 0;
        *top_bins = L > hi ? (L - hi >= 8 ? kRadix : (1u << (L - hi))) : 1u;
        *sb_fine = s_lo;
        *sb_coarse = s_lo_coarse;
    }
    __device__ __forceinline__ uint64_t super_bucket(K key, uint32_t sb_shift) const {
        return bidx(key) >> sb_shift;
    }
};

// -------------------------------------------------------- bucket state
struct BucketState {
    unsigned long long span_lo_not;  // ~(min start) of non-constant oversized super-buckets
    unsigned long long span_hi;      // max end
    uint32_t oversized;              // non-constant oversized super-buckets
    uint32_t pad;
};

// ------------------------------------------------------------------ K5
// In-smem sort: up to 10-bit digits, two 16-bit counters per 32-bit word (a
// stage holds < 2^16 keys, so a half never carries into the other).
// BLOCK threads own one counter word each in the scan: BLOCK words = 2*BLOCK bins.
template <int BLOCK>
struct SegDigits {
    static constexpr int kWords = BLOCK;
    static constexpr int kBits = BLOCK >= 1024 ? 11 : (BLOCK >= 512 ? 10 : (BLOCK >= 256 ? 9 : 8));
    static_assert((1 << (kBits - 1)) == kWords, "power-of-two block");
};

// ISORT_SEG_PREFETCH: a second stage buffer so the next stage lands during the
// sort.  Off by default: one buffer leaves room for twice the stage (16,384 keys,
// +8% measured), and the SM's other CTA covers the load latency.
#ifndef ISORT_SEG_PREFETCH
#define ISORT_SEG_PREFETCH 0
#endif
template <typename K, int BLOCK, int IPT, bool VALS>
struct SegSmem {
    static constexpr int kCap = BLOCK * IPT + 4;  // a stage + slack that keeps bulk copies 16-byte aligned
    static constexpr int kBufs = ISORT_SEG_PREFETCH ? 2 : 1;
    alignas(16) K buf[kBufs][kCap];  // the stage being sorted (in place) / the next one landing
    alignas(16) uint32_t vbuf[kBufs][VALS ? kCap : 1];
    alignas(16) uint32_t cnt[BLOCK / 32][SegDigits<BLOCK>::kWords];  // per-warp packed digit counters, then slot bases
    uint32_t scan_tot[BLOCK / 32];
    unsigned long long red[2][BLOCK / 32];
    unsigned long long pos[2];  // segment bounds, then the end of an oversized super-bucket
    alignas(8) unsigned long long bar;  // mbarrier: bulk stage load landed
    int ls;                             // start of the stage's last super-bucket
};

// ---- bulk (TMA) global -> shared copies completing on an mbarrier
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
#ifndef ISORT_SEG_BULK_STORE
#define ISORT_SEG_BULK_STORE 1
#endif

// Split of src[pos, pos + len) into a head (up to the first 16-byte boundary),
// a bulk-copyable interior of whole 16-byte blocks, and a tail.  Element j is
// staged at dst[off + j], which puts the interior on a 16-byte boundary.
struct BulkSplit {
    int off, head, body;  // body: interior elements
};
template <typename T>
__device__ __forceinline__ BulkSplit bulk_split(const T* src, uint64_t pos, int len) {
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src + pos) & 15u);
    BulkSplit b;
    b.off = static_cast<int>(mis / sizeof(T));
    const int h = static_cast<int>(((16u - mis) & 15u) / sizeof(T));
    b.head = h < len ? h : len;
    b.body = ((len - b.head) * static_cast<int>(sizeof(T)) / 16) * 16 / static_cast<int>(sizeof(T));
    return b;
}

// Start loading stage [pos, pos + len) of keys (and payload) into kd / vd: the
// interiors by bulk copies on `bar` (thread 0), heads and tails by plain loads.
// Call with the whole CTA after a barrier that freed kd / vd.
template <typename K, bool VALS>
__device__ __forceinline__ void seg_issue(const K* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t pos,
                                          int len, K* kd, uint32_t* vd, unsigned long long* bar, BulkSplit& kb,
                                          BulkSplit& vb) {
    kb = bulk_split(keys, pos, len);
    if (VALS) vb = bulk_split(vals, pos, len);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_expect_tx(bar, static_cast<uint32_t>(kb.body * sizeof(K) + (VALS ? vb.body * 4 : 0)));
        if (kb.body) bulk_g2s(kd + kb.off + kb.head, keys + pos + kb.head, kb.body * sizeof(K), bar);
        if (VALS && vb.body) bulk_g2s(vd + vb.off + vb.head, vals + pos + vb.head, vb.body * 4u, bar);
    }
    const int kplain = len - kb.body;  // head + tail elements
    if (tid < kplain) {
        const int j = tid < kb.head ? tid : kb.body + tid;
        kd[kb.off + j] = keys[pos + j];
    }
    if (VALS) {
        const int vplain = len - vb.body;
        if (tid >= 32 && tid - 32 < vplain) {
            const int t = tid - 32;
            const int j = t < vb.head ? t : vb.body + t;
            vd[vb.off + j] = vals[pos + j];
        }
    }
}

// First index in [lo, hi) where the monotone predicate holds, or hi.  Called by a
// whole warp: 32 probes per round narrow the range 32x.
template <typename Pred>
__device__ __forceinline__ uint64_t warp_first_true(uint64_t lo, uint64_t hi, Pred pred) {
    while (lo < hi) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t idx = lo + lane_id() * step;
        const bool p = idx >= hi || pred(idx);
        const uint32_t ball = __ballot_sync(ISORT_FULL_MASK, p);
        if (ball == 0) {  // every probe false, including lo + 31 * step < hi
            lo = lo + 31 * step + 1;
            continue;
        }
        const int f = __ffs(ball) - 1;
        if (f == 0) return lo;
        const uint64_t nhi = lo + static_cast<uint64_t>(f) * step < hi ? lo + static_cast<uint64_t>(f) * step : hi;
        if (step == 1) return nhi;
        lo = lo + static_cast<uint64_t>(f - 1) * step + 1;
        hi = nhi;
    }
    return hi;
}

// First super-bucket start at or after x (0 and n count as starts).  The array
// is ordered by super-bucket after K3, so this is a lower bound: gallop from x,
// then a 32-ary search.  Whole warp.
template <typename K, typename Dz>
__device__ uint64_t warp_next_start(const K* __restrict__ keys, uint64_t n, uint64_t x, const Dz& dz,
                                    uint32_t sbs) {
    if (x == 0) return 0;
    if (x >= n) return n;
    const uint64_t sbp = dz.super_bucket(keys[x - 1], sbs);
    auto differs = [&](uint64_t i) { return dz.super_bucket(keys[i], sbs) != sbp; };
    uint64_t lo = x, hi = n - x > 2048 ? x + 2048 : n;
    while (hi < n && !differs(hi - 1)) {
        lo = hi;
        const uint64_t w = (hi - x) * 16;
        hi = n - x > w ? x + w : n;
    }
    return warp_first_true(lo, hi, differs);
}

// Count / rank steps of seg_lsd for one warp's IPT x 32 positions; FULL: all in range.
template <bool FULL, typename K, int IPT, bool VALS>
__device__ __forceinline__ void seg_count(const K* ka, const uint32_t* va, int obase, int len, K kmin, uint32_t shift,
                                          uint32_t mask, uint32_t* wc, K (&kv)[IPT], uint32_t (&vv)[VALS ? IPT : 1]) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const int o = obase + i * 32;
        if (FULL || o < len) {
            kv[i] = ka[o];
            if (VALS) vv[i] = va[o];
            const uint32_t d = static_cast<uint32_t>((kv[i] - kmin) >> shift) & mask;
            atomicAdd(&wc[d >> 1], 1u << ((d & 1u) << 4));
        }
    }
}

template <bool FULL, typename K, int IPT, bool VALS>
__device__ __forceinline__ void seg_rank(K* kb, uint32_t* vb, int obase, int len, K kmin, uint32_t shift,
                                         uint32_t mask, uint32_t* wc, const K (&kv)[IPT],
                                         const uint32_t (&vv)[VALS ? IPT : 1]) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const int o = obase + i * 32;
        if (FULL || o < len) {
            const uint32_t d = static_cast<uint32_t>((kv[i] - kmin) >> shift) & mask;
            const uint32_t h = (d & 1u) << 4;
            const uint32_t slot = (atomicAdd(&wc[d >> 1], 1u << h) >> h) & 0xFFFFu;
            kb[slot] = kv[i];
            if (VALS) vb[slot] = vv[i];
        }
    }
}

// Block-wide (min, max), two barriers; the final step is a warp reduction.
template <typename K, int BLOCK>
__device__ __forceinline__ void block_minmax2(K& lo, K& hi, unsigned long long (*red)[BLOCK / 32]) {
    constexpr int kWarps = BLOCK / 32;
    const uint32_t lane = lane_id();
    unsigned long long a = warp_max<unsigned long long>(~static_cast<unsigned long long>(lo));
    unsigned long long b = warp_max<unsigned long long>(static_cast<unsigned long long>(hi));
    __syncthreads();  // previous readers of red[] are done
    if (lane == 0) {
        red[0][threadIdx.x >> 5] = a;
        red[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    a = lane < static_cast<uint32_t>(kWarps) ? red[0][lane] : 0ull;
    b = lane < static_cast<uint32_t>(kWarps) ? red[1][lane] : 0ull;
    a = warp_max<unsigned long long>(a);
    b = warp_max<unsigned long long>(b);
    lo = static_cast<K>(~a);
    hi = static_cast<K>(b);
}

// Stable LSD sort of ka[0, len) (payload va) in shared memory by key - kmin,
// `passes` r-bit digits (r <= SegDigits<BLOCK>::kBits), in place: each pass
// holds the stage in registers between its count and its scatter.
// Rank primitive of the one-sweep pass: per-warp counters pre-scanned into slot
// bases, slot = atomicAdd (lane-ordered, program-ordered => stable).  Warp w
// owns positions [w*32*IPT, (w+1)*32*IPT); keys stay in registers between the
// count and the rank step.
template <typename K, int BLOCK, int IPT, bool VALS>
__device__ __forceinline__ void seg_lsd(SegSmem<K, BLOCK, IPT, VALS>& sm, K* ka, uint32_t* va, int len, K kmin,
                                        int passes, int r) {
    constexpr int kWarps = BLOCK / 32;
    constexpr int kSegWords = SegDigits<BLOCK>::kWords;
    static_assert(BLOCK * IPT < 65536, "16-bit counters");
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint32_t nwords = 1u << (r - 1), mask = (1u << r) - 1u;
    const int obase = warp * 32 * IPT + static_cast<int>(lane);
    uint32_t* wc = sm.cnt[warp];
    for (int pass = 0; pass < passes; ++pass) {
        const uint32_t shift = static_cast<uint32_t>(pass * r);
        {
            uint4* c4 = reinterpret_cast<uint4*>(&sm.cnt[0][0]);
#pragma unroll
            for (int i = tid; i < kWarps * kSegWords / 4; i += BLOCK) c4[i] = make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
        K kv[IPT];
        uint32_t vv[VALS ? IPT : 1];
        const bool wfull = obase - static_cast<int>(lane) + 32 * IPT <= len;  // warp-uniform
        if (wfull)
            seg_count<true, K, IPT, VALS>(ka, va, obase, len, kmin, shift, mask, wc, kv, vv);
        else
            seg_count<false, K, IPT, VALS>(ka, va, obase, len, kmin, shift, mask, wc, kv, vv);
        __syncthreads();
        // thread t owns counter word t (digits 2t, 2t+1): totals over warps, scan, per-warp bases
        uint32_t lo = 0, hi = 0;
        if (static_cast<uint32_t>(tid) < nwords) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t v = sm.cnt[w][tid];
                lo += v & 0xFFFFu;
                hi += v >> 16;
            }
        }
        const uint32_t tsum = lo + hi;
        const uint32_t inc = warp_inclusive_scan(tsum);
        if (lane == 31) sm.scan_tot[warp] = inc;
        __syncthreads();
        if (static_cast<uint32_t>(tid) < nwords) {
            uint32_t base = inc - tsum;
            for (int w = 0; w < warp; ++w) base += sm.scan_tot[w];
            uint32_t blo = base, bhi = base + lo;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t v = sm.cnt[w][tid];
                sm.cnt[w][tid] = blo | (bhi << 16);
                blo += v & 0xFFFFu;
                bhi += v >> 16;
            }
        }
        __syncthreads();
        // in place: every key of the stage is in registers now
        if (wfull)
            seg_rank<true, K, IPT, VALS>(ka, va, obase, len, kmin, shift, mask, wc, kv, vv);
        else
            seg_rank<false, K, IPT, VALS>(ka, va, obase, len, kmin, shift, mask, wc, kv, vv);
        __syncthreads();
    }
}

#ifndef ISORT_SEG_MINB
#define ISORT_SEG_MINB 2  // 64 registers (a 128-register build measured 11% slower)
#endif

// K5: each persistent CTA owns the super-buckets that start in its share
// [n*b/G, n*(b+1)/G) of the array (bounds moved to the next super-bucket start).
// It walks them in steps: stage up to BLOCK*IPT keys in shared memory, sort the
// complete super-buckets of the stage stably by key, write them back in place,
// and continue from the first incomplete one.  A stable sort of whole buckets
// laid out in bucket order equals per-bucket insertion sort + concatenation,
// because bucket_index is monotone in the key.  A super-bucket longer than the
// stage is "oversized": one holding a single key value is already in arrival
// order; the others extend a span that the radix pipeline re-sorts.
template <typename K, typename Dz, int BLOCK, int IPT, bool VALS>
__global__ void __launch_bounds__(BLOCK, ISORT_SEG_MINB)
    k_bucket_segments(K* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t n,
                      const RadixState* __restrict__ rst, BucketState* __restrict__ bst, Dz dz) {
    using Smem = SegSmem<K, BLOCK, IPT, VALS>;
    constexpr int kStage = BLOCK * IPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    if (rst->descents == 0 || rst->reversed || rst->counting || rst->first_bad != 0)
        return;  // sorted / reversed / counting pass / range error

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    const uint32_t sbs = rst->sb_shift;  // the plan's super-bucket shift (fine or coarse)
    if (warp < 2) {
        const uint64_t x = n * (blockIdx.x + static_cast<uint64_t>(warp)) / gridDim.x;
        const uint64_t p = warp_next_start(keys, n, x, dz, sbs);
        if (lane == 0) sm.pos[warp] = p;
    }
    if (tid == 0) mbar_init(&sm.bar, 1);
    __syncthreads();
    uint64_t pos = sm.pos[0];
    const uint64_t seg_hi = sm.pos[1];
    auto stage_len = [&](uint64_t p) {
        return seg_hi - p < static_cast<uint64_t>(kStage) ? static_cast<int>(seg_hi - p) : kStage;
    };

    // Stage i+1 streams in (bulk copy) while stage i is sorted and written back:
    // the sort is in place, so the other buffer is free as soon as stage i's
    // extent is known.
    int cur = 0;
    uint32_t phase = 0;
    BulkSplit ksp{}, vsp{};
    if (pos < seg_hi) seg_issue<K, VALS>(keys, vals, pos, stage_len(pos), sm.buf[cur], sm.vbuf[cur], &sm.bar, ksp, vsp);
    __syncthreads();
    while (pos < seg_hi) {
        const int len = stage_len(pos);
        const bool tail = pos + len == seg_hi;  // ends on a super-bucket start: all complete
        mbar_wait(&sm.bar, phase);
        phase ^= 1u;
        K* ka = sm.buf[cur] + ksp.off;
        uint32_t* va = VALS ? sm.vbuf[cur] + vsp.off : nullptr;
        // ---- min/max of the stage (a superset of the sorted part is fine: the
        // tail super-bucket's keys are all larger than the complete ones')
        K kmin = static_cast<K>(~static_cast<K>(0)), kmax = 0;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int j = tid + i * BLOCK;
            if (j < len) {
                const K k = ka[j];
                kmin = k < kmin ? k : kmin;
                kmax = k > kmax ? k : kmax;
            }
        }
        // ---- ls = start of the last (possibly incomplete) super-bucket: a lower bound
        // over the staged keys, which are ordered by super-bucket
        if (warp == 0) {
            int l = len;
            if (!tail) {
                const uint64_t sbl = dz.super_bucket(ka[len - 1], sbs);
                l = static_cast<int>(warp_first_true(0, static_cast<uint64_t>(len), [&](uint64_t j) {
                    return dz.super_bucket(ka[j], sbs) == sbl;
                }));
            }
            if (lane == 0) sm.ls = l;
        }
        block_minmax2<K, BLOCK>(kmin, kmax, sm.red);
        int ls = sm.ls;
        if (ls == 0) {  // the whole stage is one super-bucket
            if (warp == 0) {
                const uint64_t e = warp_next_start(keys, n, pos + len, dz, sbs);
                if (lane == 0) sm.pos[0] = e;
            }
            __syncthreads();
            const uint64_t e = sm.pos[0];
            if (e == pos + static_cast<uint64_t>(len)) {  // ends exactly with the stage
                ls = len;
            } else {  // oversized: constant (nothing to do) or a span for the radix fallback
                if (ISORT_SEG_PREFETCH && e < seg_hi)
                    seg_issue<K, VALS>(keys, vals, e, stage_len(e), sm.buf[cur ^ 1], sm.vbuf[cur ^ 1], &sm.bar, ksp,
                                       vsp);
                kmin = static_cast<K>(~static_cast<K>(0));
                kmax = 0;
                for (uint64_t i = pos + tid; i < e; i += BLOCK) {
                    const K k = keys[i];
                    kmin = k < kmin ? k : kmin;
                    kmax = k > kmax ? k : kmax;
                }
                block_minmax2<K, BLOCK>(kmin, kmax, sm.red);
                if (tid == 0 && kmin != kmax) {
                    atomicAdd(&bst->oversized, 1u);
                    atomicMax(&bst->span_lo_not, ~static_cast<unsigned long long>(pos));
                    atomicMax(&bst->span_hi, static_cast<unsigned long long>(e));
                }
                pos = e;
                fence_proxy_async_smem();
                __syncthreads();
                if (ISORT_SEG_PREFETCH) {
                    cur ^= 1;
                } else if (pos < seg_hi) {
                    seg_issue<K, VALS>(keys, vals, pos, stage_len(pos), sm.buf[0], sm.vbuf[0], &sm.bar, ksp, vsp);
                    __syncthreads();
                }
                continue;
            }
        }
        const uint64_t next = pos + static_cast<uint64_t>(ls);
        // the other buffer was last read by the previous write-back (before the
        // end-of-iteration fence + barrier): the next stage can start landing now
        if (ISORT_SEG_PREFETCH && next < seg_hi)
            seg_issue<K, VALS>(keys, vals, next, stage_len(next), sm.buf[cur ^ 1], sm.vbuf[cur ^ 1], &sm.bar, ksp,
                               vsp);
        if (kmin != kmax) {  // else one key value (or one key): arrival order is the answer, in place
            // ---- stable in-smem LSD sort of ka[0, ls) by (key - min)
            const int bits = 64 - __clzll(static_cast<unsigned long long>(kmax - kmin));
            constexpr int kSegDigitBits = SegDigits<BLOCK>::kBits;
            const int passes = (bits + kSegDigitBits - 1) / kSegDigitBits;
            seg_lsd<K, BLOCK, IPT, VALS>(sm, ka, va, ls, kmin, passes, (bits + passes - 1) / passes);
            if (ISORT_SEG_BULK_STORE && !ISORT_SEG_PREFETCH) {
                // write-back by bulk copy (TMA store): the 16-byte-aligned interior of the
                // sorted stage in one transfer, the head and tail by plain stores
                fence_proxy_async_smem();  // the scatter's stores, visible to the async proxy
                __syncthreads();
                const BulkSplit kw = bulk_split(keys, pos, ls);
                if (tid == 0 && kw.body)
                    bulk_s2g(keys + pos + kw.head, ka + kw.head, static_cast<uint32_t>(kw.body * sizeof(K)));
                if (tid < ls - kw.body) {
                    const int j = tid < kw.head ? tid : kw.body + tid;
                    keys[pos + j] = ka[j];
                }
                if (VALS) {
                    const BulkSplit vw = bulk_split(vals, pos, ls);
                    if (tid == 32 && vw.body)
                        bulk_s2g(vals + pos + vw.head, va + vw.head, static_cast<uint32_t>(vw.body * 4));
                    if (tid >= 64 && tid - 64 < ls - vw.body) {
                        const int t = tid - 64;
                        const int j = t < vw.head ? t : vw.body + t;
                        vals[pos + j] = va[j];
                    }
                }
                if (tid == 0 || tid == 32) bulk_wait_read();  // the buffer is reused by the next stage
            } else {
                for (int j = tid; j < ls; j += BLOCK) {
                    keys[pos + j] = ka[j];
                    if (VALS) vals[pos + j] = va[j];
                }
            }
        }
        pos = next;
        fence_proxy_async_smem();
        __syncthreads();
        if (ISORT_SEG_PREFETCH) {
            cur ^= 1;
        } else if (pos < seg_hi) {  // one buffer: the next stage lands after the write-back
            seg_issue<K, VALS>(keys, vals, pos, stage_len(pos), sm.buf[0], sm.vbuf[0], &sm.bar, ksp, vsp);
            __syncthreads();
        }
    }
    if (ISORT_SEG_BULK_STORE && (tid == 0 || tid == 32)) bulk_wait_all();  // stores complete before exit
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
static_assert(kMaxParts <= kScatterMax, "one scatter base per destination");

template <typename K>
struct DestDigitizer {
    static constexpr int kDigits = 1;
    static constexpr bool kChecks = false;
    __device__ __forceinline__ bool needs_range_check() const { return false; }
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
    void plan_args(int*, int*, uint32_t*, uint32_t*, uint32_t*) const {}
};

static __global__ void k_copy_part_counts(const RadixState* __restrict__ st, uint64_t* __restrict__ counts, int parts) {
    if (threadIdx.x < parts) counts[threadIdx.x] = st->hist[0][threadIdx.x];
}

}  // namespace isort
