/*
 * isort_oracle.c -- CPU restatement of the reference's sorting path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 engine: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_1206_3511_b200/, libisort.so) never links or calls it.
 *
 * Every function restates the algorithm of the reference C++ library
 * (/root/reference/proj/core) in plain C, citing the file:line it follows.
 * Parity is pinned by tests/test_oracle.py against
 *   - the reference's own known-answer tests (proj/tests/test_sort.cpp,
 *     test_verify.cpp, test_rng.cpp), restated as Python asserts, and
 *   - golden vectors produced by the reference itself compiled here
 *     (oracle/_ref, see oracle/Makefile and tests/golden/make_golden.py).
 *
 * Records are the reference's 16-byte AoS {u64 key, u64 tag}
 * (record.hpp:20-25).  Errors the reference reports with
 * std::invalid_argument are returned as ORC_EINVAL with the reference's
 * message text in orc_last_error().
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 22
#define ORC_ENOMEM 12

typedef struct {
    uint64_t key;
    uint64_t tag;
} orc_record;

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return ORC_EINVAL;
}

/* ---------------------------------------------------------------- rng ---
 * SplitMix64, rng.hpp:13-47.  next(): add golden gamma, two
 * xorshift-multiply rounds (rng.hpp:17-23).  below(): reject the top
 * partial block then reduce mod bound (rng.hpp:28-41). */
#define ORC_GAMMA 0x9e3779b97f4a7c15ULL

uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t orc_splitmix_next(uint64_t* state) {
    *state += ORC_GAMMA;
    return orc_mix64(*state);
}

int orc_splitmix_below(uint64_t* state, uint64_t bound, uint64_t* out) {
    if (bound == 0) return fail("SplitMix64::below: bound must be >= 1");
    const uint64_t rem = (UINT64_MAX - bound + 1) % bound; /* 2^64 mod bound */
    for (;;) {
        const uint64_t x = orc_splitmix_next(state);
        if (x <= UINT64_MAX - rem) {
            *out = x % bound;
            return ORC_OK;
        }
    }
}

/* ---------------------------------------------------------- generator ---
 * generator.cpp:15-156.  Six cases; tag = position (generator.cpp:151-154). */
static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x > y) - (x < y);
}

uint64_t orc_default_range_bound(int case_id) { /* generator.cpp:71-80 */
    switch (case_id) {
        case 4: return 10000ULL;
        case 5: return 100000000ULL;
        default: return 1000000ULL;
    }
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
    while (b) {
        const uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* Writes n records.  has_range/has_rep mirror the std::optional fields of
 * InputSpec (generator.hpp:21-34); validation follows
 * InputSpec::resolved (generator.cpp:82-113). */
int orc_generate(int case_id, uint64_t n, int has_range, uint64_t range_bound, uint64_t seed,
                 int has_rep, uint64_t repeated_value, double sorted_fraction, orc_record* out) {
    char msg[256];
    if (case_id < 1 || case_id > 6) {
        snprintf(msg, sizeof msg, "InputSpec: case_id must be in 1..6, got %d", case_id);
        return fail(msg);
    }
    const uint64_t bound = has_range ? range_bound : orc_default_range_bound(case_id);
    if (bound > (1ULL << 40)) return fail("InputSpec: range_bound exceeds 2^40");
    if (sorted_fraction < 0.0 || sorted_fraction > 1.0)
        return fail("InputSpec: sorted_fraction must be in [0, 1]");
    uint64_t rep = 0;
    if (case_id == 6) {
        rep = has_rep ? repeated_value : bound / 2;
        if (rep > bound) return fail("InputSpec: repeated_value exceeds range_bound");
        const uint64_t need = (2 * n + 2) / 3; /* generator.cpp:15-18 */
        if (need > bound) {
            snprintf(msg, sizeof msg,
                     "InputSpec: case 6 infeasible, ceil(2n/3) = %llu exceeds range_bound %llu "
                     "(not enough distinct values)",
                     (unsigned long long)need, (unsigned long long)bound);
            return fail(msg);
        }
    }
    uint64_t* keys = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!keys) return ORC_ENOMEM;
    uint64_t st = seed;
    if (case_id != 6) {
        /* uniform_keys, generator.cpp:20-27 */
        for (uint64_t i = 0; i < n; ++i) orc_splitmix_below(&st, bound + 1, &keys[i]);
        if (case_id == 2 || case_id == 3) qsort(keys, n, sizeof(uint64_t), cmp_u64);
        if (case_id == 3) { /* generator.cpp:132-143 */
            const uint64_t swaps = (uint64_t)((1.0 - sorted_fraction) * (double)n);
            for (uint64_t s = 0; s < swaps; ++s) {
                uint64_t a, b;
                orc_splitmix_below(&st, n, &a);
                orc_splitmix_below(&st, n, &b);
                const uint64_t t = keys[a];
                keys[a] = keys[b];
                keys[b] = t;
            }
        }
    } else {
        /* duplicate_heavy_keys, generator.cpp:33-67 */
        const uint64_t dup = (n + 2) / 3;
        const uint64_t modulus = bound + 1;
        uint64_t filled = 0;
        for (; filled < dup; ++filled) keys[filled] = rep;
        if (n - dup > 0) {
            uint64_t stride = 0;
            do {
                orc_splitmix_below(&st, modulus, &stride);
            } while (stride == 0 || gcd_u64(stride, modulus) != 1);
            uint64_t v;
            orc_splitmix_below(&st, modulus, &v);
            while (filled < n) {
                if (v != rep) keys[filled++] = v;
                v += stride;
                if (v >= modulus) v -= modulus;
            }
        }
        for (uint64_t i = n; i > 1; --i) { /* Fisher-Yates, generator.cpp:61-65 */
            uint64_t j;
            orc_splitmix_below(&st, i, &j);
            const uint64_t t = keys[i - 1];
            keys[i - 1] = keys[j];
            keys[j] = t;
        }
    }
    for (uint64_t i = 0; i < n; ++i) {
        out[i].key = keys[i];
        out[i].tag = i;
    }
    free(keys);
    return ORC_OK;
}

/* Counter form of case 1 for power-of-two bounds: below(2^k) never rejects
 * (rng.hpp:33-38 with 2^64 mod 2^k = 0), so key_i = mix(seed+(i+1)*gamma)
 * & (2^k-1).  Bit-identical to orc_generate(case 1, M = 2^k-1) keys
 * (tests/test_oracle.py pins it); used to build 10^8..10^9-key inputs
 * quickly. */
void orc_gen_uniform_u32(uint64_t n, uint64_t seed, uint32_t bits, uint32_t* out) {
    const uint64_t mask = bits >= 64 ? UINT64_MAX : ((1ULL << bits) - 1);
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)(orc_mix64(seed + (i + 1) * ORC_GAMMA) & mask);
}

/* Config-5 mixture (a harness addition): stream x_j =
 * mix(seed+(j+1)*gamma).  Component = top bit of x_{3i}; uniform ->
 * low 32 bits of x_{3i+1}; normal(2^31, 2^24) by Box-Muller on
 * x_{3i+1}, x_{3i+2}, rounded and clamped to [0, 2^32-1]. */
void orc_gen_mixture_u32_range(uint64_t start, uint64_t count, uint64_t seed, uint32_t* out) {
    const double two_pi = 6.283185307179586476925286766559;
    for (uint64_t i = start; i < start + count; ++i, ++out) {
        const uint64_t x0 = orc_mix64(seed + (3 * i + 1) * ORC_GAMMA);
        const uint64_t x1 = orc_mix64(seed + (3 * i + 2) * ORC_GAMMA);
        if (!(x0 >> 63)) {
            *out = (uint32_t)x1;
        } else {
            const uint64_t x2 = orc_mix64(seed + (3 * i + 3) * ORC_GAMMA);
            const double u1 = 1.0 - (double)(x1 >> 11) * 0x1.0p-53; /* (0, 1] */
            const double u2 = (double)(x2 >> 11) * 0x1.0p-53;
            const double z = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
            double v = llround(2147483648.0 + 16777216.0 * z);
            if (v < 0) v = 0;
            if (v > 4294967295.0) v = 4294967295.0;
            *out = (uint32_t)v;
        }
    }
}

void orc_gen_mixture_u32(uint64_t n, uint64_t seed, uint32_t* out) {
    orc_gen_mixture_u32_range(0, n, seed, out);
}

/* ---------------------------------------------------------- sort core ---
 * sort.cpp:13-152. */

/* insertion_sort_in_place, sort.cpp:15-25: strict > keeps equal keys in
 * arrival order. */
static void insertion_in_place(orc_record* a, uint64_t n) {
    for (uint64_t j = 1; j < n; ++j) {
        const orc_record item = a[j];
        int64_t i = (int64_t)j - 1;
        while (i >= 0 && a[i].key > item.key) {
            a[i + 1] = a[i];
            --i;
        }
        a[i + 1] = item;
    }
}

void orc_insertion_sort(const orc_record* in, orc_record* out, uint64_t n) { /* sort.cpp:38-42 */
    if (n) memmove(out, in, n * sizeof(orc_record));
    insertion_in_place(out, n);
}

/* extract_digit, sort.cpp:44-55: repeated division, safe for any index. */
int orc_extract_digit(uint64_t key, uint32_t digit_index, uint64_t base, uint64_t* out) {
    if (base < 2) return fail("extract_digit: base must be >= 2");
    uint64_t v = key;
    for (uint32_t i = 0; i < digit_index && v != 0; ++i) v /= base;
    *out = v % base;
    return ORC_OK;
}

/* build_radix_plan, sort.cpp:57-75: max key, minimal digits with
 * base^digits > max, 1 for empty/all-zero. */
int orc_build_radix_plan(const orc_record* in, uint64_t n, uint64_t base, uint32_t* digits) {
    if (base < 2) return fail("build_radix_plan: base must be >= 2");
    uint64_t max_key = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (in[i].key > max_key) max_key = in[i].key;
    uint32_t d = 0;
    uint64_t v = max_key;
    do {
        v /= base;
        ++d;
    } while (v != 0);
    *digits = d;
    return ORC_OK;
}

/* counting_sort_by_digit, sort.cpp:77-110: count, prefix (counts[d] =
 * #records with digit <= d), reverse walk placement. */
int orc_counting_sort_by_digit(const orc_record* in, orc_record* out, uint64_t n, uint64_t base,
                               uint32_t digits, uint32_t digit_index) {
    char msg[160];
    if (base < 2) return fail("counting_sort_by_digit: base must be >= 2");
    if (digit_index >= digits) {
        snprintf(msg, sizeof msg,
                 "counting_sort_by_digit: digit_index %u out of range for a %u-digit plan",
                 digit_index, digits);
        return fail(msg);
    }
    uint64_t divisor = 1; /* pow_u64, sort.cpp:28-34 */
    for (uint32_t i = 0; i < digit_index; ++i) divisor *= base;
    /* base can reach 2^32 through the CLI (intsort_main.cpp:298-299); a
     * dense count array of that size is the reference's own cost. */
    uint64_t* counts = (uint64_t*)calloc((size_t)base, sizeof(uint64_t));
    if (!counts) return ORC_ENOMEM;
    for (uint64_t i = 0; i < n; ++i) ++counts[(in[i].key / divisor) % base];
    for (uint64_t d = 1; d < base; ++d) counts[d] += counts[d - 1];
    for (uint64_t j = n; j-- > 0;) {
        const uint64_t d = (in[j].key / divisor) % base;
        out[--counts[d]] = in[j];
    }
    free(counts);
    return ORC_OK;
}

/* radix_sort_lsd, sort.cpp:112-119. */
int orc_radix_sort_lsd(const orc_record* in, orc_record* out, uint64_t n, uint64_t base) {
    uint32_t digits;
    int rc = orc_build_radix_plan(in, n, base, &digits);
    if (rc) return rc;
    if (n == 0) return ORC_OK;
    orc_record* tmp = (orc_record*)malloc(n * sizeof(orc_record));
    if (!tmp) return ORC_ENOMEM;
    memmove(out, in, n * sizeof(orc_record)); /* RecordSeq current = input */
    for (uint32_t d = 0; d < digits; ++d) {
        rc = orc_counting_sort_by_digit(out, tmp, n, base, digits, d);
        if (rc) break;
        memcpy(out, tmp, n * sizeof(orc_record));
    }
    free(tmp);
    return rc;
}

/* bucket_index, sort.cpp:121-134: floor(count*key/(M+1)) in 128 bits. */
int orc_bucket_index(uint64_t key, uint64_t count, uint64_t range_bound, uint64_t* out) {
    char msg[200];
    if (count == 0) return fail("bucket_index: bucket_count must be >= 1");
    if (key > range_bound) {
        snprintf(msg, sizeof msg,
                 "bucket_index: key %llu exceeds range bound %llu (sequence/spec mismatch)",
                 (unsigned long long)key, (unsigned long long)range_bound);
        return fail(msg);
    }
    const unsigned __int128 p = (unsigned __int128)count * key;
    *out = (uint64_t)(p / ((unsigned __int128)range_bound + 1));
    return ORC_OK;
}

/* bucket_sort, sort.cpp:136-152: n buckets, stable append in input order,
 * insertion sort per bucket, concatenate.  The append order into each
 * bucket is restated as a stable counting distribution (same sequence per
 * bucket as push_back in input order).  *bad_index receives the position
 * of the first key > range_bound (the record the reference throws on). */
int orc_bucket_sort(const orc_record* in, orc_record* out, uint64_t n, uint64_t range_bound,
                    uint64_t* bad_index) {
    if (bad_index) *bad_index = UINT64_MAX;
    if (n == 0) return ORC_OK; /* sort.cpp:139-141: no range check on empty */
    uint64_t* bidx = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* start = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    if (!bidx || !start) {
        free(bidx);
        free(start);
        return ORC_ENOMEM;
    }
    for (uint64_t i = 0; i < n; ++i) {
        int rc = orc_bucket_index(in[i].key, n, range_bound, &bidx[i]);
        if (rc) {
            if (bad_index) *bad_index = i;
            free(bidx);
            free(start);
            return rc;
        }
        ++start[bidx[i] + 1];
    }
    for (uint64_t b = 1; b <= n; ++b) start[b] += start[b - 1];
    for (uint64_t i = 0; i < n; ++i) out[start[bidx[i]]++] = in[i];
    /* start[b] is now the end of bucket b; bucket b spans [end(b-1), end(b)) */
    uint64_t lo = 0;
    for (uint64_t b = 0; b < n; ++b) {
        insertion_in_place(out + lo, start[b] - lo);
        lo = start[b];
    }
    free(bidx);
    free(start);
    return ORC_OK;
}

/* ------------------------------------------------------------- verify ---
 * verify.cpp:15-65: independent top-down merge sort, left wins ties. */
static void merge_range(orc_record* w, orc_record* s, uint64_t lo, uint64_t hi) {
    if (hi - lo < 2) return;
    const uint64_t mid = lo + (hi - lo) / 2;
    merge_range(w, s, lo, mid);
    merge_range(w, s, mid, hi);
    uint64_t l = lo, r = mid, o = lo;
    while (l < mid && r < hi) s[o++] = (w[r].key < w[l].key) ? w[r++] : w[l++];
    while (l < mid) s[o++] = w[l++];
    while (r < hi) s[o++] = w[r++];
    memcpy(w + lo, s + lo, (hi - lo) * sizeof(orc_record));
}

int orc_oracle_sort(const orc_record* in, orc_record* out, uint64_t n) {
    if (n == 0) return ORC_OK;
    orc_record* s = (orc_record*)malloc(n * sizeof(orc_record));
    if (!s) return ORC_ENOMEM;
    memmove(out, in, n * sizeof(orc_record));
    merge_range(out, s, 0, n);
    free(s);
    return ORC_OK;
}

int orc_is_sorted(const orc_record* a, uint64_t n) { /* verify.cpp:67-74 */
    for (uint64_t i = 1; i < n; ++i)
        if (a[i - 1].key > a[i].key) return 0;
    return 1;
}

/* ------------------------------------------------ keys-only u32 oracle ---
 * For BASELINE-sized parity (10^8 keys) the record oracle is needlessly
 * slow; a stable LSD counting sort over u32 (key, index) pairs is the same
 * algorithm as radix_sort_lsd at base 256 (sort.cpp:77-119) without the
 * 16-byte AoS.  vals may be NULL (keys only). */
int orc_radix_sort_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                       uint32_t* vals_out, uint64_t n) {
    if (n == 0) return ORC_OK;
    uint32_t* tk = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* tv = vals_out ? (uint32_t*)malloc(n * sizeof(uint32_t)) : NULL;
    if (!tk || (vals_out && !tv)) {
        free(tk);
        free(tv);
        return ORC_ENOMEM;
    }
    memmove(keys_out, keys_in, n * sizeof(uint32_t));
    if (vals_out) {
        if (vals_in)
            memmove(vals_out, vals_in, n * sizeof(uint32_t));
        else
            for (uint64_t i = 0; i < n; ++i) vals_out[i] = (uint32_t)i;
    }
    for (int pass = 0; pass < 4; ++pass) {
        const int sh = 8 * pass;
        uint64_t cnt[257] = {0};
        for (uint64_t i = 0; i < n; ++i) ++cnt[((keys_out[i] >> sh) & 255) + 1];
        int trivial = 0;
        for (int d = 0; d < 256; ++d) trivial |= (cnt[d + 1] == n);
        if (trivial) continue;
        for (int d = 1; d <= 256; ++d) cnt[d] += cnt[d - 1];
        for (uint64_t i = 0; i < n; ++i) { /* forward walk == reverse walk from the end */
            const uint64_t p = cnt[(keys_out[i] >> sh) & 255]++;
            tk[p] = keys_out[i];
            if (vals_out) tv[p] = vals_out[i];
        }
        memcpy(keys_out, tk, n * sizeof(uint32_t));
        if (vals_out) memcpy(vals_out, tv, n * sizeof(uint32_t));
    }
    free(tk);
    free(tv);
    return ORC_OK;
}
