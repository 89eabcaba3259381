// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together
// with the reference's own sources (/root/reference/proj/core/src/*.cpp,
// namespace-renamed with -Dintsort=intsort_ref so it can share a process
// with the B200 engine) into oracle/_ref/libintsort_ref.so.  Used to
//   * pin the C restatement (oracle/isort_oracle.c) against the reference
//     itself (tests/golden/make_golden.py, tests/test_oracle.py), and
//   * time the reference CPU path for bench.py's cpu_baseline and
//     `--impl reference` legs.
// Nothing on the product path loads it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "intsort/bench.hpp"
#include "intsort/generator.hpp"
#include "intsort/rng.hpp"
#include "intsort/sequence_io.hpp"
#include "intsort/sort.hpp"
#include "intsort/verify.hpp"

namespace {

struct CRecord {
    std::uint64_t key;
    std::uint64_t tag;
};
static_assert(sizeof(CRecord) == sizeof(intsort::Record), "Record layout");

thread_local std::string g_err;

intsort::RecordSeq to_seq(const CRecord* in, std::uint64_t n) {
    intsort::RecordSeq s(n);
    if (n) std::memcpy(s.data(), in, n * sizeof(CRecord));
    return s;
}

void from_seq(const intsort::RecordSeq& s, CRecord* out) {
    if (!s.empty()) std::memcpy(out, s.data(), s.size() * sizeof(CRecord));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 22;
    } catch (const intsort::SequenceIoError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_radix_sort_lsd(const CRecord* in, CRecord* out, std::uint64_t n, std::uint64_t base) {
    return guarded([&] { from_seq(intsort::radix_sort_lsd(to_seq(in, n), base), out); });
}

int ref_bucket_sort(const CRecord* in, CRecord* out, std::uint64_t n, std::uint64_t range_bound) {
    return guarded([&] { from_seq(intsort::bucket_sort(to_seq(in, n), range_bound), out); });
}

int ref_insertion_sort(const CRecord* in, CRecord* out, std::uint64_t n) {
    return guarded([&] { from_seq(intsort::insertion_sort(to_seq(in, n)), out); });
}

int ref_counting_sort_by_digit(const CRecord* in, CRecord* out, std::uint64_t n, std::uint64_t base,
                               std::uint32_t digits, std::uint32_t digit_index) {
    return guarded([&] {
        from_seq(intsort::counting_sort_by_digit(to_seq(in, n), intsort::RadixPlan{base, digits},
                                                 digit_index),
                 out);
    });
}

int ref_build_radix_plan(const CRecord* in, std::uint64_t n, std::uint64_t base,
                         std::uint32_t* digits) {
    return guarded([&] { *digits = intsort::build_radix_plan(to_seq(in, n), base).digits; });
}

int ref_extract_digit(std::uint64_t key, std::uint32_t digit_index, std::uint64_t base,
                      std::uint64_t* out) {
    return guarded([&] { *out = intsort::extract_digit(key, digit_index, base); });
}

int ref_bucket_index(std::uint64_t key, std::uint64_t count, std::uint64_t range_bound,
                     std::uint64_t* out) {
    return guarded([&] { *out = intsort::bucket_index(key, count, range_bound); });
}

int ref_oracle_sort(const CRecord* in, CRecord* out, std::uint64_t n) {
    return guarded([&] { from_seq(intsort::verify::oracle_sort(to_seq(in, n)), out); });
}

int ref_generate(int case_id, std::uint64_t n, int has_range, std::uint64_t range_bound,
                 std::uint64_t seed, int has_rep, std::uint64_t rep, double sorted_fraction,
                 CRecord* out) {
    return guarded([&] {
        intsort::InputSpec spec;
        spec.case_id = case_id;
        spec.n = n;
        if (has_range) spec.range_bound = range_bound;
        spec.seed = seed;
        if (has_rep) spec.repeated_value = rep;
        spec.sorted_fraction = sorted_fraction;
        from_seq(intsort::generate(spec), out);
    });
}

// write_sequence_file / read_sequence_file (sequence_io.cpp:45-128).  hdr: case_id,
// n, range_bound, seed.  read: header always filled when it parses; records
// only when the whole file reads (capacity permitting).
int ref_write_sequence_file(const char* path, const std::uint64_t* hdr, const CRecord* in, std::uint64_t n) {
    return guarded([&] {
        intsort::write_sequence_file({hdr[0], hdr[1], hdr[2], hdr[3]}, to_seq(in, n), path);
    });
}

int ref_read_sequence_file(const char* path, std::uint64_t* hdr, CRecord* out, std::uint64_t capacity) {
    return guarded([&] {
        const intsort::SequenceFile f = intsort::read_sequence_file(path);
        hdr[0] = f.header.case_id;
        hdr[1] = f.header.n;
        hdr[2] = f.header.range_bound;
        hdr[3] = f.header.seed;
        if (f.records.size() > capacity) throw std::runtime_error("capacity");
        from_seq(f.records, out);
    });
}

std::uint64_t ref_splitmix_next(std::uint64_t seed, std::uint64_t skip) {
    intsort::SplitMix64 rng(seed);
    for (std::uint64_t i = 0; i < skip; ++i) rng.next();
    return rng.next();
}

// One timed sort of a private copy (the region time_sort times,
// bench.cpp:81-84).  algorithm: 0 bucket, 1 radix, 2 insertion
// (AlgorithmId order, bench.hpp:15).  Returns seconds or -1 on error.
double ref_time_one(int algorithm, const CRecord* in, std::uint64_t n, std::uint64_t range_bound,
                    std::uint64_t base) {
    double secs = -1.0;
    guarded([&] {
        const intsort::SortFn fn = intsort::make_sort_fn(
            static_cast<intsort::AlgorithmId>(algorithm), range_bound, base);
        intsort::RecordSeq copy = to_seq(in, n);
        const auto t0 = std::chrono::steady_clock::now();
        intsort::RecordSeq out = fn(copy);
        const auto t1 = std::chrono::steady_clock::now();
        if (!intsort::verify::is_sorted(out)) throw std::runtime_error("unsorted output");
        secs = std::chrono::duration<double>(t1 - t0).count();
    });
    return secs;
}

// The reference's own harness: warm-up + repeats, median (bench.cpp:67-99).
int ref_time_sort(int algorithm, const CRecord* in, std::uint64_t n, std::uint64_t range_bound,
                  std::uint64_t base, int repeats, double* median_s, double* spread) {
    return guarded([&] {
        const intsort::SortFn fn = intsort::make_sort_fn(
            static_cast<intsort::AlgorithmId>(algorithm), range_bound, base);
        const intsort::TimingStats st = intsort::time_sort(fn, to_seq(in, n), repeats);
        *median_s = st.median_s;
        *spread = st.relative_spread;
    });
}

}  // extern "C"
