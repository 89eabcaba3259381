// sort_b200.cpp -- drop-in replacement for proj/core/src/sort.cpp.
//
// Implements every declaration of the reference header intsort/sort.hpp
// (proj/core/include/intsort/sort.hpp:13-53) with unchanged signatures, so a
// maintainer swaps this file in for sort.cpp and links libisort.so
// (INTEGRATION.md).  Every sort runs on the B200 through the C ABI
// (include/isort.h); the two scalar helpers (extract_digit, bucket_index) are
// single-key integer arithmetic and stay on the host.  There is no CPU
// fallback: without a usable device the sorts throw std::runtime_error.
//
// Error behaviour follows the reference: std::invalid_argument with the same
// messages for base < 2 (sort.cpp:45-47, 58-60, 79-81), digit_index >= digits
// (sort.cpp:82-86), bucket_count == 0 and key > range_bound (sort.cpp:122-129).
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "intsort/sort.hpp"
#include "isort.h"

namespace intsort {

namespace {

static_assert(sizeof(Record) == sizeof(isort_record), "Record must stay the 16-byte {key, tag} layout");

int device_ordinal() {
    const char* env = std::getenv("ISORT_DEVICE");
    return env ? std::atoi(env) : 0;
}

void check(int rc) {
    if (rc == ISORT_OK) return;
    const std::string msg = isort_last_error();
    if (rc == ISORT_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("isort: " + msg);
}

const isort_record* in_ptr(const RecordSeq& s) { return reinterpret_cast<const isort_record*>(s.data()); }
isort_record* out_ptr(RecordSeq& s) { return reinterpret_cast<isort_record*>(s.data()); }

}  // namespace

RecordSeq insertion_sort(const RecordSeq& input) {
    // The quadratic shift-insert loop is the reference's cost model, not its
    // contract: the result is the unique stable sort by key.
    RecordSeq out(input.size());
    check(isort_radix_sort_records(in_ptr(input), out_ptr(out), input.size(), 256, device_ordinal()));
    return out;
}

std::uint64_t extract_digit(Key key, std::uint32_t digit_index, std::uint64_t base) {
    if (base < 2) throw std::invalid_argument("extract_digit: base must be >= 2");
    Key rest = key;  // divide digit_index times; stops early once nothing is left
    for (std::uint32_t i = 0; rest != 0 && i < digit_index; ++i) rest /= base;
    return rest % base;
}

RadixPlan build_radix_plan(const RecordSeq& input, std::uint64_t base) {
    std::uint32_t digits = 0;
    check(isort_build_radix_plan_records(in_ptr(input), input.size(), base, &digits, device_ordinal()));
    return RadixPlan{base, digits};
}

RecordSeq counting_sort_by_digit(const RecordSeq& input, const RadixPlan& plan, std::uint32_t digit_index) {
    RecordSeq out(input.size());
    check(isort_counting_sort_by_digit_records(in_ptr(input), out_ptr(out), input.size(), plan.base, plan.digits,
                                               digit_index, device_ordinal()));
    return out;
}

RecordSeq radix_sort_lsd(const RecordSeq& input, std::uint64_t base) {
    RecordSeq out(input.size());
    check(isort_radix_sort_records(in_ptr(input), out_ptr(out), input.size(), base, device_ordinal()));
    return out;
}

std::size_t bucket_index(Key key, std::size_t bucket_count, Key range_bound) {
    if (bucket_count == 0) throw std::invalid_argument("bucket_index: bucket_count must be >= 1");
    if (key > range_bound)
        throw std::invalid_argument("bucket_index: key " + std::to_string(key) + " exceeds range bound " +
                                    std::to_string(range_bound) + " (sequence/spec mismatch)");
    // floor(count * key / (M + 1)); up to 2^32 * 2^40 needs 128-bit arithmetic
    const unsigned __int128 num = static_cast<unsigned __int128>(bucket_count) * key;
    const unsigned __int128 den = static_cast<unsigned __int128>(range_bound) + 1u;
    return static_cast<std::size_t>(num / den);
}

RecordSeq bucket_sort(const RecordSeq& input, Key range_bound) {
    RecordSeq out(input.size());
    if (input.empty()) return out;  // no range check on empty input (sort.cpp:139-141)
    check(isort_bucket_sort_records(in_ptr(input), out_ptr(out), input.size(), range_bound, device_ordinal()));
    return out;
}

}  // namespace intsort
