// radix_sort.cpp (B200 drop-in) -- replaces the reference's src/radix_sort.cpp:
// radix_sort and RadixSorter::sort (inc/radix_sort.hpp:15-27) on the device
// through dpdb_radix_sort (stable LSD radix sort, 8-bit digits; the same
// contract: stable, deterministic, bit_length a multiple of 4 and <= 32).
#include "b200_session.hpp"
#include "dpd/radix_sort.hpp"

namespace dpd {

void radix_sort(std::span<std::uint32_t> keys, std::span<std::uint32_t> values, int bit_length, WorkerPool&) {
    if (keys.size() != values.size()) fail(ErrorCategory::config, "radix_sort: keys and values differ in length");
    if (bit_length < 0 || bit_length > 32 || bit_length % 4)
        fail(ErrorCategory::config, "radix_sort: bit_length must be a multiple of 4 in [0, 32]");
    if (keys.empty() || bit_length == 0) return;
    b200::check(dpdb_radix_sort(0, keys.data(), values.data(), keys.size(), bit_length), nullptr, "radix_sort");
}

void RadixSorter::sort(std::span<std::uint32_t> keys, std::span<std::uint32_t> values, int bit_length,
                       WorkerPool& pool) {
    radix_sort(keys, values, bit_length, pool);  // device scratch lives in libdpdb
}

}  // namespace dpd
