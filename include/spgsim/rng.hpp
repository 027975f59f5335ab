// SplitMix64 stream used by the synthetic generators; identical sequence to the
// reference's (proj/include/spgsim/rng.hpp:10-34) so seeded inputs match bit for bit.
#pragma once

#include <cstdint>

namespace spgsim {

class SplitMix64 {
public:
    explicit SplitMix64(std::uint64_t seed) : s_(seed) {}
    std::uint64_t next() { return mix(s_ += kGamma); }
    // [0,1) with 53 random bits
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    // (0,1]
    double uniform_pos() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; }
    std::uint64_t below(std::uint64_t bound) { return next() % bound; }
    // Value of the t-th call (t >= 1) of a stream seeded with `seed`, without
    // advancing anything: the stream is counter-based, which lets generators
    // run in parallel.
    static std::uint64_t at(std::uint64_t seed, std::uint64_t t) { return mix(seed + t * kGamma); }
    static std::uint64_t mix(std::uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }

private:
    static constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
    std::uint64_t s_;
};

inline std::uint64_t mix64(std::uint64_t x) { return SplitMix64::mix(x); }

}  // namespace spgsim
