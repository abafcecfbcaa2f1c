// cachegram-b200: splitmix64 stream, bit-identical to the reference generator
// (rng.hpp:13-43) because init_model, subsampling and window draws of the
// deterministic mode must consume the same numbers. The device side uses the
// same mixing function (csrc/cg_device.cuh) as a counter-based generator.
#pragma once

#include <cstdint>

namespace cachegram {

namespace rngdetail {
inline constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
inline constexpr std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
}  // namespace rngdetail

class Rng {
public:
    explicit Rng(std::uint64_t seed) : s_(seed) {}

    std::uint64_t next_u64() {
        s_ += rngdetail::kGolden;
        return rngdetail::mix64(s_);
    }
    // [0,1) from the top 24 bits; exact in float.
    float next_float() { return static_cast<float>(next_u64() >> 40) * 0x1.0p-24f; }
    // [0,n), n > 0, by modulo (the reference's convention, bias included).
    std::uint32_t next_below(std::uint32_t n) { return static_cast<std::uint32_t>(next_u64() % n); }

private:
    std::uint64_t s_;
};

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) {
    return Rng(seed ^ (0x632be59bd9b4e019ull * (stream + 1))).next_u64();
}

}  // namespace cachegram
