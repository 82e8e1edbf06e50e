// sptucker/rng.hpp -- the seeded random source.
//
// Stream-compatible with the reference Rng (proj/include/sptucker/rng.hpp:
// std::mt19937_64 engine, unbiased rejection next_below, 53-bit next_unit,
// Box-Muller with one cached spare), but the engine is spelled out here so
// its 312-word state can cross the C-ABI: the device sampler consumes the
// very same outputs and hands the advanced state back (sgdt_set_rng /
// sgdt_get_rng).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>

namespace sptucker {

class Rng {
 public:
  static constexpr int kWords = 312;

  explicit Rng(std::uint64_t seed) { reseed(seed); }

  void reseed(std::uint64_t seed) {
    mt_[0] = seed;
    for (int i = 1; i < kWords; ++i)
      mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + static_cast<std::uint64_t>(i);
    pos_ = kWords;
    has_spare_ = false;
    spare_ = 0.0;
  }

  std::uint64_t next_u64() {
    if (pos_ >= kWords) twist();
    std::uint64_t z = mt_[pos_++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    return z ^ (z >> 43);
  }

  // Uniform in [0, bound): reject raw draws below 2^64 mod bound.
  std::uint64_t next_below(std::uint64_t bound) {
    const std::uint64_t reject_below = (0ULL - bound) % bound;
    std::uint64_t r;
    do {
      r = next_u64();
    } while (r < reject_below);
    return r % bound;
  }

  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

  double next_gaussian(double mean, double stddev) {
    if (has_spare_) {
      has_spare_ = false;
      return mean + stddev * spare_;
    }
    const double u1 = 1.0 - next_unit();
    const double u2 = next_unit();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * 3.141592653589793 * u2;
    spare_ = rad * std::sin(ang);
    has_spare_ = true;
    return mean + stddev * rad * std::cos(ang);
  }

  // Engine state exchange with the device (Box-Muller spare stays host-side).
  const std::array<std::uint64_t, kWords>& state_words() const { return mt_; }
  std::uint32_t state_pos() const { return pos_; }
  void set_state(const std::uint64_t* words, std::uint32_t pos) {
    for (int i = 0; i < kWords; ++i) mt_[i] = words[i];
    pos_ = pos;
  }

 private:
  void twist() {
    constexpr std::uint64_t kA = 0xB5026F5AA96619E9ULL, kHi = 0xFFFFFFFF80000000ULL, kLo = 0x7FFFFFFFULL;
    auto mix = [&](std::uint64_t cur, std::uint64_t nxt, std::uint64_t far) {
      const std::uint64_t y = (cur & kHi) | (nxt & kLo);
      return far ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
    };
    int k = 0;
    for (; k < kWords - 156; ++k) mt_[k] = mix(mt_[k], mt_[k + 1], mt_[k + 156]);
    for (; k < kWords - 1; ++k) mt_[k] = mix(mt_[k], mt_[k + 1], mt_[k - (kWords - 156)]);
    mt_[kWords - 1] = mix(mt_[kWords - 1], mt_[0], mt_[155]);
    pos_ = 0;
  }

  std::array<std::uint64_t, kWords> mt_{};
  std::uint32_t pos_ = kWords;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

}  // namespace sptucker
