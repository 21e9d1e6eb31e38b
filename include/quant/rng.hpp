// quant/rng.hpp -- drop-in for /root/reference/proj/include/quant/rng.hpp:17-64:
// the seeded mt19937_64 stream with portable derived draws. Every seeded law of
// the device initialisers (csrc/init.cu) consumes this exact stream.
#ifndef QUANT_RNG_HPP
#define QUANT_RNG_HPP

#include <cstdint>
#include <random>
#include <span>
#include <stdexcept>
#include <vector>

namespace quant {

class Rng {
  public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    std::uint64_t next_u64() { return gen_(); }
    // uniform in [0, n) by rejection (no modulo bias); n == 0 throws
    std::uint64_t next_below(std::uint64_t n);
    // uniform in [0, 1) with 53 random bits
    double next_unit() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }

  private:
    std::mt19937_64 gen_;
};

// index drawn with probability mass[i] / sum(mass) by a sequential prefix
std::size_t weighted_draw(std::span<const double> mass, Rng &rng);

// k distinct indices of [0, n), uniform, in selection order (partial Fisher-Yates)
std::vector<std::size_t> sample_indices_uniform(std::size_t n, std::size_t k, Rng &rng);

// k distinct indices drawn proportionally to positive weights without
// replacement (exponential keys log(u)/w, largest first)
std::vector<std::size_t> sample_indices_weighted(std::span<const double> weights, std::size_t k, Rng &rng);

} // namespace quant

#endif
