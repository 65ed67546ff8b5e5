// Deterministic random source of /root/reference/proj/core/include/ufpgd/rng.hpp:15-50
// and generate_channel (channel.hpp:9-11): seeded harness inputs.
#pragma once

#include <cstdint>
#include <random>
#include <utility>
#include <vector>

#include "ufpgd/system_config.hpp"
#include "ufpgd/types.hpp"

namespace ufpgd {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  static Rng stream(std::uint64_t seed, std::uint64_t stream_index);
  std::uint64_t next_u64() { return gen_(); }
  double uniform();
  double uniform_open();
  std::size_t index_below(std::size_t n);
  Complex complex_gaussian();

 private:
  std::mt19937_64 gen_;
};

ChannelMatrix generate_channel(const SystemConfig& cfg, Rng& rng);

// In-place Fisher-Yates shuffle driven by `rng` (rng.hpp:43-50): the order
// train's mini-batches are drawn in.
template <class T>
void shuffle(std::vector<T>& items, Rng& rng) {
  for (std::size_t i = items.size(); i > 1; --i) {
    const std::size_t j = rng.index_below(i);
    std::swap(items[i - 1], items[j]);
  }
}

}  // namespace ufpgd
