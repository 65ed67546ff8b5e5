// Deterministic random source of /root/reference/proj/core/include/ufpgd/rng.hpp:15-50
// and generate_channel (channel.hpp:9-11): seeded harness inputs.
#pragma once

#include <cstdint>
#include <random>

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

}  // namespace ufpgd
