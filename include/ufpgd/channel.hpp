// ufpgd/channel.hpp of the reference (/root/reference/proj/core/include/ufpgd/channel.hpp:9-18):
// generate_channel is declared with the random source in ufpgd/rng.hpp; seeded
// batches come from ufpgd_generate_channels / ufpgd_gpu_generate_channels.
#pragma once

#include "ufpgd/rng.hpp"
#include "ufpgd/system_config.hpp"
#include "ufpgd/types.hpp"

namespace ufpgd {

// Received vector r = H W^T s + n, n ~ CN(0, sigma_nu^2 I) (channel.cpp:18-34);
// std::invalid_argument on a shape mismatch. A host helper for link-level
// simulation, not part of the solver path.
ComplexVector simulate_received(const ChannelMatrix& channel, const PrecoderMatrix& precoder,
                                const ComplexVector& symbols, const SystemConfig& cfg, Rng& rng);

}  // namespace ufpgd
