// ufpgd/channel.hpp of the reference (/root/reference/proj/core/include/ufpgd/channel.hpp:9-11):
// generate_channel is declared with the random source in ufpgd/rng.hpp; seeded
// batches come from ufpgd_generate_channels / ufpgd_gpu_generate_channels.
#pragma once

#include "ufpgd/rng.hpp"
