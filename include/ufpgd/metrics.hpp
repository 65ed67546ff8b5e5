// Summary metrics of /root/reference/proj/core/include/ufpgd/metrics.hpp:10-42
// that the batched path reports (host FP64 on single matrices).
#pragma once

#include "ufpgd/system_config.hpp"
#include "ufpgd/types.hpp"

namespace ufpgd {

double l21_norm(const PrecoderMatrix& precoder);
double tx_power(const PrecoderMatrix& precoder);
double consumed_power(const PrecoderMatrix& precoder, double alpha);
double constraint_residual(const ChannelMatrix& channel, const PrecoderMatrix& precoder,
                           const SystemConfig& cfg);
int count_active_columns(const PrecoderMatrix& precoder);

}  // namespace ufpgd
