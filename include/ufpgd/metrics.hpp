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

// Device-evaluated (FP64) metrics of metrics.hpp:18-58 / zf.hpp:9-18.
PrecoderMatrix zf_precoder(const ChannelMatrix& channel, const SystemConfig& cfg);  // SingularChannelError
RealVector sinr_per_user(const ChannelMatrix& channel, const PrecoderMatrix& precoder, const SystemConfig& cfg);
double sum_rate(const RealVector& sinr);
double pcg(const ChannelMatrix& channel, const PrecoderMatrix& precoder, const SystemConfig& cfg);
double pcg_from_reference(const PrecoderMatrix& zf_reference, const PrecoderMatrix& precoder);

struct MetricsReport {
  double tx_power = 0.0;
  double cons_power = 0.0;
  RealVector sinr;
  double sum_rate = 0.0;
  double pcg = 0.0;
  double residual = 0.0;
};

// compute_metrics with the ZF reference computed on the device for `channel`
// (the reference takes a precomputed zf_reference; evaluate computes it per
// channel right before, training.cpp:328).
MetricsReport compute_metrics(const ChannelMatrix& channel, const PrecoderMatrix& precoder,
                              const SystemConfig& cfg);

}  // namespace ufpgd
