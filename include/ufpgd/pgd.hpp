// Reference-compatible PGD API (/root/reference/proj/core/include/ufpgd/pgd.hpp:16-115),
// executed on the B200 through the C ABI (include/ufpgd_gpu.h). Results are
// computed in FP32 on the device (parity bar: 1e-4 relative Frobenius against
// the FP64 reference), except lipschitz_bound, which runs the reference's
// converged rule in FP64 on the device.
#pragma once

#include <optional>
#include <vector>

#include "ufpgd/system_config.hpp"
#include "ufpgd/types.hpp"

namespace ufpgd {

struct PgdParams {
  double lambda = 1.0 / 15.0;
  double eta = 0.0;
  long max_iters = 0;
  double residual_tol = 0.0;
  long trace_every = 0;  // > 0: record a TraceRecord every trace_every iterations (pgd.cpp:196-223)

  void validate() const;  // pgd.cpp:33-49
};

struct TraceRecord {
  long index = 0;
  double lagrangian = 0.0;
  double residual = 0.0;
  double pcg = 0.0;
  double sum_rate = 0.0;
  double active_columns = 0.0;
};

struct SolveTrace {
  std::vector<TraceRecord> records;
};

// grad f(W) = (W H^T) H^* - (sigma_nu D^{1/2}) H^*  (pgd.hpp:41-46).
ComplexMatrix grad_f(const PrecoderMatrix& precoder, const ChannelMatrix& channel,
                     const SystemConfig& cfg);

// pgd.hpp:48-62. The pieces are kept for API compatibility; apply() runs on
// the device with the constraint folded into the K x K residual.
struct SmoothGradient {
  ComplexMatrix h_trans;  // M x K
  ComplexMatrix h_conj;   // K x M
  ComplexMatrix offset;   // K x M, diag(c) H^*
  ChannelMatrix channel;
  RealVector c;

  static SmoothGradient make(const ChannelMatrix& channel, const SystemConfig& cfg);
  ComplexMatrix apply(const PrecoderMatrix& precoder) const;
  void apply_into(const PrecoderMatrix& precoder, ComplexMatrix& scratch, ComplexMatrix& out) const;
};

PrecoderMatrix prox_l21(const ComplexMatrix& input, double t);
PrecoderMatrix pgd_step(const PrecoderMatrix& precoder, const ChannelMatrix& channel,
                        const SystemConfig& cfg, double lambda, double eta);

struct LipschitzBound {
  double exact = 0.0;
  double mp = 0.0;
};

double mp_bound(int num_users, int num_antennas);
LipschitzBound lipschitz_bound(const ChannelMatrix& channel);
double lagrangian_value(const PrecoderMatrix& precoder, const ChannelMatrix& channel,
                        const SystemConfig& cfg, double lambda);

struct PgdResult {
  PrecoderMatrix precoder;
  SolveTrace trace;
  long iterations = 0;
};

PgdResult solve_pgd(const ChannelMatrix& channel, const SystemConfig& cfg, const PgdParams& params,
                    const std::optional<PrecoderMatrix>& start = std::nullopt);

PrecoderMatrix oracle_solve(const ChannelMatrix& channel, const SystemConfig& cfg, double lambda);

// Device selection for the calls above (default 0).
void set_device(int device);
int device();

}  // namespace ufpgd
