// Batched entry points: the reason this library exists. They take the
// reference's per-channel storage stacked into one [B][M][K] complex<float>
// array (what `parallel_for` over channels did on the CPU, parallel.hpp:12-18)
// and run the whole batch on the device(s).
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

#include "ufpgd/metrics.hpp"
#include "ufpgd/pgd.hpp"
#include "ufpgd/system_config.hpp"
#include "ufpgd/training.hpp"
#include "ufpgd/unfolded.hpp"

namespace ufpgd {

enum class StartMode { Zero = 0, ConjChannel = 1, Given = 2 };

struct BatchResult {
  std::vector<std::complex<float>> precoders;  // [B][M][K]
  std::vector<std::int32_t> diverged_at;       // -1 = ok
  std::vector<float> steps;                    // PGD: the 1/L step used per realization
  double consumed_power_sum = 0.0;             // sum over non-diverged of alpha ||W||_{2,1}
  double active_sum = 0.0;                     // sum of active antennas
  long diverged = 0;
};

// forward over B channels (unfolded.cpp:83-146 per channel). Validates the
// network exactly like forward (projected steps, matching K, M); does not
// throw on divergence — per-realization indices are returned.
BatchResult forward_batch(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                          const SystemConfig& cfg, StartMode start = StartMode::ConjChannel,
                          const std::complex<float>* W0 = nullptr);

// solve_pgd over B channels with eta_b = 1 / (power_steps-step power iteration)
// and threshold lambda * eta_b (BASELINE config 3), W0 = H^*.
BatchResult solve_pgd_batch(const std::complex<float>* channels, std::int64_t B, const SystemConfig& cfg,
                            double lambda, long iterations, int power_steps = 30);

// forward_batch sharded over `ngpus` devices of this process (one NCCL
// all-reduce of the statistics).
BatchResult forward_batch_multi_gpu(const UnfoldedNetwork& net, const std::complex<float>* channels,
                                    std::int64_t B, const SystemConfig& cfg, int ngpus);

// The per-sample body of train (training.cpp:205-246) for one mini-batch on
// the device: taped forward from H^*, loss, loss gradient, backward, then the
// deterministic batch mean. grads are packed (d_lambda_0, d_eta_0, ...) as
// pack_params orders them (training.hpp:50-51), ready for adam_update.
// (LossKind and EvaluationSummary are declared in ufpgd/training.hpp.)

struct TrainGradients {
  double loss = 0.0;          // batch mean loss
  std::vector<double> grads;  // batch mean gradient, size 2L
};

TrainGradients train_gradients(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                               const SystemConfig& cfg, LossKind kind = LossKind::Unsupervised,
                               double lambda_cost = 1.0 / 15.0, const std::complex<float>* labels = nullptr);

// oracle_solve (pgd.cpp:270-279) over many channels in FP64 on the device —
// the supervised labels of train (commands.cpp:163-168): converged power
// iteration, then PGD with the 1e-10 relative-change stop, one warp per
// channel retiring on convergence. Same results as the per-channel call;
// ConvergenceError / DivergenceError name the first failing channel.
std::vector<PrecoderMatrix> oracle_solve_batch(const std::vector<ChannelMatrix>& channels, const SystemConfig& cfg,
                                               double lambda);

// evaluate (training.cpp:310-421) over a stacked complex<float> batch without
// per-layer curves: singular channels are counted in `singular` and skipped
// instead of throwing.
EvaluationSummary evaluate_batch(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                                 const SystemConfig& cfg);

}  // namespace ufpgd
