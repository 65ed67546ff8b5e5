// C++ API with the reference's signatures (include/ufpgd/*.hpp), implemented
// on the C ABI (include/ufpgd_gpu.h). Validation and exceptions follow the
// reference (pgd.cpp, unfolded.cpp, system_config.cpp); all precoder math runs
// on the device. Scalar helpers (mp_bound, project_params, constraint_diag,
// metrics of one matrix) are host code, as in the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <complex>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <limits>
#include <numbers>
#include <numeric>
#include <string>
#include <vector>

#include "ufpgd/batch.hpp"
#include "ufpgd/dataset.hpp"
#include "ufpgd/errors.hpp"
#include "ufpgd/metrics.hpp"
#include "ufpgd/pgd.hpp"
#include "ufpgd/rng.hpp"
#include "ufpgd/system_config.hpp"
#include "ufpgd/training.hpp"
#include "ufpgd/unfolded.hpp"
#include "ufpgd_gpu.h"

namespace ufpgd {
namespace {

int g_device = 0;

[[noreturn]] void raise(int rc, long index = -1) {
  const std::string msg = ufpgd_gpu_last_error();
  switch (rc) {
    case UFPGD_EINVAL_SHAPE:
    case UFPGD_EINVAL_PARAM:
      throw std::invalid_argument(msg);
    case UFPGD_EDIVERGED:
      throw DivergenceError(msg, index);
    case UFPGD_ECONVERGENCE:
      throw ConvergenceError(msg);
    default:
      throw DeviceError("ufpgd device error " + std::to_string(rc) + ": " + msg);
  }
}

void check(int rc) {
  if (rc != UFPGD_OK) raise(rc);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer.
template <class T>
struct DeviceBuffer {
  T* p = nullptr;
  std::size_t n = 0;
  explicit DeviceBuffer(std::size_t count) : n(count) {
    if (n) cuda_check(cudaMalloc(&p, sizeof(T) * n), "cudaMalloc");
  }
  ~DeviceBuffer() {
    if (p) cudaFree(p);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void upload(const T* h) { cuda_check(cudaMemcpy(p, h, sizeof(T) * n, cudaMemcpyHostToDevice), "H2D"); }
  void download(T* h) const { cuda_check(cudaMemcpy(h, p, sizeof(T) * n, cudaMemcpyDeviceToHost), "D2H"); }
};

struct DeviceScope {
  int prev = 0;
  DeviceScope() {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(g_device), "cudaSetDevice");
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

// K x M complex<double> (col-major) -> complex64 [M][K] (same element order).
std::vector<ufpgd_c64> to_c64(const ComplexMatrix& A) {
  std::vector<ufpgd_c64> out(static_cast<std::size_t>(A.size()));
  const Complex* d = A.data();
  for (std::size_t i = 0; i < out.size(); ++i)
    out[i] = {static_cast<float>(d[i].real()), static_cast<float>(d[i].imag())};
  return out;
}

ComplexMatrix from_c64(const ufpgd_c64* d, std::ptrdiff_t K, std::ptrdiff_t M) {
  ComplexMatrix A(K, M);
  Complex* o = A.data();
  for (std::ptrdiff_t i = 0; i < K * M; ++i) o[i] = Complex(d[i].re, d[i].im);
  return A;
}

void check_shapes(const ChannelMatrix& channel, const SystemConfig& cfg) {  // pgd.cpp:16-21
  cfg.validate();
  if (channel.rows() != cfg.K || channel.cols() != cfg.M)
    throw std::invalid_argument("channel shape does not match SystemConfig");
}

constexpr double kBoundSlack = 1e-12;  // unfolded.cpp:17

void check_projected(const UnfoldedNetwork& net) {  // unfolded.cpp:19-35
  const double hi = 1.0 / net.mp_bound, lo = 0.5 * hi;
  for (std::size_t i = 0; i < net.layers.size(); ++i) {
    const LayerParams& l = net.layers[i];
    if (!(l.lambda_i >= 0.0) || !std::isfinite(l.lambda_i))
      throw std::invalid_argument("UnfoldedNetwork: layer " + std::to_string(i) + " lambda_i < 0");
    if (!(l.eta_i >= lo * (1.0 - kBoundSlack)) || !(l.eta_i <= hi * (1.0 + kBoundSlack)))
      throw std::invalid_argument("UnfoldedNetwork: layer " + std::to_string(i) + " eta_i outside [1/(2L), 1/L]");
  }
}

// Runs the FP64 general-shape layer sweep on one realization: the reference's
// own precision, on the device. A ComplexMatrix (col-major complex<double>)
// is already the kernel's interleaved [M][K] FP64 layout.
struct LayerRun {
  PrecoderMatrix W;
  int32_t diverged = -1;
  int64_t iterations = 0;
  std::vector<double> iterates, tape_v, tape_norms, tape_shrink;
};

LayerRun run_layers(const ChannelMatrix& H, const RealVector& c, const std::vector<double>& eta,
                    const std::vector<double>& thr, int w0_mode, const ComplexMatrix* W0, int mode,
                    double residual_tol, int index_base, bool iterates, bool tape) {
  const int K = static_cast<int>(H.rows()), M = static_cast<int>(H.cols());
  const int L = mode == 1 ? 1 : static_cast<int>(eta.size());
  const std::size_t n = static_cast<std::size_t>(K) * M;
  DeviceScope scope;
  DeviceBuffer<double> dH(2 * n), dW(2 * n), dW0(W0 ? 2 * n : 0);
  DeviceBuffer<int32_t> ddiv(1);
  DeviceBuffer<int64_t> dits(1);
  DeviceBuffer<double> ditr(iterates ? 2 * (L + 1) * n : 0), dtv(tape ? 2 * L * n : 0);
  DeviceBuffer<double> dtn(tape ? static_cast<std::size_t>(L) * M : 0), dts(tape ? static_cast<std::size_t>(L) * M : 0);
  dH.upload(reinterpret_cast<const double*>(H.data()));
  if (W0) dW0.upload(reinterpret_cast<const double*>(W0->data()));
  check(ufpgd_gpu_layers_general64(dH.p, 1, K, M, eta.data(), thr.data(), L, c.data(), w0_mode, dW0.p, mode,
                                   residual_tol, index_base, dW.p, ddiv.p, dits.p, ditr.p, dtv.p, dtn.p, dts.p,
                                   g_device, nullptr));
  cuda_check(cudaDeviceSynchronize(), "layers_general64");
  LayerRun r;
  r.W = ComplexMatrix(K, M);
  dW.download(reinterpret_cast<double*>(r.W.data()));
  ddiv.download(&r.diverged);
  dits.download(&r.iterations);
  if (iterates) {
    r.iterates.resize(2 * (L + 1) * n);
    ditr.download(r.iterates.data());
  }
  if (tape) {
    r.tape_v.resize(2 * L * n);
    r.tape_norms.resize(static_cast<std::size_t>(L) * M);
    r.tape_shrink.resize(static_cast<std::size_t>(L) * M);
    dtv.download(r.tape_v.data());
    dtn.download(r.tape_norms.data());
    dts.download(r.tape_shrink.data());
  }
  return r;
}

ComplexMatrix from_f64(const double* d, std::ptrdiff_t K, std::ptrdiff_t M) {
  ComplexMatrix A(K, M);
  std::memcpy(static_cast<void*>(A.data()), d, sizeof(double) * 2 * K * M);
  return A;
}

std::uint64_t mix64(std::uint64_t x) {  // rng.cpp:10-15
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

}  // namespace

// ---- system_config.cpp -------------------------------------------------------
SystemConfig SystemConfig::uniform(int num_users, int num_antennas, double sinr_target, double noise_std,
                                   double pa_scale) {
  SystemConfig cfg;
  cfg.K = num_users;
  cfg.M = num_antennas;
  cfg.sigma_nu = noise_std;
  cfg.gamma = RealVector::Constant(std::max(num_users, 0), sinr_target);
  cfg.alpha = pa_scale;
  cfg.validate();
  return cfg;
}

void SystemConfig::validate() const {
  if (K < 1) throw std::invalid_argument("SystemConfig: K must be >= 1");
  if (M < K)
    throw std::invalid_argument("SystemConfig: need K <= M, got K=" + std::to_string(K) + " M=" + std::to_string(M));
  if (!(sigma_nu >= 0.0)) throw std::invalid_argument("SystemConfig: sigma_nu must be >= 0");
  if (gamma.size() != K) throw std::invalid_argument("SystemConfig: gamma must have K entries");
  for (std::ptrdiff_t k = 0; k < gamma.size(); ++k)
    if (!(gamma[k] > 0.0)) throw std::invalid_argument("SystemConfig: gamma[" + std::to_string(k) + "] must be > 0");
  if (!(alpha > 0.0)) throw std::invalid_argument("SystemConfig: alpha must be > 0");
}

RealVector SystemConfig::constraint_diag() const {
  RealVector c(gamma.size());
  for (std::ptrdiff_t k = 0; k < gamma.size(); ++k) c[k] = sigma_nu * std::sqrt(gamma[k]);
  return c;
}

// ---- rng.cpp / channel.cpp ------------------------------------------------------
Rng Rng::stream(std::uint64_t seed, std::uint64_t stream_index) { return Rng(mix64(seed ^ mix64(stream_index))); }
double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double Rng::uniform_open() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
std::size_t Rng::index_below(std::size_t n) { return static_cast<std::size_t>(next_u64() % n); }
Complex Rng::complex_gaussian() {
  const double radius = std::sqrt(-std::log(uniform_open()));
  const double angle = 2.0 * std::numbers::pi * uniform();
  return {radius * std::cos(angle), radius * std::sin(angle)};
}

ChannelMatrix generate_channel(const SystemConfig& cfg, Rng& rng) {
  cfg.validate();
  ChannelMatrix h(cfg.K, cfg.M);
  for (int k = 0; k < cfg.K; ++k)
    for (int m = 0; m < cfg.M; ++m) h(k, m) = rng.complex_gaussian();
  return h;
}

// ---- pgd.cpp ------------------------------------------------------------------
void set_device(int d) { g_device = d; }
int device() { return g_device; }

void PgdParams::validate() const {
  if (!(lambda >= 0.0)) throw std::invalid_argument("PgdParams: lambda must be >= 0");
  if (!(eta > 0.0)) throw std::invalid_argument("PgdParams: eta must be > 0");
  if (max_iters < 0) throw std::invalid_argument("PgdParams: max_iters must be >= 0");
  if (!(residual_tol >= 0.0)) throw std::invalid_argument("PgdParams: residual_tol must be >= 0");
  if (trace_every < 0) throw std::invalid_argument("PgdParams: trace_every must be >= 0");
}

SmoothGradient SmoothGradient::make(const ChannelMatrix& channel, const SystemConfig& cfg) {
  check_shapes(channel, cfg);
  SmoothGradient g;
  g.h_trans = channel.transpose();
  g.h_conj = channel.conjugate();
  g.c = cfg.constraint_diag();
  g.offset = g.h_conj;
  for (std::ptrdiff_t m = 0; m < g.offset.cols(); ++m)
    for (std::ptrdiff_t k = 0; k < g.offset.rows(); ++k) g.offset(k, m) *= g.c[k];
  g.channel = channel;
  return g;
}

ComplexMatrix SmoothGradient::apply(const PrecoderMatrix& precoder) const {
  if (precoder.rows() != channel.rows() || precoder.cols() != channel.cols())
    throw std::invalid_argument("SmoothGradient: precoder shape mismatch");
  return run_layers(channel, c, {0.0}, {0.0}, UFPGD_W0_GIVEN, &precoder, 1, 0.0, 0, false, false).W;
}

void SmoothGradient::apply_into(const PrecoderMatrix& precoder, ComplexMatrix& scratch, ComplexMatrix& out) const {
  scratch = ComplexMatrix(precoder.rows(), precoder.rows());
  out = apply(precoder);
}

ComplexMatrix grad_f(const PrecoderMatrix& precoder, const ChannelMatrix& channel, const SystemConfig& cfg) {
  if (precoder.rows() != channel.rows() || precoder.cols() != channel.cols())
    throw std::invalid_argument("grad_f: precoder/channel shape mismatch");
  return SmoothGradient::make(channel, cfg).apply(precoder);
}

PrecoderMatrix prox_l21(const ComplexMatrix& input, double t) {
  if (!(t >= 0.0)) throw std::invalid_argument("prox_l21: threshold must be >= 0");
  // eta = 0 leaves V = W; the channel is irrelevant (a zero K x M channel).
  ChannelMatrix zero(input.rows(), input.cols());
  RealVector c(input.rows(), 0.0);
  return run_layers(zero, c, {0.0}, {t}, UFPGD_W0_GIVEN, &input, 0, 0.0, 0, false, false).W;
}

PrecoderMatrix pgd_step(const PrecoderMatrix& precoder, const ChannelMatrix& channel, const SystemConfig& cfg,
                        double lambda, double eta) {
  if (!(lambda >= 0.0) || !(eta > 0.0)) throw std::invalid_argument("pgd_step: need lambda >= 0 and eta > 0");
  check_shapes(channel, cfg);
  if (precoder.rows() != cfg.K || precoder.cols() != cfg.M)
    throw std::invalid_argument("grad_f: precoder/channel shape mismatch");
  return run_layers(channel, cfg.constraint_diag(), {eta}, {lambda * eta}, UFPGD_W0_GIVEN, &precoder, 0, 0.0, 0,
                    false, false)
      .W;
}

double mp_bound(int num_users, int num_antennas) {  // pgd.cpp:111-118
  if (num_users < 1 || num_antennas < 1) throw std::invalid_argument("mp_bound: dimensions must be positive");
  const double edge = std::sqrt(static_cast<double>(num_users)) + std::sqrt(static_cast<double>(num_antennas));
  return edge * edge;
}

LipschitzBound lipschitz_bound(const ChannelMatrix& channel) {
  if (channel.rows() < 1 || channel.cols() < 1) throw std::invalid_argument("lipschitz_bound: empty channel");
  LipschitzBound b;
  b.mp = mp_bound(static_cast<int>(channel.rows()), static_cast<int>(channel.cols()));
  DeviceScope scope;
  const std::size_t n = static_cast<std::size_t>(channel.size());
  DeviceBuffer<double> dH(2 * n), dL(1);
  DeviceBuffer<int32_t> dst(1);
  dH.upload(reinterpret_cast<const double*>(channel.data()));
  check(ufpgd_gpu_lipschitz_exact(dH.p, 1, static_cast<int>(channel.rows()), static_cast<int>(channel.cols()), dL.p,
                                  dst.p, g_device, nullptr));
  int32_t st = 0;
  dst.download(&st);
  if (st != 0)
    throw ConvergenceError("lipschitz_bound: power iteration did not reach tolerance 1e-8 within 10000 iterations");
  dL.download(&b.exact);
  return b;
}

double lagrangian_value(const PrecoderMatrix& precoder, const ChannelMatrix& channel, const SystemConfig& cfg,
                        double lambda) {
  const double r = constraint_residual(channel, precoder, cfg);
  return lambda * l21_norm(precoder) + r * r;
}

PgdResult solve_pgd(const ChannelMatrix& channel, const SystemConfig& cfg, const PgdParams& params,
                    const std::optional<PrecoderMatrix>& start) {  // pgd.cpp:178-268
  check_shapes(channel, cfg);
  params.validate();
  if (start && (start->rows() != cfg.K || start->cols() != cfg.M))
    throw std::invalid_argument("solve_pgd: W0 shape mismatch");
  PgdResult result;
  const bool tracing = params.trace_every > 0;
  PrecoderMatrix zf_reference;
  if (tracing) zf_reference = zf_precoder(channel, cfg);  // SingularChannelError as in the reference
  PrecoderMatrix w = start ? *start : channel.conjugate();
  // Trace record (pgd.cpp:204-221): FP64 on the host from the device iterate,
  // exactly the reference's formulae (diagnostics, off the solver path).
  auto record = [&](long index) {
    const int K = cfg.K, M = cfg.M;
    const RealVector c = cfg.constraint_diag();
    TraceRecord rec;
    rec.index = index;
    double res2 = 0.0;
    RealVector sinr(K);
    const double noise = cfg.sigma_nu * cfg.sigma_nu;
    for (int k = 0; k < K; ++k) {
      double row2 = 0.0, signal = 0.0;
      for (int j = 0; j < K; ++j) {
        Complex e = 0.0;  // effective channel (H W^T)(k, j)
        for (int m = 0; m < M; ++m) e += channel(k, m) * w(j, m);
        const double p2 = std::norm(e);
        row2 += p2;
        if (j == k) signal = p2;
        res2 += std::norm(j == k ? e - c[k] : e);
      }
      sinr[k] = signal / (row2 - signal + noise);
    }
    rec.residual = std::sqrt(res2);
    rec.lagrangian = params.lambda * l21_norm(w) + rec.residual * rec.residual;
    rec.pcg = pcg_from_reference(zf_reference, w);
    rec.sum_rate = sum_rate(sinr);
    rec.active_columns = count_active_columns(w);
    result.trace.records.push_back(rec);
  };
  if (tracing) record(0);
  if (params.max_iters == 0) {
    result.precoder = w;
    return result;
  }
  const int K = cfg.K, M = cfg.M;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  DeviceScope scope;
  DeviceBuffer<double> dH(2 * n), dW(2 * n), dW0(2 * n), deta(1);
  DeviceBuffer<int32_t> ddiv(1);
  DeviceBuffer<int64_t> dits(1);
  dH.upload(reinterpret_cast<const double*>(channel.data()));
  deta.upload(&params.eta);
  const RealVector c = cfg.constraint_diag();
  // Without tracing one launch runs every iteration; with tracing the solve
  // runs in chunks of trace_every iterations, each restarting from the last
  // iterate (the iteration is memoryless), with a record after every chunk.
  const long chunk = tracing ? params.trace_every : params.max_iters;
  long done = 0, last_recorded = 0;
  while (done < params.max_iters) {
    const long its_now = std::min(chunk, params.max_iters - done);
    dW0.upload(reinterpret_cast<const double*>(w.data()));
    check(ufpgd_gpu_solve_pgd64(dH.p, 1, K, M, c.data(), params.lambda, deta.p, its_now, params.residual_tol, dW0.p,
                                dW.p, dits.p, ddiv.p, g_device, nullptr));
    cuda_check(cudaDeviceSynchronize(), "solve_pgd");
    int32_t div = -1;
    ddiv.download(&div);
    if (div >= 0) throw DivergenceError("solve_pgd: non-finite iterate", done + div);
    w = ComplexMatrix(K, M);
    dW.download(reinterpret_cast<double*>(w.data()));
    int64_t its = 0;
    dits.download(&its);
    done += its;
    result.iterations = done;
    if (tracing && done % params.trace_every == 0) {
      record(done);
      last_recorded = done;
    }
    if (its < its_now) break;  // residual_tol stop inside the chunk
  }
  if (tracing && result.iterations > last_recorded) record(result.iterations);
  result.precoder = std::move(w);
  return result;
}

PrecoderMatrix oracle_solve(const ChannelMatrix& channel, const SystemConfig& cfg, double lambda) {
  check_shapes(channel, cfg);
  if (!(lambda >= 0.0)) throw std::invalid_argument("PgdParams: lambda must be >= 0");
  const int K = cfg.K, M = cfg.M;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  DeviceScope scope;
  DeviceBuffer<double> dH(2 * n), dW(2 * n);
  DeviceBuffer<int32_t> dst(1);
  dH.upload(reinterpret_cast<const double*>(channel.data()));
  const RealVector c = cfg.constraint_diag();
  check(ufpgd_gpu_oracle_solve(dH.p, 1, K, M, c.data(), lambda, 100000, 1e-10, dW.p, nullptr, nullptr, dst.p, g_device,
                               nullptr));
  int32_t st = 0;
  dst.download(&st);
  if (st == UFPGD_ECONVERGENCE)
    throw ConvergenceError("lipschitz_bound: power iteration did not reach tolerance 1e-8 within 10000 iterations");
  if (st == UFPGD_EDIVERGED) throw DivergenceError("solve_pgd: non-finite iterate", -1);
  ComplexMatrix W(K, M);
  dW.download(reinterpret_cast<double*>(W.data()));
  return W;
}

std::vector<PrecoderMatrix> oracle_solve_batch(const std::vector<ChannelMatrix>& channels, const SystemConfig& cfg,
                                               double lambda) {
  cfg.validate();
  if (!(lambda >= 0.0)) throw std::invalid_argument("PgdParams: lambda must be >= 0");
  for (const ChannelMatrix& h : channels) check_shapes(h, cfg);
  const int K = cfg.K, M = cfg.M;
  const std::size_t n = static_cast<std::size_t>(K) * M, B = channels.size();
  std::vector<PrecoderMatrix> out;
  if (B == 0) return out;
  DeviceScope scope;
  DeviceBuffer<double> dH(2 * n * B), dW(2 * n * B);
  DeviceBuffer<int32_t> dst(B);
  std::vector<double> stage(2 * n * B);
  for (std::size_t b = 0; b < B; ++b)
    std::memcpy(&stage[2 * n * b], static_cast<const void*>(channels[b].data()), 2 * n * sizeof(double));
  dH.upload(stage.data());
  const RealVector c = cfg.constraint_diag();
  check(ufpgd_gpu_oracle_solve(dH.p, static_cast<int64_t>(B), K, M, c.data(), lambda, 100000, 1e-10, dW.p, nullptr,
                               nullptr, dst.p, g_device, nullptr));
  std::vector<int32_t> st(B);
  dst.download(st.data());
  for (std::size_t b = 0; b < B; ++b) {
    if (st[b] == UFPGD_ECONVERGENCE)
      throw ConvergenceError("lipschitz_bound: power iteration did not reach tolerance 1e-8 within 10000 iterations "
                             "(channel " + std::to_string(b) + ")");
    if (st[b] == UFPGD_EDIVERGED) throw DivergenceError("solve_pgd: non-finite iterate (channel " + std::to_string(b) + ")", -1);
  }
  dW.download(stage.data());
  out.reserve(B);
  for (std::size_t b = 0; b < B; ++b) {
    ComplexMatrix W(K, M);
    std::memcpy(static_cast<void*>(W.data()), &stage[2 * n * b], 2 * n * sizeof(double));
    out.push_back(std::move(W));
  }
  return out;
}

// ---- unfolded.cpp -------------------------------------------------------------
UnfoldedNetwork UnfoldedNetwork::pgd_init(int num_users, int num_antennas, int num_layers, double lambda) {
  if (num_layers < 1) throw std::invalid_argument("pgd_init: need at least one layer");
  if (!(lambda >= 0.0)) throw std::invalid_argument("pgd_init: lambda must be >= 0");
  UnfoldedNetwork net;
  net.num_users = num_users;
  net.num_antennas = num_antennas;
  net.mp_bound = ufpgd::mp_bound(num_users, num_antennas);
  net.layers.assign(static_cast<std::size_t>(num_layers), LayerParams{lambda, 1.0 / net.mp_bound});
  net.validate();
  return net;
}

void UnfoldedNetwork::validate() const {
  if (num_users < 1 || num_antennas < num_users) throw std::invalid_argument("UnfoldedNetwork: bad dimensions");
  if (layers.empty()) throw std::invalid_argument("UnfoldedNetwork: no layers");
  const double expected = ufpgd::mp_bound(num_users, num_antennas);
  if (!(std::abs(mp_bound - expected) <= 1e-9 * expected))
    throw std::invalid_argument("UnfoldedNetwork: mp_bound does not match (K, M)");
}

UnfoldedNetwork project_params(const UnfoldedNetwork& net) {
  net.validate();
  UnfoldedNetwork p = net;
  const double hi = 1.0 / p.mp_bound, lo = 0.5 * hi;
  for (LayerParams& l : p.layers) {
    l.lambda_i = std::max(0.0, l.lambda_i);
    l.eta_i = std::min(std::max(l.eta_i, lo), hi);
  }
  return p;
}

ForwardResult forward(const UnfoldedNetwork& net, const ChannelMatrix& channel, const SystemConfig& cfg,
                      const std::optional<PrecoderMatrix>& start, const ForwardOptions& options) {
  net.validate();
  check_projected(net);
  cfg.validate();
  if (cfg.K != net.num_users || cfg.M != net.num_antennas || channel.rows() != cfg.K || channel.cols() != cfg.M)
    throw std::invalid_argument("forward: dimension mismatch");
  if (start && (start->rows() != cfg.K || start->cols() != cfg.M))
    throw std::invalid_argument("forward: W0 shape mismatch");
  const int L = static_cast<int>(net.layers.size());
  std::vector<double> eta, thr;
  for (const LayerParams& l : net.layers) {
    eta.push_back(l.eta_i);
    thr.push_back(l.lambda_i * l.eta_i);
  }
  ForwardResult result;
  // Networks deeper than one launch's parameter block are chained.
  if (L > UFPGD_MAX_LAYERS && !options.with_tape && !options.with_iterates) {
    PrecoderMatrix w = start ? *start : channel.conjugate();
    for (int l0 = 0; l0 < L; l0 += UFPGD_MAX_LAYERS) {
      const int l1 = std::min(L, l0 + UFPGD_MAX_LAYERS);
      LayerRun r = run_layers(channel, cfg.constraint_diag(), {eta.begin() + l0, eta.begin() + l1},
                              {thr.begin() + l0, thr.begin() + l1}, UFPGD_W0_GIVEN, &w, 0, 0.0, 0, false, false);
      if (r.diverged >= 0) throw DivergenceError("forward: non-finite iterate at layer", l0 + r.diverged);
      w = r.W;
    }
    result.output = w;
    return result;
  }
  if (L > UFPGD_MAX_LAYERS) throw std::invalid_argument("forward: tapes support at most UFPGD_MAX_LAYERS layers");
  LayerRun r = run_layers(channel, cfg.constraint_diag(), eta, thr, start ? UFPGD_W0_GIVEN : UFPGD_W0_CONJ_H,
                          start ? &*start : nullptr, 0, 0.0, 0, options.with_iterates || options.with_tape,
                          options.with_tape);
  if (r.diverged >= 0) throw DivergenceError("forward: non-finite iterate at layer", r.diverged);
  result.output = r.W;
  const std::ptrdiff_t K = cfg.K, M = cfg.M, n = K * M;
  if (options.with_iterates)
    for (int i = 0; i <= L; ++i) result.iterates.push_back(from_f64(r.iterates.data() + 2 * i * n, K, M));
  if (options.with_tape) {
    result.tape.layers.resize(static_cast<std::size_t>(L));
    for (int i = 0; i < L; ++i) {
      LayerTape& t = result.tape.layers[static_cast<std::size_t>(i)];
      t.input = from_f64(r.iterates.data() + 2 * i * n, K, M);
      t.step_image = from_f64(r.tape_v.data() + 2 * i * n, K, M);
      t.column_norms.resize(M);
      t.shrink_factors.resize(M);
      for (std::ptrdiff_t m = 0; m < M; ++m) {
        t.column_norms[m] = r.tape_norms[static_cast<std::size_t>(i * M + m)];
        t.shrink_factors[m] = r.tape_shrink[static_cast<std::size_t>(i * M + m)];
      }
    }
  }
  return result;
}

PrecoderMatrix forward_infer(const UnfoldedNetwork& net, const ChannelMatrix& channel, const SystemConfig& cfg) {
  return forward(net, channel, cfg).output;
}

ParamGradients backward(const ForwardTape& tape, const UnfoldedNetwork& net, const ChannelMatrix& channel,
                        const SystemConfig& cfg, const ComplexMatrix& dcost_dw) {  // unfolded.cpp:158-239
  net.validate();
  cfg.validate();
  const std::size_t depth = net.layers.size();
  if (tape.layers.size() != depth) throw TrainingError("backward: tape depth does not match network");
  if (dcost_dw.rows() != cfg.K || dcost_dw.cols() != cfg.M || channel.rows() != cfg.K || channel.cols() != cfg.M)
    throw TrainingError("backward: shape mismatch");
  for (const LayerTape& layer : tape.layers)
    if (layer.input.rows() != cfg.K || layer.input.cols() != cfg.M || layer.step_image.rows() != cfg.K ||
        layer.step_image.cols() != cfg.M || layer.column_norms.size() != cfg.M ||
        layer.shrink_factors.size() != cfg.M)
      throw TrainingError("backward: malformed tape layer");
  const int K = cfg.K, M = cfg.M, L = static_cast<int>(depth);
  const std::size_t n = static_cast<std::size_t>(K) * M;
  std::vector<double> lam, eta;
  for (const LayerParams& l : net.layers) {
    lam.push_back(l.lambda_i);
    eta.push_back(l.eta_i);
  }
  const RealVector c = cfg.constraint_diag();
  DeviceScope scope;
  DeviceBuffer<double> dH(2 * n), dW0(2 * n), dG(2 * n), dgr(2 * static_cast<std::size_t>(L));
  dH.upload(reinterpret_cast<const double*>(channel.data()));
  dW0.upload(reinterpret_cast<const double*>(tape.layers[0].input.data()));
  dG.upload(reinterpret_cast<const double*>(dcost_dw.data()));
  check(ufpgd_gpu_unfolded_backward64(dH.p, 1, K, M, lam.data(), eta.data(), L, c.data(), UFPGD_W0_GIVEN, dW0.p,
                                      dG.p, dgr.p, g_device, nullptr));
  cuda_check(cudaDeviceSynchronize(), "backward");
  std::vector<double> g(2 * static_cast<std::size_t>(L));
  dgr.download(g.data());
  ParamGradients out;
  for (int i = 0; i < L; ++i) {
    out.d_lambda.push_back(g[2 * static_cast<std::size_t>(i)]);
    out.d_eta.push_back(g[2 * static_cast<std::size_t>(i) + 1]);
  }
  return out;
}

// ---- metrics.cpp ----------------------------------------------------------------
double l21_norm(const PrecoderMatrix& precoder) {
  double total = 0.0;
  for (std::ptrdiff_t m = 0; m < precoder.cols(); ++m) total += precoder.colNorm(m);
  return total;
}

double tx_power(const PrecoderMatrix& precoder) { return precoder.squaredNorm(); }

double consumed_power(const PrecoderMatrix& precoder, double alpha) {
  if (!(alpha > 0.0)) throw std::invalid_argument("consumed_power: alpha must be > 0");
  return alpha * l21_norm(precoder);
}

double constraint_residual(const ChannelMatrix& channel, const PrecoderMatrix& precoder, const SystemConfig& cfg) {
  const RealVector c = cfg.constraint_diag();
  double s = 0.0;
  for (std::ptrdiff_t k = 0; k < channel.rows(); ++k)
    for (std::ptrdiff_t j = 0; j < precoder.rows(); ++j) {
      Complex acc = 0.0;
      for (std::ptrdiff_t m = 0; m < channel.cols(); ++m) acc += channel(k, m) * precoder(j, m);
      if (k == j) acc -= c[k];
      s += std::norm(acc);
    }
  return std::sqrt(s);
}

int count_active_columns(const PrecoderMatrix& precoder) {
  int a = 0;
  for (std::ptrdiff_t m = 0; m < precoder.cols(); ++m)
    if (precoder.colNorm(m) > 0.0) ++a;
  return a;
}

namespace {
// out = {tx, cons, sum_rate, pcg, residual, zf_ok, sinr[K]} for one pair.
std::vector<double> device_metrics(const ChannelMatrix& channel, const PrecoderMatrix& precoder,
                                   const SystemConfig& cfg, PrecoderMatrix* zf_out) {
  cfg.validate();
  if (channel.rows() != cfg.K || channel.cols() != cfg.M || precoder.rows() != cfg.K || precoder.cols() != cfg.M)
    throw std::invalid_argument("sinr_per_user: shape mismatch");
  const int K = cfg.K, M = cfg.M;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  DeviceScope scope;
  DeviceBuffer<ufpgd_c64> dH(n), dW(n), dZ(zf_out ? n : 0);
  DeviceBuffer<double> dout(6 + K);
  const auto h = to_c64(channel);
  const auto w = to_c64(precoder);
  dH.upload(h.data());
  dW.upload(w.data());
  const RealVector c = cfg.constraint_diag();
  check(ufpgd_gpu_metrics(dH.p, dW.p, 1, K, M, c.data(), cfg.sigma_nu, cfg.alpha, dout.p, dZ.p, g_device, nullptr));
  std::vector<double> out(6 + K);
  dout.download(out.data());
  if (zf_out) {
    std::vector<ufpgd_c64> z(n);
    dZ.download(z.data());
    *zf_out = from_c64(z.data(), K, M);
  }
  return out;
}
}  // namespace

PrecoderMatrix zf_precoder(const ChannelMatrix& channel, const SystemConfig& cfg) {
  PrecoderMatrix z;
  const auto out = device_metrics(channel, channel.conjugate(), cfg, &z);
  if (out[5] == 0.0) throw SingularChannelError("zf_precoder: channel Gram matrix is singular");
  return z;
}

RealVector sinr_per_user(const ChannelMatrix& channel, const PrecoderMatrix& precoder, const SystemConfig& cfg) {
  const auto out = device_metrics(channel, precoder, cfg, nullptr);
  RealVector s(cfg.K);
  for (int k = 0; k < cfg.K; ++k) s[k] = out[6 + k];
  return s;
}

double sum_rate(const RealVector& sinr) {  // metrics.cpp:48-54
  double total = 0.0;
  for (std::ptrdiff_t k = 0; k < sinr.size(); ++k) total += std::log2(1.0 + sinr[k]);
  return total;
}

double pcg_from_reference(const PrecoderMatrix& zf_reference, const PrecoderMatrix& precoder) {
  const double denom = l21_norm(precoder);
  if (!(denom > 0.0)) throw std::invalid_argument("pcg: precoder consumes zero power");
  return l21_norm(zf_reference) / denom;
}

double pcg(const ChannelMatrix& channel, const PrecoderMatrix& precoder, const SystemConfig& cfg) {
  if (!(l21_norm(precoder) > 0.0)) throw std::invalid_argument("pcg: precoder consumes zero power");
  const auto out = device_metrics(channel, precoder, cfg, nullptr);
  if (out[5] == 0.0) throw SingularChannelError("zf_precoder: channel Gram matrix is singular");
  return out[3];
}

MetricsReport compute_metrics(const ChannelMatrix& channel, const PrecoderMatrix& precoder, const SystemConfig& cfg) {
  const auto out = device_metrics(channel, precoder, cfg, nullptr);
  if (out[5] == 0.0) throw SingularChannelError("zf_precoder: channel Gram matrix is singular");
  MetricsReport r;
  r.tx_power = out[0];
  r.cons_power = out[1];
  r.sum_rate = out[2];
  r.pcg = out[3];
  r.residual = out[4];
  r.sinr = RealVector(cfg.K);
  for (int k = 0; k < cfg.K; ++k) r.sinr[k] = out[6 + k];
  return r;
}

// ---- batch.hpp ------------------------------------------------------------------
BatchResult forward_batch(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                          const SystemConfig& cfg, StartMode start, const std::complex<float>* W0) {
  net.validate();
  check_projected(net);
  cfg.validate();
  if (cfg.K != net.num_users || cfg.M != net.num_antennas) throw std::invalid_argument("forward: dimension mismatch");
  if (start == StartMode::Given && !W0) throw std::invalid_argument("forward_batch: W0 required");
  std::vector<double> lam, eta;
  for (const LayerParams& l : net.layers) {
    lam.push_back(l.lambda_i);
    eta.push_back(l.eta_i);
  }
  BatchResult r;
  const std::size_t n = static_cast<std::size_t>(B) * cfg.K * cfg.M;
  r.precoders.resize(n);
  r.diverged_at.resize(static_cast<std::size_t>(B));
  double stats[3] = {0, 0, 0};
  const RealVector c = cfg.constraint_diag();
  const int rc = ufpgd_gpu_unfolded_forward_host(
      reinterpret_cast<const ufpgd_c64*>(channels), B, cfg.K, cfg.M, lam.data(), eta.data(),
      static_cast<int>(lam.size()), c.data(), static_cast<int>(start), reinterpret_cast<const ufpgd_c64*>(W0),
      reinterpret_cast<ufpgd_c64*>(r.precoders.data()), r.diverged_at.data(), stats, cfg.alpha, g_device);
  if (rc != UFPGD_OK && rc != UFPGD_EDIVERGED) raise(rc);
  r.consumed_power_sum = stats[0];
  r.active_sum = stats[1];
  r.diverged = static_cast<long>(stats[2]);
  return r;
}

BatchResult solve_pgd_batch(const std::complex<float>* channels, std::int64_t B, const SystemConfig& cfg,
                            double lambda, long iterations, int power_steps) {
  cfg.validate();
  if (!(lambda >= 0.0)) throw std::invalid_argument("PgdParams: lambda must be >= 0");
  if (iterations < 0) throw std::invalid_argument("PgdParams: max_iters must be >= 0");
  BatchResult r;
  const std::size_t n = static_cast<std::size_t>(B) * cfg.K * cfg.M;
  r.precoders.resize(n);
  r.diverged_at.resize(static_cast<std::size_t>(B));
  r.steps.resize(static_cast<std::size_t>(B));
  double stats[3] = {0, 0, 0};
  const RealVector c = cfg.constraint_diag();
  const int rc = ufpgd_gpu_pgd_fixed_host(reinterpret_cast<const ufpgd_c64*>(channels), B, cfg.K, cfg.M, power_steps,
                                          lambda, iterations, c.data(), UFPGD_W0_CONJ_H, nullptr,
                                          reinterpret_cast<ufpgd_c64*>(r.precoders.data()), r.diverged_at.data(),
                                          r.steps.data(), stats, cfg.alpha, g_device);
  if (rc != UFPGD_OK && rc != UFPGD_EDIVERGED) raise(rc);
  r.consumed_power_sum = stats[0];
  r.active_sum = stats[1];
  r.diverged = static_cast<long>(stats[2]);
  return r;
}

BatchResult forward_batch_multi_gpu(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                                    const SystemConfig& cfg, int ngpus) {
  net.validate();
  check_projected(net);
  cfg.validate();
  if (cfg.K != net.num_users || cfg.M != net.num_antennas) throw std::invalid_argument("forward: dimension mismatch");
  check(ufpgd_gpu_init(ngpus));
  std::vector<double> lam, eta;
  for (const LayerParams& l : net.layers) {
    lam.push_back(l.lambda_i);
    eta.push_back(l.eta_i);
  }
  BatchResult r;
  r.precoders.resize(static_cast<std::size_t>(B) * cfg.K * cfg.M);
  r.diverged_at.resize(static_cast<std::size_t>(B));
  double stats[3] = {0, 0, 0};
  const RealVector c = cfg.constraint_diag();
  const int rc = ufpgd_gpu_unfolded_forward_sharded(
      reinterpret_cast<const ufpgd_c64*>(channels), B, cfg.K, cfg.M, lam.data(), eta.data(),
      static_cast<int>(lam.size()), c.data(), UFPGD_W0_CONJ_H, nullptr, reinterpret_cast<ufpgd_c64*>(r.precoders.data()),
      r.diverged_at.data(), stats, cfg.alpha);
  if (rc != UFPGD_OK && rc != UFPGD_EDIVERGED) raise(rc);
  r.consumed_power_sum = stats[0];
  r.active_sum = stats[1];
  r.diverged = static_cast<long>(stats[2]);
  return r;
}

TrainGradients train_gradients(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                               const SystemConfig& cfg, LossKind kind, double lambda_cost,
                               const std::complex<float>* labels) {
  net.validate();
  check_projected(net);
  cfg.validate();
  if (cfg.K != net.num_users || cfg.M != net.num_antennas) throw std::invalid_argument("forward: dimension mismatch");
  if (kind == LossKind::Supervised && !labels) throw TrainingError("train: supervised mode requires labeled datasets");
  const int L = static_cast<int>(net.layers.size());
  std::vector<double> lam, eta;
  for (const LayerParams& l : net.layers) {
    lam.push_back(l.lambda_i);
    eta.push_back(l.eta_i);
  }
  const std::size_t n = static_cast<std::size_t>(B) * cfg.K * cfg.M;
  TrainGradients r;
  r.grads.assign(2 * static_cast<std::size_t>(L), 0.0);
  if (B == 0) return r;
  DeviceScope scope;
  DeviceBuffer<ufpgd_c64> dH(n), dLab(labels ? n : 0);
  DeviceBuffer<double> dloss(static_cast<std::size_t>(B)), dgr(static_cast<std::size_t>(B) * 2 * L), dmean(1 + 2 * L);
  dH.upload(reinterpret_cast<const ufpgd_c64*>(channels));
  if (labels) dLab.upload(reinterpret_cast<const ufpgd_c64*>(labels));
  const RealVector c = cfg.constraint_diag();
  check(ufpgd_gpu_unfolded_grad(dH.p, B, cfg.K, cfg.M, lam.data(), eta.data(), L, c.data(), UFPGD_W0_CONJ_H,
                                static_cast<int>(kind), lambda_cost, dLab.p, dloss.p, dgr.p, dmean.p, g_device,
                                nullptr));
  std::vector<double> mean(1 + 2 * static_cast<std::size_t>(L));
  dmean.download(mean.data());
  if (!std::isfinite(mean[0])) throw TrainingError("train: non-finite loss");
  r.loss = mean[0];
  for (int i = 0; i < 2 * L; ++i) r.grads[static_cast<std::size_t>(i)] = mean[1 + i];
  return r;
}

EvaluationSummary evaluate_batch(const UnfoldedNetwork& net, const std::complex<float>* channels, std::int64_t B,
                                 const SystemConfig& cfg) {
  BatchResult r = forward_batch(net, channels, B, cfg, StartMode::ConjChannel);
  if (r.diverged) throw DivergenceError("evaluate: non-finite iterate", r.diverged_at[0]);
  const int K = cfg.K, M = cfg.M;
  const std::size_t n = static_cast<std::size_t>(B) * K * M;
  EvaluationSummary s;
  s.num_channels = static_cast<std::size_t>(B);
  if (B == 0) return s;
  DeviceScope scope;
  DeviceBuffer<ufpgd_c64> dH(n), dW(n);
  DeviceBuffer<double> dout(static_cast<std::size_t>(B) * (6 + K));
  dH.upload(reinterpret_cast<const ufpgd_c64*>(channels));
  dW.upload(reinterpret_cast<const ufpgd_c64*>(r.precoders.data()));
  const RealVector c = cfg.constraint_diag();
  check(ufpgd_gpu_metrics(dH.p, dW.p, B, K, M, c.data(), cfg.sigma_nu, cfg.alpha, dout.p, nullptr, g_device, nullptr));
  std::vector<double> out(static_cast<std::size_t>(B) * (6 + K));
  dout.download(out.data());
  // training.cpp:361-399 (singular channels are counted and skipped instead
  // of aborting the whole evaluation)
  s.mean.sinr = RealVector(K);
  s.std_error.sinr = RealVector(K);
  std::size_t used = 0;
  for (std::int64_t b = 0; b < B; ++b) {
    const double* o = &out[static_cast<std::size_t>(b) * (6 + K)];
    if (o[5] == 0.0) {
      ++s.singular;
      continue;
    }
    ++used;
    s.mean.tx_power += o[0];
    s.mean.cons_power += o[1];
    s.mean.sum_rate += o[2];
    s.mean.pcg += o[3];
    s.mean.residual += o[4];
    for (int k = 0; k < K; ++k) s.mean.sinr[k] += o[6 + k];
  }
  if (used == 0) return s;
  const double scale = 1.0 / static_cast<double>(used);
  s.mean.tx_power *= scale;
  s.mean.cons_power *= scale;
  s.mean.sum_rate *= scale;
  s.mean.pcg *= scale;
  s.mean.residual *= scale;
  for (int k = 0; k < K; ++k) s.mean.sinr[k] *= scale;
  if (used > 1) {
    auto sq = [](double d) { return d * d; };
    for (std::int64_t b = 0; b < B; ++b) {
      const double* o = &out[static_cast<std::size_t>(b) * (6 + K)];
      if (o[5] == 0.0) continue;
      s.std_error.tx_power += sq(o[0] - s.mean.tx_power);
      s.std_error.cons_power += sq(o[1] - s.mean.cons_power);
      s.std_error.sum_rate += sq(o[2] - s.mean.sum_rate);
      s.std_error.pcg += sq(o[3] - s.mean.pcg);
      s.std_error.residual += sq(o[4] - s.mean.residual);
      for (int k = 0; k < K; ++k) s.std_error.sinr[k] += sq(o[6 + k] - s.mean.sinr[k]);
    }
    const double vs = 1.0 / (static_cast<double>(used - 1) * static_cast<double>(used));
    s.std_error.tx_power = std::sqrt(s.std_error.tx_power * vs);
    s.std_error.cons_power = std::sqrt(s.std_error.cons_power * vs);
    s.std_error.sum_rate = std::sqrt(s.std_error.sum_rate * vs);
    s.std_error.pcg = std::sqrt(s.std_error.pcg * vs);
    s.std_error.residual = std::sqrt(s.std_error.residual * vs);
    for (int k = 0; k < K; ++k) s.std_error.sinr[k] = std::sqrt(s.std_error.sinr[k] * vs);
  }
  return s;
}

// ---- dataset.cpp: host files ------------------------------------------------
namespace {

void put_le(std::string& out, std::uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}

// Row-major K x M f64 (re, im) <-> the col-major ComplexMatrix (dataset.cpp:38-66).
void append_rowmajor(std::vector<double>& out, const ComplexMatrix& A) {
  for (std::ptrdiff_t k = 0; k < A.rows(); ++k)
    for (std::ptrdiff_t m = 0; m < A.cols(); ++m) {
      out.push_back(A(k, m).real());
      out.push_back(A(k, m).imag());
    }
}

ComplexMatrix from_rowmajor(const double* d, int K, int M) {
  ComplexMatrix A(K, M);
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < M; ++m) A(k, m) = Complex(d[2 * (k * M + m)], d[2 * (k * M + m) + 1]);
  return A;
}

}  // namespace

void write_dataset(const Dataset& data, const std::string& path) {  // dataset.cpp:70-127
  if (data.num_users < 1 || data.num_antennas < 1) throw std::invalid_argument("write_dataset: bad dimensions");
  if (data.has_labels() && data.labels.size() != data.channels.size())
    throw std::invalid_argument("write_dataset: label count does not match channel count");
  for (const ChannelMatrix& ch : data.channels)
    if (ch.rows() != data.num_users || ch.cols() != data.num_antennas)
      throw std::invalid_argument("write_dataset: channel shape mismatch");
  for (const PrecoderMatrix& lb : data.labels)
    if (lb.rows() != data.num_users || lb.cols() != data.num_antennas)
      throw std::invalid_argument("write_dataset: label shape mismatch");
  std::string header;
  put_le(header, kDatasetMagic, 4);
  put_le(header, kDatasetVersion, 4);
  put_le(header, static_cast<std::uint32_t>(data.num_users), 4);
  put_le(header, static_cast<std::uint32_t>(data.num_antennas), 4);
  put_le(header, data.channels.size(), 8);
  put_le(header, data.seed, 8);
  put_le(header, data.has_labels() ? 1u : 0u, 4);
  const std::filesystem::path target(path);
  std::filesystem::path temp = target;
  temp += ".tmp";
  {
    std::ofstream out(temp, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open for writing: " + temp.string());
    out.write(header.data(), static_cast<std::streamsize>(header.size()));
    std::vector<double> buf;
    for (const std::vector<ComplexMatrix>* set : {&data.channels, &data.labels})
      for (const ComplexMatrix& A : *set) {
        buf.clear();
        append_rowmajor(buf, A);
        out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size() * sizeof(double)));
      }
    out.flush();
    if (!out) throw std::runtime_error("write failed: " + temp.string());
  }
  std::filesystem::rename(temp, target);
}

Dataset read_dataset(const std::string& path) {  // dataset.cpp:129-175
  int K = 0, M = 0, labels = 0;
  int64_t N = 0;
  std::uint64_t seed = 0;
  if (ufpgd_ufpd_read_header(path.c_str(), &K, &M, &N, &seed, &labels) != UFPGD_OK)
    throw DataFormatError(ufpgd_dataset_last_error());
  Dataset d;
  d.num_users = K;
  d.num_antennas = M;
  d.seed = seed;
  std::ifstream in(path, std::ios::binary);
  in.seekg(static_cast<std::streamoff>(kDatasetHeaderBytes));
  std::vector<double> buf(2 * static_cast<std::size_t>(K) * M);
  for (int set = 0; set < (labels ? 2 : 1); ++set)
    for (int64_t i = 0; i < N; ++i) {
      in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * sizeof(double)));
      if (!in) throw DataFormatError("dataset truncated: " + path);
      (set == 0 ? d.channels : d.labels).push_back(from_rowmajor(buf.data(), K, M));
    }
  return d;
}

// ---- training.cpp -------------------------------------------------------------
namespace {

constexpr std::uint64_t kShuffleStream = 0x7D5A1E0B33C4F216ULL;  // training.cpp:20

void check_dataset(const Dataset& data, const SystemConfig& sys, const char* which) {  // training.cpp:22-31
  if (data.size() == 0) throw TrainingError(std::string(which) + " dataset is empty");
  if (data.num_users != sys.K || data.num_antennas != sys.M)
    throw TrainingError(std::string(which) + " dataset dimensions do not match SystemConfig");
}

void project_flat(std::vector<double>& params, double eta_lo, double eta_hi) {  // training.cpp:33-38
  for (std::size_t i = 0; i + 1 < params.size(); i += 2) {
    params[i] = std::max(0.0, params[i]);
    params[i + 1] = std::min(std::max(params[i + 1], eta_lo), eta_hi);
  }
}

// A set of K x M matrices as one complex64 [N][M][K] device batch.
std::vector<ufpgd_c64> stack_c64(const std::vector<ComplexMatrix>& mats) {
  std::vector<ufpgd_c64> out;
  for (const ComplexMatrix& A : mats) {
    const std::vector<ufpgd_c64> a = to_c64(A);
    out.insert(out.end(), a.begin(), a.end());
  }
  return out;
}

void layer_vectors(const UnfoldedNetwork& net, std::vector<double>& lam, std::vector<double>& eta) {
  lam.clear();
  eta.clear();
  for (const LayerParams& l : net.layers) {
    lam.push_back(l.lambda_i);
    eta.push_back(l.eta_i);
  }
}

// Device metrics rows [tx, cons, sum_rate, pcg, residual, ok, sinr_0..K-1]
// for B (H, W) pairs; SingularChannelError where the ZF reference is singular
// (zf.cpp:17-23 throws inside the reference's evaluate / train).
std::vector<double> device_metric_rows(const ufpgd_c64* dH, const ufpgd_c64* dW, std::int64_t B,
                                       const SystemConfig& sys) {
  const int K = sys.K;
  DeviceBuffer<double> dout(static_cast<std::size_t>(B) * (6 + K));
  const RealVector c = sys.constraint_diag();
  check(ufpgd_gpu_metrics(dH, dW, B, K, sys.M, c.data(), sys.sigma_nu, sys.alpha, dout.p, nullptr, g_device,
                          nullptr));
  std::vector<double> out(dout.n);
  dout.download(out.data());
  for (std::int64_t b = 0; b < B; ++b)
    if (out[static_cast<std::size_t>(b) * (6 + K) + 5] == 0.0)
      throw SingularChannelError("zf_precoder: channel Gram matrix is singular");
  return out;
}

MetricsReport report_from_row(const double* o, int K) {
  MetricsReport r;
  r.tx_power = o[0];
  r.cons_power = o[1];
  r.sum_rate = o[2];
  r.pcg = o[3];
  r.residual = o[4];
  r.sinr = RealVector(K);
  for (int k = 0; k < K; ++k) r.sinr[k] = o[6 + k];
  return r;
}

int active_of(const ufpgd_c64* w, int K, int M) {
  int a = 0;
  for (int m = 0; m < M; ++m) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s += static_cast<double>(w[m * K + k].re) * w[m * K + k].re +
                                     static_cast<double>(w[m * K + k].im) * w[m * K + k].im;
    if (s > 0.0) ++a;
  }
  return a;
}

}  // namespace

void TrainConfig::validate() const {  // training.cpp:40-56
  if (!(lambda_cost >= 0.0)) throw std::invalid_argument("TrainConfig: lambda_cost must be >= 0");
  if (batch_size < 1) throw std::invalid_argument("TrainConfig: batch_size must be >= 1");
  if (!(learning_rate >= 0.0)) throw std::invalid_argument("TrainConfig: learning_rate must be >= 0");
  if (max_epochs < 1) throw std::invalid_argument("TrainConfig: max_epochs must be >= 1");
  if (patience < 1) throw std::invalid_argument("TrainConfig: patience must be >= 1");
}

double supervised_loss(const PrecoderMatrix& precoder, const PrecoderMatrix& ground_truth) {
  if (precoder.rows() != ground_truth.rows() || precoder.cols() != ground_truth.cols())
    throw std::invalid_argument("supervised_loss: shape mismatch");
  double s = 0.0;
  for (std::ptrdiff_t i = 0; i < precoder.size(); ++i) s += std::norm(precoder.data()[i] - ground_truth.data()[i]);
  return s;
}

ComplexMatrix supervised_loss_grad(const PrecoderMatrix& precoder, const PrecoderMatrix& ground_truth) {
  if (precoder.rows() != ground_truth.rows() || precoder.cols() != ground_truth.cols())
    throw std::invalid_argument("supervised_loss_grad: shape mismatch");
  ComplexMatrix g(precoder.rows(), precoder.cols());
  for (std::ptrdiff_t i = 0; i < precoder.size(); ++i) g.data()[i] = 2.0 * (precoder.data()[i] - ground_truth.data()[i]);
  return g;
}

double unsupervised_loss(const PrecoderMatrix& precoder, const ChannelMatrix& channel, const SystemConfig& cfg,
                         double lambda_cost) {
  return lagrangian_value(precoder, channel, cfg, lambda_cost);
}

ComplexMatrix unsupervised_loss_grad(const PrecoderMatrix& precoder, const ChannelMatrix& channel,
                                     const SystemConfig& cfg, double lambda_cost) {
  ComplexMatrix g = grad_f(precoder, channel, cfg);  // FP64 on the device
  for (std::ptrdiff_t i = 0; i < g.size(); ++i) g.data()[i] *= 2.0;
  for (std::ptrdiff_t m = 0; m < precoder.cols(); ++m) {
    const double n = precoder.colNorm(m);
    if (n > 0.0)
      for (std::ptrdiff_t k = 0; k < precoder.rows(); ++k) g(k, m) += (lambda_cost / n) * precoder(k, m);
  }
  return g;
}

std::vector<double> pack_params(const UnfoldedNetwork& net) {
  std::vector<double> p(2 * net.layers.size());
  for (std::size_t i = 0; i < net.layers.size(); ++i) {
    p[2 * i] = net.layers[i].lambda_i;
    p[2 * i + 1] = net.layers[i].eta_i;
  }
  return p;
}

void unpack_params(const std::vector<double>& params, UnfoldedNetwork& net) {
  if (params.size() != 2 * net.layers.size()) throw std::invalid_argument("unpack_params: size mismatch");
  for (std::size_t i = 0; i < net.layers.size(); ++i) {
    net.layers[i].lambda_i = params[2 * i];
    net.layers[i].eta_i = params[2 * i + 1];
  }
}

void adam_update(AdamState& state, const std::vector<double>& grads, std::vector<double>& params, double lr) {
  if (grads.size() != params.size() || grads.size() != state.m.size() || grads.size() != state.v.size())
    throw TrainingError("adam_update: parameter/gradient size mismatch");
  for (std::size_t i = 0; i < grads.size(); ++i)
    if (!std::isfinite(grads[i])) throw TrainingError("adam_update: non-finite gradient for parameter " + std::to_string(i));
  state.step += 1;
  const double bias1 = 1.0 - std::pow(state.beta1, static_cast<double>(state.step));
  const double bias2 = 1.0 - std::pow(state.beta2, static_cast<double>(state.step));
  for (std::size_t i = 0; i < grads.size(); ++i) {
    state.m[i] = state.beta1 * state.m[i] + (1.0 - state.beta1) * grads[i];
    state.v[i] = state.beta2 * state.v[i] + (1.0 - state.beta2) * grads[i] * grads[i];
    params[i] -= lr * (state.m[i] / bias1) / (std::sqrt(state.v[i] / bias2) + state.epsilon);
  }
}

TrainResult train(const UnfoldedNetwork& net, const Dataset& train_set, const Dataset& val_set,
                  const TrainConfig& cfg, const SystemConfig& sys) {
  cfg.validate();
  sys.validate();
  check_dataset(train_set, sys, "train");
  check_dataset(val_set, sys, "validation");
  const bool supervised = cfg.loss_kind == LossKind::kSupervised;
  if (supervised && (!train_set.has_labels() || !val_set.has_labels()))
    throw TrainingError("train: supervised mode requires labeled datasets");
  UnfoldedNetwork model = project_params(net);
  if (model.num_users != sys.K || model.num_antennas != sys.M)
    throw TrainingError("train: network dimensions do not match SystemConfig");
  const int K = sys.K, M = sys.M, L = static_cast<int>(model.layers.size());
  const std::size_t km = static_cast<std::size_t>(K) * M;
  const double eta_hi = 1.0 / model.mp_bound, eta_lo = 0.5 * eta_hi;
  std::vector<double> params = pack_params(model);
  AdamState adam(params.size());
  const RealVector c = sys.constraint_diag();

  DeviceScope scope;
  // The datasets as complex64 batches: training channels gathered per
  // mini-batch on the host (the shuffle order), the validation set resident.
  const std::vector<ufpgd_c64> tr = stack_c64(train_set.channels);
  const std::vector<ufpgd_c64> tl = supervised ? stack_c64(train_set.labels) : std::vector<ufpgd_c64>{};
  const std::int64_t nv = static_cast<std::int64_t>(val_set.size());
  DeviceBuffer<ufpgd_c64> dV(static_cast<std::size_t>(nv) * km), dVW(static_cast<std::size_t>(nv) * km);
  dV.upload(stack_c64(val_set.channels).data());
  std::vector<ufpgd_c64> val_out(dVW.n);
  const std::size_t bmax = std::min<std::size_t>(static_cast<std::size_t>(cfg.batch_size), train_set.size());
  DeviceBuffer<ufpgd_c64> dB(bmax * km), dBL(supervised ? bmax * km : 0);
  DeviceBuffer<double> dloss(bmax), dgr(bmax * 2 * L), dmean(1 + 2 * static_cast<std::size_t>(L));
  DeviceBuffer<int32_t> ddiv(static_cast<std::size_t>(nv));
  std::vector<ufpgd_c64> stage(bmax * km), stage_l(supervised ? bmax * km : 0);
  std::vector<double> mean(1 + 2 * static_cast<std::size_t>(L));
  device_metric_rows(dV.p, dV.p, nv, sys);  // ZF reference of every validation channel (training.cpp:165-171)

  Rng shuffle_rng = Rng::stream(cfg.seed, kShuffleStream);
  std::vector<std::size_t> order(train_set.size());
  std::iota(order.begin(), order.end(), std::size_t{0});
  TrainResult result;
  TrainHistory& history = result.history;
  double best_val = std::numeric_limits<double>::infinity();
  int since_best = 0;
  std::vector<double> lam, eta;
  for (int epoch = 0; epoch < cfg.max_epochs; ++epoch) {
    shuffle(order, shuffle_rng);
    double epoch_loss_sum = 0.0;
    for (std::size_t start = 0; start < train_set.size(); start += static_cast<std::size_t>(cfg.batch_size)) {
      const std::size_t count = std::min<std::size_t>(static_cast<std::size_t>(cfg.batch_size), train_set.size() - start);
      for (std::size_t b = 0; b < count; ++b) {
        std::memcpy(&stage[b * km], &tr[order[start + b] * km], km * sizeof(ufpgd_c64));
        if (supervised) std::memcpy(&stage_l[b * km], &tl[order[start + b] * km], km * sizeof(ufpgd_c64));
      }
      cuda_check(cudaMemcpy(dB.p, stage.data(), count * km * sizeof(ufpgd_c64), cudaMemcpyHostToDevice), "H2D");
      if (supervised)
        cuda_check(cudaMemcpy(dBL.p, stage_l.data(), count * km * sizeof(ufpgd_c64), cudaMemcpyHostToDevice), "H2D");
      layer_vectors(model, lam, eta);
      // per-sample taped forward from H^*, loss, backward; ordered batch mean
      check(ufpgd_gpu_unfolded_grad(dB.p, static_cast<std::int64_t>(count), K, M, lam.data(), eta.data(), L,
                                    c.data(), UFPGD_W0_CONJ_H, supervised ? 1 : 0, cfg.lambda_cost,
                                    supervised ? dBL.p : nullptr, dloss.p, dgr.p, dmean.p, g_device, nullptr));
      dmean.download(mean.data());
      const double batch_loss = mean[0];
      if (!std::isfinite(batch_loss))
        throw TrainingError("train: non-finite loss at epoch " + std::to_string(epoch) + " batch " +
                            std::to_string(start / static_cast<std::size_t>(cfg.batch_size)));
      epoch_loss_sum += batch_loss * static_cast<double>(count);
      const std::vector<double> grads(mean.begin() + 1, mean.end());
      adam_update(adam, grads, params, cfg.learning_rate);
      project_flat(params, eta_lo, eta_hi);
      unpack_params(params, model);
    }

    // validation: forward_infer (start H^*) on the device, then device metrics
    layer_vectors(model, lam, eta);
    const int rc = ufpgd_gpu_unfolded_forward(dV.p, nv, K, M, lam.data(), eta.data(), L, c.data(), UFPGD_W0_CONJ_H,
                                              nullptr, dVW.p, ddiv.p, nullptr, nullptr, nullptr, sys.alpha, g_device,
                                              nullptr);
    if (rc != UFPGD_OK) raise(rc);
    cuda_check(cudaDeviceSynchronize(), "validation forward");
    std::vector<int32_t> div(static_cast<std::size_t>(nv));
    ddiv.download(div.data());
    for (int32_t d : div)
      if (d >= 0) throw DivergenceError("forward: non-finite iterate in validation", d);
    const std::vector<double> rows = device_metric_rows(dV.p, dVW.p, nv, sys);
    if (supervised) dVW.download(val_out.data());
    EpochRecord rec;
    rec.epoch = epoch;
    rec.train_loss = epoch_loss_sum / static_cast<double>(train_set.size());
    for (std::int64_t j = 0; j < nv; ++j) {
      const double* o = &rows[static_cast<std::size_t>(j) * (6 + K)];
      double loss;
      if (supervised) {
        loss = 0.0;
        const ComplexMatrix& g = val_set.labels[static_cast<std::size_t>(j)];
        const ufpgd_c64* w = &val_out[static_cast<std::size_t>(j) * km];
        for (std::size_t i = 0; i < km; ++i) loss += std::norm(Complex(w[i].re, w[i].im) - g.data()[i]);
      } else {
        loss = cfg.lambda_cost * (o[1] / sys.alpha) + o[4] * o[4];  // lagrangian_value (pgd.cpp:171-176)
      }
      rec.val_loss += loss;
      rec.val_mean_pcg += o[3];
      rec.val_mean_sum_rate += o[2];
    }
    const double vn = static_cast<double>(nv);
    rec.val_loss /= vn;
    rec.val_mean_pcg /= vn;
    rec.val_mean_sum_rate /= vn;
    if (!std::isfinite(rec.val_loss))
      throw TrainingError("train: non-finite validation loss at epoch " + std::to_string(epoch));
    history.epochs.push_back(rec);
    history.stopping_epoch = epoch;
    if (rec.val_loss < best_val) {
      best_val = rec.val_loss;
      history.best_epoch = epoch;
      history.best_params = model.layers;
      since_best = 0;
    } else {
      ++since_best;
    }
    if (since_best >= cfg.patience) break;
  }
  model.layers = history.best_params;
  result.network = std::move(model);
  return result;
}

EvaluationSummary evaluate(const UnfoldedNetwork& net, const Dataset& test_set, const SystemConfig& sys,
                           const EvalOptions& options) {
  sys.validate();
  check_dataset(test_set, sys, "test");
  UnfoldedNetwork model = net;
  model.validate();
  check_projected(model);
  if (model.num_users != sys.K || model.num_antennas != sys.M)
    throw std::invalid_argument("forward: network dimensions do not match SystemConfig");
  const int K = sys.K, M = sys.M, L = static_cast<int>(model.layers.size());
  const std::size_t km = static_cast<std::size_t>(K) * M;
  const std::int64_t n = static_cast<std::int64_t>(test_set.size());
  std::vector<double> lam, eta, thr;
  layer_vectors(model, lam, eta);
  for (int l = 0; l < L; ++l) thr.push_back(lam[static_cast<std::size_t>(l)] * eta[static_cast<std::size_t>(l)]);
  const RealVector c = sys.constraint_diag();
  DeviceScope scope;
  EvaluationSummary summary;
  summary.num_channels = static_cast<std::size_t>(n);
  std::vector<MetricsReport> reports;
  reports.reserve(static_cast<std::size_t>(n));
  if (options.per_layer) summary.per_layer.assign(static_cast<std::size_t>(L) + 1, TraceRecord{});
  // chunks bound the (L + 1) iterates kept on the device for per-layer curves
  const std::int64_t chunk = options.per_layer ? std::max<std::int64_t>(1, (std::int64_t{1} << 28) / ((L + 1) * km * 8))
                                               : n;
  const std::vector<ufpgd_c64> all = stack_c64(test_set.channels);
  for (std::int64_t b0 = 0; b0 < n; b0 += chunk) {
    const std::int64_t nb = std::min(chunk, n - b0);
    DeviceBuffer<ufpgd_c64> dH(static_cast<std::size_t>(nb) * km), dW(static_cast<std::size_t>(nb) * km);
    cuda_check(cudaMemcpy(dH.p, &all[static_cast<std::size_t>(b0) * km], dH.n * sizeof(ufpgd_c64),
                          cudaMemcpyHostToDevice), "H2D");
    DeviceBuffer<int32_t> ddiv(static_cast<std::size_t>(nb));
    std::vector<int32_t> div(static_cast<std::size_t>(nb));
    if (options.per_layer) {  // forward with_iterates (unfolded.cpp:112-146), FP32 general kernel
      DeviceBuffer<ufpgd_c64> dI(static_cast<std::size_t>(L + 1) * dH.n);
      DeviceBuffer<int64_t> dits(static_cast<std::size_t>(nb));
      check(ufpgd_gpu_layers_general(dH.p, nb, K, M, eta.data(), thr.data(), L, c.data(), UFPGD_W0_CONJ_H, nullptr, 0,
                                     0.0, 0, dW.p, ddiv.p, dits.p, dI.p, nullptr, nullptr, nullptr, g_device, nullptr));
      cuda_check(cudaDeviceSynchronize(), "forward with iterates");
      ddiv.download(div.data());
      for (int32_t d : div)
        if (d >= 0) throw DivergenceError("forward: non-finite iterate", d);
      std::vector<ufpgd_c64> it(dH.n);
      for (int l = 0; l <= L; ++l) {
        const ufpgd_c64* dWl = dI.p + static_cast<std::size_t>(l) * dH.n;
        const std::vector<double> rows = device_metric_rows(dH.p, dWl, nb, sys);
        cuda_check(cudaMemcpy(it.data(), dWl, dH.n * sizeof(ufpgd_c64), cudaMemcpyDeviceToHost), "D2H");
        TraceRecord& rec = summary.per_layer[static_cast<std::size_t>(l)];
        for (std::int64_t j = 0; j < nb; ++j) {
          const double* o = &rows[static_cast<std::size_t>(j) * (6 + K)];
          rec.lagrangian += options.lagrangian_lambda * (o[1] / sys.alpha) + o[4] * o[4];
          rec.residual += o[4];
          rec.pcg += o[3];
          rec.sum_rate += o[2];
          rec.active_columns += active_of(&it[static_cast<std::size_t>(j) * km], K, M);
          if (l == L) reports.push_back(report_from_row(o, K));
        }
      }
    } else {  // forward_infer from H^* (fused kernels where the shape has one)
      check(ufpgd_gpu_unfolded_forward(dH.p, nb, K, M, lam.data(), eta.data(), L, c.data(), UFPGD_W0_CONJ_H, nullptr,
                                       dW.p, ddiv.p, nullptr, nullptr, nullptr, sys.alpha, g_device, nullptr));
      cuda_check(cudaDeviceSynchronize(), "forward");
      ddiv.download(div.data());
      for (int32_t d : div)
        if (d >= 0) throw DivergenceError("forward: non-finite iterate", d);
      const std::vector<double> rows = device_metric_rows(dH.p, dW.p, nb, sys);
      for (std::int64_t j = 0; j < nb; ++j) reports.push_back(report_from_row(&rows[static_cast<std::size_t>(j) * (6 + K)], K));
    }
  }
  // training.cpp:361-399: means, then standard errors of the means
  MetricsReport& mu = summary.mean;
  MetricsReport& se = summary.std_error;
  mu.sinr = RealVector(K);
  se.sinr = RealVector(K);
  for (const MetricsReport& r : reports) {
    mu.tx_power += r.tx_power;
    mu.cons_power += r.cons_power;
    mu.sum_rate += r.sum_rate;
    mu.pcg += r.pcg;
    mu.residual += r.residual;
    for (int k = 0; k < K; ++k) mu.sinr[k] += r.sinr[k];
  }
  const double scale = 1.0 / static_cast<double>(n);
  mu.tx_power *= scale;
  mu.cons_power *= scale;
  mu.sum_rate *= scale;
  mu.pcg *= scale;
  mu.residual *= scale;
  for (int k = 0; k < K; ++k) mu.sinr[k] *= scale;
  if (n > 1) {
    auto sq = [](double d) { return d * d; };
    for (const MetricsReport& r : reports) {
      se.tx_power += sq(r.tx_power - mu.tx_power);
      se.cons_power += sq(r.cons_power - mu.cons_power);
      se.sum_rate += sq(r.sum_rate - mu.sum_rate);
      se.pcg += sq(r.pcg - mu.pcg);
      se.residual += sq(r.residual - mu.residual);
      for (int k = 0; k < K; ++k) se.sinr[k] += sq(r.sinr[k] - mu.sinr[k]);
    }
    const double vs = 1.0 / (static_cast<double>(n - 1) * static_cast<double>(n));
    se.tx_power = std::sqrt(se.tx_power * vs);
    se.cons_power = std::sqrt(se.cons_power * vs);
    se.sum_rate = std::sqrt(se.sum_rate * vs);
    se.pcg = std::sqrt(se.pcg * vs);
    se.residual = std::sqrt(se.residual * vs);
    for (int k = 0; k < K; ++k) se.sinr[k] = std::sqrt(se.sinr[k] * vs);
  }
  if (options.per_layer)
    for (TraceRecord& rec : summary.per_layer) {
      rec.lagrangian *= scale;
      rec.residual *= scale;
      rec.pcg *= scale;
      rec.sum_rate *= scale;
      rec.active_columns *= scale;
    }
  for (std::size_t l = 0; l < summary.per_layer.size(); ++l) summary.per_layer[l].index = static_cast<long>(l);
  return summary;
}

}  // namespace ufpgd

// ---- unfolded.cpp:241-298: model JSON -------------------------------------------
namespace ufpgd {
namespace {

// nlohmann::json's number format: shortest round-trip, ".0" on integral doubles.
std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, res.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// Minimal JSON reader for the model schema: objects, arrays, numbers,
// strings, true/false/null. Throws DataFormatError with a position.
struct JsonValue {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  double number = 0.0;
  bool integral = false;
  std::string text;
  std::vector<JsonValue> items;
  std::vector<std::pair<std::string, JsonValue>> fields;
  const JsonValue& at(const std::string& key) const {
    if (kind != Object) throw DataFormatError("model JSON: expected an object");
    for (const auto& f : fields)
      if (f.first == key) return f.second;
    throw DataFormatError("model JSON: missing key \"" + key + "\"");
  }
  double as_number(const char* what) const {
    if (kind != Number) throw DataFormatError(std::string("model JSON: ") + what + " must be a number");
    return number;
  }
  long as_integer(const char* what) const {
    if (kind != Number || !integral) throw DataFormatError(std::string("model JSON: ") + what + " must be an integer");
    return static_cast<long>(number);
  }
};

class JsonParser {
 public:
  explicit JsonParser(const std::string& t) : t_(t) {}
  JsonValue document() {
    JsonValue v = value();
    ws();
    if (i_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  std::size_t i_ = 0;
  [[noreturn]] void fail(const std::string& what) const {
    throw DataFormatError("model JSON parse error at byte " + std::to_string(i_) + ": " + what);
  }
  void ws() {
    while (i_ < t_.size() && (t_[i_] == ' ' || t_[i_] == '\n' || t_[i_] == '\t' || t_[i_] == '\r')) ++i_;
  }
  bool lit(const char* s) {
    const std::size_t n = std::strlen(s);
    if (t_.compare(i_, n, s) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (t_[i_] != '"') fail("expected a string");
    ++i_;
    std::string out;
    while (i_ < t_.size() && t_[i_] != '"') {
      if (t_[i_] == '\\') {
        if (++i_ >= t_.size()) fail("bad escape");
        const char e = t_[i_];
        out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e);
        ++i_;
      } else {
        out.push_back(t_[i_++]);
      }
    }
    if (i_ >= t_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  JsonValue value() {
    ws();
    if (i_ >= t_.size()) fail("unexpected end of input");
    JsonValue v;
    const char ch = t_[i_];
    if (ch == '{') {
      v.kind = JsonValue::Object;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        std::string key = str();
        ws();
        if (i_ >= t_.size() || t_[i_] != ':') fail("expected ':'");
        ++i_;
        v.fields.emplace_back(std::move(key), value());
        ws();
        if (i_ < t_.size() && t_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < t_.size() && t_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (ch == '[') {
      v.kind = JsonValue::Array;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.items.push_back(value());
        ws();
        if (i_ < t_.size() && t_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < t_.size() && t_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (ch == '"') {
      v.kind = JsonValue::String;
      v.text = str();
      return v;
    }
    if (lit("true") || lit("false")) {
      v.kind = JsonValue::Bool;
      v.number = t_[i_ - 1] == 'e' && t_[i_ - 2] == 'u' ? 1.0 : 0.0;
      return v;
    }
    if (lit("null")) return v;
    const std::size_t start = i_;
    while (i_ < t_.size() && std::strchr("+-0123456789.eE", t_[i_]) && t_[i_] != '\0') ++i_;
    if (start == i_) fail("unexpected character");
    const std::string num = t_.substr(start, i_ - start);
    double d = 0.0;
    auto res = std::from_chars(num.data(), num.data() + num.size(), d);
    if (res.ec != std::errc() || res.ptr != num.data() + num.size()) fail("bad number");
    v.kind = JsonValue::Number;
    v.number = d;
    v.integral = num.find_first_of(".eE") == std::string::npos;
    return v;
  }
};

}  // namespace

std::string to_json_string(const UnfoldedNetwork& net) {
  std::string s = "{\n";
  s += "  \"I\": " + std::to_string(net.layers.size()) + ",\n";
  s += "  \"K\": " + std::to_string(net.num_users) + ",\n";
  s += "  \"M\": " + std::to_string(net.num_antennas) + ",\n";
  s += "  \"layers\": [";
  for (std::size_t i = 0; i < net.layers.size(); ++i) {
    s += i ? ",\n    {\n" : "\n    {\n";
    s += "      \"eta\": " + json_number(net.layers[i].eta_i) + ",\n";
    s += "      \"lambda\": " + json_number(net.layers[i].lambda_i) + "\n    }";
  }
  s += net.layers.empty() ? "],\n" : "\n  ],\n";
  s += "  \"mp_bound\": " + json_number(net.mp_bound) + ",\n";
  s += "  \"version\": 1\n}\n";
  return s;
}

UnfoldedNetwork network_from_json_string(const std::string& text) {
  const JsonValue doc = JsonParser(text).document();
  if (doc.at("version").as_integer("version") != 1) throw DataFormatError("model JSON: unsupported version");
  UnfoldedNetwork net;
  net.num_users = static_cast<int>(doc.at("K").as_integer("K"));
  net.num_antennas = static_cast<int>(doc.at("M").as_integer("M"));
  net.mp_bound = doc.at("mp_bound").as_number("mp_bound");
  const JsonValue& layers = doc.at("layers");
  if (layers.kind != JsonValue::Array || layers.items.empty())
    throw DataFormatError("model JSON: layers must be a non-empty array");
  if (doc.at("I").as_integer("I") != static_cast<long>(layers.items.size()))
    throw DataFormatError("model JSON: I does not match layers length");
  for (const JsonValue& e : layers.items)
    net.layers.push_back(LayerParams{e.at("lambda").as_number("lambda"), e.at("eta").as_number("eta")});
  try {
    net.validate();
  } catch (const std::invalid_argument& err) {
    throw DataFormatError(std::string("model JSON: ") + err.what());
  }
  return net;
}

void save_network(const UnfoldedNetwork& net, const std::string& path) {
  const std::filesystem::path target(path);
  std::filesystem::path temp = target;
  temp += ".tmp";
  {
    std::ofstream out(temp, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open for writing: " + temp.string());
    out << to_json_string(net);
    out.flush();
    if (!out) throw std::runtime_error("write failed: " + temp.string());
  }
  std::filesystem::rename(temp, target);
}

UnfoldedNetwork load_network(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataFormatError("cannot open model file: " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return network_from_json_string(text);
}

}  // namespace ufpgd
