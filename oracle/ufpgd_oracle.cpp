// ============================================================================
// ufpgd FP64 CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// This file is the parity checker for the B200 product path, not part of it.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// legs may load it. The product library (paper_2304_12745_b200/) never links,
// loads or calls anything under oracle/.
//
// It restates, in double precision, the reference's hot path
// (/root/reference/proj/core/src/*.cpp), function by function, in the same
// operation order where that matters. Eigen (the reference's only dependency,
// un-vendored and absent from this container) is replaced by explicit loops.
// The reference cannot be compiled here (no Eigen), so the
// oracle is pinned by the reference's own known-answer tests, restated in
// tests/test_oracle_*.py.
//
// Storage: a K x M complex matrix (Eigen col-major, column m = antenna m) is
// an interleaved double array of M*K complex values, element (k, m) at index
// m*K + k — i.e. row-major [M][K], the same layout the GPU uses.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;

enum Status : int {
  ORA_OK = 0,
  ORA_EINVAL = -1,
  ORA_EDIVERGED = -3,
  ORA_ECONVERGENCE = -4,
  ORA_ESINGULAR = -5,
};

// --- rng.cpp:9-40 ----------------------------------------------------------
// splitmix64 finalizer (rng.cpp:10-15).
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

struct Rng {
  std::mt19937_64 gen;
  explicit Rng(std::uint64_t seed) : gen(seed) {}
  // rng.cpp:19-21
  static Rng stream(std::uint64_t seed, std::uint64_t idx) { return Rng(mix64(seed ^ mix64(idx))); }
  std::uint64_t next_u64() { return gen(); }
  // rng.cpp:23-25
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  // rng.cpp:27-29
  double uniform_open() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
  // rng.cpp:35-40 (Box-Muller, E|z|^2 = 1; radius drawn first)
  cd complex_gaussian() {
    double radius = std::sqrt(-std::log(uniform_open()));
    double angle = 2.0 * std::numbers::pi * uniform();
    return {radius * std::cos(angle), radius * std::sin(angle)};
  }
};

// pgd.cpp:14
constexpr std::uint64_t kPowerIterationSeed = 0x1F2E3D4C5B6A7988ULL;

inline cd* as_c(double* p) { return reinterpret_cast<cd*>(p); }
inline const cd* as_c(const double* p) { return reinterpret_cast<const cd*>(p); }

// --- parallel.cpp:13-59 ----------------------------------------------------
int default_thread_count() {
  if (const char* env = std::getenv("UFPGD_THREADS")) {
    char* end = nullptr;
    long parsed = std::strtol(env, &end, 10);
    if (end != env && *end == '\0' && parsed >= 1) return static_cast<int>(parsed);
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

void parallel_for(std::size_t n, const std::function<void(std::size_t)>& body, int threads) {
  if (n == 0) return;
  if (threads <= 0) threads = default_thread_count();
  if (static_cast<std::size_t>(threads) > n) threads = static_cast<int>(n);
  if (threads == 1) {
    for (std::size_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  std::exception_ptr first_error;
  std::mutex error_mutex;
  auto worker = [&] {
    for (;;) {
      std::size_t i = next.fetch_add(1);
      if (i >= n) return;
      try {
        body(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(error_mutex);
        if (!first_error) first_error = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(static_cast<std::size_t>(threads));
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  if (first_error) std::rethrow_exception(first_error);
}

// --- pgd.cpp:51-99: the smooth gradient pieces and the prox -----------------
// scratch = W H^T (K x K): scratch(k, j) = sum_m W(k, m) H(j, m)  (pgd.cpp:71)
void w_times_ht(const cd* W, const cd* H, int K, int M, cd* X) {
  for (int i = 0; i < K * K; ++i) X[i] = 0.0;
  for (int m = 0; m < M; ++m) {
    const cd* w = W + static_cast<std::size_t>(m) * K;
    const cd* h = H + static_cast<std::size_t>(m) * K;
    for (int j = 0; j < K; ++j) {
      const cd hj = h[j];
      for (int k = 0; k < K; ++k) X[j * K + k] += w[k] * hj;  // X col-major (k, j)
    }
  }
}

// One gradient step image in the reference's order (pgd.cpp:227-230,
// unfolded.cpp:116-119): V = W; V -= eta * (X H^*); V += eta * offset,
// offset = diag(c) H^*. Returns false when V has a non-finite entry
// (pgd.cpp:231-235 / unfolded.cpp:120-125).
bool step_image(const cd* W, const cd* H, const double* c, int K, int M, double eta,
                std::vector<cd>& X, cd* V) {
  X.resize(static_cast<std::size_t>(K) * K);
  w_times_ht(W, H, K, M, X.data());
  bool finite = true;
  for (int m = 0; m < M; ++m) {
    const cd* h = H + static_cast<std::size_t>(m) * K;
    const cd* w = W + static_cast<std::size_t>(m) * K;
    cd* v = V + static_cast<std::size_t>(m) * K;
    for (int k = 0; k < K; ++k) {
      cd g = 0.0;
      for (int j = 0; j < K; ++j) g += X[j * K + k] * std::conj(h[j]);
      cd val = w[k];
      val -= eta * g;
      val += eta * (c[k] * std::conj(h[k]));
      v[k] = val;
      if (!std::isfinite(val.real()) || !std::isfinite(val.imag())) finite = false;
    }
  }
  return finite;
}

// Column 2-norm as Eigen computes it: sqrt(squaredNorm()).
inline double col_norm(const cd* col, int K) {
  double s = 0.0;
  for (int k = 0; k < K; ++k) s += std::norm(col[k]);
  return std::sqrt(s);
}

// Per-column block soft threshold (pgd.cpp:85-99; unfolded.cpp:135-143).
// Strict '>': a column whose norm equals t maps to zero (test_pgd.cpp:180-183).
// Optionally records the column norms / shrink factors (the LayerTape fields,
// unfolded.hpp:42-47) and the smallest relative distance |n - t| / t.
void prox_cols(const cd* V, int K, int M, double t, cd* out, double* norms, double* shrinks,
               double* tie_margin) {
  for (int m = 0; m < M; ++m) {
    const cd* v = V + static_cast<std::size_t>(m) * K;
    cd* o = out + static_cast<std::size_t>(m) * K;
    double n = col_norm(v, K);
    double shrink = n > t ? 1.0 - t / n : 0.0;
    for (int k = 0; k < K; ++k) o[k] = shrink * v[k];
    if (norms) norms[m] = n;
    if (shrinks) shrinks[m] = shrink;
    if (tie_margin && t > 0.0) *tie_margin = std::min(*tie_margin, std::abs(n - t) / t);
  }
}

// Rayleigh-quotient power iteration on H^T H^* (pgd.cpp:120-169).
// fixed_steps == 0: the reference's converged rule (tol 1e-8, refine to
// 1e-13, cap 1e4, ConvergenceError). fixed_steps > 0: exactly that many
// applications of H^T(H^* v), estimate = Re(v^H w) of the last one (the
// BASELINE "30-step power iteration", SURVEY.md §0 finding 6b).
int lipschitz(const cd* H, int K, int M, int fixed_steps, const cd* v0, double* exact) {
  std::vector<cd> v(v0, v0 + M), u(K), w(M);
  const long max_iters = fixed_steps > 0 ? fixed_steps : 10000;
  constexpr double kTol = 1e-8;
  constexpr double kRefineTol = 1e-13;
  double estimate = 0.0, previous = -1.0;
  bool reached_tol = false;
  for (long iter = 0; iter < max_iters; ++iter) {
    // u = H^* v  (K)
    for (int j = 0; j < K; ++j) u[j] = 0.0;
    for (int m = 0; m < M; ++m)
      for (int j = 0; j < K; ++j) u[j] += std::conj(H[static_cast<std::size_t>(m) * K + j]) * v[m];
    // w = H^T u  (M)
    for (int m = 0; m < M; ++m) {
      cd acc = 0.0;
      for (int j = 0; j < K; ++j) acc += H[static_cast<std::size_t>(m) * K + j] * u[j];
      w[m] = acc;
    }
    cd dot = 0.0;  // Eigen v.dot(w) conjugates v
    double wn2 = 0.0;
    for (int m = 0; m < M; ++m) {
      dot += std::conj(v[m]) * w[m];
      wn2 += std::norm(w[m]);
    }
    estimate = dot.real();
    double w_norm = std::sqrt(wn2);
    if (w_norm == 0.0) {
      *exact = 0.0;
      return ORA_OK;
    }
    for (int m = 0; m < M; ++m) v[m] = w[m] / w_norm;
    if (fixed_steps == 0 && previous >= 0.0) {
      double change = std::abs(estimate - previous) / std::max(std::abs(estimate), 1e-300);
      if (change <= kTol) reached_tol = true;
      if (change <= kRefineTol) break;
    }
    previous = estimate;
  }
  if (fixed_steps == 0 && !reached_tol) return ORA_ECONVERGENCE;
  *exact = estimate;
  return ORA_OK;
}

void power_v0(int M, cd* v0) {
  Rng rng(kPowerIterationSeed);  // pgd.cpp:131-134
  double s = 0.0;
  for (int i = 0; i < M; ++i) {
    v0[i] = rng.complex_gaussian();
    s += std::norm(v0[i]);
  }
  double n = std::sqrt(s);
  for (int i = 0; i < M; ++i) v0[i] /= n;
}

double l21(const cd* W, int K, int M) {  // metrics.cpp:10-16
  double total = 0.0;
  for (int m = 0; m < M; ++m) total += col_norm(W + static_cast<std::size_t>(m) * K, K);
  return total;
}

int active_columns(const cd* W, int K, int M) {  // pgd.cpp:23-29
  int active = 0;
  for (int m = 0; m < M; ++m) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s += std::norm(W[static_cast<std::size_t>(m) * K + k]);
    if (s > 0.0) ++active;
  }
  return active;
}

// metrics.cpp:71-77: || H W^T - diag(c) ||_F
double residual(const cd* H, const cd* W, const double* c, int K, int M) {
  std::vector<cd> R(static_cast<std::size_t>(K) * K, 0.0);  // R(k, j) = sum_m H(k,m) W(j,m)
  for (int m = 0; m < M; ++m)
    for (int j = 0; j < K; ++j)
      for (int k = 0; k < K; ++k)
        R[j * K + k] += H[static_cast<std::size_t>(m) * K + k] * W[static_cast<std::size_t>(m) * K + j];
  for (int k = 0; k < K; ++k) R[k * K + k] -= c[k];
  double s = 0.0;
  for (const cd& r : R) s += std::norm(r);
  return std::sqrt(s);
}

// The unfolded forward pass (unfolded.cpp:83-146) for one realization.
// Returns the 0-based diverging layer or -1.
long forward_one(const cd* H, const double* c, int K, int M, const double* lambda,
                 const double* eta, int L, const cd* W0, cd* Wout, cd* iterates, cd* tape_in,
                 cd* tape_v, double* tape_norms, double* tape_shrink, double* tie_margin) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  std::vector<cd> w(n), v(n), X;
  if (W0)
    std::copy(W0, W0 + n, w.begin());
  else
    for (std::size_t i = 0; i < n; ++i) w[i] = std::conj(H[i]);  // unfolded.cpp:96
  if (iterates) std::copy(w.begin(), w.end(), iterates);
  for (int i = 0; i < L; ++i) {
    const double threshold = lambda[i] * eta[i];
    if (!step_image(w.data(), H, c, K, M, eta[i], X, v.data())) return i;
    if (tape_in) std::copy(w.begin(), w.end(), tape_in + i * n);
    if (tape_v) std::copy(v.begin(), v.end(), tape_v + i * n);
    prox_cols(v.data(), K, M, threshold, w.data(), tape_norms ? tape_norms + static_cast<std::size_t>(i) * M : nullptr,
              tape_shrink ? tape_shrink + static_cast<std::size_t>(i) * M : nullptr, tie_margin);
    if (iterates) std::copy(w.begin(), w.end(), iterates + (i + 1) * n);
  }
  std::copy(w.begin(), w.end(), Wout);
  return -1;
}

// solve_pgd's loop (pgd.cpp:178-268) without tracing. Returns the 1-based
// diverging iteration or -1; *iterations = steps actually taken.
long pgd_one(const cd* H, const double* c, int K, int M, double lambda, double eta, long max_iters,
             double residual_tol, const cd* W0, cd* Wout, long* iterations, double* tie_margin) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  std::vector<cd> w(n), v(n), wn(n), X;
  if (W0)
    std::copy(W0, W0 + n, w.begin());
  else
    for (std::size_t i = 0; i < n; ++i) w[i] = std::conj(H[i]);  // pgd.cpp:184
  const double threshold = lambda * eta;
  long taken = 0;
  for (long iter = 1; iter <= max_iters; ++iter) {
    if (!step_image(w.data(), H, c, K, M, eta, X, v.data())) {
      if (iterations) *iterations = taken;
      return iter;
    }
    prox_cols(v.data(), K, M, threshold, wn.data(), nullptr, nullptr, tie_margin);
    double rel = -1.0;
    if (residual_tol > 0.0) {  // pgd.cpp:246-250
      double d = 0.0, s = 0.0;
      for (std::size_t i = 0; i < n; ++i) {
        d += std::norm(wn[i] - w[i]);
        s += std::norm(w[i]);
      }
      rel = std::sqrt(d) / std::max(std::sqrt(s), 1e-12);
    }
    w.swap(wn);
    taken = iter;
    if (rel >= 0.0 && rel < residual_tol) break;  // pgd.cpp:258-260
  }
  if (iterations) *iterations = taken;
  std::copy(w.begin(), w.end(), Wout);
  return -1;
}

// Hermitian eigenvalues by cyclic Jacobi (for the ZF condition check,
// zf.cpp:15-23; K is small).
std::vector<double> hermitian_eigenvalues(std::vector<cd> A, int n) {
  auto at = [&](int r, int c) -> cd& { return A[c * n + r]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += std::norm(at(p, q));
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        cd apq = at(p, q);
        double a = std::abs(apq);
        if (a < 1e-300) continue;
        double app = at(p, p).real(), aqq = at(q, q).real();
        cd phase = apq / a;
        double theta = 0.5 * std::atan2(2.0 * a, aqq - app);
        double cs = std::cos(theta), sn = std::sin(theta);
        // Rotation acting on columns p, q: G = [[c, s*phase], [-s*conj(phase), c]]
        for (int k = 0; k < n; ++k) {
          cd akp = at(k, p), akq = at(k, q);
          at(k, p) = cs * akp - sn * std::conj(phase) * akq;
          at(k, q) = sn * phase * akp + cs * akq;
        }
        for (int k = 0; k < n; ++k) {
          cd apk = at(p, k), aqk = at(q, k);
          at(p, k) = cs * apk - sn * phase * aqk;
          at(q, k) = sn * std::conj(phase) * apk + cs * aqk;
        }
      }
    }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = at(i, i).real();
  return ev;
}

// zf.cpp:9-30: W = diag(c) conj((H H^H)^{-1} H), Cholesky solve.
int zf(const cd* H, const double* c, int K, int M, cd* W) {
  std::vector<cd> G(static_cast<std::size_t>(K) * K, 0.0);  // G(k, j) = sum_m H(k,m) conj(H(j,m))
  for (int m = 0; m < M; ++m)
    for (int j = 0; j < K; ++j)
      for (int k = 0; k < K; ++k)
        G[j * K + k] += H[static_cast<std::size_t>(m) * K + k] * std::conj(H[static_cast<std::size_t>(m) * K + j]);
  std::vector<double> ev = hermitian_eigenvalues(G, K);
  double mn = *std::min_element(ev.begin(), ev.end());
  double mx = *std::max_element(ev.begin(), ev.end());
  if (!(mn > 0.0) || mx > 1e12 * mn) return ORA_ESINGULAR;  // zf.hpp:10
  // Cholesky G = L L^H (lower), col-major.
  std::vector<cd> Lc(static_cast<std::size_t>(K) * K, 0.0);
  auto l = [&](int r, int cc) -> cd& { return Lc[cc * K + r]; };
  for (int j = 0; j < K; ++j) {
    double d = G[j * K + j].real();
    for (int p = 0; p < j; ++p) d -= std::norm(l(j, p));
    if (!(d > 0.0)) return ORA_ESINGULAR;
    double djj = std::sqrt(d);
    l(j, j) = djj;
    for (int i = j + 1; i < K; ++i) {
      cd s = G[j * K + i];
      for (int p = 0; p < j; ++p) s -= l(i, p) * std::conj(l(j, p));
      l(i, j) = s / djj;
    }
  }
  // Solve G S = H column by column (S is K x M), then W = diag(c) conj(S).
  std::vector<cd> y(K), x(K);
  for (int m = 0; m < M; ++m) {
    const cd* h = H + static_cast<std::size_t>(m) * K;
    for (int i = 0; i < K; ++i) {
      cd s = h[i];
      for (int p = 0; p < i; ++p) s -= l(i, p) * y[p];
      y[i] = s / l(i, i);
    }
    for (int i = K - 1; i >= 0; --i) {
      cd s = y[i];
      for (int p = i + 1; p < K; ++p) s -= std::conj(l(p, i)) * x[p];
      x[i] = s / l(i, i).real();
    }
    for (int k = 0; k < K; ++k) W[static_cast<std::size_t>(m) * K + k] = c[k] * std::conj(x[k]);
  }
  return ORA_OK;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument&) {
    return ORA_EINVAL;
  } catch (...) {
    return ORA_EINVAL;
  }
}

void promote(const float* src, std::size_t n_complex, std::vector<cd>& dst) {
  dst.resize(n_complex);
  for (std::size_t i = 0; i < n_complex; ++i) dst[i] = cd(src[2 * i], src[2 * i + 1]);
}

}  // namespace

extern "C" {

int ora_default_thread_count() { return default_thread_count(); }

// pgd.cpp:111-118
int ora_mp_bound(int K, int M, double* out) {
  if (K < 1 || M < 1) return ORA_EINVAL;
  double edge = std::sqrt(static_cast<double>(K)) + std::sqrt(static_cast<double>(M));
  *out = edge * edge;
  return ORA_OK;
}

// Rng draws for known-answer checks. kind: 0 = next_u64 (as two uint32 halves
// in out_u64), 1 = uniform, 2 = uniform_open, 3 = complex_gaussian (2 doubles).
int ora_rng_draw(std::uint64_t seed, std::uint64_t stream, int use_stream, int kind, int n,
                 double* out, std::uint64_t* out_u64) {
  Rng rng = use_stream ? Rng::stream(seed, stream) : Rng(seed);
  for (int i = 0; i < n; ++i) {
    switch (kind) {
      case 0: out_u64[i] = rng.next_u64(); break;
      case 1: out[i] = rng.uniform(); break;
      case 2: out[i] = rng.uniform_open(); break;
      case 3: {
        cd z = rng.complex_gaussian();
        out[2 * i] = z.real();
        out[2 * i + 1] = z.imag();
        break;
      }
      default: return ORA_EINVAL;
    }
  }
  return ORA_OK;
}

// channel.cpp:7-16: K x M, drawn row by row (k outer, m inner).
int ora_generate_channel(std::uint64_t seed, std::uint64_t stream, int use_stream, int K, int M,
                         double* H) {
  if (K < 1 || M < K) return ORA_EINVAL;
  Rng rng = use_stream ? Rng::stream(seed, stream) : Rng(seed);
  cd* h = as_c(H);
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < M; ++m) h[static_cast<std::size_t>(m) * K + k] = rng.complex_gaussian();
  return ORA_OK;
}

// The BASELINE workloads' inputs, for the reference arm of
// bench.py so that it touches nothing of the product library: realization
// first+b is generate_channel(Rng::stream(seed_h, first+b)) (channel.cpp:7-16)
// with row k scaled in FP64 by 10^(-u_k R / 20), u_k drawn from
// Rng::stream(seed_g, first+b), then rounded once to complex64 [B][M][K].
int ora_generate_channels_batch_f32(std::uint64_t seed_h, std::uint64_t seed_g, double gain_range_db,
                                    std::int64_t first, std::int64_t B, int K, int M, float* H, int threads) {
  if (B < 0 || K < 1 || M < K || !(gain_range_db >= 0.0)) return ORA_EINVAL;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
    const std::uint64_t idx = static_cast<std::uint64_t>(first) + b;
    std::vector<double> gain(K, 1.0);
    if (gain_range_db > 0.0) {
      Rng g = Rng::stream(seed_g, idx);
      for (int k = 0; k < K; ++k) gain[k] = std::pow(10.0, -g.uniform() * gain_range_db / 20.0);
    }
    Rng r = Rng::stream(seed_h, idx);
    float* h = H + 2 * n * b;
    for (int k = 0; k < K; ++k)
      for (int m = 0; m < M; ++m) {
        const cd z = r.complex_gaussian();
        h[2 * (static_cast<std::size_t>(m) * K + k)] = static_cast<float>(z.real() * gain[k]);
        h[2 * (static_cast<std::size_t>(m) * K + k) + 1] = static_cast<float>(z.imag() * gain[k]);
      }
  }, threads);
  return ORA_OK;
}

// Seeded layer parameters of the BASELINE configs, pack order (lambda_0,
// mu_0, lambda_1, ...) from Rng::stream(seed_p, 0): lambda = 0.01 + 0.09 u,
// mu = (0.5 + u) / mp_bound(K, M) — raw, before project_params. No FMA
// contraction (-march=x86-64-v3 would fuse 0.01 + 0.09 u into one rounding).
__attribute__((optimize("fp-contract=off"))) int ora_layer_params(std::uint64_t seed_p, int L, int K, int M, double* lambda, double* eta) {
  if (L < 0 || K < 1 || M < 1) return ORA_EINVAL;
  const double edge = std::sqrt(static_cast<double>(K)) + std::sqrt(static_cast<double>(M));
  const double mp = edge * edge;
  Rng r = Rng::stream(seed_p, 0);
  for (int l = 0; l < L; ++l) {
    lambda[l] = 0.01 + 0.09 * r.uniform();
    eta[l] = (0.5 + r.uniform()) / mp;
  }
  return ORA_OK;
}

int ora_power_v0(int M, double* v0) {
  if (M < 1) return ORA_EINVAL;
  power_v0(M, as_c(v0));
  return ORA_OK;
}

int ora_prox_l21(const double* V, int K, int M, double t, double* out) {
  if (!(t >= 0.0)) return ORA_EINVAL;  // pgd.cpp:86-88
  prox_cols(as_c(V), K, M, t, as_c(out), nullptr, nullptr, nullptr);
  return ORA_OK;
}

// grad_f (pgd.cpp:68-83): X H^* - diag(c) H^*
int ora_grad_f(const double* W, const double* H, const double* c, int K, int M, double* out) {
  std::vector<cd> X(static_cast<std::size_t>(K) * K);
  w_times_ht(as_c(W), as_c(H), K, M, X.data());
  const cd* h = as_c(H);
  cd* g = as_c(out);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      cd acc = 0.0;
      for (int j = 0; j < K; ++j) acc += X[j * K + k] * std::conj(h[static_cast<std::size_t>(m) * K + j]);
      acc -= c[k] * std::conj(h[static_cast<std::size_t>(m) * K + k]);
      g[static_cast<std::size_t>(m) * K + k] = acc;
    }
  return ORA_OK;
}

// pgd_step (pgd.cpp:101-109): prox(W - eta grad_f(W), lambda eta).
int ora_pgd_step(const double* W, const double* H, const double* c, int K, int M, double lambda,
                 double eta, double* out) {
  if (!(lambda >= 0.0) || !(eta > 0.0)) return ORA_EINVAL;
  std::vector<cd> g(static_cast<std::size_t>(K) * M);
  ora_grad_f(W, H, c, K, M, reinterpret_cast<double*>(g.data()));
  const cd* w = as_c(W);
  for (std::size_t i = 0; i < g.size(); ++i) g[i] = w[i] - eta * g[i];
  prox_cols(g.data(), K, M, lambda * eta, as_c(out), nullptr, nullptr, nullptr);
  return ORA_OK;
}

int ora_lipschitz(const double* H, int K, int M, int fixed_steps, double* exact) {
  if (K < 1 || M < 1 || fixed_steps < 0) return ORA_EINVAL;
  std::vector<cd> v0(M);
  power_v0(M, v0.data());
  return lipschitz(as_c(H), K, M, fixed_steps, v0.data(), exact);
}

double ora_l21_norm(const double* W, int K, int M) { return l21(as_c(W), K, M); }
int ora_active_columns(const double* W, int K, int M) { return active_columns(as_c(W), K, M); }
double ora_constraint_residual(const double* H, const double* W, const double* c, int K, int M) {
  return residual(as_c(H), as_c(W), c, K, M);
}
// pgd.cpp:171-176
double ora_lagrangian(const double* W, const double* H, const double* c, int K, int M, double lambda) {
  double r = residual(as_c(H), as_c(W), c, K, M);
  return lambda * l21(as_c(W), K, M) + r * r;
}

// metrics.cpp:29-91 + zf.cpp:9-30 for one realization. out = [tx_power,
// cons_power, sum_rate, pcg, residual, zf_ok, sinr[K]]; zf_ok = 0 when
// zf_precoder throws SingularChannelError (then pcg = NaN).
int ora_metrics(const double* Hp, const double* Wp, const double* c, double sigma_nu, double alpha, int K,
                int M, double* out) {
  const cd* H = as_c(Hp);
  const cd* W = as_c(Wp);
  double tx = 0.0;
  for (int i = 0; i < K * M; ++i) tx += std::norm(W[i]);
  const double l21w = l21(W, K, M);
  // effective channel H W^T (K x K): E(k, j) = sum_m H(k, m) W(j, m)
  std::vector<cd> E(static_cast<std::size_t>(K) * K, 0.0);
  for (int m = 0; m < M; ++m)
    for (int j = 0; j < K; ++j)
      for (int k = 0; k < K; ++k) E[j * K + k] += H[static_cast<std::size_t>(m) * K + k] * W[static_cast<std::size_t>(m) * K + j];
  const double noise = sigma_nu * sigma_nu;
  double rate = 0.0;
  for (int k = 0; k < K; ++k) {
    const double signal = std::norm(E[k * K + k]);
    double row = 0.0;
    for (int j = 0; j < K; ++j) row += std::norm(E[j * K + k]);
    const double sinr = signal / ((row - signal) + noise);
    out[6 + k] = sinr;
    rate += std::log2(1.0 + sinr);
  }
  double res = 0.0;
  for (int j = 0; j < K; ++j)
    for (int k = 0; k < K; ++k) {
      cd e = E[j * K + k];
      if (k == j) e -= c[k];
      res += std::norm(e);
    }
  std::vector<cd> Z(static_cast<std::size_t>(K) * M);
  const int zrc = zf(H, c, K, M, Z.data());
  out[0] = tx;
  out[1] = alpha * l21w;
  out[2] = rate;
  out[3] = zrc == ORA_OK && l21w > 0.0 ? l21(Z.data(), K, M) / l21w : std::nan("");
  out[4] = std::sqrt(res);
  out[5] = zrc == ORA_OK ? 1.0 : 0.0;
  return ORA_OK;
}

int ora_metrics_batch_f32(const float* H, const float* W, std::int64_t B, const double* c, double sigma_nu,
                          double alpha, int K, int M, double* out, int threads) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h, w;
      promote(H + 2 * n * b, n, h);
      promote(W + 2 * n * b, n, w);
      ora_metrics(reinterpret_cast<const double*>(h.data()), reinterpret_cast<const double*>(w.data()), c,
                  sigma_nu, alpha, K, M, out + b * (6 + K));
    }, threads);
    return ORA_OK;
  });
}

// backward (unfolded.cpp:158-239) over the tape of forward_one. dcost is the
// real-pair cost gradient dC/dRe(W) + i dC/dIm(W) of the output.
int ora_backward(const double* Hp, int K, int M, const double* lambda, const double* eta, int L,
                 const double* tape_in, const double* tape_v, const double* tape_norms,
                 const double* tape_shrink, const double* dcost, double* d_lambda, double* d_eta) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  const cd* H = as_c(Hp);
  std::vector<cd> g(as_c(dcost), as_c(dcost) + n), gimg(n), S(static_cast<std::size_t>(K) * K);
  for (int idx = L - 1; idx >= 0; --idx) {
    const cd* Win = as_c(tape_in) + n * idx;
    const cd* V = as_c(tape_v) + n * idx;
    const double* norms = tape_norms + static_cast<std::size_t>(M) * idx;
    const double* shrink = tape_shrink + static_cast<std::size_t>(M) * idx;
    const double lam = lambda[idx], et = eta[idx];
    if (!(et > 0.0)) return ORA_EINVAL;  // TrainingError (unfolded.cpp:189-191)
    const double t = lam * et;
    double d_t = 0.0;
    for (int m = 0; m < M; ++m) {
      const double nrm = norms[m];
      const cd* v = V + static_cast<std::size_t>(m) * K;
      const cd* gm = g.data() + static_cast<std::size_t>(m) * K;
      cd* gi = gimg.data() + static_cast<std::size_t>(m) * K;
      if (nrm > t) {
        cd dot = 0.0;
        for (int k = 0; k < K; ++k) dot += std::conj(v[k]) * gm[k];
        const double inner = dot.real();
        d_t -= inner / nrm;
        for (int k = 0; k < K; ++k) gi[k] = shrink[m] * gm[k] + (t / (nrm * nrm * nrm)) * inner * v[k];
      } else {
        for (int k = 0; k < K; ++k) gi[k] = 0.0;
      }
    }
    double d_eta_direct = 0.0;
    for (int m = 0; m < M; ++m) {
      cd dot = 0.0;
      for (int k = 0; k < K; ++k) {
        const std::size_t e = static_cast<std::size_t>(m) * K + k;
        dot += std::conj(gimg[e]) * (Win[e] - V[e]);
      }
      d_eta_direct -= dot.real() / et;
    }
    d_lambda[idx] = et * d_t;
    d_eta[idx] = lam * d_t + d_eta_direct;
    w_times_ht(gimg.data(), H, K, M, S.data());  // S(k, j) = sum_m gimg(k, m) H(j, m)
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) {
        cd acc = 0.0;
        for (int j = 0; j < K; ++j) acc += S[j * K + k] * std::conj(H[static_cast<std::size_t>(m) * K + j]);
        const std::size_t e = static_cast<std::size_t>(m) * K + k;
        g[e] = gimg[e] - et * acc;
      }
  }
  return ORA_OK;
}

// The per-sample body of train's parallel_for (training.cpp:205-234): taped
// forward from H^*, loss, loss gradient (training.cpp:59-95), backward.
// loss_kind 0 = unsupervised (lagrangian with lambda_cost), 1 = supervised
// (||W - label||^2). grads = (d_lambda_0, d_eta_0, d_lambda_1, ...).
int ora_train_sample(const double* Hp, const double* c, int K, int M, const double* lambda, const double* eta, int L,
                     int loss_kind, double lambda_cost, const double* label, double* loss, double* grads) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  const cd* H = as_c(Hp);
  std::vector<cd> W(n), tin(n * L), tv(n * L);
  std::vector<double> tn(static_cast<std::size_t>(M) * L), ts(static_cast<std::size_t>(M) * L);
  const long d = forward_one(H, c, K, M, lambda, eta, L, nullptr, W.data(), nullptr, tin.data(), tv.data(), tn.data(),
                             ts.data(), nullptr);
  if (d >= 0) return ORA_EDIVERGED;
  std::vector<cd> dc(n);
  if (loss_kind == 1) {
    const cd* lab = as_c(label);
    double l = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
      l += std::norm(W[i] - lab[i]);
      dc[i] = 2.0 * (W[i] - lab[i]);
    }
    *loss = l;
  } else {
    const double r = residual(H, W.data(), c, K, M);
    *loss = lambda_cost * l21(W.data(), K, M) + r * r;
    ora_grad_f(reinterpret_cast<const double*>(W.data()), Hp, c, K, M, reinterpret_cast<double*>(dc.data()));
    for (int m = 0; m < M; ++m) {
      const cd* w = W.data() + static_cast<std::size_t>(m) * K;
      const double nrm = col_norm(w, K);
      for (int k = 0; k < K; ++k) {
        cd& e = dc[static_cast<std::size_t>(m) * K + k];
        e = 2.0 * e;
        if (nrm > 0.0) e += (lambda_cost / nrm) * w[k];
      }
    }
  }
  std::vector<double> dl(L), de(L);
  const int rc = ora_backward(Hp, K, M, lambda, eta, L, reinterpret_cast<const double*>(tin.data()),
                              reinterpret_cast<const double*>(tv.data()), tn.data(), ts.data(),
                              reinterpret_cast<const double*>(dc.data()), dl.data(), de.data());
  for (int i = 0; i < L; ++i) {
    grads[2 * i] = dl[i];
    grads[2 * i + 1] = de[i];
  }
  return rc;
}

int ora_train_batch_f32(const float* H, std::int64_t B, const double* c, int K, int M, const double* lambda,
                        const double* eta, int L, int loss_kind, double lambda_cost, const float* labels,
                        double* loss, double* grads, std::int32_t* status, int threads) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h, lab;
      promote(H + 2 * n * b, n, h);
      if (labels) promote(labels + 2 * n * b, n, lab);
      const int rc = ora_train_sample(reinterpret_cast<const double*>(h.data()), c, K, M, lambda, eta, L, loss_kind,
                                      lambda_cost, labels ? reinterpret_cast<const double*>(lab.data()) : nullptr,
                                      loss + b, grads + 2 * L * b);
      if (status) status[b] = rc;
    }, threads);
    return ORA_OK;
  });
}

int ora_zf_precoder(const double* H, const double* c, int K, int M, double* W) {
  if (K < 1 || M < K) return ORA_EINVAL;
  return zf(as_c(H), c, K, M, as_c(W));
}

// forward (unfolded.cpp:83-146) for one realization, raw (no validation; the
// Python mirror in oracle/oracle.py performs the reference's checks).
// W0 == nullptr selects the default start H^*. Returns ORA_EDIVERGED with
// *diverged_layer set (0-based) on a non-finite step image.
int ora_forward(const double* H, const double* c, int K, int M, const double* lambda,
                const double* eta, int L, const double* W0, double* W, long* diverged_layer,
                double* iterates, double* tape_in, double* tape_v, double* tape_norms,
                double* tape_shrink) {
  long d = forward_one(as_c(H), c, K, M, lambda, eta, L, W0 ? as_c(W0) : nullptr, as_c(W),
                       iterates ? as_c(iterates) : nullptr, tape_in ? as_c(tape_in) : nullptr,
                       tape_v ? as_c(tape_v) : nullptr, tape_norms, tape_shrink, nullptr);
  if (diverged_layer) *diverged_layer = d;
  return d >= 0 ? ORA_EDIVERGED : ORA_OK;
}

int ora_solve_pgd(const double* H, const double* c, int K, int M, double lambda, double eta,
                  long max_iters, double residual_tol, const double* W0, double* W, long* iterations,
                  long* diverged_iter) {
  long d = pgd_one(as_c(H), c, K, M, lambda, eta, max_iters, residual_tol, W0 ? as_c(W0) : nullptr,
                   as_c(W), iterations, nullptr);
  if (diverged_iter) *diverged_iter = d;
  return d >= 0 ? ORA_EDIVERGED : ORA_OK;
}

// ---------------------------------------------------------------------------
// Batched drivers over complex64 inputs [B][M][K] (promoted to FP64 once), run
// with the restated parallel_for on `threads` host threads. Per realization
// outputs are optional (nullptr skips): W (FP64), diverged index, l21 norm,
// active columns, tie margin (min over layers and antennas of |n - t| / t).
// w0_mode: 0 = zero, 1 = H^* (reference default), 2 = given (W0 complex64).
// ---------------------------------------------------------------------------
int ora_forward_batch_f32(const float* H, std::int64_t B, const double* c, int K, int M,
                          const double* lambda, const double* eta, int L, int w0_mode,
                          const float* W0, double* W, std::int32_t* diverged_at, double* l21_out,
                          std::int32_t* active_out, double* tie_margin, int threads) {
  if (B < 0 || K < 1 || M < 1 || L < 0 || w0_mode < 0 || w0_mode > 2) return ORA_EINVAL;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h, w0, w(n);
      promote(H + 2 * n * b, n, h);
      const cd* start = nullptr;
      if (w0_mode == 0) {
        w0.assign(n, cd(0.0, 0.0));
        start = w0.data();
      } else if (w0_mode == 2) {
        promote(W0 + 2 * n * b, n, w0);
        start = w0.data();
      }
      double tie = std::numeric_limits<double>::infinity();
      long d = forward_one(h.data(), c, K, M, lambda, eta, L, start, w.data(), nullptr, nullptr,
                           nullptr, nullptr, nullptr, &tie);
      if (diverged_at) diverged_at[b] = static_cast<std::int32_t>(d);
      if (W) std::copy(w.begin(), w.end(), as_c(W) + n * b);
      if (l21_out) l21_out[b] = d >= 0 ? std::nan("") : l21(w.data(), K, M);
      if (active_out) active_out[b] = d >= 0 ? -1 : active_columns(w.data(), K, M);
      if (tie_margin) tie_margin[b] = tie;
    }, threads);
    return ORA_OK;
  });
}

// Plain PGD per realization with its own step eta[b] (config 3) and shared
// lambda; diverged_at holds the 1-based iteration or -1.
int ora_pgd_batch_f32(const float* H, std::int64_t B, const double* c, int K, int M, double lambda,
                      const double* eta, long max_iters, double residual_tol, int w0_mode,
                      const float* W0, double* W, std::int32_t* diverged_at, std::int64_t* iterations,
                      double* l21_out, std::int32_t* active_out, double* tie_margin, int threads) {
  if (B < 0 || K < 1 || M < 1 || max_iters < 0 || w0_mode < 0 || w0_mode > 2) return ORA_EINVAL;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h, w0, w(n);
      promote(H + 2 * n * b, n, h);
      const cd* start = nullptr;
      if (w0_mode == 0) {
        w0.assign(n, cd(0.0, 0.0));
        start = w0.data();
      } else if (w0_mode == 2) {
        promote(W0 + 2 * n * b, n, w0);
        start = w0.data();
      }
      double tie = std::numeric_limits<double>::infinity();
      long it = 0;
      long d = pgd_one(h.data(), c, K, M, lambda, eta[b], max_iters, residual_tol, start, w.data(),
                       &it, &tie);
      if (diverged_at) diverged_at[b] = static_cast<std::int32_t>(d);
      if (iterations) iterations[b] = it;
      if (W) std::copy(w.begin(), w.end(), as_c(W) + n * b);
      if (l21_out) l21_out[b] = d >= 0 ? std::nan("") : l21(w.data(), K, M);
      if (active_out) active_out[b] = d >= 0 ? -1 : active_columns(w.data(), K, M);
      if (tie_margin) tie_margin[b] = tie;
    }, threads);
    return ORA_OK;
  });
}

// Fixed-step (steps > 0) or converged (steps == 0) power iteration per
// realization; status per realization in `status` (0 ok, ORA_ECONVERGENCE).
int ora_power_iteration_batch_f32(const float* H, std::int64_t B, int K, int M, int steps,
                                  double* L, std::int32_t* status, int threads) {
  if (B < 0 || K < 1 || M < 1 || steps < 0) return ORA_EINVAL;
  const std::size_t n = static_cast<std::size_t>(K) * M;
  std::vector<cd> v0(M);
  power_v0(M, v0.data());
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h;
      promote(H + 2 * n * b, n, h);
      double est = 0.0;
      int st = lipschitz(h.data(), K, M, steps, v0.data(), &est);
      L[b] = est;
      if (status) status[b] = st;
    }, threads);
    return ORA_OK;
  });
}

// FP64 objective / residual of complex64 precoders against complex64 channels
// for a batch (parity metric helper).
int ora_lagrangian_batch_f32(const float* H, const float* W, std::int64_t B, const double* c, int K,
                             int M, double lambda, double* out, int threads) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h, w;
      promote(H + 2 * n * b, n, h);
      promote(W + 2 * n * b, n, w);
      double r = residual(h.data(), w.data(), c, K, M);
      out[b] = lambda * l21(w.data(), K, M) + r * r;
    }, threads);
    return ORA_OK;
  });
}

int ora_lagrangian_batch_f64(const float* H, const double* W, std::int64_t B, const double* c, int K,
                             int M, double lambda, double* out, int threads) {
  const std::size_t n = static_cast<std::size_t>(K) * M;
  return guarded([&] {
    parallel_for(static_cast<std::size_t>(B), [&](std::size_t b) {
      std::vector<cd> h;
      promote(H + 2 * n * b, n, h);
      const cd* w = as_c(W) + n * b;
      double r = residual(h.data(), w, c, K, M);
      out[b] = lambda * l21(w, K, M) + r * r;
    }, threads);
    return ORA_OK;
  });
}

}  // extern "C"
