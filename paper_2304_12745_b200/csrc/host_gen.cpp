// Seeded synthetic inputs for the batched solver — the
// harness side of the path, run on the host and never timed. Restates the
// reference random source (rng.cpp:9-40) and channel draw (channel.cpp:7-16)
// so realization i of a batch is bit-identical to the reference's
// generate_channel(cfg, Rng::stream(seed, i)) before the single rounding to
// complex64. std::mt19937_64 is fully specified by the C++ standard.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

#include "ufpgd_gpu.h"

namespace {

std::uint64_t mix64(std::uint64_t x) {  // rng.cpp:10-15
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

struct Rng {
  std::mt19937_64 gen;
  explicit Rng(std::uint64_t s) : gen(s) {}
  static Rng stream(std::uint64_t seed, std::uint64_t i) { return Rng(mix64(seed ^ mix64(i))); }
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform_open() { return static_cast<double>((gen() >> 11) + 1) * 0x1.0p-53; }
  void complex_gaussian(double& re, double& im) {  // rng.cpp:35-40
    const double radius = std::sqrt(-std::log(uniform_open()));
    const double angle = 2.0 * std::numbers::pi * uniform();
    re = radius * std::cos(angle);
    im = radius * std::sin(angle);
  }
};

int hw_threads(int threads) {
  if (threads > 0) return threads;
  unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

}  // namespace

extern "C" int ufpgd_generate_channels(uint64_t seed_h, uint64_t seed_g, double gain_range_db,
                                       int64_t first_index, int64_t B, int K, int M, ufpgd_c64* H,
                                       int threads) {
  if (B < 0 || K < 1 || M < K || !H || !(gain_range_db >= 0.0)) return UFPGD_EINVAL_SHAPE;
  const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(hw_threads(threads), std::max<int64_t>(B, 1))));
  auto work = [&](int t) {
    std::vector<double> gain(K, 1.0);
    for (int64_t b = t; b < B; b += nt) {
      const uint64_t idx = static_cast<uint64_t>(first_index + b);
      if (gain_range_db > 0.0) {
        Rng g = Rng::stream(seed_g, idx);
        for (int k = 0; k < K; ++k) gain[k] = std::pow(10.0, -g.uniform() * gain_range_db / 20.0);
      }
      Rng r = Rng::stream(seed_h, idx);
      ufpgd_c64* h = H + b * static_cast<int64_t>(K) * M;
      for (int k = 0; k < K; ++k)  // channel.cpp:10-14: k outer, m inner
        for (int m = 0; m < M; ++m) {
          double re, im;
          r.complex_gaussian(re, im);
          h[static_cast<int64_t>(m) * K + k] = {static_cast<float>(re * gain[k]),
                                                static_cast<float>(im * gain[k])};
        }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return UFPGD_OK;
}

extern "C" int ufpgd_power_v0_f64(int M, double* v0) {
  if (M < 1 || !v0) return UFPGD_EINVAL_SHAPE;
  Rng rng(0x1F2E3D4C5B6A7988ULL);  // pgd.cpp:14, :131-134
  double s = 0.0;
  for (int i = 0; i < M; ++i) {
    rng.complex_gaussian(v0[2 * i], v0[2 * i + 1]);
    s += v0[2 * i] * v0[2 * i] + v0[2 * i + 1] * v0[2 * i + 1];
  }
  const double n = std::sqrt(s);
  for (int i = 0; i < 2 * M; ++i) v0[i] /= n;
  return UFPGD_OK;
}

extern "C" int ufpgd_power_v0(int M, ufpgd_c64* v0) {
  if (M < 1 || !v0) return UFPGD_EINVAL_SHAPE;
  Rng rng(0x1F2E3D4C5B6A7988ULL);  // pgd.cpp:14, :131-134
  std::vector<double> re(M), im(M);
  double s = 0.0;
  for (int i = 0; i < M; ++i) {
    rng.complex_gaussian(re[i], im[i]);
    s += re[i] * re[i] + im[i] * im[i];
  }
  const double n = std::sqrt(s);
  for (int i = 0; i < M; ++i) v0[i] = {static_cast<float>(re[i] / n), static_cast<float>(im[i] / n)};
  return UFPGD_OK;
}

extern "C" int ufpgd_layer_params(uint64_t seed_p, int L, int K, int M, double* lambda, double* eta) {
  if (L < 0 || K < 1 || M < 1 || (L > 0 && (!lambda || !eta))) return UFPGD_EINVAL_PARAM;
  const double edge = std::sqrt(static_cast<double>(K)) + std::sqrt(static_cast<double>(M));
  const double mp = edge * edge;  // pgd.cpp:111-118
  Rng r = Rng::stream(seed_p, 0);
  for (int l = 0; l < L; ++l) {  // pack order lambda_0, eta_0, ... (training.hpp:50-51)
    lambda[l] = 0.01 + 0.09 * r.uniform();
    eta[l] = (0.5 + r.uniform()) / mp;
  }
  return UFPGD_OK;
}
