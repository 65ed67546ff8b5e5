// FP64 warp-per-realization PGD (oracle_solve at scale,
// and the batched FP64 solve_pgd). One warp owns one realization for all its
// iterations with W and its rows of X' in registers and H in shared memory,
// and retires on its own the moment the realization meets the reference's
// relative-change stop (pgd.cpp:246-260) or diverges — no CTA-wide barriers,
// so converged realizations free their slot for the next block. Same
// arithmetic as pgd.cpp:226-244 in FP64 with the constraint folded into X'
// (X' = W H^T - diag c, V = W - eta X' H^*), exact sqrt / division in the prox.
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "device_common.cuh"

namespace ufpgd_gpu_impl {
namespace {

// Thread (a, b) of the warp: users k = a*KA + kk, antennas m = i*TM + b.
template <int K_, int M_, int TK_, int TM_>
struct Team64 {
  static constexpr int K = K_, M = M_, TK = TK_, TM = TM_;
  static constexpr int KA = K / TK, MB = M / TM;
  static constexpr int U = K;                 // 16-byte units (one complex double) per H row
  static constexpr int RPP = U >= 8 ? 1 : 8 / U;  // rows per 128-byte bank period
  static_assert(TK * TM == 32, "one warp per realization");
  static_assert(K % TK == 0 && M % TM == 0, "team must tile (K, M)");
  // H(j, m) lives at unit j ^ swz(m) of row m: the TM rows an LDS.128 phase
  // touches (same unit j) land on distinct bank groups.
  static __device__ __forceinline__ int swz(int m) { return (m / RPP) & (U >= 8 ? 7 : U - 1); }
  static __device__ __forceinline__ int hoff(int m, int j) { return m * U + (j ^ swz(m)); }
};

template <class S>
#ifndef UFPGD_T64_MINB
#define UFPGD_T64_MINB 1
#endif
__global__ void __launch_bounds__(32, UFPGD_T64_MINB) pgd64_team_kernel(const __grid_constant__ GeneralArgs64 p) {
  __shared__ double2 hs[S::M * S::K];
  const int lane = threadIdx.x, a = lane / S::TM, b = lane % S::TM;
  const long long rid = blockIdx.x;
  const double2* hg = p.H + rid * (S::M * S::K);
  for (int e = lane; e < S::M * S::K; e += 32) hs[S::hoff(e / S::K, e % S::K)] = hg[e];
  __syncwarp();

  // W(k, m) for the thread's users and antennas
  double wr[S::MB][S::KA], wi[S::MB][S::KA];
#pragma unroll
  for (int i = 0; i < S::MB; ++i)
#pragma unroll
    for (int kk = 0; kk < S::KA; ++kk) {
      const int m = i * S::TM + b, k = a * S::KA + kk;
      double2 w;
      if (p.w0_mode == UFPGD_W0_ZERO) {
        w = make_double2(0.0, 0.0);
      } else if (p.w0_mode == UFPGD_W0_GIVEN) {
        w = p.W0[rid * (S::M * S::K) + m * S::K + k];
      } else {
        const double2 h = hs[S::hoff(m, k)];
        w = make_double2(h.x, -h.y);
      }
      wr[i][kk] = w.x;
      wi[i][kk] = w.y;
    }
  const double eta = p.eta_b ? p.eta_b[rid] : 1.0 / p.lip_b[rid];
  const double thr = p.lambda * eta;
  if (p.eta_out && lane == 0) p.eta_out[rid] = eta;

  double xr[S::KA][S::K], xi[S::KA][S::K];
  // X' = W H^T - diag(c): partial over the thread's antennas, then all-reduce
  // across the TM lanes of the row group (the b == 0 lane carries -c).
  auto stage1 = [&]() {
#pragma unroll
    for (int kk = 0; kk < S::KA; ++kk)
#pragma unroll
      for (int j = 0; j < S::K; ++j) {
        xr[kk][j] = (b == 0 && j == a * S::KA + kk) ? -p.c[j] : 0.0;
        xi[kk][j] = 0.0;
      }
#pragma unroll
    for (int i = 0; i < S::MB; ++i) {
      const int m = i * S::TM + b;
#pragma unroll
      for (int j = 0; j < S::K; ++j) {
        const double2 h = hs[S::hoff(m, j)];
#pragma unroll
        for (int kk = 0; kk < S::KA; ++kk) {  // X'(k, j) += W(k, m) H(j, m)
          xr[kk][j] = fma(wr[i][kk], h.x, xr[kk][j]);
          xr[kk][j] = fma(-wi[i][kk], h.y, xr[kk][j]);
          xi[kk][j] = fma(wr[i][kk], h.y, xi[kk][j]);
          xi[kk][j] = fma(wi[i][kk], h.x, xi[kk][j]);
        }
      }
    }
#pragma unroll
    for (int kk = 0; kk < S::KA; ++kk)
#pragma unroll
      for (int j = 0; j < S::K; ++j)
#pragma unroll
        for (int off = 1; off < S::TM; off <<= 1) {
          xr[kk][j] += __shfl_xor_sync(kFull, xr[kk][j], off);
          xi[kk][j] += __shfl_xor_sync(kFull, xi[kk][j], off);
        }
  };

  long long taken = 0;
  int first_bad = -1;
  for (long long it = 0; it < p.iters; ++it) {
    stage1();
#pragma unroll
    for (int kk = 0; kk < S::KA; ++kk)
#pragma unroll
      for (int j = 0; j < S::K; ++j) {
        xr[kk][j] *= -eta;
        xi[kk][j] *= -eta;
      }
    bool bad = false;
    double d2 = 0.0, s2 = 0.0;
#pragma unroll
    for (int i = 0; i < S::MB; ++i) {
      const int m = i * S::TM + b;
      double vr[S::KA], vi[S::KA];
#pragma unroll
      for (int kk = 0; kk < S::KA; ++kk) {
        vr[kk] = wr[i][kk];
        vi[kk] = wi[i][kk];
      }
#pragma unroll
      for (int j = 0; j < S::K; ++j) {
        const double2 h = hs[S::hoff(m, j)];
#pragma unroll
        for (int kk = 0; kk < S::KA; ++kk) {  // V = W + (-eta X') conj(H)
          vr[kk] = fma(h.x, xr[kk][j], vr[kk]);
          vr[kk] = fma(h.y, xi[kk][j], vr[kk]);
          vi[kk] = fma(h.x, xi[kk][j], vi[kk]);
          vi[kk] = fma(-h.y, xr[kk][j], vi[kk]);
        }
      }
      double sq = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KA; ++kk) sq = fma(vr[kk], vr[kk], fma(vi[kk], vi[kk], sq));
#pragma unroll
      for (int off = S::TM; off < 32; off <<= 1) sq += __shfl_xor_sync(kFull, sq, off);
      bad |= !(sq <= DBL_MAX);  // non-finite step image (pgd.cpp:231-235)
      const double nrm = sqrt(sq);
      const bool on = nrm > thr;  // prox (pgd.cpp:85-99), exact
      const double sh = on ? 1.0 - thr / nrm : 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KA; ++kk) {
        const double nr = on ? sh * vr[kk] : 0.0, ni = on ? sh * vi[kk] : 0.0;
        if (p.residual_tol > 0.0) {
          d2 += (nr - wr[i][kk]) * (nr - wr[i][kk]) + (ni - wi[i][kk]) * (ni - wi[i][kk]);
          s2 += wr[i][kk] * wr[i][kk] + wi[i][kk] * wi[i][kk];
        }
        wr[i][kk] = nr;
        wi[i][kk] = ni;
      }
    }
    taken = it + 1;
    if (__any_sync(kFull, bad)) {
      first_bad = static_cast<int>(it);
      break;  // solve_pgd stops at the first non-finite step image
    }
    if (p.residual_tol > 0.0) {
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        d2 += __shfl_xor_sync(kFull, d2, off);
        s2 += __shfl_xor_sync(kFull, s2, off);
      }
      if (sqrt(d2) / fmax(sqrt(s2), 1e-12) < p.residual_tol) break;  // warp-uniform: all lanes hold the sums
    }
  }

  double* Wg = reinterpret_cast<double*>(p.W + rid * (S::M * S::K));
  double l21 = 0.0, act = 0.0;
#pragma unroll
  for (int i = 0; i < S::MB; ++i) {
    const int m = i * S::TM + b;
    double sq = 0.0;
#pragma unroll
    for (int kk = 0; kk < S::KA; ++kk) {
      const int k = a * S::KA + kk;
      Wg[2 * (m * S::K + k)] = wr[i][kk];
      Wg[2 * (m * S::K + k) + 1] = wi[i][kk];
      sq = fma(wr[i][kk], wr[i][kk], fma(wi[i][kk], wi[i][kk], sq));
    }
#pragma unroll
    for (int off = S::TM; off < 32; off <<= 1) sq += __shfl_xor_sync(kFull, sq, off);
    if (a == 0) {
      l21 += sqrt(sq);
      act += sq > 0.0 ? 1.0 : 0.0;
    }
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    l21 += __shfl_xor_sync(kFull, l21, off);
    act += __shfl_xor_sync(kFull, act, off);
  }
  if (lane == 0) {
    const bool diverged = first_bad >= 0;
    if (p.diverged_at) p.diverged_at[rid] = diverged ? first_bad + p.index_base : -1;
    if (p.iterations) p.iterations[rid] = taken;
    if (p.l21) p.l21[rid] = diverged ? __longlong_as_double(0x7ff8000000000000LL) : l21;
    if (p.active) p.active[rid] = diverged ? -1 : static_cast<int32_t>(act);
    if (p.block_partials) {
      p.block_partials[rid * 3 + 0] = diverged ? 0.0 : p.alpha * l21;
      p.block_partials[rid * 3 + 1] = diverged ? 0.0 : act;
      p.block_partials[rid * 3 + 2] = diverged ? 1.0 : 0.0;
    }
  }
}

template <class S>
cudaError_t launch_pgd64_team(const GeneralArgs64& a, cudaStream_t s) {
  pgd64_team_kernel<S><<<static_cast<unsigned>(a.B), 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool pgd64_team_supported(const GeneralArgs64& a) {
  if (option(UFPGD_OPT_FP64_TEAM) == 0) return false;
  const bool shape = (a.K == 8 && a.M == 64) || (a.K == 4 && a.M == 32);
  return shape && a.pgd == 1 && a.mode == 0 && a.index_base == 1 && !a.iterates && !a.tape_v && !a.tape_norms &&
         !a.tape_shrink;
}

cudaError_t launch_pgd64_team(const GeneralArgs64& a, cudaStream_t s) {
  if (a.K == 8 && a.M == 64) return launch_pgd64_team<Team64<8, 64, 4, 8>>(a, s);
  if (a.K == 4 && a.M == 32) return launch_pgd64_team<Team64<4, 32, 2, 16>>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace ufpgd_gpu_impl
