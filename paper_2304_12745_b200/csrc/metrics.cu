// FP64 metrics epilogue: compute_metrics + zf_precoder per realization.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <algorithm>

#include "device_common.cuh"

namespace ufpgd_gpu_impl {
namespace {

// ---------------------------------------------------------------------------
// Batched metrics epilogue: the consumer side of forward
// in evaluate (training.cpp:310-421) — compute_metrics (metrics.cpp:79-91)
// with the ZF reference (zf.cpp:9-30) per realization. One CTA per
// realization. The ZF reference (Gram H H^H, its eigenvalue condition check,
// Cholesky and the per-antenna solves) runs in FP64: it is a precision-
// critical K x K solve; the effective channel H W^T for SINR / residual too.
// out[b] = {tx_power, cons_power, sum_rate, pcg, residual, zf_ok, sinr[K]}.
// ---------------------------------------------------------------------------
constexpr int kMetThreads = 128;

__device__ __forceinline__ double2 dcmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 dconj(double2 a) { return make_double2(a.x, -a.y); }

__device__ double block_sum_d(double v, double* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += scratch[q];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kMetThreads) metrics_kernel(const float2* __restrict__ H,
                                                              const float2* __restrict__ W, int K, int M,
                                                              const double* __restrict__ c, double sigma2,
                                                              double alpha, double* __restrict__ out,
                                                              float2* __restrict__ Wzf) {
  extern __shared__ __align__(16) double2 msm[];
  __shared__ double scratch[kMetThreads / 32];
  __shared__ int s_ok;
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long rid = blockIdx.x;
  const int n = K * M;
  double2* G = msm;            // K x K, G(k, j) at [j * K + k]
  double2* E = G + K * K;      // effective channel H W^T
  double2* Lc = E + K * K;     // Cholesky factor (lower)
  double2* vec = Lc + K * K;   // 2K scratch for the eigenvalue iterations
  float2* hs = reinterpret_cast<float2*>(vec + 2 * K);
  const float2* hg = H + rid * n;
  const float2* wg = W + rid * n;
  for (int e = tid; e < n; e += nt) hs[e] = hg[e];
  __syncthreads();
  for (int e = tid; e < K * K; e += nt) {
    const int k = e % K, j = e / K;
    double2 g = make_double2(0.0, 0.0), f = make_double2(0.0, 0.0);
    for (int m = 0; m < M; ++m) {
      const float2 a = hs[m * K + k], b = hs[m * K + j];
      const float2 w = wg[m * K + j];
      g.x += (double)a.x * b.x + (double)a.y * b.y;  // H(k,m) conj(H(j,m))
      g.y += (double)a.y * b.x - (double)a.x * b.y;
      f.x += (double)a.x * w.x - (double)a.y * w.y;  // H(k,m) W(j,m)
      f.y += (double)a.x * w.y + (double)a.y * w.x;
    }
    G[e] = g;
    E[e] = f;
  }
  // W statistics
  double l21w = 0.0, tx = 0.0;
  for (int m = tid; m < M; m += nt) {
    double sm = 0.0;
    for (int k = 0; k < K; ++k) {
      const float2 w = wg[m * K + k];
      sm += (double)w.x * w.x + (double)w.y * w.y;
    }
    tx += sm;
    l21w += sqrt(sm);
  }
  l21w = block_sum_d(l21w, scratch);
  tx = block_sum_d(tx, scratch);
  // Cholesky G = L L^H (thread 0; K <= 32)
  if (tid == 0) {
    int ok = 1;
    for (int j = 0; j < K && ok; ++j) {
      double d = G[j * K + j].x;
      for (int q = 0; q < j; ++q) d -= Lc[q * K + j].x * Lc[q * K + j].x + Lc[q * K + j].y * Lc[q * K + j].y;
      if (!(d > 0.0)) {
        ok = 0;
        break;
      }
      const double ljj = sqrt(d);
      Lc[j * K + j] = make_double2(ljj, 0.0);
      for (int i = j + 1; i < K; ++i) {
        double2 s2 = G[j * K + i];  // G(i, j)
        for (int q = 0; q < j; ++q) {
          const double2 t = dcmul(Lc[q * K + i], dconj(Lc[q * K + j]));
          s2.x -= t.x;
          s2.y -= t.y;
        }
        Lc[j * K + i] = make_double2(s2.x / ljj, s2.y / ljj);
      }
    }
    // Condition check of zf.cpp:17-23 (min_eig > 0, max <= 1e12 min): largest
    // eigenvalue by power iteration on G, smallest by inverse iteration with
    // the Cholesky factor; 200 iterations each (K <= 32).
    if (ok) {
      double2* x = vec;
      double2* y = vec + K;
      double lmax = 0.0, lmin_inv = 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = 0; k < K; ++k) x[k] = make_double2(1.0 + 0.1 * k, 0.05 * k);
        double lam = 0.0;
        for (int it = 0; it < 200; ++it) {
          if (pass == 0) {  // y = G x
            for (int k = 0; k < K; ++k) {
              double2 acc = make_double2(0.0, 0.0);
              for (int j = 0; j < K; ++j) {
                const double2 t = dcmul(G[j * K + k], x[j]);
                acc.x += t.x;
                acc.y += t.y;
              }
              y[k] = acc;
            }
          } else {  // y = G^{-1} x: L z = x, L^H y = z
            for (int i = 0; i < K; ++i) {
              double2 acc = x[i];
              for (int q = 0; q < i; ++q) {
                const double2 t = dcmul(Lc[q * K + i], y[q]);
                acc.x -= t.x;
                acc.y -= t.y;
              }
              y[i] = make_double2(acc.x / Lc[i * K + i].x, acc.y / Lc[i * K + i].x);
            }
            for (int i = K - 1; i >= 0; --i) {
              double2 acc = y[i];
              for (int q = i + 1; q < K; ++q) {
                const double2 t = dcmul(dconj(Lc[i * K + q]), y[q]);
                acc.x -= t.x;
                acc.y -= t.y;
              }
              y[i] = make_double2(acc.x / Lc[i * K + i].x, acc.y / Lc[i * K + i].x);
            }
          }
          double nx = 0.0, ny = 0.0, dot = 0.0;
          for (int k = 0; k < K; ++k) {
            nx += x[k].x * x[k].x + x[k].y * x[k].y;
            ny += y[k].x * y[k].x + y[k].y * y[k].y;
            dot += x[k].x * y[k].x + x[k].y * y[k].y;
          }
          lam = dot / nx;
          const double inv = 1.0 / sqrt(ny);
          for (int k = 0; k < K; ++k) x[k] = make_double2(y[k].x * inv, y[k].y * inv);
        }
        if (pass == 0)
          lmax = lam;
        else
          lmin_inv = lam;
      }
      const double lmin = lmin_inv > 0.0 ? 1.0 / lmin_inv : 0.0;
      if (!(lmin > 0.0) || lmax > 1e12 * lmin) ok = 0;  // zf.hpp:10 kSingularConditionLimit
    }
    s_ok = ok;
  }
  __syncthreads();
  const int ok = s_ok;
  // ZF columns: G x = h_m, w_zf(:, m) = diag(c) conj(x)
  double l21zf = 0.0;
  if (ok) {
    for (int m = tid; m < M; m += nt) {
      double2 z[UFPGD_MAX_USERS];
      for (int i = 0; i < K; ++i) {
        const float2 hv = hs[m * K + i];
        double2 acc = make_double2(hv.x, hv.y);
        for (int q = 0; q < i; ++q) {
          const double2 t = dcmul(Lc[q * K + i], z[q]);
          acc.x -= t.x;
          acc.y -= t.y;
        }
        z[i] = make_double2(acc.x / Lc[i * K + i].x, acc.y / Lc[i * K + i].x);
      }
      for (int i = K - 1; i >= 0; --i) {
        double2 acc = z[i];
        for (int q = i + 1; q < K; ++q) {
          const double2 t = dcmul(dconj(Lc[i * K + q]), z[q]);
          acc.x -= t.x;
          acc.y -= t.y;
        }
        z[i] = make_double2(acc.x / Lc[i * K + i].x, acc.y / Lc[i * K + i].x);
      }
      double sm = 0.0;
      for (int k = 0; k < K; ++k) {
        const double2 w = make_double2(c[k] * z[k].x, -c[k] * z[k].y);
        sm += w.x * w.x + w.y * w.y;
        if (Wzf) Wzf[rid * n + m * K + k] = make_float2((float)w.x, (float)w.y);
      }
      l21zf += sqrt(sm);
    }
  }
  l21zf = block_sum_d(l21zf, scratch);
  if (tid == 0) {
    double* o = out + rid * (6 + K);
    double rate = 0.0, res = 0.0;
    for (int k = 0; k < K; ++k) {
      const double sig = E[k * K + k].x * E[k * K + k].x + E[k * K + k].y * E[k * K + k].y;
      double row = 0.0;
      for (int j = 0; j < K; ++j) {
        const double2 e = E[j * K + k];
        row += e.x * e.x + e.y * e.y;
        const double2 r = make_double2(e.x - (j == k ? c[k] : 0.0), e.y);
        res += r.x * r.x + r.y * r.y;
      }
      const double sinr = sig / ((row - sig) + sigma2);
      o[6 + k] = sinr;
      rate += log2(1.0 + sinr);
    }
    o[0] = tx;
    o[1] = alpha * l21w;
    o[2] = rate;
    o[3] = (ok && l21w > 0.0) ? l21zf / l21w : __longlong_as_double(0x7ff8000000000000LL);
    o[4] = sqrt(res);
    o[5] = ok ? 1.0 : 0.0;
  }
}

}  // namespace

size_t metrics_smem_bytes(int K, int M) {
  return (3ull * K * K + 2ull * K) * sizeof(double2) + static_cast<size_t>(K) * M * sizeof(float2);
}

cudaError_t launch_metrics(const float2* H, const float2* W, long long B, int K, int M, const double* c,
                           double sigma2, double alpha, double* out, float2* Wzf, cudaStream_t s) {
  const size_t smem = metrics_smem_bytes(K, M);
  cudaError_t e = cudaFuncSetAttribute(metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  metrics_kernel<<<static_cast<unsigned>(B), kMetThreads, smem, s>>>(H, W, K, M, c, sigma2, alpha, out, Wzf);
  return cudaGetLastError();
}

}  // namespace ufpgd_gpu_impl
