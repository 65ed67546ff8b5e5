// Training-step gradients: taped forward, loss, reverse sweep, batch mean.
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
// Training-step gradients: the per-sample body of train's
// parallel_for (training.cpp:205-234) — taped forward (unfolded.cpp:83-146),
// loss and loss gradient (training.cpp:59-95), reverse sweep (backward,
// unfolded.cpp:158-239) — one CTA per realization, any shape the general
// kernel takes. The tape (layer inputs and step images, FP32) goes to a global
// workspace; a mini-batch of 64 (8,64) realizations is 10 MB, L2-resident.
// out_loss[b], out_grads[b][2L] = (d_lambda_0, d_eta_0, d_lambda_1, ...).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kGenThreads) grad_kernel(const __grid_constant__ GradArgs p) {
  extern __shared__ __align__(16) float2 gsm2[];
  __shared__ double dscratch[kGenThreads / 32];
  const int K = p.K, M = p.M, n = K * M, tid = threadIdx.x, nt = blockDim.x, L = p.L;
  const long long rid = blockIdx.x;
  float2* hs = gsm2;
  float2* ws = hs + n;
  float2* vs = ws + n;
  float2* xs = vs + n;
  float* ns = reinterpret_cast<float*>(xs + K * K);  // column norms (M)
  float2* tin = p.tape + rid * 2LL * L * n;
  float2* tv = tin + static_cast<long long>(L) * n;
  const float2* hg = p.H + rid * n;
  for (int e = tid; e < n; e += nt) {
    const float2 h = hg[e];
    hs[e] = h;
    ws[e] = p.w0_mode == UFPGD_W0_ZERO ? make_float2(0.f, 0.f) : make_float2(h.x, -h.y);
  }
  __syncthreads();
  // stage 1 into xs: X'(k, j) = sum_m A(k, m) H(j, m) - csub * c_k [k == j]
  auto stage1 = [&](const float2* A, float csub) {
    for (int o = tid; o < K * K; o += nt) {
      const int k = o % K, j = o / K;
      float2 acc = make_float2(0.f, 0.f);
      for (int m = 0; m < M; ++m) cmac(acc, A[m * K + k], hs[m * K + j]);
      if (k == j) acc.x -= csub * p.c[k];
      xs[o] = acc;
    }
  };
  // G(k, m) = sum_j X'(k, j) conj(H(j, m))
  auto stage2 = [&](int e) {
    const int m = e / K, k = e % K;
    float2 g = make_float2(0.f, 0.f);
    for (int j = 0; j < K; ++j) cmac_conj(g, xs[j * K + k], hs[m * K + j]);
    return g;
  };
  // ---- taped forward ----
  for (int l = 0; l < L; ++l) {
    stage1(ws, 1.f);
    __syncthreads();
    const float eta = p.eta[l], thr = p.thr[l];
    for (int e = tid; e < n; e += nt) {
      const float2 g = stage2(e);
      const float2 v = make_float2(fmaf(-eta, g.x, ws[e].x), fmaf(-eta, g.y, ws[e].y));
      vs[e] = v;
      tin[static_cast<long long>(l) * n + e] = ws[e];
      tv[static_cast<long long>(l) * n + e] = v;
    }
    __syncthreads();
    for (int m = tid; m < M; m += nt) {
      float sq = 0.f;
      for (int k = 0; k < K; ++k) sq = fmaf(vs[m * K + k].x, vs[m * K + k].x, fmaf(vs[m * K + k].y, vs[m * K + k].y, sq));
      const float nrm = sqrtf(sq);
      const float sh = nrm > thr ? 1.f - thr / nrm : 0.f;
      for (int k = 0; k < K; ++k) ws[m * K + k] = nrm > thr ? make_float2(sh * vs[m * K + k].x, sh * vs[m * K + k].y)
                                                              : make_float2(0.f, 0.f);
    }
    __syncthreads();
  }
  // ---- loss and dC/dW into vs ----
  double loss = 0.0;
  if (p.loss_kind == 1) {
    const float2* lab = p.labels + rid * n;
    for (int e = tid; e < n; e += nt) {
      const float2 d = make_float2(ws[e].x - lab[e].x, ws[e].y - lab[e].y);
      loss += static_cast<double>(d.x) * d.x + static_cast<double>(d.y) * d.y;
      vs[e] = make_float2(2.f * d.x, 2.f * d.y);
    }
  } else {
    stage1(ws, 1.f);  // X' of the output: residual and grad_f
    __syncthreads();
    for (int o = tid; o < K * K; o += nt) loss += static_cast<double>(xs[o].x) * xs[o].x + static_cast<double>(xs[o].y) * xs[o].y;
    for (int m = tid; m < M; m += nt) {
      float sq = 0.f;
      for (int k = 0; k < K; ++k) sq = fmaf(ws[m * K + k].x, ws[m * K + k].x, fmaf(ws[m * K + k].y, ws[m * K + k].y, sq));
      ns[m] = sqrtf(sq);
      loss += static_cast<double>(p.lambda_cost) * ns[m];
    }
    __syncthreads();
    for (int e = tid; e < n; e += nt) {
      const int m = e / K;
      const float2 g = stage2(e);
      float2 d = make_float2(2.f * g.x, 2.f * g.y);
      if (ns[m] > 0.f) {
        const float f = p.lambda_cost / ns[m];
        d.x = fmaf(f, ws[e].x, d.x);
        d.y = fmaf(f, ws[e].y, d.y);
      }
      vs[e] = d;
    }
  }
  // block sum of the loss (double)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) loss += __shfl_xor_sync(kFull, loss, off);
  __syncthreads();
  if ((tid & 31) == 0) dscratch[tid >> 5] = loss;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < nt / 32; ++q) t += dscratch[q];
    p.out_loss[rid] = t;
  }
  __syncthreads();
  for (int e = tid; e < n; e += nt) ws[e] = vs[e];  // g = dC/dW
  __syncthreads();
  // ---- reverse sweep ----
  for (int idx = L - 1; idx >= 0; --idx) {
    const float eta = p.eta[idx], thr = p.thr[idx];
    const float2* Vt = tv + static_cast<long long>(idx) * n;
    const float2* Wt = tin + static_cast<long long>(idx) * n;
    double d_t = 0.0, d_dir = 0.0;
    for (int m = tid; m < M; m += nt) {
      float sq = 0.f, inner = 0.f;
      for (int k = 0; k < K; ++k) {
        const float2 v = Vt[m * K + k], g = ws[m * K + k];
        sq = fmaf(v.x, v.x, fmaf(v.y, v.y, sq));
        inner = fmaf(v.x, g.x, fmaf(v.y, g.y, inner));  // Re(conj(v) g)
      }
      const float nrm = sqrtf(sq);
      if (nrm > thr) {
        const float sh = 1.f - thr / nrm;
        const float f = thr / (nrm * nrm * nrm) * inner;
        d_t -= static_cast<double>(inner) / nrm;
        for (int k = 0; k < K; ++k) {
          const float2 v = Vt[m * K + k], g = ws[m * K + k];
          vs[m * K + k] = make_float2(fmaf(f, v.x, sh * g.x), fmaf(f, v.y, sh * g.y));
        }
      } else {
        for (int k = 0; k < K; ++k) vs[m * K + k] = make_float2(0.f, 0.f);
      }
    }
    __syncthreads();
    for (int e = tid; e < n; e += nt) {
      const float2 gi = vs[e], w = Wt[e], v = Vt[e];
      // Re(conj(gimg) (Win - V))
      d_dir -= (static_cast<double>(gi.x) * (w.x - v.x) + static_cast<double>(gi.y) * (w.y - v.y)) / eta;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      d_t += __shfl_xor_sync(kFull, d_t, off);
      d_dir += __shfl_xor_sync(kFull, d_dir, off);
    }
    if ((tid & 31) == 0) {
      dscratch[tid >> 5] = d_t;
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < nt / 32; ++q) t += dscratch[q];
      d_t = t;
    }
    __syncthreads();
    if ((tid & 31) == 0) dscratch[tid >> 5] = d_dir;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < nt / 32; ++q) t += dscratch[q];
      const double lam = p.lam[idx], et = p.eta64[idx];
      p.out_grads[rid * 2LL * L + 2 * idx] = et * d_t;
      p.out_grads[rid * 2LL * L + 2 * idx + 1] = lam * d_t + t;
    }
    // g = gimg - eta (gimg H^T) H^*
    stage1(vs, 0.f);
    __syncthreads();
    for (int e = tid; e < n; e += nt) {
      const float2 g = stage2(e);
      ws[e] = make_float2(fmaf(-eta, g.x, vs[e].x), fmaf(-eta, g.y, vs[e].y));
    }
    __syncthreads();
  }
}

// Deterministic batch mean of [loss, grads...] rows: out[c] = sum_b rows[b][c] / B.
__global__ void __launch_bounds__(128) row_mean_kernel(const double* __restrict__ loss,
                                                       const double* __restrict__ grads, long long B, int G,
                                                       double* __restrict__ out) {
  for (int col = threadIdx.x; col <= G; col += blockDim.x) {
    double s = 0.0;
    for (long long b = 0; b < B; ++b) s += col == 0 ? loss[b] : grads[b * G + col - 1];
    out[col] = B > 0 ? s / static_cast<double>(B) : 0.0;
  }
}

}  // namespace

size_t grad_smem_bytes(int K, int M) {
  return (3ull * K * M + static_cast<size_t>(K) * K) * sizeof(float2) + static_cast<size_t>(M) * sizeof(float);
}

cudaError_t launch_grad(const GradArgs& a, double* mean, cudaStream_t s) {
  const size_t smem = grad_smem_bytes(a.K, a.M);
  cudaError_t e = cudaFuncSetAttribute(grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  grad_kernel<<<static_cast<unsigned>(a.B), kGenThreads, smem, s>>>(a);
  e = cudaGetLastError();
  if (e == cudaSuccess && mean) {
    row_mean_kernel<<<1, 128, 0, s>>>(a.out_loss, a.out_grads, a.B, 2 * a.L, mean);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace ufpgd_gpu_impl
