// Training-step gradients: taped forward, loss, reverse sweep, batch mean —
// in FP32 (the batched training path) and FP64 (the reference's precision, for
// the per-channel backward() of the C++ API).
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <algorithm>

#include "device_common.cuh"

namespace ufpgd_gpu_impl {
namespace {

// acc += a * b and acc += a * conj(b) for float2 / double2.
template <class V2>
__device__ __forceinline__ void cmac_t(V2& acc, V2 a, V2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
template <class V2>
__device__ __forceinline__ void cmac_conj_t(V2& acc, V2 a, V2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
}

// ---------------------------------------------------------------------------
// Training-step gradients: the per-sample body of train's
// parallel_for (training.cpp:205-234) — taped forward (unfolded.cpp:83-146),
// loss and loss gradient (training.cpp:59-95), reverse sweep (backward,
// unfolded.cpp:158-239) — one CTA per realization, any shape the general
// kernel takes. The tape (layer inputs and step images) goes to a global
// workspace; a mini-batch of 64 (8,64) realizations is 10 MB in FP32,
// L2-resident. loss_kind 2 takes the output gradient dC/dW as an input (the
// reference's backward(tape, net, channel, cfg, dcost_dw)); the tape is then
// the forward recomputed on the device from the same start point.
// out_loss[b], out_grads[b][2L] = (d_lambda_0, d_eta_0, d_lambda_1, ...).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kGenThreads) grad_kernel_t(const __grid_constant__ GradArgsT<T> p) {
  using V2 = typename Vec2<T>::type;
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  __shared__ double dscratch[kGenThreads / 32];
  const int K = p.K, M = p.M, n = K * M, tid = threadIdx.x, nt = blockDim.x, L = p.L;
  const long long rid = blockIdx.x;
  V2* hs = reinterpret_cast<V2*>(gsm_raw);
  V2* ws = hs + n;
  V2* vs = ws + n;
  V2* xs = vs + n;
  T* ns = reinterpret_cast<T*>(xs + K * K);  // column norms (M)
  V2* tin = p.tape + rid * 2LL * L * n;
  V2* tv = tin + static_cast<long long>(L) * n;
  const V2* hg = p.H + rid * n;
  const V2 zero{T(0), T(0)};
  for (int e = tid; e < n; e += nt) {
    const V2 h = hg[e];
    hs[e] = h;
    ws[e] = p.w0_mode == UFPGD_W0_ZERO    ? zero
            : p.w0_mode == UFPGD_W0_GIVEN ? p.W0[rid * n + e]
                                          : V2{h.x, -h.y};
  }
  __syncthreads();
  // stage 1 into xs: X'(k, j) = sum_m A(k, m) H(j, m) - csub * c_k [k == j]
  auto stage1 = [&](const V2* A, T csub) {
    for (int o = tid; o < K * K; o += nt) {
      const int k = o % K, j = o / K;
      V2 acc = zero;
      for (int m = 0; m < M; ++m) cmac_t(acc, A[m * K + k], hs[m * K + j]);
      if (k == j) acc.x -= csub * p.c[k];
      xs[o] = acc;
    }
  };
  // G(k, m) = sum_j X'(k, j) conj(H(j, m))
  auto stage2 = [&](int e) {
    const int m = e / K, k = e % K;
    V2 g = zero;
    for (int j = 0; j < K; ++j) cmac_conj_t(g, xs[j * K + k], hs[m * K + j]);
    return g;
  };
  // ---- taped forward ----
  for (int l = 0; l < L; ++l) {
    stage1(ws, T(1));
    __syncthreads();
    const T eta = p.eta[l], thr = p.thr[l];
    for (int e = tid; e < n; e += nt) {
      const V2 g = stage2(e);
      const V2 v{fma(-eta, g.x, ws[e].x), fma(-eta, g.y, ws[e].y)};
      vs[e] = v;
      tin[static_cast<long long>(l) * n + e] = ws[e];
      tv[static_cast<long long>(l) * n + e] = v;
    }
    __syncthreads();
    for (int m = tid; m < M; m += nt) {
      T sq = 0;
      for (int k = 0; k < K; ++k) sq = fma(vs[m * K + k].x, vs[m * K + k].x, fma(vs[m * K + k].y, vs[m * K + k].y, sq));
      const T nrm = sqrt(sq);
      const T sh = nrm > thr ? T(1) - thr / nrm : T(0);
      for (int k = 0; k < K; ++k) ws[m * K + k] = nrm > thr ? V2{sh * vs[m * K + k].x, sh * vs[m * K + k].y} : zero;
    }
    __syncthreads();
  }
  // ---- loss and dC/dW into vs ----
  double loss = 0.0;
  if (p.loss_kind == 2) {
    const V2* dc = p.dcost + rid * n;
    for (int e = tid; e < n; e += nt) vs[e] = dc[e];
  } else if (p.loss_kind == 1) {
    const V2* lab = p.labels + rid * n;
    for (int e = tid; e < n; e += nt) {
      const V2 d{ws[e].x - lab[e].x, ws[e].y - lab[e].y};
      loss += static_cast<double>(d.x) * d.x + static_cast<double>(d.y) * d.y;
      vs[e] = V2{T(2) * d.x, T(2) * d.y};
    }
  } else {
    stage1(ws, T(1));  // X' of the output: residual and grad_f
    __syncthreads();
    for (int o = tid; o < K * K; o += nt) loss += static_cast<double>(xs[o].x) * xs[o].x + static_cast<double>(xs[o].y) * xs[o].y;
    for (int m = tid; m < M; m += nt) {
      T sq = 0;
      for (int k = 0; k < K; ++k) sq = fma(ws[m * K + k].x, ws[m * K + k].x, fma(ws[m * K + k].y, ws[m * K + k].y, sq));
      ns[m] = sqrt(sq);
      loss += static_cast<double>(p.lambda_cost) * ns[m];
    }
    __syncthreads();
    for (int e = tid; e < n; e += nt) {
      const int m = e / K;
      const V2 g = stage2(e);
      V2 d{T(2) * g.x, T(2) * g.y};
      if (ns[m] > T(0)) {
        const T f = p.lambda_cost / ns[m];
        d.x = fma(f, ws[e].x, d.x);
        d.y = fma(f, ws[e].y, d.y);
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
    const T eta = p.eta[idx], thr = p.thr[idx];
    const V2* Vt = tv + static_cast<long long>(idx) * n;
    const V2* Wt = tin + static_cast<long long>(idx) * n;
    double d_t = 0.0, d_dir = 0.0;
    for (int m = tid; m < M; m += nt) {
      T sq = 0, inner = 0;
      for (int k = 0; k < K; ++k) {
        const V2 v = Vt[m * K + k], g = ws[m * K + k];
        sq = fma(v.x, v.x, fma(v.y, v.y, sq));
        inner = fma(v.x, g.x, fma(v.y, g.y, inner));  // Re(conj(v) g)
      }
      const T nrm = sqrt(sq);
      if (nrm > thr) {
        const T sh = T(1) - thr / nrm;
        const T f = thr / (nrm * nrm * nrm) * inner;
        d_t -= static_cast<double>(inner) / nrm;
        for (int k = 0; k < K; ++k) {
          const V2 v = Vt[m * K + k], g = ws[m * K + k];
          vs[m * K + k] = V2{fma(f, v.x, sh * g.x), fma(f, v.y, sh * g.y)};
        }
      } else {
        for (int k = 0; k < K; ++k) vs[m * K + k] = zero;
      }
    }
    __syncthreads();
    for (int e = tid; e < n; e += nt) {
      const V2 gi = vs[e], w = Wt[e], v = Vt[e];
      // Re(conj(gimg) (Win - V))
      d_dir -= (static_cast<double>(gi.x) * (w.x - v.x) + static_cast<double>(gi.y) * (w.y - v.y)) / eta;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      d_t += __shfl_xor_sync(kFull, d_t, off);
      d_dir += __shfl_xor_sync(kFull, d_dir, off);
    }
    if ((tid & 31) == 0) dscratch[tid >> 5] = d_t;
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
    stage1(vs, T(0));
    __syncthreads();
    for (int e = tid; e < n; e += nt) {
      const V2 g = stage2(e);
      ws[e] = V2{fma(-eta, g.x, vs[e].x), fma(-eta, g.y, vs[e].y)};
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

template <class T>
size_t grad_smem_t(int K, int M) {
  using V2 = typename Vec2<T>::type;
  return (3ull * K * M + static_cast<size_t>(K) * K) * sizeof(V2) + static_cast<size_t>(M) * sizeof(T);
}

template <class T>
cudaError_t launch_grad_t(const GradArgsT<T>& a, double* mean, cudaStream_t s) {
  const size_t smem = grad_smem_t<T>(a.K, a.M);
  cudaError_t e = cudaFuncSetAttribute(grad_kernel_t<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  grad_kernel_t<T><<<static_cast<unsigned>(a.B), kGenThreads, smem, s>>>(a);
  e = cudaGetLastError();
  if (e == cudaSuccess && mean) {
    row_mean_kernel<<<1, 128, 0, s>>>(a.out_loss, a.out_grads, a.B, 2 * a.L, mean);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace

size_t grad_smem_bytes(int K, int M) { return grad_smem_t<float>(K, M); }
size_t grad64_smem_bytes(int K, int M) { return grad_smem_t<double>(K, M); }
cudaError_t launch_grad(const GradArgs& a, double* mean, cudaStream_t s) { return launch_grad_t<float>(a, mean, s); }
cudaError_t launch_grad64(const GradArgs64& a, double* mean, cudaStream_t s) { return launch_grad_t<double>(a, mean, s); }

}  // namespace ufpgd_gpu_impl
