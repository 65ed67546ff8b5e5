// General-shape FP32 / FP64 kernel (any K <= 64 within shared memory), the
// standalone power iterations (fixed-step FP32, converged FP64) and the
// deterministic statistics finaliser.
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
// General-shape kernel: one CTA per realization, H / W / V / X' in shared
// memory. Serves every (K, M) without a fused team specialisation, the
// reference's per-realization helpers (grad_f, prox_l21, pgd_step) and the
// taped forward (unfolded.cpp:127-143). Exact FP32 sqrt/div in the prox.
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T t = 0;
  for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += scratch[q];
  return t;
}

template <class V2, class T>
__device__ __forceinline__ V2 mk2(T x, T y) {
  V2 r;
  r.x = x;
  r.y = y;
  return r;
}

template <class T>
__device__ __forceinline__ T nan_of();
template <>
__device__ __forceinline__ float nan_of<float>() {
  return __int_as_float(0x7fc00000);
}
template <>
__device__ __forceinline__ double nan_of<double>() {
  return __longlong_as_double(0x7ff8000000000000LL);
}

// Generic-precision body: T = float (the general FP32 kernel) or double (the
// FP64 precision path). Plain loops; serves every shape.
template <class T>
__global__ void __launch_bounds__(kGenThreads) general_kernel_t(const __grid_constant__ GeneralArgsT<T> p) {
  using V2 = typename Vec2<T>::type;
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  __shared__ T scratch[kGenThreads / 32];
  V2* gsm = reinterpret_cast<V2*>(gsm_raw);
  const int K = p.K, M = p.M, n = K * M, tid = threadIdx.x, nt = blockDim.x;
  const long long rid = blockIdx.x;
  V2* hs = gsm;
  V2* ws = hs + n;
  V2* vs = ws + n;
  V2* xs = vs + n;
  const V2* hg = p.H + rid * n;
  for (int e = tid; e < n; e += nt) {
    const V2 h = hg[e];
    hs[e] = h;
    ws[e] = p.w0_mode == UFPGD_W0_ZERO ? mk2<V2, T>(0, 0)
            : p.w0_mode == UFPGD_W0_CONJ_H ? mk2<V2, T>(h.x, -h.y)
                                           : p.W0[rid * n + e];
  }
  __syncthreads();
  if (p.iterates)
    for (int e = tid; e < n; e += nt) p.iterates[rid * n + e] = ws[e];

  int first_bad = -1;
  long long taken = 0;
  T eta_r = 0, thr_r = 0;
  if (p.pgd) {
    eta_r = p.eta_b ? p.eta_b[rid] : T(1) / p.lip_b[rid];
    thr_r = p.lambda * eta_r;
    if (p.eta_out && tid == 0) p.eta_out[rid] = eta_r;
  }
  const long long layers = p.mode == 1 ? 1 : (p.pgd ? p.iters : p.L);
  for (long long l = 0; l < layers; ++l) {
    // stage 1: X'(k, j) = sum_m W(k, m) H(j, m) - c_k [k == j]
    for (int o = tid; o < K * K; o += nt) {
      const int k = o % K, j = o / K;
      T ar = 0, ai = 0;
      for (int m = 0; m < M; ++m) {
        const V2 a = ws[m * K + k], b = hs[m * K + j];
        ar = fma(a.x, b.x, ar);
        ar = fma(-a.y, b.y, ar);
        ai = fma(a.x, b.y, ai);
        ai = fma(a.y, b.x, ai);
      }
      if (k == j) ar -= p.c[k];
      xs[o] = mk2<V2, T>(ar, ai);
    }
    __syncthreads();
    // stage 2: G = X' H^*, V = W - eta G
    const T eta = p.pgd ? eta_r : p.eta[l], thr = p.pgd ? thr_r : p.thr[l];
    for (int e = tid; e < n; e += nt) {
      const int m = e / K, k = e % K;
      T gr = 0, gi = 0;
      for (int j = 0; j < K; ++j) {
        const V2 a = xs[j * K + k], b = hs[m * K + j];  // a * conj(b)
        gr = fma(a.x, b.x, gr);
        gr = fma(a.y, b.y, gr);
        gi = fma(a.y, b.x, gi);
        gi = fma(-a.x, b.y, gi);
      }
      if (p.mode == 1) {
        p.W[rid * n + e] = mk2<V2, T>(gr, gi);
      } else {
        vs[e] = mk2<V2, T>(fma(-eta, gr, ws[e].x), fma(-eta, gi, ws[e].y));
      }
    }
    if (p.mode == 1) return;
    __syncthreads();
    // prox per antenna (pgd.cpp:85-99, exact sqrt and division)
    T bad = 0, d2 = 0, s2 = 0;
    for (int m = tid; m < M; m += nt) {
      T s = 0;
      for (int k = 0; k < K; ++k) {
        const V2 v = vs[m * K + k];
        if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
        s = fma(v.x, v.x, fma(v.y, v.y, s));
      }
      const T nrm = sqrt(s);
      const bool on = nrm > thr;
      const T sh = on ? T(1) - thr / nrm : T(0);
      for (int k = 0; k < K; ++k) {
        const V2 v = vs[m * K + k];
        const V2 wn = on ? mk2<V2, T>(sh * v.x, sh * v.y) : mk2<V2, T>(0, 0);
        if (p.residual_tol > T(0)) {
          const V2 wo = ws[m * K + k];
          d2 += (wn.x - wo.x) * (wn.x - wo.x) + (wn.y - wo.y) * (wn.y - wo.y);
          s2 += wo.x * wo.x + wo.y * wo.y;
        }
        ws[m * K + k] = wn;
      }
      if (p.tape_norms) p.tape_norms[(l * p.B + rid) * M + m] = nrm;
      if (p.tape_shrink) p.tape_shrink[(l * p.B + rid) * M + m] = sh;
    }
    if (p.tape_v)
      for (int e = tid; e < n; e += nt) p.tape_v[(l * p.B + rid) * n + e] = vs[e];
    bad = block_sum<T>(bad, scratch);
    if (bad > T(0) && first_bad < 0) first_bad = static_cast<int>(l);
    taken = l + 1;
    if (p.iterates)
      for (int e = tid; e < n; e += nt) p.iterates[((l + 1) * p.B + rid) * n + e] = ws[e];
    // solve_pgd stops at the first non-finite step image (pgd.cpp:231-235)
    if (first_bad >= 0 && p.index_base == 1) break;
    if (p.residual_tol > T(0)) {
      d2 = block_sum<T>(d2, scratch);
      s2 = block_sum<T>(s2, scratch);
      if (sqrt(d2) / fmax(sqrt(s2), T(1e-12)) < p.residual_tol) break;
    }
    __syncthreads();
  }
  __syncthreads();
  for (int e = tid; e < n; e += nt) p.W[rid * n + e] = ws[e];
  // statistics
  T l21 = 0, act = 0;
  for (int m = tid; m < M; m += nt) {
    T s = 0;
    for (int k = 0; k < K; ++k) s = fma(ws[m * K + k].x, ws[m * K + k].x, fma(ws[m * K + k].y, ws[m * K + k].y, s));
    l21 += sqrt(s);
    act += s > T(0) ? T(1) : T(0);
  }
  l21 = block_sum<T>(l21, scratch);
  act = block_sum<T>(act, scratch);
  if (tid == 0) {
    const bool diverged = first_bad >= 0;
    if (p.diverged_at) p.diverged_at[rid] = diverged ? first_bad + p.index_base : -1;
    if (p.iterations) p.iterations[rid] = taken;
    if (p.l21) p.l21[rid] = diverged ? nan_of<T>() : l21;
    if (p.active) p.active[rid] = diverged ? -1 : static_cast<int32_t>(act);
    if (p.block_partials) {
      p.block_partials[rid * 3 + 0] = diverged ? 0.0 : static_cast<double>(p.alpha) * l21;
      p.block_partials[rid * 3 + 1] = diverged ? 0.0 : static_cast<double>(act);
      p.block_partials[rid * 3 + 2] = diverged ? 1.0 : 0.0;
    }
  }
}


// Standalone fixed-step power iteration, one warp per realization, any shape
// (H read straight from global memory; it is tiny next to the PGD loop).
__global__ void __launch_bounds__(128) power_kernel(const __grid_constant__ PowerArgs p) {
  const int lane = threadIdx.x & 31;
  const long long rid = static_cast<long long>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (rid >= p.B) return;  // warp-uniform
  const int K = p.K, M = p.M;
  const float2* h = p.H + rid * static_cast<long long>(K) * M;
  extern __shared__ float2 psm[];
  float2* v = psm + (threadIdx.x >> 5) * (M + UFPGD_MAX_USERS);
  float2* u = v + M;
  for (int m = lane; m < M; m += 32) v[m] = p.v0[m];
  __syncwarp();
  float est = 0.f;
  for (int st = 0; st < p.steps; ++st) {
    // u = H^* v
    for (int j = 0; j < K; ++j) {
      float2 acc = make_float2(0.f, 0.f);
      for (int m = lane; m < M; m += 32) {
        const float2 hv = h[m * K + j];
        cmac(acc, make_float2(hv.x, -hv.y), v[m]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(kFull, acc.x, off);
        acc.y += __shfl_xor_sync(kFull, acc.y, off);
      }
      if (lane == 0) u[j] = acc;
    }
    __syncwarp();
    float dot = 0.f, wn2 = 0.f;
    for (int m = lane; m < M; m += 32) {
      float2 acc = make_float2(0.f, 0.f);
      for (int j = 0; j < K; ++j) cmac(acc, h[m * K + j], u[j]);
      dot = fmaf(v[m].x, acc.x, fmaf(v[m].y, acc.y, dot));
      wn2 = fmaf(acc.x, acc.x, fmaf(acc.y, acc.y, wn2));
      v[m] = acc;  // unnormalised; scaled below
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dot += __shfl_xor_sync(kFull, dot, off);
      wn2 += __shfl_xor_sync(kFull, wn2, off);
    }
    if (wn2 == 0.f) {
      est = 0.f;
      break;  // warp-uniform
    }
    est = dot;
    const float inv = 1.f / sqrtf(wn2);
    __syncwarp();
    for (int m = lane; m < M; m += 32) v[m] = make_float2(v[m].x * inv, v[m].y * inv);
    __syncwarp();
  }
  if (lane == 0) p.Lout[rid] = est;
}

// FP64 power iteration with the reference's converged rule (pgd.cpp:120-169):
// relative change <= 1e-8 marks convergence, iteration continues to 1e-13 or
// the 1e4 cap; status = UFPGD_ECONVERGENCE when 1e-8 was never reached. One
// warp per realization; serves the per-channel lipschitz_bound of the C++ API.
__global__ void __launch_bounds__(128) lipschitz_exact_kernel(const double2* __restrict__ H, long long B, int K,
                                                              int M, const double2* __restrict__ v0,
                                                              double* Lout, int32_t* status) {
  extern __shared__ double2 lsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long rid = static_cast<long long>(blockIdx.x) * 4 + wid;
  if (rid >= B) return;  // warp-uniform
  double2* v = lsm + wid * (2 * M + K);
  double2* w = v + M;
  double2* u = w + M;
  const double2* h = H + rid * static_cast<long long>(K) * M;
  for (int m = lane; m < M; m += 32) v[m] = v0[m];
  __syncwarp();
  double estimate = 0.0, previous = -1.0;
  bool reached = false, zero = false;
  for (int iter = 0; iter < 10000; ++iter) {
    for (int j = 0; j < K; ++j) {  // u = H^* v
      double re = 0.0, im = 0.0;
      for (int m = lane; m < M; m += 32) {
        const double2 a = h[m * K + j], b = v[m];
        re += a.x * b.x + a.y * b.y;
        im += a.x * b.y - a.y * b.x;
      }
      for (int off = 16; off > 0; off >>= 1) {
        re += __shfl_xor_sync(kFull, re, off);
        im += __shfl_xor_sync(kFull, im, off);
      }
      if (lane == 0) u[j] = make_double2(re, im);
    }
    __syncwarp();
    double dot = 0.0, wn2 = 0.0;
    for (int m = lane; m < M; m += 32) {  // w = H^T u
      double re = 0.0, im = 0.0;
      for (int j = 0; j < K; ++j) {
        const double2 a = h[m * K + j], b = u[j];
        re += a.x * b.x - a.y * b.y;
        im += a.x * b.y + a.y * b.x;
      }
      w[m] = make_double2(re, im);
      dot += v[m].x * re + v[m].y * im;  // Re(conj(v) w)
      wn2 += re * re + im * im;
    }
    for (int off = 16; off > 0; off >>= 1) {
      dot += __shfl_xor_sync(kFull, dot, off);
      wn2 += __shfl_xor_sync(kFull, wn2, off);
    }
    estimate = dot;
    const double wn = sqrt(wn2);
    if (wn == 0.0) {
      zero = true;
      break;
    }
    __syncwarp();
    for (int m = lane; m < M; m += 32) v[m] = make_double2(w[m].x / wn, w[m].y / wn);
    __syncwarp();
    if (previous >= 0.0) {
      const double change = fabs(estimate - previous) / fmax(fabs(estimate), 1e-300);
      if (change <= 1e-8) reached = true;
      if (change <= 1e-13) break;
    }
    previous = estimate;
  }
  if (lane == 0) {
    Lout[rid] = zero ? 0.0 : estimate;
    if (status) status[rid] = (zero || reached) ? 0 : UFPGD_ECONVERGENCE;
  }
}

// Deterministic sum of per-block partials [n][3] -> stats[3].
// Small partial counts (config 1, config 2: up to 16 Ki): one 256-thread block,
// thread-strided triples, fixed tree.
__global__ void __launch_bounds__(256) stats_finalize_small_kernel(const double* __restrict__ part, long long n,
                                                                   double* __restrict__ stats) {
  __shared__ double acc[3][256];
  double s[3] = {0.0, 0.0, 0.0};
  for (long long i = threadIdx.x; i < n; i += 256)
#pragma unroll
    for (int c = 0; c < 3; ++c) s[c] += part[i * 3 + c];
#pragma unroll
  for (int c = 0; c < 3; ++c) acc[c][threadIdx.x] = s[c];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c][threadIdx.x] += acc[c][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 3) stats[threadIdx.x] = acc[threadIdx.x][0];
}

// Deterministic sum of n partial triples (block partials of the fused kernels)
// over the range [i0, i1): the triples are read as one coalesced stream of
// doubles (thread t takes doubles t, t + T, ...; double e belongs to column
// e % 3), each thread keeps one sum per column in a fixed order, then a fixed
// shared-memory tree combines the threads. Grid-wide: block b sums its range
// into out[3 b]; a single block (out = stats) finishes.
template <int kFinT>
__global__ void __launch_bounds__(kFinT) stats_finalize_kernel(const double* __restrict__ part, long long n,
                                                               long long per_block, double* __restrict__ out) {
  static_assert(kFinT % 3 == 1, "column bookkeeping: thread t's next double is in column (c + 1) % 3");
  __shared__ double acc[3][kFinT];
  const long long i0 = static_cast<long long>(blockIdx.x) * per_block;
  const long long i1 = min(n, i0 + per_block);
  double s[3] = {0.0, 0.0, 0.0};
  if (i1 > i0) {
    const double* p = part + 3 * i0;
    const long long nd = 3 * (i1 - i0);
    int c = static_cast<int>(threadIdx.x % 3);  // column of double threadIdx.x + j kFinT (kFinT % 3 == 1)
#pragma unroll 4
    for (long long e = threadIdx.x; e < nd; e += kFinT) {
      const double v = p[e];
      s[0] += c == 0 ? v : 0.0;
      s[1] += c == 1 ? v : 0.0;
      s[2] += c == 2 ? v : 0.0;
      c = c == 2 ? 0 : c + 1;
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) acc[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int w = kFinT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc[q][threadIdx.x] += acc[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 3) out[3 * blockIdx.x + threadIdx.x] = acc[threadIdx.x][0];
}

}  // namespace

size_t general_smem_bytes(int K, int M) {
  return (3ull * K * M + static_cast<size_t>(K) * K) * sizeof(float2);
}

cudaError_t launch_general(const GeneralArgs& a, cudaStream_t s) {
  const size_t smem = general_smem_bytes(a.K, a.M);
  cudaError_t e = cudaFuncSetAttribute(general_kernel_t<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  general_kernel_t<float><<<static_cast<unsigned>(a.B), kGenThreads, smem, s>>>(a);
  return cudaGetLastError();
}

size_t general64_smem_bytes(int K, int M) {
  return (3ull * K * M + static_cast<size_t>(K) * K) * sizeof(double2);
}

cudaError_t launch_general64(const GeneralArgs64& a, cudaStream_t s) {
  if (pgd64_team_supported(a)) return launch_pgd64_team(a, s);
  const size_t smem = general64_smem_bytes(a.K, a.M);
  cudaError_t e = cudaFuncSetAttribute(general_kernel_t<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  general_kernel_t<double><<<static_cast<unsigned>(a.B), kGenThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_power(const PowerArgs& a, cudaStream_t s) {
  const size_t smem = 4 * (a.M + UFPGD_MAX_USERS) * sizeof(float2);
  cudaError_t e = cudaFuncSetAttribute(power_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  power_kernel<<<static_cast<unsigned>((a.B + 3) / 4), 128, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lipschitz_exact(const double2* H, long long B, int K, int M, const double2* v0, double* Lout,
                                   int32_t* status, cudaStream_t s) {
  const size_t smem = 4 * (2 * M + K) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(lipschitz_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  lipschitz_exact_kernel<<<static_cast<unsigned>((B + 3) / 4), 128, smem, s>>>(H, B, K, M, v0, Lout, status);
  return cudaGetLastError();
}

namespace {
__global__ void fill_i64_kernel(int64_t* p, long long n, int64_t v) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) p[i] = v;
}
}  // namespace

cudaError_t launch_fill_i64(int64_t* p, long long n, int64_t value, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  fill_i64_kernel<<<static_cast<unsigned>(std::min<long long>((n + 255) / 256, 1024)), 256, 0, s>>>(p, n, value);
  return cudaGetLastError();
}

cudaError_t launch_stats_finalize(const double* partials, long long n, double* stats, cudaStream_t s) {
  // Up to 64 Ki partials (config 2: 8,192 blocks): one block. Beyond (the
  // tcgen05 kernel writes one triple per realization: 2^20 at config 5), a
  // first pass of up to 296 blocks over contiguous ranges, then one block over
  // their sums — the order of every addition is fixed, so the result is
  // deterministic and independent of scheduling.
  // Small n: the 256-thread strided kernel (its latency is lowest at config 1).
  constexpr long long kOneBlock = 1LL << 16;
  if (n <= 16384) {
    stats_finalize_small_kernel<<<1, 256, 0, s>>>(partials, n, stats);
    return cudaGetLastError();
  }
  if (n <= kOneBlock) {
    stats_finalize_kernel<1024><<<1, 1024, 0, s>>>(partials, n, n, stats);
    return cudaGetLastError();
  }
  const long long G = std::min<long long>(296, (n + kOneBlock / 8 - 1) / (kOneBlock / 8));
  const long long per = (n + G - 1) / G;
  double* mid = nullptr;
  cudaError_t e = scratch_alloc_async(reinterpret_cast<void**>(&mid), sizeof(double) * 3 * G, s);
  if (e != cudaSuccess) return e;
  stats_finalize_kernel<1024><<<static_cast<unsigned>(G), 1024, 0, s>>>(partials, n, per, mid);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    stats_finalize_kernel<256><<<1, 256, 0, s>>>(mid, G, G, stats);
    e = cudaGetLastError();
  }
  cudaFreeAsync(mid, s);
  return e;
}

}  // namespace ufpgd_gpu_impl
