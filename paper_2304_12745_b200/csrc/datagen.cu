// On-device seeded channel generation and UFPD layout conversion.
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
// On-device seeded channel generation. Realization
// i = first_index + b is the reference's generate_channel(cfg,
// Rng::stream(seed_h, i)) (channel.cpp:7-16, rng.cpp:19-40): a 64-bit
// Mersenne Twister (std::mt19937_64, fully specified by the C++ standard)
// seeded with splitmix(seed ^ splitmix(i)), drawn k-outer / m-inner, each
// complex entry Box-Muller from (uniform_open, uniform). One warp owns one
// realization at a time: lane 0 runs the 312-step (inherently sequential)
// seeding, the twist is split into its two data-parallel halves across the
// lanes, and tempering + the FP64 transforms run one complex entry per lane.
// The integer stream is bit-identical to the host's; log / sincos / pow are
// CUDA's FP64 routines (a few ulp from glibc), so FP64 entries agree to
// ~1e-15 relative and the complex64 rounding almost always bit-for-bit.
// ---------------------------------------------------------------------------
namespace mt {
constexpr int N = 312, MID = 156;
constexpr unsigned long long A = 0xB5026F5AA96619E9ULL, F = 6364136223846793005ULL;
constexpr unsigned long long UPPER = ~0ULL << 31, LOWER = (1ULL << 31) - 1;

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {  // rng.cpp:10-15
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ unsigned long long temper(unsigned long long y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  return y ^ (y >> 43);
}

__device__ __forceinline__ double uniform(unsigned long long y) { return static_cast<double>(temper(y) >> 11) * 0x1.0p-53; }
__device__ __forceinline__ double uniform_open(unsigned long long y) {
  return static_cast<double>((temper(y) >> 11) + 1) * 0x1.0p-53;
}

// Rng::stream(seed, index) state into x[0..N).
__device__ __forceinline__ void seed_stream(unsigned long long* x, unsigned long long seed, unsigned long long index,
                                            int lane) {
  if (lane == 0) {
    unsigned long long v = mix64(seed ^ mix64(index));
    x[0] = v;
    for (int i = 1; i < N; ++i) {
      v = F * (v ^ (v >> 62)) + static_cast<unsigned long long>(i);
      x[i] = v;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ unsigned long long twist1(unsigned long long cur, unsigned long long next,
                                                     unsigned long long far) {
  const unsigned long long y = (cur & UPPER) | (next & LOWER);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}

// One full regeneration of the N-word state. Words [0, MID) read only old
// words; words [MID, N) read the new words k - MID (and word N-1 the new
// word 0). Within a half, each 32-word round reads before it writes, and the
// only word a round reads that a later round writes is the next round's
// first, so one __syncwarp between read and write suffices.
__device__ __forceinline__ void twist(unsigned long long* x, int lane) {
#pragma unroll 1
  for (int k0 = 0; k0 < MID; k0 += 32) {
    const int k = k0 + lane;
    unsigned long long v = 0;
    if (k < MID) v = twist1(x[k], x[k + 1], x[k + MID]);
    __syncwarp();
    if (k < MID) x[k] = v;
    __syncwarp();
  }
#pragma unroll 1
  for (int k0 = MID; k0 < N; k0 += 32) {
    const int k = k0 + lane;
    unsigned long long v = 0;
    if (k < N) v = twist1(x[k], x[k + 1 == N ? 0 : k + 1], x[k - MID]);
    __syncwarp();
    if (k < N) x[k] = v;
    __syncwarp();
  }
}
}  // namespace mt

template <class OUT>
__device__ __forceinline__ void store_entry(OUT* H, long long off, double re, double im);
template <>
__device__ __forceinline__ void store_entry<float2>(float2* H, long long off, double re, double im) {
  H[off] = make_float2(static_cast<float>(re), static_cast<float>(im));
}
template <>
__device__ __forceinline__ void store_entry<double2>(double2* H, long long off, double re, double im) {
  H[off] = make_double2(re, im);
}

constexpr int kGenWarps = 8;

template <class OUT>
__global__ void __launch_bounds__(kGenWarps * 32) channel_gen_kernel(unsigned long long seed_h, unsigned long long seed_g,
                                                                     double gain_range_db, long long first_index,
                                                                     long long B, int K, int M, OUT* __restrict__ H) {
  __shared__ unsigned long long state[kGenWarps][mt::N];
  __shared__ double gain[kGenWarps][UFPGD_MAX_USERS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* x = state[warp];
  double* g = gain[warp];
  const long long KM = static_cast<long long>(K) * M;
  const double two_pi = 2.0 * 3.14159265358979323846;  // 2 * std::numbers::pi, exact doubling
  for (long long b = static_cast<long long>(blockIdx.x) * kGenWarps + warp; b < B;
       b += static_cast<long long>(gridDim.x) * kGenWarps) {
    const unsigned long long idx = static_cast<unsigned long long>(first_index + b);
    if (gain_range_db > 0.0) {  // per-user large-scale gain from its own stream (K <= MAX_USERS < N)
      mt::seed_stream(x, seed_g, idx, lane);
      mt::twist(x, lane);
      for (int k = lane; k < K; k += 32) g[k] = pow(10.0, -mt::uniform(x[k]) * gain_range_db / 20.0);
    } else {
      for (int k = lane; k < K; k += 32) g[k] = 1.0;
    }
    __syncwarp();  // gain draws read x before lane 0 reseeds it
    mt::seed_stream(x, seed_h, idx, lane);
    OUT* Hb = H + b * KM;
    for (long long t0 = 0; t0 < KM; t0 += mt::N / 2) {  // N / 2 complex entries per regeneration
      mt::twist(x, lane);
      const int cnt = static_cast<int>(KM - t0 < mt::N / 2 ? KM - t0 : mt::N / 2);
      for (int tl = lane; tl < cnt; tl += 32) {
        const double radius = sqrt(-log(mt::uniform_open(x[2 * tl])));  // rng.cpp:35-40
        const double angle = two_pi * mt::uniform(x[2 * tl + 1]);
        double sn, cs;
        sincos(angle, &sn, &cs);
        const long long t = t0 + tl;
        const int k = static_cast<int>(t / M), m = static_cast<int>(t % M);
        store_entry(Hb, static_cast<long long>(m) * K + k, radius * cs * g[k], radius * sn * g[k]);
      }
      __syncwarp();
    }
  }
}


// ---------------------------------------------------------------------------
// Dataset layout conversion: the reference's UFPD payload
// stores each K x M matrix row-major with interleaved f64 (re, im)
// (dataset.cpp:38-45, dataset.hpp:28-33); the device batches are complex64
// [B][M][K]. One CTA per realization transposes through shared memory so both
// the f64 reads (along m) and the c64 writes (along k) are coalesced. Pure
// HBM traffic: 16KM bytes in, 8KM out (or the reverse for the writer).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) f64_rowmajor_to_c64_kernel(const double2* __restrict__ src, float2* __restrict__ dst,
                                                                  int K, int M) {
  extern __shared__ float2 tsm[];  // [K][M + 1]
  const long long r = blockIdx.x;
  const double2* s = src + r * K * M;
  float2* d = dst + r * K * M;
  for (int e = threadIdx.x; e < K * M; e += blockDim.x) {
    const int k = e / M, m = e % M;
    const double2 v = s[e];
    tsm[k * (M + 1) + m] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * M; e += blockDim.x) {
    const int m = e / K, k = e % K;
    d[e] = tsm[k * (M + 1) + m];
  }
}

__global__ void __launch_bounds__(256) c64_to_f64_rowmajor_kernel(const float2* __restrict__ src, double2* __restrict__ dst,
                                                                  int K, int M) {
  extern __shared__ float2 tsm[];  // [M][K + 1]
  const long long r = blockIdx.x;
  const float2* s = src + r * K * M;
  double2* d = dst + r * K * M;
  for (int e = threadIdx.x; e < K * M; e += blockDim.x) {
    const int m = e / K, k = e % K;
    tsm[m * (K + 1) + k] = s[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * M; e += blockDim.x) {
    const int k = e / M, m = e % M;
    const float2 v = tsm[m * (K + 1) + k];
    d[e] = make_double2(v.x, v.y);
  }
}

// Zero-padding repack between [B][Ms][Ks] and [B][Md][Kd] complex64 batches:
// dst(b, m, k) = src(b, m, k) inside the source shape, 0 outside. Pads a
// batch up to a fused-kernel shape and crops the result back. Blocks stride
// over realizations, threads over a realization's destination elements
// (coalesced stores, 32-bit index arithmetic).
__global__ void __launch_bounds__(256) repack_c64_kernel(const float2* __restrict__ src, float2* __restrict__ dst,
                                                         long long B, int Ms, int Ks, int Md, int Kd) {
  const int per = Md * Kd;
  for (long long b = blockIdx.x; b < B; b += gridDim.x) {
    const float2* sb = src + b * Ms * Ks;
    float2* db = dst + b * per;
    for (int r = threadIdx.x; r < per; r += 256) {
      const int m = r / Kd, k = r - m * Kd;
      db[r] = (m < Ms && k < Ks) ? sb[m * Ks + k] : make_float2(0.f, 0.f);
    }
  }
}

}  // namespace

cudaError_t launch_repack_c64(const float2* src, int Ms, int Ks, float2* dst, int Md, int Kd, long long B,
                              cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(B < 16LL * sms ? B : 16LL * sms);
  repack_c64_kernel<<<grid, 256, 0, s>>>(src, dst, B, Ms, Ks, Md, Kd);
  return cudaGetLastError();
}

cudaError_t launch_channel_gen(unsigned long long seed_h, unsigned long long seed_g, double gain_range_db,
                               long long first_index, long long B, int K, int M, void* H, bool f64, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long need = (B + kGenWarps - 1) / kGenWarps;
  const unsigned grid = static_cast<unsigned>(need < 8LL * sms ? need : 8LL * sms);
  if (f64)
    channel_gen_kernel<double2><<<grid, kGenWarps * 32, 0, s>>>(seed_h, seed_g, gain_range_db, first_index, B, K, M,
                                                                static_cast<double2*>(H));
  else
    channel_gen_kernel<float2><<<grid, kGenWarps * 32, 0, s>>>(seed_h, seed_g, gain_range_db, first_index, B, K, M,
                                                               static_cast<float2*>(H));
  return cudaGetLastError();
}

cudaError_t launch_convert(const void* src, void* dst, long long B, int K, int M, bool to_c64, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(K + 1) * (M + 1) * sizeof(float2);
  if (to_c64) {
    cudaError_t e = cudaFuncSetAttribute(f64_rowmajor_to_c64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    f64_rowmajor_to_c64_kernel<<<static_cast<unsigned>(B), 256, smem, s>>>(static_cast<const double2*>(src),
                                                                            static_cast<float2*>(dst), K, M);
  } else {
    cudaError_t e = cudaFuncSetAttribute(c64_to_f64_rowmajor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    c64_to_f64_rowmajor_kernel<<<static_cast<unsigned>(B), 256, smem, s>>>(static_cast<const float2*>(src),
                                                                            static_cast<double2*>(dst), K, M);
  }
  return cudaGetLastError();
}

}  // namespace ufpgd_gpu_impl
