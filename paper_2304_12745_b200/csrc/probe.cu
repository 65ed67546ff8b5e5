// FP32 FFMA2 throughput probe (the roofline denominator of bench.py).
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <algorithm>

#include "device_common.cuh"

namespace ufpgd_gpu_impl {
namespace {

// FP32 roofline probe: independent FFMA2 outer-product chains (the fused
// kernel's instruction form, scalar broadcast operand) with the SM clock read
// in-kernel (clock64 vs %globaltimer). Used by bench.py for the measured FP32
// FMA denominator; MEASURED_PEAKS.json has no FP32 figure.
__global__ void __launch_bounds__(256) fp32_peak_kernel(const float* __restrict__ in, float* out, int iters,
                                                       unsigned long long* clk) {
  float2 b[4], acc[16];
  float a[4];
  for (int i = 0; i < 4; ++i) {
    a[i] = in[(threadIdx.x + i) & 255];
    b[i] = make_float2(in[(threadIdx.x + 32 + i) & 255], in[(threadIdx.x + 64 + i) & 255]);
  }
  for (int i = 0; i < 16; ++i) acc[i] = make_float2(in[(threadIdx.x + 96 + i) & 255], 0.f);
  unsigned long long c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i * 4 + j] = ffma2(a[i], b[j], acc[i * 4 + j]);
  }
  unsigned long long c1 = clock64(), t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  float sacc = 0.f;
  for (int i = 0; i < 16; ++i) sacc += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = sacc;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    clk[0] = c1 - c0;
    clk[1] = t1 - t0;
  }
}

}  // namespace

cudaError_t measure_fp32_peak(double* tflops, double* sm_ghz) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float *in = nullptr, *out = nullptr;
  unsigned long long* clk = nullptr;
  const int blocks = sms * 8, tpb = 256, iters = 8192;
  cudaError_t e = cudaMalloc(&in, 256 * sizeof(float));
  if (e == cudaSuccess) e = cudaMemset(in, 0, 256 * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&out, sizeof(float) * blocks * tpb);
  if (e == cudaSuccess) e = cudaMalloc(&clk, 2 * sizeof(unsigned long long));
  cudaEvent_t a = nullptr, b = nullptr;
  if (e == cudaSuccess) e = cudaEventCreate(&a);
  if (e == cudaSuccess) e = cudaEventCreate(&b);
  float best_ms = 1e30f;
  unsigned long long h[2] = {1, 1};
  for (int rep = 0; rep < 3 && e == cudaSuccess; ++rep) {
    fp32_peak_kernel<<<blocks, tpb>>>(in, out, rep == 0 ? 64 : iters, clk);
    if (rep == 0) {
      e = cudaDeviceSynchronize();
      continue;
    }
    cudaEventRecord(a);
    fp32_peak_kernel<<<blocks, tpb>>>(in, out, iters, clk);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_ms) {
      best_ms = ms;
      cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    }
  }
  if (e == cudaSuccess) {
    const double fma = 2.0 * 16.0 * iters * static_cast<double>(blocks) * tpb;  // 2 FMA per FFMA2
    *tflops = 2.0 * fma / (best_ms * 1e-3) / 1e12;
    *sm_ghz = static_cast<double>(h[0]) / static_cast<double>(h[1]);
  }
  cudaFree(in);
  cudaFree(out);
  cudaFree(clk);
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  return e;
}

}  // namespace ufpgd_gpu_impl
