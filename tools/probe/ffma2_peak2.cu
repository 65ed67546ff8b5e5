// FFMA2 peak with larger unrolled bodies (8x8 and 4x16 outer products).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gtimer() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <int NA, int NB>
__global__ void probe(const float* __restrict__ in, float* out, int iters, unsigned long long* clk) {
  float a[NA]; float2 b[NB], acc[NA][NB];
  for (int i = 0; i < NA; ++i) a[i] = in[(threadIdx.x + i) & 255];
  for (int j = 0; j < NB; ++j) b[j] = make_float2(in[(threadIdx.x + 7 * j) & 255], in[(threadIdx.x + 3 * j + 1) & 255]);
  for (int i = 0; i < NA; ++i) for (int j = 0; j < NB; ++j) acc[i][j] = make_float2(0.f, 0.f);
  unsigned long long c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
  }
  unsigned long long c1 = clock64(), t1 = gtimer();
  float s = 0.f;
  for (int i = 0; i < NA; ++i) for (int j = 0; j < NB; ++j) s += acc[i][j].x + acc[i][j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}
template <int NA, int NB>
void run(float* in, float* out, unsigned long long* clk, int sms, int tpb, int bps) {
  int blocks = sms * bps, iters = 4096;
  probe<NA, NB><<<blocks, tpb>>>(in, out, 16, clk); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); probe<NA, NB><<<blocks, tpb>>>(in, out, iters, clk); cudaEventRecord(b);
  cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
  double ghz = (double)h[0] / h[1];
  double fma = 2.0 * NA * NB * iters * (double)blocks * tpb;
  printf("FFMA2 %dx%d tpb %d x %d/SM: %.2f TFLOP/s at %.3f GHz -> %.1f FMA/clk/SM\n", NA, NB, tpb, bps,
         2 * fma / ms / 1e9, ghz, fma / (ms * 1e-3) / sms / (ghz * 1e9));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  float *in, *out; unsigned long long* clk;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4); cudaMalloc(&out, p.multiProcessorCount * 16 * 256 * 4); cudaMalloc(&clk, 16);
  run<4, 4>(in, out, clk, p.multiProcessorCount, 256, 4);
  run<8, 8>(in, out, clk, p.multiProcessorCount, 256, 2);
  run<8, 8>(in, out, clk, p.multiProcessorCount, 128, 4);
  run<4, 16>(in, out, clk, p.multiProcessorCount, 256, 2);
  run<2, 16>(in, out, clk, p.multiProcessorCount, 256, 4);
  run<8, 8>(in, out, clk, p.multiProcessorCount, 64, 8);
  return 0;
}
