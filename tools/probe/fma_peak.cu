// FP32 FMA-pipe peak probe on B200 with the SM clock measured in-kernel
// (clock64 vs %globaltimer), so FFMA/clk/SM is known independently of DVFS.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

// MODE 0: acc = fma(acc, a[j], b[j])  — 3 distinct registers
// MODE 1: acc = fma(acc, a[j], 1.5f)  — immediate operand
// MODE 2: acc = fma(a[j], b[j], acc) with 16 accumulators sharing a, b pairs (outer-product reuse)
template <int MODE>
__global__ void probe(const float* __restrict__ in, float* out, int iters, unsigned long long* clk) {
  float a[4], b[4], acc[16];
  for (int i = 0; i < 4; ++i) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 32 + i]; }
  for (int i = 0; i < 16; ++i) acc[i] = in[threadIdx.x + 64 + i];
  unsigned long long c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (MODE == 0) acc[i * 4 + j] = fmaf(acc[i * 4 + j], a[i], b[j]);
        if (MODE == 1) acc[i * 4 + j] = fmaf(acc[i * 4 + j], a[j], 1.5f);
        if (MODE == 2) acc[i * 4 + j] = fmaf(a[i], b[j], acc[i * 4 + j]);
      }
  }
  unsigned long long c1 = clock64(), t1 = gtimer();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

template <int MODE>
void run(const char* name, float* in, float* out, unsigned long long* clk, int sms) {
  int tpb = 256, blocks = sms * 8, iters = 8192;
  probe<MODE><<<blocks, tpb>>>(in, out, 64, clk); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); probe<MODE><<<blocks, tpb>>>(in, out, iters, clk); cudaEventRecord(b);
  cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
  double ghz = (double)h[0] / (double)h[1];
  double fma = 16.0 * iters * (double)blocks * tpb;
  double tflops = 2 * fma / ms / 1e9;
  printf("%-28s %.2f TFLOP/s  clock %.3f GHz  -> %.1f FFMA/clk/SM (nominal 128)\n", name, tflops, ghz,
         fma / (ms * 1e-3) / sms / (ghz * 1e9));
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  float *in, *out; unsigned long long* clk;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, p.multiProcessorCount * 8 * 256 * 4); cudaMalloc(&clk, 16);
  run<0>("fma(acc, a, b) 3-reg", in, out, clk, p.multiProcessorCount);
  run<1>("fma(acc, a, imm)", in, out, clk, p.multiProcessorCount);
  run<2>("fma(a, b, acc) outer-prod", in, out, clk, p.multiProcessorCount);
  run<0>("fma(acc, a, b) 3-reg (again)", in, out, clk, p.multiProcessorCount);
  return 0;
}
