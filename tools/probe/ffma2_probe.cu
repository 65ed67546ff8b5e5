// Does sm_100a's packed fma.rn.f32x2 (FFMA2) lift the 3-register FFMA limit?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gtimer() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned long long pack(float a, float b) { unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(unsigned long long r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a + b; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

template <int MODE>
__global__ void probe(const float* __restrict__ in, float* out, int iters, unsigned long long* clk) {
  unsigned long long a[4], b[4], acc[16];
  for (int i = 0; i < 4; ++i) { a[i] = pack(in[threadIdx.x + i], in[threadIdx.x + 8 + i]); b[i] = pack(in[threadIdx.x + 32 + i], in[threadIdx.x + 40 + i]); }
  for (int i = 0; i < 16; ++i) acc[i] = pack(in[threadIdx.x + 64 + i], in[threadIdx.x + 96 + i]);
  unsigned long long c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (MODE == 0) acc[i * 4 + j] = fma2(a[i], b[j], acc[i * 4 + j]);
        if (MODE == 1) { float sa = lo(a[i]); acc[i * 4 + j] = fma2(pack(sa, sa), b[j], acc[i * 4 + j]); }
      }
  }
  unsigned long long c1 = clock64(), t1 = gtimer();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += lo(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  float *in, *out; unsigned long long* clk;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, p.multiProcessorCount * 8 * 256 * 4); cudaMalloc(&clk, 16);
  for (int rep = 0; rep < 4; ++rep) {
    int tpb = 256, blocks = p.multiProcessorCount * 8, iters = 8192;
    if (rep & 1) probe<1><<<blocks, tpb>>>(in, out, 64, clk); else probe<0><<<blocks, tpb>>>(in, out, 64, clk); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); if (rep & 1) probe<1><<<blocks, tpb>>>(in, out, iters, clk); else probe<0><<<blocks, tpb>>>(in, out, iters, clk); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    double ghz = (double)h[0] / (double)h[1];
    double fma = 2.0 * 16.0 * iters * (double)blocks * tpb;  // 2 FMAs per FFMA2
    printf(rep & 1 ? "FFMA2 scalar-bcast operand:" : "FFMA2 3 pairs:");
    printf(" %.2f TFLOP/s clock %.3f GHz -> %.1f FMA/clk/SM (nominal 128) err=%s\n",
           2 * fma / ms / 1e9, ghz, fma / (ms * 1e-3) / p.multiProcessorCount / (ghz * 1e9),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
