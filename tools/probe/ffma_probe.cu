// Throughput probes for the B200 FP32 pipe, SHFL and LDS.128 (broadcast) —
// the three resources the fused unfolded-PGD kernel lives on.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// Complex outer-product accumulate: 2 x 8 complex accumulators, like stage 1.
__global__ void ffma_cplx(float* out, int iters, float s) {
  float ar[2], ai[2], br[8], bi[8], xr[2][8], xi[2][8];
  for (int i = 0; i < 2; ++i) { ar[i] = threadIdx.x * 1e-3f + i; ai[i] = s * i; }
  for (int j = 0; j < 8; ++j) { br[j] = j * 1e-2f; bi[j] = s + j; }
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) { xr[i][j] = 0.f; xi[i][j] = 0.f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        xr[i][j] = fmaf(ar[i], br[j], xr[i][j]);
        xr[i][j] = fmaf(-ai[i], bi[j], xr[i][j]);
        xi[i][j] = fmaf(ar[i], bi[j], xi[i][j]);
        xi[i][j] = fmaf(ai[i], br[j], xi[i][j]);
      }
#pragma unroll
    for (int j = 0; j < 8; ++j) { br[j] += 1e-7f; }
  }
  float acc = 0.f;
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) acc += xr[i][j] + xi[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void shfl_probe(float* out, int iters) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 1 << (i & 3));
  }
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// LDS.128 where 4 lanes share an address (the fused kernel's H read pattern).
__global__ void lds_probe(float* out, int iters) {
  __shared__ float4 sm[4096 / 16 * 4];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int r = lane >> 4, b = lane & 3;
  const float4* base = sm + ((warp * 2 + r) & 3) * 256;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float4 v = base[((4 * i + b) * 5 + (it & 1)) & 255];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock(kHz) %d smem/SM %zu regs/SM %d\n", p.name, p.multiProcessorCount, clk,
         p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  float* out; CK(cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float)));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int tpb : {128, 256, 512}) {
    int blocks = p.multiProcessorCount * (2048 / tpb);
    int iters = 4096;
    ffma_cplx<<<blocks, tpb>>>(out, 16, 1.f);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    ffma_cplx<<<blocks, tpb>>>(out, iters, 1.f);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 64.0 * iters * (double)blocks * tpb;
    printf("ffma_cplx tpb=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, blocks, flops / ms / 1e9, ms);
  }
  {
    int tpb = 256, blocks = p.multiProcessorCount * 8, iters = 4096;
    shfl_probe<<<blocks, tpb>>>(out, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); shfl_probe<<<blocks, tpb>>>(out, iters); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr = 8.0 * iters * blocks * (tpb / 32);
    printf("shfl: %.3f warp-instr/clk/SM (at %d MHz nominal; %.3f ms)\n",
           warp_instr / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3), clk / 1000, ms);
  }
  {
    int tpb = 256, blocks = p.multiProcessorCount * 8, iters = 4096;
    lds_probe<<<blocks, tpb>>>(out, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); lds_probe<<<blocks, tpb>>>(out, iters); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr = 16.0 * iters * blocks * (tpb / 32);
    printf("lds128 (4-lane broadcast): %.3f warp-instr/clk/SM (%.3f ms)\n",
           warp_instr / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3), ms);
  }
  return 0;
}
