// tcgen05.mma kind::f16 issue-to-completion throughput probe on B200 (development aid):
// clocks per MMA for the operand layouts the tensor-core kernel (csrc/mma.cu) can use.
//   variant 0: A MN-major no-swizzle, B K-major no-swizzle (the kernel's stage 1)
//   variant 1: A K-major no-swizzle,  B K-major no-swizzle
//   variant 2: A K-major 128B-swizzle, B K-major 128B-swizzle
//   variant 3: A MN-major 128B-swizzle, B K-major 128B-swizzle
// M = 128, N in {64, 128, 256}, K = 16 per instruction, KS instructions per chain,
// one chain = issue KS MMAs -> commit -> mbarrier wait. One CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_probe.cu -o umma_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}

template <int VAR, int N, int KS>
__global__ void __launch_bounds__(128, 1) probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 200 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;  // 1.0h
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot, sb = su32(sm);
  constexpr uint32_t IDESC = (1u << 4) | ((VAR == 0 || VAR == 3) ? (1u << 15) : 0u) | ((N >> 3) << 17) | ((128 >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  uint32_t ph = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int ks = 0; ks < KS; ++ks) {
        uint64_t a, b;
        if (VAR == 0) {  // A MN-major: cores (mg, kg), LBO = K-group stride, SBO = MN-group stride
          a = sdesc(sb + ks * 2 * 16 * 128, 16 * 128, 128, 0);
          b = sdesc(sb + 96 * 1024 + ks * 256, 128, 16 * KS * 16, 0);
        } else if (VAR == 1) {  // A K-major: cores (mg, kg): LBO = K-group stride 128, SBO = 8-row group stride
          a = sdesc(sb + ks * 256, 128, 16 * KS * 16, 0);
          b = sdesc(sb + 96 * 1024 + ks * 256, 128, 16 * KS * 16, 0);
        } else if (VAR == 2) {  // K-major SW128: 64-element (128 B) rows, 8-row atoms of 1 KB; K advance 32 B
          const int atom = ks / 4, kin = ks % 4;
          a = sdesc(sb + atom * 128 * 128 + kin * 32, 16, 1024, 2);
          b = sdesc(sb + 96 * 1024 + atom * N * 128 + kin * 32, 16, 1024, 2);
        } else {  // A MN-major SW128: 64 MN elements per 128 B row, 8 K-rows per atom; LBO = MN-atom stride
          a = sdesc(sb + ks * 2 * 1024, 1024 * (16 * KS / 8), 1024, 2);
          const int atom = ks / 4, kin = ks % 4;
          b = sdesc(sb + 96 * 1024 + atom * N * 128 + kin * 32, 16, 1024, 2);
        }
        const uint32_t acc = ks > 0;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(a), "l"(b), "r"(IDESC), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(su32(&bar)), "r"(ph));
      ph ^= 1;
    }
    t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int VAR, int N, int KS>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto k = probe<VAR, N, KS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int reps = 200;
  k<<<148, 128, 200 * 1024>>>(reps, d);
  k<<<148, 128, 200 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = static_cast<double>(c) / reps / KS;
  printf("%-34s N=%3d KS=%2d: %7.1f clk/MMA  %6.0f clk/chain  %5.0f MAC/clk  (%s)\n", name, N, KS, per,
         static_cast<double>(c) / reps, 128.0 * N * 16 / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 128, 16>("A MN-major, B K-major (no swizzle)");
  run<1, 128, 16>("A K-major, B K-major (no swizzle)");
  run<2, 128, 16>("A K-major, B K-major (SW128)");
  run<3, 128, 16>("A MN-major SW128, B K-major SW128");
  run<0, 64, 16>("A MN-major, B K-major (no swizzle)");
  run<1, 64, 16>("A K-major, B K-major (no swizzle)");
  run<2, 64, 16>("A K-major, B K-major (SW128)");
  run<0, 256, 8>("A MN-major, B K-major (no swizzle)");
  run<1, 256, 8>("A K-major, B K-major (no swizzle)");
  run<2, 256, 8>("A K-major, B K-major (SW128)");
  run<1, 128, 4>("A K-major, B K-major (no swizzle)");
  run<0, 128, 4>("A MN-major, B K-major (no swizzle)");
  return 0;
}
