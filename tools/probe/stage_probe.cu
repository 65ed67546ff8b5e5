// Per-layer MMA sequences of the (32,256) tensor-core kernel (csrc/mma.cu) in
// isolation (development aid): same shared-memory layouts, descriptors and
// instruction shapes, one CTA per SM, clock64 from issue to each commit's
// mbarrier completion, averaged over reps.
//   s1      : stage 1, 2 antenna tiles x 8 K-steps of M = 128, N = 128, commit per tile
//   s2-int  : stage 2 as issued today: per tile, per K-step [N = 128 main|corr] then [N = 64 corr]
//   s2-grp  : stage 2 grouped: per tile, 4 x N = 128 then 4 x N = 64
//   s2-n128 : stage 2 without the corr MMAs (4 x N = 128 per tile) - the floor
//   lat     : one M = 128, N = 128, K = 16 MMA -> commit -> wait (latency)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 stage_probe.cu -o stage_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace {
constexpr int K = 32, M = 256, R = 2 * K, Q = 2 * R;
constexpr int OFF_HH = 0, OFF_HL = R * M * 2, OFF_W = OFF_HL + R * M * 2;
constexpr int BSBO = 16 * R;
constexpr int OFF_BH = OFF_W + Q * M * 2, OFF_BL = OFF_BH + (R / 8) * BSBO;
constexpr int SMEM = OFF_BL + (R / 8) * BSBO + 1024;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
template <int MM, int NN>
__device__ constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 15) | (static_cast<uint32_t>(NN >> 3) << 17) | (static_cast<uint32_t>(MM >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// warp-wide issue: every lane executes, one elected lane issues (descriptors warp-uniform)
__device__ __forceinline__ void mma_w(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_w(uint32_t bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(ph)
        : "memory");
}

template <int SEQ>
__global__ void __launch_bounds__(128, 1) probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < SMEM / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
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
  const uint32_t tmem = slot, sb = su32(sm), b0 = su32(&bar[0]), b1 = su32(&bar[1]);
  unsigned long long a0 = 0, a1 = 0, a2 = 0;
  uint32_t ph = 0;
  const int wu = __shfl_sync(0xffffffffu, tid >> 5, 0);
  if (SEQ >= 300 && wu == 0) {
    for (int r = 0; r < reps; ++r) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const unsigned long long t0 = clock64();
      constexpr int n = 2 * ((SEQ - 300) / 10), v = SEQ % 10;
      constexpr uint32_t ID = v == 0 ? idesc<64, 64>() : v == 1 ? idesc<128, 64>() : v == 2 ? idesc<64, 32>() : v == 3 ? idesc<128, 32>() : idesc<64, 128>();
      for (int i = 0; i < n; ++i)
        mma_w(tmem, sdesc(sb + OFF_W + i * 2 * 16 * Q, 16 * Q, 128), sdesc(sb + OFF_HH + i * 256, 128, 16 * M), ID, i > 0);
      commit_w(b0);
      commit_w(b1);
      const unsigned long long ti = clock64();
      wait(b0, ph);
      const unsigned long long tw0 = clock64();
      wait(b1, ph);
      const unsigned long long tw1 = clock64();
      ph ^= 1;
      a0 += ti - t0;
      a1 += tw0 - t0;
      a2 += tw1 - t0;
    }
    if (blockIdx.x == 0 && tid == 0) {
      out[0] = a0;
      out[1] = a1;
      out[2] = a2;
    }
  }
  if (SEQ >= 200 && SEQ < 300 && wu == 0) {
    for (int r = 0; r < reps; ++r) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const unsigned long long t0 = clock64();
      constexpr int n = (SEQ - 200) / 10;
      for (int i = 0; i < n; ++i)
        mma_w(tmem, sdesc(sb + OFF_W + i * 2 * 16 * Q, 16 * Q, 128), sdesc(sb + OFF_HH + i * 256, 128, 16 * M), idesc<Q, 2 * R>(), i > 0);
      commit_w(b0);
      commit_w(b1);
      const unsigned long long ti = clock64();
      wait(b0, ph);
      const unsigned long long tw0 = clock64();
      wait(b1, ph);
      const unsigned long long tw1 = clock64();
      ph ^= 1;
      a0 += ti - t0;
      a1 += tw0 - t0;
      a2 += tw1 - t0;
    }
    if (blockIdx.x == 0 && tid == 0) {
      out[0] = a0;
      out[1] = a1;
      out[2] = a2;
    }
  }
  if (SEQ < 200 && tid == 0) {
    for (int r = 0; r < reps; ++r) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const unsigned long long t0 = clock64();
      if (SEQ == 0) {  // s1
        for (int t = 0; t < 2; ++t) {
          for (int ks = t * 8; ks < (t + 1) * 8; ++ks)
            mma(tmem + t * 2 * R, sdesc(sb + OFF_W + ks * 2 * 16 * Q, 16 * Q, 128), sdesc(sb + OFF_HH + ks * 256, 128, 16 * M),
                idesc<Q, 2 * R>(), ks > t * 8);
          commit(t ? b1 : b0);
        }
      } else if (SEQ >= 100) {  // SEQ 100 + 10 n + big: n MMAs, tiny (M=64, N=8) or M=128 N=128
        constexpr int n = (SEQ - 100) / 10;
        constexpr bool big = (SEQ % 10) != 0;
        for (int i = 0; i < n; ++i) {
          if (big)
            mma(tmem, sdesc(sb + OFF_W + i * 2 * 16 * Q, 16 * Q, 128), sdesc(sb + OFF_HH + i * 256, 128, 16 * M), idesc<Q, 2 * R>(), i > 0);
          else
            mma(tmem, sdesc(sb + OFF_W + i * 2 * 16 * Q, 16 * Q, 128), sdesc(sb + OFF_HH + i * 256, 128, 16 * M), idesc<64, 8>(), i > 0);
        }
        commit(b0);
        commit(b1);
      } else if (SEQ == 4) {
        mma(tmem, sdesc(sb + OFF_W, 16 * Q, 128), sdesc(sb + OFF_HH, 128, 16 * M), idesc<Q, 2 * R>(), 0);
        commit(b0);
        commit(b1);
      } else {
        for (int t = 0; t < 2; ++t) {
          const uint32_t dm = tmem + t * 2 * R, dc = dm + R;
          auto ah = [&](int ks) { return sdesc(sb + OFF_HH + t * 16 * 128 + ks * 2 * 16 * M, 16 * M, 128); };
          auto al = [&](int ks) { return sdesc(sb + OFF_HL + t * 16 * 128 + ks * 2 * 16 * M, 16 * M, 128); };
          auto bh = [&](int ks) { return sdesc(sb + OFF_BH + ks * 256, 128, BSBO); };
          if (SEQ == 1) {
            for (int ks = 0; ks < R / 16; ++ks) {
              mma(dm, ah(ks), bh(ks), idesc<128, 2 * R>(), ks > 0);
              mma(dc, al(ks), bh(ks), idesc<128, R>(), 1);
            }
          } else if (SEQ == 2) {
            for (int ks = 0; ks < R / 16; ++ks) mma(dm, ah(ks), bh(ks), idesc<128, 2 * R>(), ks > 0);
            for (int ks = 0; ks < R / 16; ++ks) mma(dc, al(ks), bh(ks), idesc<128, R>(), 1);
          } else {
            for (int ks = 0; ks < R / 16; ++ks) mma(dm, ah(ks), bh(ks), idesc<128, 2 * R>(), ks > 0);
          }
          commit(t ? b1 : b0);
        }
      }
      const unsigned long long ti = clock64();
      wait(b0, ph);
      const unsigned long long tw0 = clock64();
      wait(b1, ph);
      const unsigned long long tw1 = clock64();
      ph ^= 1;
      a0 += ti - t0;
      a1 += tw0 - t0;
      a2 += tw1 - t0;
    }
    if (blockIdx.x == 0) {
      out[0] = a0;
      out[1] = a1;
      out[2] = a2;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int SEQ>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 24);
  auto k = probe<SEQ>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int reps = 500;
  k<<<148, 128, SMEM>>>(reps, d);
  k<<<148, 128, SMEM>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[3] = {0, 0, 0};
  cudaMemcpy(c, d, 24, cudaMemcpyDeviceToHost);
  printf("%-8s issue %6.0f  tile0 done %6.0f  tile1 done %6.0f clk  (%s)\n", name, (double)c[0] / reps,
         (double)c[1] / reps, (double)c[2] / reps, cudaGetErrorString(e));
  cudaFree(d);
}
}  // namespace

int main() {
  run<4>("lat");
  run<110>("1 tiny");
  run<120>("2 tiny");
  run<140>("4 tiny");
  run<180>("8 tiny");
  run<111>("1 big");
  run<121>("2 big");
  run<141>("4 big");
  run<181>("8 big");
  run<210>("w 1 big");
  run<220>("w 2 big");
  run<240>("w 4 big");
  run<280>("w 8 big");
  run<380>("16 M64N64");
  run<381>("16 M128N64");
  run<382>("16 M64N32");
  run<383>("16 M128N32");
  run<384>("16 M64N128");
  run<0>("s1");
  run<1>("s2-int");
  run<2>("s2-grp");
  run<3>("s2-n128");
  run<1>("s2-int");
  run<0>("s1");
  return 0;
}
