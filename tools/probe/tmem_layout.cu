// Probe of the tcgen05.ld shapes' thread/register layout (development aid):
// TMEM lanes 0..31 x columns 0..31 are written with value 1000 * lane + column
// (32x32b stores: thread = lane), then read back with .16x256b / .16x128b /
// .16x64b and each thread's registers printed as (lane, column).
#include <cstdio>
#include <cstdint>
__global__ void probe(int* out) {
  __shared__ uint32_t slot;
  const int lane = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(&slot))) : "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;
  for (int c = 0; c < 32; ++c) {
    const uint32_t v = 1000 * lane + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t + c), "r"(v) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 8; ++i) out[lane * 8 + i] = r[i];
  uint32_t q[4];
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 4; ++i) out[256 + lane * 4 + i] = q[i];
  uint32_t u[2];
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(u[0]), "=r"(u[1]) : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 2; ++i) out[384 + lane * 2 + i] = u[i];
  __syncthreads();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t) : "memory");
}
int main() {
  int* d;
  cudaMalloc(&d, 448 * sizeof(int));
  probe<<<1, 32>>>(d);
  int h[448];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  const char* names[3] = {"16x256b.x2", "16x128b.x2", "16x64b.x2"};
  const int base[3] = {0, 256, 384}, n[3] = {8, 4, 2};
  for (int s = 0; s < 3; ++s) {
    printf("%s:\n", names[s]);
    for (int l = 0; l < 32; ++l) {
      printf(" t%02d:", l);
      for (int i = 0; i < n[s]; ++i) printf(" (%d,%d)", h[base[s] + l * n[s] + i] / 1000, h[base[s] + l * n[s] + i] % 1000);
      printf("\n");
    }
  }
  return 0;
}
