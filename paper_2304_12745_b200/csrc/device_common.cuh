// Device helpers shared by the sm_100a kernels of this directory (team.cu,
// tile.cu, general.cu, metrics.cu, grad.cu, datagen.cu, probe.cu): streaming
// global loads / stores, complex MACs and the packed FP32x2 (FFMA2 / FMUL2 /
// FADD2) forms every FP32 kernel computes in.
#pragma once

#include <cuda_runtime.h>

#include "ufpgd_internal.h"

namespace ufpgd_gpu_impl {
namespace {
constexpr int kFusedMaxWarps = 8;  // fused blocks have 1..8 warps (chosen per launch)
constexpr int kGenThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// acc += a * b
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}

// Packed FP32x2 arithmetic (sm_100a FFMA2 / FMUL2 / FADD2). A complex matrix
// is held split into real and imaginary parts, each packed over the thread's
// user PAIR (rows k, k+1): re = (Re W(k,m), Re W(k+1,m)), im likewise. A
// complex MAC with a broadcast scalar complex h then costs two FFMA2 per part
// and ptxas folds the broadcast (and its negation) into the scalar operand of
// FFMA2, so no shuffled or rotated copies are ever materialised.
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) { return __ffma2_rn(bc(a), b, c); }
__device__ __forceinline__ float2 fmul2(float a, float2 b) { return __fmul2_rn(bc(a), b); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 zero2() { return make_float2(0.f, 0.f); }
// MUFU.RSQ without the subnormal-range fix-up rsqrtf() adds (same accuracy
// for normal inputs; callers clamp the argument to >= FLT_MIN).
__device__ __forceinline__ float rsqrt_ftz(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

}  // namespace
}  // namespace ufpgd_gpu_impl
