// sm_100a kernels for the batched PA-aware precoder solver.
//
// Hot path: per realization
// and per layer
//     X' = W H^T - diag(c)            (K x K, contraction over the M antennas)
//     V  = W - eta X' H^*             (K x M, contraction over the K users)
//     w_m = max(0, 1 - t/||v_m||) v_m  (per-antenna group soft threshold)
// which is unfolded.cpp:112-146 / pgd.cpp:226-244 with the constraint term
// folded into X' (diag(c) H^* = (diag(c)) H^*, so X' H^* = grad_f(W),
// pgd.hpp:41-47). The fold is exact algebra; it removes the K x M offset
// matrix of SmoothGradient (pgd.cpp:51-59) and keeps FP32 error small over
// thousands of iterations.
//
// Fused team kernel (fused_kernel): a team of T = TK*TM threads owns one
// realization for ALL layers. Thread (a, b) of the team holds, in registers,
//   w[i][kk] = W(k = a*KA + kk, m = i*TM + b)     (KA users x MB antennas)
//   x[kk][j] = X'(a*KA + kk, j)                   (its KA rows of X')
// packed over user pairs for FFMA2, and H lives in shared memory (unpadded
// rows, 16-byte units XOR-swizzled so the quarter-warp LDS.128 phases are
// bank-conflict free). Per layer: stage 2 + prox over the thread's antennas,
// then (two-sweep mode) stage 1 over them again, building the NEXT layer's X'
// — so X' and the next X' are never live at once and the unfolded kernel fits
// 168 registers (12 warps/SM). Warp shuffles do the two reductions: the
// per-antenna norm across the TK threads sharing an antenna, and the X'
// all-reduce across the TM threads sharing rows (once per layer). H is read
// from HBM once (ld.global.nc, streaming) and W written once (st.global.cs).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "device_common.cuh"

namespace ufpgd_gpu_impl {
namespace {

// 1: two sweeps per layer (stage 2 + prox, then stage 1 re-reading H), so X'
// and the next X' are never live together (A/B knob; 0 = one fused sweep).
#ifndef UFPGD_TWO_SWEEP
#define UFPGD_TWO_SWEEP 1
#endif

template <int K_, int M_, int TK_, int TM_, int MAXT_ = 256, int MINB_ = 1, bool WSMEM_ = false,
          bool TWO_SWEEP_ = UFPGD_TWO_SWEEP>
struct Team {
  // WSMEM: W lives in shared memory (one 16-byte unit per thread and antenna)
  // instead of registers; TWO_SWEEP: see UFPGD_TWO_SWEEP.
  static constexpr bool WSMEM = WSMEM_, TWO_SWEEP = TWO_SWEEP_;
  static constexpr int K = K_, M = M_, TK = TK_, TM = TM_;
  // launch bounds: register cap = 64K / (MAXT * MINB)
  static constexpr int MAXT = MAXT_, MINB = MINB_;
  static constexpr int T = TK * TM;     // threads per realization
  static constexpr int R = 32 / T;      // realizations per warp
  static constexpr int KA = K / TK;     // users per thread
  static constexpr int P = KA / 2;      // user pairs per thread (FFMA2 lanes)
  static constexpr int MB = M / TM;     // antennas per thread
  static constexpr int HS = 2 * K;      // H row stride in floats (XOR-swizzled units, no padding)
  static constexpr int U = K / 2;       // 16-byte units per H row
  static constexpr int SMEM_PER_WARP = R * M * HS * 4;          // H tiles
  static constexpr int WSMEM_PER_WARP = WSMEM ? R * M * TK * P * 16 : 0;  // W tiles (bytes)
  // Unit swizzle of row m: with U >= 4 units per row, rows m and m + 2 of a
  // quarter-warp LDS.128 phase would hit the same banks; XOR-ing the unit
  // index with (m >> 1) mod U separates them. U <= 2 is conflict-free as is.
  static __device__ __forceinline__ int swz(int m) { return U >= 4 ? (m >> 1) & (U - 1) : 0; }
  // Address of complex H(c, m) (user c, antenna m) in the tile.
  static __device__ __forceinline__ const float* hat(const float* hs, int m, int c) {
    return hs + m * HS + 4 * ((c >> 1) ^ swz(m)) + 2 * (c & 1);
  }
  static_assert(32 % T == 0, "a team must divide the warp");
  static_assert(K % TK == 0 && M % TM == 0, "team must tile (K, M)");
  static_assert(KA % 2 == 0 && K % 2 == 0, "users are processed in FFMA2 pairs");
};


// Per-thread H row pointers: with TM even, the unit swizzle of antenna
// m = i * TM + b splits into a compile-time part (from i) XOR a per-thread part
// (from b), so u[q] = row b, unit q ^ swz_b, and column i, unit q is
// u[q ^ swz_i] + i * TM * HS: an immediate offset from one of U registers, no
// per-load address arithmetic in the unrolled layer loop.
template <class S>
struct ColPtr {
  const float* u[S::U];
  __device__ __forceinline__ ColPtr(const float* hs, int b) {
    const int fb = S::U >= 4 ? (b >> 1) & (S::U - 1) : 0;
#pragma unroll
    for (int q = 0; q < S::U; ++q) u[q] = hs + b * S::HS + 4 * (q ^ fb);
  }
};

// LDS.128 the compiler may not merge with an identical earlier load.
__device__ __forceinline__ float4 lds128_fresh(const float* p) {
  float4 v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

template <class S, bool FRESH = false>
__device__ __forceinline__ void load_col(const ColPtr<S>& cp, int i, float2 (&h)[S::K]) {
  static_assert(S::TM % 2 == 0, "swizzle split needs an even TM");
  const int ci = S::U >= 4 ? (i * (S::TM / 2)) & (S::U - 1) : 0;  // folds: i is unrolled
#pragma unroll
  for (int q = 0; q < S::U; ++q) {
    const float* ptr = cp.u[q ^ ci] + i * S::TM * S::HS;
    const float4 t = FRESH ? lds128_fresh(ptr) : *reinterpret_cast<const float4*>(ptr);
    h[2 * q] = make_float2(t.x, t.y);
    h[2 * q + 1] = make_float2(t.z, t.w);
  }
}

// Split-complex accumulators of the thread's rows of X' (stage 1 output).
template <class S>
struct XAcc {
  float2 re[S::P][S::K], im[S::P][S::K];
};

// W(a*KA + 2p + {0,1}, i*TM + b) split into real / imaginary user pairs, in
// registers (WReg) or in a shared-memory tile (WSm).
template <class S>
struct WReg {
  float2 r[S::MB][S::P], im[S::MB][S::P];
  __device__ __forceinline__ void ld(int i, int p, float2& wr, float2& wi) const {
    wr = r[i][p];
    wi = im[i][p];
  }
  __device__ __forceinline__ void st(int i, int p, float2 wr, float2 wi) {
    r[i][p] = wr;
    im[i][p] = wi;
  }
};

// Shared-memory W tile: row m holds the TK user-pair units (re pair, im pair)
// of antenna m; unit a is XOR-ed with ((m >> 1) & 1) << 1 so the 8 lanes of a
// quarter-warp LDS.128 / STS.128 phase (a in {0,1}, b in 0..3) hit 8 distinct
// units. With TM = 4 the swizzle depends on b only: one base pointer per thread.
template <class S>
struct WSm {
  static_assert(S::P == 1 && S::TK == 4 && S::TM == 4, "WSm covers the (TK, TM) = (4, 4), one-pair team");
  float* base;
  __device__ __forceinline__ WSm(float* tile, int a, int b)
      : base(tile + b * S::TK * 4 + 4 * (a ^ (((b >> 1) & 1) << 1))) {}
  __device__ __forceinline__ void ld(int i, int p, float2& wr, float2& wi) const {
    const float4 t = *reinterpret_cast<const float4*>(base + i * S::TM * S::TK * 4);
    wr = make_float2(t.x, t.y);
    wi = make_float2(t.z, t.w);
  }
  __device__ __forceinline__ void st(int i, int p, float2 wr, float2 wi) {
    *reinterpret_cast<float4*>(base + i * S::TM * S::TK * 4) = make_float4(wr.x, wr.y, wi.x, wi.y);
  }
};

// Stage 1 contribution of antenna m: X'(k, j) += W(k, m) H(j, m).
template <class S>
__device__ __forceinline__ void stage1_accumulate(XAcc<S>& xn, const float2 (&wr)[S::P],
                                                  const float2 (&wi)[S::P], const float2 (&h)[S::K]) {
#pragma unroll
  for (int p = 0; p < S::P; ++p)
#pragma unroll
    for (int j = 0; j < S::K; ++j) {
      xn.re[p][j] = ffma2(h[j].x, wr[p], xn.re[p][j]);
      xn.re[p][j] = ffma2(-h[j].y, wi[p], xn.re[p][j]);
      xn.im[p][j] = ffma2(h[j].x, wi[p], xn.im[p][j]);
      xn.im[p][j] = ffma2(h[j].y, wr[p], xn.im[p][j]);
    }
}

// All-reduce of the stage-1 partials across the TM threads sharing rows. The
// constraint fold X'(k, k) -= c_k is already in the partials: the b == 0
// thread of each row group starts its accumulation from -diag(c) (xacc_init).
template <class S>
__device__ __forceinline__ void allreduce(XAcc<S>& xn, XAcc<S>& x) {
#pragma unroll
  for (int p = 0; p < S::P; ++p)
#pragma unroll
    for (int j = 0; j < S::K; ++j) {
      float2 r = xn.re[p][j], i = xn.im[p][j];
#pragma unroll
      for (int off = 1; off < S::TM; off <<= 1) {
        const float2 ro = make_float2(__shfl_xor_sync(kFull, r.x, off), __shfl_xor_sync(kFull, r.y, off));
        const float2 io = make_float2(__shfl_xor_sync(kFull, i.x, off), __shfl_xor_sync(kFull, i.y, off));
        r = fadd2(r, ro);
        i = fadd2(i, io);
      }
      x.re[p][j] = r;
      x.im[p][j] = i;
    }
}

// Start value of the stage-1 accumulators: -diag(c) on the thread's rows for
// the b == 0 thread (so the all-reduce applies the fold exactly once), zero
// elsewhere. cdiag[p] = (-c_k0, -c_k0+1) or zero, precomputed per thread.
template <class S>
__device__ __forceinline__ void xacc_init(XAcc<S>& x, const float2 (&cdiag)[S::P], int a) {
#pragma unroll
  for (int p = 0; p < S::P; ++p)
#pragma unroll
    for (int j = 0; j < S::K; ++j) {
      // j is compile-time; the row pair (k0, k0+1) = (a*KA + 2p, +1) is not:
      // only j in that pair gets a non-zero start, selected with one compare.
      const int k0 = a * S::KA + 2 * p;
      x.re[p][j] = make_float2(j == k0 ? cdiag[p].x : 0.f, j == k0 + 1 ? cdiag[p].y : 0.f);
      x.im[p][j] = zero2();
    }
}

template <class S, bool FRESH = false, class WS>
__device__ __forceinline__ void team_stage1(const WS& w, XAcc<S>& x, const float* hs, int a, int b,
                                            const float2 (&cdiag)[S::P]) {
  XAcc<S> xn;
  xacc_init<S>(xn, cdiag, a);
  const ColPtr<S> cp(hs, b);
#pragma unroll
  for (int i = 0; i < S::MB; ++i) {
    float2 h[S::K];
    load_col<S, FRESH>(cp, i, h);
    float2 wr[S::P], wi[S::P];
#pragma unroll
    for (int p = 0; p < S::P; ++p) w.ld(i, p, wr[p], wi[p]);
    stage1_accumulate<S>(xn, wr, wi, h);
  }
  allreduce<S>(xn, x);
}

// One layer (or PGD iteration). STAGE1: also build X' for the next layer.
// STATS: accumulate ||W||_{2,1} and the active count for this thread's
// antennas (counted on the a == 0 threads only).
// Antennas go in pairs (their stage-2 contractions, norm shuffles and prox
// tails are independent), so the two squared column norms reduce as one
// packed FP32x2. Each stage-2 output part is ONE K-deep FFMA2 chain started
// at W (no merge adds) — measured fastest at 3 warps per scheduler, against
// 2- and 4-chain splits.

// Tape rows of one layer of one realization (ForwardOptions::with_tape /
// with_iterates, unfolded.cpp:127-143): step image V, column norms and shrink
// factors of layer l, and iterate l + 1. Null members are not written (absent
// tape, padding team).
struct TapeRow {
  float2* v;
  float* nrm;
  float* shr;
  float2* it;
};

template <class S>
__device__ __forceinline__ TapeRow tape_row(const FusedArgs& p, long long l, long long rid, bool valid) {
  if (!valid) return TapeRow{nullptr, nullptr, nullptr, nullptr};
  const long long o = l * p.B + rid;
  return TapeRow{p.tape_v ? p.tape_v + o * (S::M * S::K) : nullptr, p.tape_norms ? p.tape_norms + o * S::M : nullptr,
                 p.tape_shrink ? p.tape_shrink + o * S::M : nullptr,
                 p.iterates ? p.iterates + (o + p.B) * (S::M * S::K) : nullptr};
}

// RESID: also accumulate sum |W_new - W|^2 and sum |W|^2 over the thread's
// entries (user pairs packed) into dd / ss — solve_pgd's relative iterate
// change (pgd.cpp:246-260).
// TAPE: also store the layer's tape rows (tr): V and the new W as 16-byte
// user-pair units (the team's TK threads cover an antenna's K entries, so a
// warp's stores are contiguous), the column norm sqrt(s) and the shrink factor
// actually applied (0 when the column is cut).
template <class S, bool STAGE1, bool STATS, class WS, bool RESID = false, bool TAPE = false>
__device__ __forceinline__ void team_layer(WS& w, XAcc<S>& x,
                                           const float* hs, int a, int b, float eta, float thr,
                                           const float2 (&cdiag)[S::P], bool& nonfinite, float& l21,
                                           int& act, float2* dd = nullptr, float2* ss = nullptr,
                                           TapeRow tr = TapeRow{nullptr, nullptr, nullptr, nullptr}) {
  constexpr int AB = 2;
  static_assert(S::MB % AB == 0, "antennas are processed in pairs");
  XAcc<S> xn;
  if (STAGE1) xacc_init<S>(xn, cdiag, a);
  const float thr2 = thr * thr;
  const ColPtr<S> cp(hs, b);
  // Fold the step into X' once per layer (X' <- -eta X'), so each antenna's
  // stage-2 chains start from W and V = W - eta G needs no extra FFMA2.
#pragma unroll
  for (int p = 0; p < S::P; ++p)
#pragma unroll
    for (int j = 0; j < S::K; ++j) {
      x.re[p][j] = fmul2(-eta, x.re[p][j]);
      x.im[p][j] = fmul2(-eta, x.im[p][j]);
    }
#pragma unroll
  for (int i0 = 0; i0 < S::MB; i0 += AB) {
    float2 h[AB][S::K];
    float2 vr[AB][S::P], vi[AB][S::P];
    float2 wor[AB][S::P], woi[AB][S::P];  // RESID: the W entries before the update
    float2 s2p[AB];
#pragma unroll
    for (int u = 0; u < AB; ++u) {
      const int i = i0 + u;
      load_col<S>(cp, i, h[u]);
      // stage 2: G(k, m) = sum_j X'(k, j) conj(H(j, m)); V = W - eta G
      float2 s2 = zero2();
#pragma unroll
      for (int p = 0; p < S::P; ++p) {
        float2 gr, gi;
        w.ld(i, p, gr, gi);
        if (RESID) {
          wor[u][p] = gr;
          woi[u][p] = gi;
        }
#pragma unroll
        for (int j = 0; j < S::K; ++j) {
          gr = ffma2(h[u][j].x, x.re[p][j], gr);
          gr = ffma2(h[u][j].y, x.im[p][j], gr);
          gi = ffma2(h[u][j].x, x.im[p][j], gi);
          gi = ffma2(-h[u][j].y, x.re[p][j], gi);
        }
        vr[u][p] = gr;
        vi[u][p] = gi;
        s2 = __ffma2_rn(vr[u][p], vr[u][p], s2);
        s2 = __ffma2_rn(vi[u][p], vi[u][p], s2);
      }
      s2p[u] = s2;
    }
    // the pair's squared norms as one packed FP32x2: partial sum, then the
    // shuffle levels across the TK threads holding each antenna
    float2 sp = fadd2(make_float2(s2p[0].x, s2p[1].x), make_float2(s2p[0].y, s2p[1].y));
#pragma unroll
    for (int off = S::TM; off < S::T; off <<= 1)
      sp = fadd2(sp, make_float2(__shfl_xor_sync(kFull, sp.x, off), __shfl_xor_sync(kFull, sp.y, off)));
    const float s[AB] = {sp.x, sp.y};
#pragma unroll
    for (int u = 0; u < AB; ++u) {
      const int i = i0 + u;
      // Non-finite step image (unfolded.cpp:120-125): any NaN/Inf entry of
      // v_m makes its squared column norm NaN/Inf. (A finite column whose
      // squared norm overflows FP32, |v| > ~6e18, is flagged too.)
      nonfinite |= !(s[u] <= FLT_MAX);
      // prox (pgd.cpp:85-99): strict ||v|| > t, i.e. s > t^2
      const bool on = s[u] > thr2;
      const float r = rsqrt_ftz(fmaxf(s[u], FLT_MIN));  // s = 0 or subnormal only matters at thr = 0
      const float scale = on ? fmaf(-thr, r, 1.f) : 0.f;
      float2 nwr[S::P], nwi[S::P];
#pragma unroll
      for (int p = 0; p < S::P; ++p) {
        nwr[p] = fmul2(scale, vr[u][p]);
        nwi[p] = fmul2(scale, vi[u][p]);
        w.st(i, p, nwr[p], nwi[p]);
        if (RESID) {
          const float2 dr = __ffma2_rn(make_float2(-1.f, -1.f), wor[u][p], nwr[p]);
          const float2 di = __ffma2_rn(make_float2(-1.f, -1.f), woi[u][p], nwi[p]);
          *dd = __ffma2_rn(dr, dr, __ffma2_rn(di, di, *dd));
          *ss = __ffma2_rn(wor[u][p], wor[u][p], __ffma2_rn(woi[u][p], woi[u][p], *ss));
        }
      }
      if (TAPE) {
        const int m = i * S::TM + b, ko = m * S::K + a * S::KA;
#pragma unroll
        for (int p = 0; p < S::P; ++p) {
          if (tr.v)
            stg_stream(reinterpret_cast<float4*>(tr.v + ko + 2 * p),
                       make_float4(vr[u][p].x, vi[u][p].x, vr[u][p].y, vi[u][p].y));
          if (tr.it)
            stg_stream(reinterpret_cast<float4*>(tr.it + ko + 2 * p), make_float4(nwr[p].x, nwi[p].x, nwr[p].y, nwi[p].y));
        }
        if (a == 0) {
          if (tr.nrm) tr.nrm[m] = sqrtf(s[u]);
          if (tr.shr) tr.shr[m] = scale;
        }
      }
      if (STATS) {
        if (a == 0 && on) {
          l21 += fmaf(s[u], r, -thr);  // ||w_m|| = ||v_m|| - t
          act += 1;
        }
      }
      if (STAGE1) stage1_accumulate<S>(xn, nwr, nwi, h[u]);
    }
  }
  if (STAGE1) allreduce<S>(xn, x);
}

// Layer 0 from W0 = 0 (BASELINE configs 1, 2): X' = -diag(c) exactly, so
// V = W0 - eta X' H^* is eta c_k conj(H(k, m)) — the K x K x M contraction of
// a diagonal matrix reduces to two FMUL2 per antenna on the thread's own rows
// (bit-identical to running the contraction on the exact zeros). ceta holds
// (eta c_k0, eta c_k0+1) per user pair.
template <class S, bool STATS, class WS>
__device__ __forceinline__ void team_layer0_diag(WS& w, const float* hs, int a, int b, float thr,
                                                 const float2 (&ceta)[S::P], bool& nonfinite, float& l21,
                                                 int& act) {
  const float thr2 = thr * thr;
#pragma unroll
  for (int i0 = 0; i0 < S::MB; i0 += 2) {
    float2 vr[2][S::P], vi[2][S::P], s2p[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int m = (i0 + u) * S::TM + b;
      float2 s2 = zero2();
#pragma unroll
      for (int p = 0; p < S::P; ++p) {
        // H(k0, m), H(k0 + 1, m): one 16-byte unit of the swizzled row
        const float4 h = *reinterpret_cast<const float4*>(S::hat(hs, m, a * S::KA + 2 * p));
        vr[u][p] = __fmul2_rn(ceta[p], make_float2(h.x, h.z));
        vi[u][p] = __fmul2_rn(ceta[p], make_float2(-h.y, -h.w));
        s2 = __ffma2_rn(vr[u][p], vr[u][p], s2);
        s2 = __ffma2_rn(vi[u][p], vi[u][p], s2);
      }
      s2p[u] = s2;
    }
    float2 sp = fadd2(make_float2(s2p[0].x, s2p[1].x), make_float2(s2p[0].y, s2p[1].y));
#pragma unroll
    for (int off = S::TM; off < S::T; off <<= 1)
      sp = fadd2(sp, make_float2(__shfl_xor_sync(kFull, sp.x, off), __shfl_xor_sync(kFull, sp.y, off)));
    const float sv[2] = {sp.x, sp.y};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u;
      nonfinite |= !(sv[u] <= FLT_MAX);
      const bool on = sv[u] > thr2;
      const float r = rsqrt_ftz(fmaxf(sv[u], FLT_MIN));
      const float scale = on ? fmaf(-thr, r, 1.f) : 0.f;
#pragma unroll
      for (int p = 0; p < S::P; ++p) w.st(i, p, fmul2(scale, vr[u][p]), fmul2(scale, vi[u][p]));
      if (STATS && a == 0 && on) {
        l21 += fmaf(sv[u], r, -thr);
        act += 1;
      }
    }
  }
}

// Fixed-step power iteration on H^T H^* (pgd.cpp:146-162 with the BASELINE
// 30-step rule) for the team's realization; every team thread returns the
// Rayleigh quotient Re(v^H w) of the last step. Control flow is uniform
// across the warp (all teams run `steps` steps) so the shuffles stay legal.
template <class S>
__device__ float team_power(const float* hs, const float2* v0, int steps, int a, int b) {
  float2 v[S::MB];
#pragma unroll
  for (int i = 0; i < S::MB; ++i) v[i] = v0[i * S::TM + b];
  float est = 0.f;
  bool zero = false;
  for (int st = 0; st < steps; ++st) {
    float2 u[S::KA];
#pragma unroll
    for (int jj = 0; jj < S::KA; ++jj) u[jj] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < S::MB; ++i) {
#pragma unroll
      for (int jj = 0; jj < S::KA; ++jj) {
        const float2 hv = *reinterpret_cast<const float2*>(S::hat(hs, i * S::TM + b, a * S::KA + jj));
        cmac(u[jj], v[i], make_float2(hv.x, -hv.y));
      }
    }
#pragma unroll
    for (int jj = 0; jj < S::KA; ++jj)
#pragma unroll
      for (int off = 1; off < S::TM; off <<= 1) {
        u[jj].x += __shfl_xor_sync(kFull, u[jj].x, off);
        u[jj].y += __shfl_xor_sync(kFull, u[jj].y, off);
      }
    float dot = 0.f, wn2 = 0.f;
    float2 wv[S::MB];
#pragma unroll
    for (int i = 0; i < S::MB; ++i) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < S::KA; ++jj)
        cmac(acc, *reinterpret_cast<const float2*>(S::hat(hs, i * S::TM + b, a * S::KA + jj)), u[jj]);
#pragma unroll
      for (int off = S::TM; off < S::T; off <<= 1) {
        acc.x += __shfl_xor_sync(kFull, acc.x, off);
        acc.y += __shfl_xor_sync(kFull, acc.y, off);
      }
      wv[i] = acc;
      dot = fmaf(v[i].x, acc.x, fmaf(v[i].y, acc.y, dot));
      wn2 = fmaf(acc.x, acc.x, fmaf(acc.y, acc.y, wn2));
    }
#pragma unroll
    for (int off = 1; off < S::TM; off <<= 1) {
      dot += __shfl_xor_sync(kFull, dot, off);
      wn2 += __shfl_xor_sync(kFull, wn2, off);
    }
    if (!zero) {
      if (wn2 == 0.f) {
        zero = true;  // pgd.cpp:150-153: an all-zero channel has L = 0
        est = 0.f;
      } else {
        est = dot;
        const float inv = 1.f / sqrtf(wn2);
#pragma unroll
        for (int i = 0; i < S::MB; ++i) v[i] = make_float2(wv[i].x * inv, wv[i].y * inv);
      }
    }
  }
  return est;
}

// W storage of the thread: registers, or its units of the team's W tile (W
// tiles follow all the warps' H tiles in dynamic shared memory).
template <class S>
__device__ __forceinline__ typename std::conditional<S::WSMEM, WSm<S>, WReg<S>>::type make_wstore(
    float* smem, int warp, int team, int nwarps, int a, int b) {
  if constexpr (S::WSMEM) {
    float* tiles = smem + nwarps * (S::SMEM_PER_WARP / 4);
    return WSm<S>(tiles + (warp * S::R + team) * (S::M * S::TK * S::P * 4), a, b);
  } else {
    return WReg<S>{};
  }
}

// RESID (PGD only): solve_pgd's residual_tol early stop per realization; a
// realization that met it keeps its W (steps 0 from then on: exactly the
// identity) while the other team of its warp runs on, and the warp leaves the
// loop when both have stopped.
// TAPE (unfolded only): every layer from layer 0 through team_layer (no
// layer-0 shortcut), with its tape rows, iterate 0 = W0 and iterations = L.
template <class S, bool PGD, int MAXT, int MINB, bool RESID = false, bool TAPE = false>
__global__ void __launch_bounds__(MAXT, MINB) fused_kernel(const __grid_constant__ FusedArgs p) {
  extern __shared__ __align__(16) float smem[];
  __shared__ double red[kFusedMaxWarps][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int team = lane / S::T, tl = lane % S::T, a = tl / S::TM, b = tl % S::TM;
  const long long rid = (static_cast<long long>(blockIdx.x) * nwarps + warp) * S::R + team;
  const bool valid = rid < p.B;
  float* hs = smem + (warp * S::R + team) * (S::M * S::HS);

  // Stage H once: coalesced streaming float4 loads into the swizzled tile.
  {
    constexpr int NV = S::M * S::K / 2;
    const float4* hg = reinterpret_cast<const float4*>(p.H) + (valid ? rid : 0LL) * NV;
    float4 buf[NV / S::T];
#pragma unroll
    for (int q = 0; q < NV / S::T; ++q)
      buf[q] = valid ? ldg_stream(hg + tl + q * S::T) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < NV / S::T; ++q) {
      const int e = 2 * (tl + q * S::T);
      *reinterpret_cast<float4*>(const_cast<float*>(S::hat(hs, e / S::K, e % S::K))) = buf[q];
    }
    __syncwarp();
  }

  // W(a*KA + 2p + {0,1}, i*TM + b), split into real / imaginary user pairs.
  using WS = typename std::conditional<S::WSMEM, WSm<S>, WReg<S>>::type;
  WS w = make_wstore<S>(smem, warp, team, nwarps, a, b);
  XAcc<S> x;
  float2 cdiag[S::P];
#pragma unroll
  for (int q = 0; q < S::P; ++q) {
    const int k0 = a * S::KA + 2 * q;
    cdiag[q] = b == 0 ? make_float2(-p.c[k0], -p.c[k0 + 1]) : zero2();
  }
  if (p.w0_mode == UFPGD_W0_ZERO) {
#pragma unroll
    for (int i = 0; i < S::MB; ++i)
#pragma unroll
      for (int q = 0; q < S::P; ++q) w.st(i, q, zero2(), zero2());
    // X' = 0 H^T - diag(c): the layer-0 product is identically zero.
#pragma unroll
    for (int q = 0; q < S::P; ++q)
#pragma unroll
      for (int j = 0; j < S::K; ++j) {
        const int k0 = a * S::KA + 2 * q;
        x.re[q][j] = make_float2(j == k0 ? -p.c[j] : 0.f, j == k0 + 1 ? -p.c[j] : 0.f);
        x.im[q][j] = zero2();
      }
  } else {
    if (p.w0_mode == UFPGD_W0_CONJ_H) {
#pragma unroll
      for (int i = 0; i < S::MB; ++i) {
#pragma unroll
        for (int q = 0; q < S::P; ++q) {
          const float4 t = *reinterpret_cast<const float4*>(S::hat(hs, i * S::TM + b, a * S::KA + 2 * q));
          w.st(i, q, make_float2(t.x, t.z), make_float2(-t.y, -t.w));
        }
      }
    } else {
      const float2* w0 = p.W0 + (valid ? rid : 0LL) * (S::M * S::K);
#pragma unroll
      for (int i = 0; i < S::MB; ++i)
#pragma unroll
        for (int q = 0; q < S::P; ++q) {
          const float4 t = valid ? ldg_stream(reinterpret_cast<const float4*>(
                                       w0 + (i * S::TM + b) * S::K + a * S::KA + 2 * q))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
          w.st(i, q, make_float2(t.x, t.z), make_float2(t.y, t.w));
        }
    }
    team_stage1<S>(w, x, hs, a, b, cdiag);
  }

  float eta_b = 0.f, thr_b = 0.f;
  if (PGD) {
    if (p.eta_in) {
      eta_b = valid ? p.eta_in[rid] : 1.f;
    } else {
      const float Lb = team_power<S>(hs, p.v0, p.power_steps, a, b);
      eta_b = 1.f / Lb;
    }
    thr_b = p.lambda * eta_b;
    if (p.eta_out && valid && tl == 0) p.eta_out[rid] = eta_b;
  }

  bool nonfinite = false;
  long long first_bad = -1;
  float l21 = 0.f;
  int act = 0;
  const long long L = p.L;
  long long l0 = 0;
  if constexpr (TAPE) {
    static_assert(!PGD && !RESID, "tapes are a forward option");
    if (valid && p.iterates) {
      float2* it = p.iterates + rid * (S::M * S::K);
#pragma unroll
      for (int i = 0; i < S::MB; ++i)
#pragma unroll
        for (int q = 0; q < S::P; ++q) {
          float2 wr, wi;
          w.ld(i, q, wr, wi);
          stg_stream(reinterpret_cast<float4*>(it + (i * S::TM + b) * S::K + a * S::KA + 2 * q),
                     make_float4(wr.x, wi.x, wr.y, wi.y));
        }
    }
  }
  if (!PGD && !TAPE && p.w0_mode == UFPGD_W0_ZERO && L >= 1) {
    static_assert(S::MB % 2 == 0, "layer-0 path pairs antennas");
    float2 ceta[S::P];
#pragma unroll
    for (int q = 0; q < S::P; ++q) {
      const int k0 = a * S::KA + 2 * q;
      ceta[q] = make_float2(p.eta[0] * p.c[k0], p.eta[0] * p.c[k0 + 1]);
    }
    if (L == 1) {
      team_layer0_diag<S, true>(w, hs, a, b, p.thr[0], ceta, nonfinite, l21, act);
    } else {
      team_layer0_diag<S, false>(w, hs, a, b, p.thr[0], ceta, nonfinite, l21, act);
      team_stage1<S, true>(w, x, hs, a, b, cdiag);  // X' for layer 1
    }
    if (nonfinite) first_bad = 0;
    l0 = 1;
  }
  if constexpr (RESID) {
    static_assert(PGD, "residual_tol is a solve_pgd option");
    const float tol2 = p.residual_tol * p.residual_tol;
    bool stopped = false;
    long long taken = 0;
    float eta_r = eta_b, thr_r = thr_b;
    for (long long l = 0; l < L; ++l) {
      float2 dd = zero2(), ss = zero2();
      float l21_l = 0.f;
      int act_l = 0;
      team_layer<S, false, true, decltype(w), true>(w, x, hs, a, b, eta_r, thr_r, cdiag, nonfinite, l21_l, act_l,
                                                    &dd, &ss);
      if (nonfinite && first_bad < 0) first_bad = l;
      float2 ds = make_float2(dd.x + dd.y, ss.x + ss.y);
#pragma unroll
      for (int off = 1; off < S::T; off <<= 1)
        ds = fadd2(ds, make_float2(__shfl_xor_sync(kFull, ds.x, off), __shfl_xor_sync(kFull, ds.y, off)));
      if (!stopped) {
        taken = l + 1;
        l21 = l21_l;
        act = act_l;
        // ||W_new - W|| / max(||W||, 1e-12) < tol, in squares (pgd.cpp:246-260)
        if (ds.x < tol2 * fmaxf(ds.y, 1e-24f)) {
          stopped = true;
          eta_r = 0.f;  // from now on V = W and the prox is the identity: W stays
          thr_r = 0.f;
        }
      }
      if (__all_sync(kFull, stopped)) break;
      __syncwarp();
      team_stage1<S, true>(w, x, hs, a, b, cdiag);
    }
    if (valid && tl == 0 && p.iterations) p.iterations[rid] = taken;
  }
  for (long long l = l0; !RESID && l + 1 < L; ++l) {
    const float eta = PGD ? eta_b : p.eta[l];
    const float thr = PGD ? thr_b : p.thr[l];
    if constexpr (S::TWO_SWEEP) {
      team_layer<S, false, false, WS, false, TAPE>(w, x, hs, a, b, eta, thr, cdiag, nonfinite, l21, act, nullptr,
                                                   nullptr, TAPE ? tape_row<S>(p, l, rid, valid) : TapeRow{});
      __syncwarp();  // scheduling fence: the next X' is built only after every prox
      team_stage1<S, true>(w, x, hs, a, b, cdiag);
    } else {
      team_layer<S, true, false, WS, false, TAPE>(w, x, hs, a, b, eta, thr, cdiag, nonfinite, l21, act, nullptr,
                                                  nullptr, TAPE ? tape_row<S>(p, l, rid, valid) : TapeRow{});
    }
    if (nonfinite && first_bad < 0) first_bad = l;
  }
  if (!RESID && L >= 1 && L > l0) {
    const float eta = PGD ? eta_b : p.eta[L - 1];
    const float thr = PGD ? thr_b : p.thr[L - 1];
    team_layer<S, false, true, WS, false, TAPE>(w, x, hs, a, b, eta, thr, cdiag, nonfinite, l21, act, nullptr, nullptr,
                                                TAPE ? tape_row<S>(p, L - 1, rid, valid) : TapeRow{});
    if (nonfinite && first_bad < 0) first_bad = L - 1;
  }
  if (TAPE && valid && tl == 0 && p.iterations) p.iterations[rid] = L;  // layers_general's step count

  // Team-wide first divergence (min over the team, -1 = none).
  long long fb = first_bad < 0 ? LLONG_MAX : first_bad;
#pragma unroll
  for (int off = 1; off < S::T; off <<= 1) fb = min(fb, __shfl_xor_sync(kFull, fb, off));
#pragma unroll
  for (int off = 1; off < S::TM; off <<= 1) {
    l21 += __shfl_xor_sync(kFull, l21, off);
    act += __shfl_xor_sync(kFull, act, off);
  }
  const bool diverged = fb != LLONG_MAX;

  if (valid) {
    float2* wg = p.W + rid * (S::M * S::K);
#pragma unroll
    for (int i = 0; i < S::MB; ++i)
#pragma unroll
      for (int q = 0; q < S::P; ++q)
      {
        float2 wr, wi;
        w.ld(i, q, wr, wi);
        stg_stream(reinterpret_cast<float4*>(wg + (i * S::TM + b) * S::K + a * S::KA + 2 * q),
                   make_float4(wr.x, wi.x, wr.y, wi.y));
      }
    if (tl == 0) {
      if (p.diverged_at) p.diverged_at[rid] = diverged ? static_cast<int32_t>(fb + (PGD ? 1 : 0)) : -1;
      if (p.l21) p.l21[rid] = diverged ? __int_as_float(0x7fc00000) : l21;
      if (p.active) p.active[rid] = diverged ? -1 : act;
    }
  }

  if (p.block_partials) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (valid && tl == 0) {
      if (diverged) {
        s2 = 1.0;
      } else {
        s0 = static_cast<double>(p.alpha) * static_cast<double>(l21);
        s1 = static_cast<double>(act);
      }
    }
#pragma unroll
    for (int off = S::T; off < 32; off <<= 1) {
      s0 += __shfl_xor_sync(kFull, s0, off);
      s1 += __shfl_xor_sync(kFull, s1, off);
      s2 += __shfl_xor_sync(kFull, s2, off);
    }
    if (lane == 0) {
      red[warp][0] = s0;
      red[warp][1] = s1;
      red[warp][2] = s2;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      double t = 0.0;
      for (int q = 0; q < nwarps; ++q) t += red[q][threadIdx.x];
      p.block_partials[blockIdx.x * 3LL + threadIdx.x] = t;
    }
  }
}


// Block geometry. A realization stays resident for all its layers and each
// warp runs close to its own dependency-latency limit, so the kernel wants the
// register-limited maximum of 8 resident warps per SM and every SM busy. A
// sweep of 1..8 warps per block on B200 (tools/sweep_warps.sh)
// found 1, 2 and 8 equally fast when the grid covers the SMs, so: the largest
// of {8, 4, 2, 1} whose grid still has at least one block per SM.
int pick_warps(int rpw, long long B) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Measured on B200 (tools/nw_sweep.py, quick_time): with many waves 4-warp
  // blocks beat 8-warp ones by ~2% (a finished block's slot refills sooner);
  // with under ~4 waves (config 3: 1.7) whole-SM 8-warp blocks are ~2% ahead.
  const auto blocks = [&](int nw) { return (B + static_cast<long long>(nw) * rpw - 1) / (static_cast<long long>(nw) * rpw); };
  if (blocks(8) >= sms && blocks(8) < 4LL * sms) return 8;
  for (int nw = 4; nw > 1; nw >>= 1)
    if (blocks(nw) >= sms) return nw;
  return 1;
}

#ifndef UFPGD_PGD_MAXT
#define UFPGD_PGD_MAXT 256
#endif
#ifndef UFPGD_PGD_MINB
#define UFPGD_PGD_MINB 1
#endif
template <class S>
cudaError_t launch_team(const FusedArgs& a, bool pgd, cudaStream_t s, long long* nblocks, bool taped = false) {
  // The unfolded kernel takes the Team's launch bounds; the PGD kernel (power
  // iteration prologue, more live state) keeps 256 x 1 (no register cap).
  auto kern = pgd ? (a.residual_tol > 0.f ? fused_kernel<S, true, UFPGD_PGD_MAXT, UFPGD_PGD_MINB, true>
                                          : fused_kernel<S, true, UFPGD_PGD_MAXT, UFPGD_PGD_MINB>)
                  : taped ? fused_kernel<S, false, S::MAXT, S::MINB, false, true> : fused_kernel<S, false, S::MAXT, S::MINB>;
  const int maxt = pgd ? UFPGD_PGD_MAXT : S::MAXT;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kFusedMaxWarps * (S::SMEM_PER_WARP + S::WSMEM_PER_WARP));
  if (e != cudaSuccess) return e;
  int nw = pick_warps(S::R, a.B);
  if (const int64_t f = option(UFPGD_OPT_FUSED_WARPS); f > 0) nw = static_cast<int>(f);
  nw = std::min(nw, maxt / 32);
  const long long rpb = static_cast<long long>(nw) * S::R;
  const long long blocks = (a.B + rpb - 1) / rpb;
  if (nblocks) *nblocks = blocks;
  kern<<<static_cast<unsigned>(blocks), nw * 32, nw * (S::SMEM_PER_WARP + S::WSMEM_PER_WARP), s>>>(a);
  return cudaGetLastError();
}

// Team shapes (K, M) -> (TK, TM): KA = K/TK = 2 users and MB = M/TM antennas
// per thread keep W, X' and the next X' in registers.
using Team_4_32 = Team<4, 32, 2, 4>;
// Small (4,32) batches (BASELINE config 1: 1,024 realizations = 256 four-team
// warps, under 2 per SM) are latency-bound: 16-thread teams (2 per warp, 4
// antennas per thread) give twice the warps — 14.0 vs 16.0 us at config 1
// (CUDA-graph replay, B200); at many waves the 8-thread team's shorter X'
// all-reduce wins.
using Team_4_32w = Team<4, 32, 2, 8>;
// Config 2's unfolded kernel: two sweeps per layer fit 168 registers without
// spills, so 3 resident 4-warp blocks (12 warps/SM) — 3% over 8 warps at 255.
#ifndef UFPGD_T864_MAXT
#define UFPGD_T864_MAXT 128
#endif
#ifndef UFPGD_T864_MINB
#define UFPGD_T864_MINB 3
#endif
#ifndef UFPGD_T864_TK
#define UFPGD_T864_TK 4
#endif
#ifndef UFPGD_T864_WSMEM
#define UFPGD_T864_WSMEM 0
#endif
using Team_8_64 = Team<8, 64, UFPGD_T864_TK, 16 / UFPGD_T864_TK, UFPGD_T864_MAXT, UFPGD_T864_MINB, UFPGD_T864_WSMEM,
                       UFPGD_T864_WSMEM ? false : UFPGD_TWO_SWEEP>;
// Neighbouring shapes of the BASELINE ones (the paper sweeps users and
// antennas around K = 8, M = 64) get the same fused kernel instead of the
// general one: 2 users x M/TM antennas per thread.
using Team_4_16 = Team<4, 16, 2, 4>;
using Team_4_64 = Team<4, 64, 2, 4>;
using Team_8_32 = Team<8, 32, 4, 4>;
using Team_8_128 = Team<8, 128, 4, 8, 128, 3>;

}  // namespace

bool fused_taped_supported(int K, int M) {
  return (K == 4 && (M == 16 || M == 32 || M == 64)) || (K == 8 && (M == 32 || M == 64 || M == 128));
}

cudaError_t launch_fused_taped(const FusedArgs& a, int K, int M, cudaStream_t s) {
  constexpr bool t = true;  // the taped instance
  if (K == 4 && M == 16) return launch_team<Team_4_16>(a, false, s, nullptr, t);
  if (K == 4 && M == 32) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (a.B / Team_4_32::R < 8LL * sms) return launch_team<Team_4_32w>(a, false, s, nullptr, t);
    return launch_team<Team_4_32>(a, false, s, nullptr, t);
  }
  if (K == 4 && M == 64) return launch_team<Team_4_64>(a, false, s, nullptr, t);
  if (K == 8 && M == 32) return launch_team<Team_8_32>(a, false, s, nullptr, t);
  if (K == 8 && M == 64) return launch_team<Team_8_64>(a, false, s, nullptr, t);
  if (K == 8 && M == 128) return launch_team<Team_8_128>(a, false, s, nullptr, t);
  return cudaErrorInvalidValue;
}

bool fused_supported(int K, int M) {
  return (K == 4 && (M == 16 || M == 32 || M == 64)) || (K == 8 && (M == 32 || M == 64 || M == 128)) ||
         (K == 16 && M == 128) || (K == 32 && M == 256);
}

// Upper bound on realizations per block (partials are sized with the smallest
// block the geometry chooser can pick: one warp).

int fused_realizations_per_block(int K, int M) {
  if (K == 4 && M == 16) return Team_4_16::R;
  if (K == 4 && M == 32) return Team_4_32w::R;  // the smaller of the two (4,32) teams' R
  if (K == 4 && M == 64) return Team_4_64::R;
  if (K == 8 && M == 32) return Team_8_32::R;
  if (K == 8 && M == 64) return 1;  // the tcgen05 pair kernel writes one partial per realization
  if (K == 8 && M == 128) return Team_8_128::R;
  return 1;  // tile kernels: one realization per block
}

cudaError_t launch_fused(const FusedArgs& a, bool pgd, int K, int M, cudaStream_t s, long long* nblocks) {
  if (K == 4 && M == 16) return launch_team<Team_4_16>(a, pgd, s, nblocks);
  if (K == 4 && M == 32) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (a.B / Team_4_32::R < 8LL * sms) return launch_team<Team_4_32w>(a, pgd, s, nblocks);
    return launch_team<Team_4_32>(a, pgd, s, nblocks);
  }
  if (K == 4 && M == 64) return launch_team<Team_4_64>(a, pgd, s, nblocks);
  if (K == 8 && M == 32) return launch_team<Team_8_32>(a, pgd, s, nblocks);
  if (K == 8 && M == 64) {
    if (mma_supported(K, M, pgd)) return launch_mma(a, pgd, K, M, s, nblocks);  // mma.cu: realization pairs
    return launch_team<Team_8_64>(a, pgd, s, nblocks);
  }
  if (K == 8 && M == 128) return launch_team<Team_8_128>(a, pgd, s, nblocks);
  return launch_tiled(a, pgd, K, M, s, nblocks);  // tile.cu: (16,128), (32,256)
}

}  // namespace ufpgd_gpu_impl
