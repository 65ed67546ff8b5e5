// Tensor-core (tcgen05 / TMEM) kernel for the unfolded forward and the
// fixed-step PGD at (K, M) = (32, 256) and (16, 128) — BASELINE configs 4 and
// 5, the "larger M x K x K complex contractions" north_star reserves the
// tensor cores for — and at (8, 64) (configs 2 and 3) as pairs of
// realizations in the (16, 128) frame (MmaShape PAIR). One CTA (thread =
// antenna) owns a realization (a pair) for all layers / iterations
// (unfolded.cpp:112-146, pgd.cpp:226-244):
//
//   stage 1  X  = W H^T           tcgen05.mma  M=4K N=4K K=M, by 128-antenna tile into one accumulator
//   stage 2  G  = (-eta X') H^*   tcgen05.mma  M=128 N=4K + N=2K, K=2K, per 128-antenna tile,
//                                              A = H from TMEM
//   prox     per-antenna group soft threshold on V = W + G, in registers
//
// Precision: FP32 products are split into f16 pairs, x = hi + 2^-11 lo
// (lo = f16((x - hi) * 2^11)), and every real product is formed as
// hi*hi + 2^-11 (hi*lo + lo*hi) with FP32 accumulation in TMEM — the
// "3-term split" whose error (~2^-22 relative) matches FP32 arithmetic (a
// numpy emulation of the whole 20-layer forward at config 4 gives 1.5e-7
// W relative error against the FP64 oracle vs 1.4e-7 for plain FP32). Each
// realization is scaled by an exact power of two g (max |g H| in [1, 2)) so
// the f16 range of H is never approached: X is invariant (W_s = W / g), the
// step becomes eta / g^2 and the threshold thr / g; realizations whose W or Bs
// operands would still leave the f16 range go to a range-robust instance.
//
// Real forms (rows r = (part, k), part 0 = Re, 1 = Im, r in [0, 2K)):
//   stage 1: D1[q][(p', k')] = sum_m Wop[q][m] Hop[(p', k')][m], q = (hilo, p, k)
//            (A = [W_hi; W_lo] 4K x M, MN-major; B = [H_hi | H_lo], K-major)
//            X_r = P[(0,k),(0,k')] - P[(1,k),(1,k')], X_i = P[(0,k),(1,k')] + P[(1,k),(0,k')]
//   stage 2: D2[m][(p, k)] = sum_(p', k') Hop[(p', k')][m] Bs[(p', k')][(p, k)]
//            (A = H as M x 2K, K-major f16 pairs in TMEM, staged once per
//            realization from the thread's own H row; Bs = the real form of
//            -eta X'^T in shared memory)
// so H (hi and lo, f16) is staged once, in shared memory for stage 1 and in
// TMEM for stage 2.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include <cuda_fp16.h>

#include "device_common.cuh"

namespace ufpgd_gpu_impl {
namespace {

// Shape of the tensor-core kernel: one thread per antenna (NT = M), 2K
// real-form rows r = (part, k), Q = 4K operand rows q = (hilo, part, k) for
// stage 1 (MMA M = Q: 128 at K = 32, 64 at K = 16), M / 128 stage-2 tiles.
// PAIR: the (16,128) frame holds two (8,64) realizations block-diagonally
// (BASELINE config 2's shape): H_pair = diag(H_a, H_b), so X, X' H^* and the
// per-antenna prox never mix the blocks. Thread m works on antenna m % 64 of
// realization m / 64 and holds only its realization's 8 users. Each
// realization's MMAs touch only its own operand blocks (stage 1: one N = 32
// chain over its antennas and H rows; stage 2: one K-step against its own Bs
// tile), and the split, drains, Bs build and prox cover only its 8 users: the
// frame's off-diagonal blocks are never staged, multiplied or read.
#ifndef UFPGD_MMA_DBS
#define UFPGD_MMA_DBS 1  // 0: the F / G shared-memory exchange between the stage-1 drain and the Bs build (A/B)
#endif
template <int K_, int M_, int MINB_, bool PAIR_ = false>
struct MmaShape {
  static constexpr int K = K_, M = M_, NT = M_, MINB = MINB_;
  static constexpr bool PAIR = PAIR_;
  // DBS ("direct Bs", the M = 64 stage-1 shapes): the stage-1 operand rows are
  // ordered q = (k / 4, part, hilo, k % 4), so TMEM lane quadrant w holds all
  // 16 rows of users 4w .. 4w+3 and the 16x256b drain gives thread i rows
  // i / 4 = (hilo, k % 4) of part 0 and part 1 together: the thread forms its
  // hi- or lo-row share of X(k, .) in registers, adds its partner's (lane ^ 16:
  // one shuffle per value) and splits / stores its Bs chunk at once. No F / G
  // exchange through shared memory and one CTA barrier less per layer.
  static constexpr bool DBS = (4 * K_ == 64) && UFPGD_MMA_DBS;
  static constexpr int KX = PAIR ? K_ / 2 : K_, MX = PAIR ? M_ / 2 : M_;  // per-realization users, antennas
  static_assert(!PAIR || (K_ == 16 && M_ == 128), "pairs of (8,64) realizations in the (16,128) frame");
  static constexpr int R = 2 * K;     // real-form rows (part, k)
  static constexpr int Q = 2 * R;     // stage-1 A rows (hilo, part, k) = stage-1 MMA M
  static constexpr int NTILE = M / 128;
  static constexpr int NW = NT / 32;
  static_assert(Q == 64 || Q == 128, "stage-1 MMA M must be 64 or 128");
  static_assert(M % 128 == 0 && NW <= 8 && K % 16 == 0, "");
  // shared-memory byte offsets (16-byte aligned, as the no-swizzle layouts need)
  static constexpr int OFF_HH = 0;                       // H hi  [R x M] f16, core layout hoff()
  static constexpr int OFF_HL = OFF_HH + R * M * 2;      // H lo
  // PAIR: H is only staged per realization (hoffp(): 8 KB instead of 16), so
  // the W operand follows right after it
  static constexpr int OFF_W = PAIR ? OFF_HH + 2 * 4 * 8 * 128 : OFF_HL + R * M * 2;  // [W_hi; W_lo] [Q x M] f16, woff()
  // Bs builder chunk width: 4 values of an X' row per thread, or 2 when K^2/4
  // chunks would leave threads idle (chunk() maps either conflict-free).
  static constexpr int CWD = (K * K / 4 >= NT) ? 4 : 2;
  // Bs K-group stride (descriptor LBO). DBS: 192 — the two half-warps of a
  // put write K-groups that differ by one, and 128 + 64 bytes apart they land
  // in different bank halves (conflict-free 4-byte stores).
  static constexpr int BLBO = DBS ? 192 : 128;
  static constexpr int BSBO = (R / 8) * BLBO;            // Bs N-group stride (descriptor SBO)
  static constexpr int BSBOP = 2 * BLBO, BST = 4 * BSBOP;  // PAIR: per-realization Bs tiles (boffp())
  static constexpr int OFF_BH = OFF_W + Q * M * 2;       // Bs hi [R x R] f16, boff()
  static constexpr int OFF_BL = OFF_BH + (R / 8) * BSBO; // Bs lo (continues Bs hi along N)
  // fp32 exchange rows (floats): 4 mod 32 words at CWD 4, 8 mod 32 at CWD 2 (see chunk())
  static constexpr int FSTR = R + (CWD == 4 ? 4 : 8);
  // F [R][FSTR] (hi rows of P) and G (lo rows) alias the W operand: they are
  // written after the stage-1 MMAs retire and read before W is rewritten.
  // PAIR: their own region after the two 1 KB Bs tiles, since the W operand
  // keeps the zeros of the other realization's users at each antenna (see the
  // shared accumulators below); 45.6 KB in all, so 5 CTAs fit an SM.
  // (PAIR with DBS: F is only the power iteration's 256-byte scratch and
  // aliases the Bs tiles, which are first written in the layer loop)
  static constexpr int OFF_F = PAIR ? (DBS ? OFF_BH : OFF_BH + 2 * BST) : OFF_W;
  // PAIR: only the diagonal 8 x 8 blocks of P are exchanged — rows (part, k)
  // with the 16 columns (part', k' of k's realization), 16 floats per row,
  // 8-word halves swapped on rows (row >> 1) odd (fx()): conflict-free for the
  // drain's stores and the Bs build's loads, 4 KB for F and G together.
  static constexpr int FROW = PAIR ? 16 : FSTR;  // floats per exchange row
  static constexpr int OFF_G = OFF_F + R * FROW * 4;
  static_assert(2 * R * FSTR * 4 <= Q * M * 2, "");
  static constexpr int OFF_BAR = PAIR ? (DBS ? OFF_BH + 2 * BST : OFF_G + R * FROW * 4)
                                      : OFF_BL + (R / 8) * BSBO;  // mbarriers, TMEM slot, reductions
  // exchange-row index of P(row, col): row = (part, k), col = (part', k'), frame indices
  static __device__ __forceinline__ int fx(int row, int col) {
    if constexpr (PAIR)
      return row * 16 + (((col / K) * 8 + col % 8) ^ (((row >> 1) & 1) << 3));
    else
      return row * FSTR + col;
  }
  static constexpr int SMEM = OFF_BAR + 512;
  // TMEM columns (fp32 accumulators)
  // D1: [X-part with H_hi | with H_lo] (2R columns; each antenna tile's K-steps
  // are issued as soon as that tile's W operand is written, tile 1's after tile
  // 0's); D2 per tile t: [main | corr] at column 2R t. D1 overlaps D2 tile 0:
  // tile 0's threads drain D2 tile 0 before its stage-1 MMAs are issued (tile
  // 1's wait for tile 0's issue), and D1 is drained behind a CTA barrier
  // before the stage-2 MMAs.
  static constexpr uint32_t T_D1A = 0, T_D1B = R, T_D2 = 0;
  // Stage 2's A operand (H hi / lo, K-major f16 pairs: R / 2 columns each per
  // tile) lives in TMEM from the prologue on, so the stage-2 MMAs read only
  // Bs from shared memory: shared-memory bandwidth (LSU traffic plus the MMAs'
  // operand reads) is what the (16,128) kernel runs out of first.
  static constexpr uint32_t T_HA = 2 * NTILE * R;
  static constexpr uint32_t T_USED = T_HA + NTILE * R;
  static constexpr uint32_t T_COLS = T_USED <= 32 ? 32 : T_USED <= 64 ? 64 : T_USED <= 128 ? 128 : T_USED <= 256 ? 256 : 512;
  static_assert(T_USED <= 512, "");
  // PAIR, fast path ("shared"): both realizations' stage-1 chains accumulate
  // into one 32-column D1 and both stage-2 K-steps into one 32-column D2 — the
  // other realization's terms are exact zeros (zero W-operand entries, zero
  // TMEM A columns) — so a CTA needs 64 TMEM columns and 5 CTAs fit an SM.
  // Exact only while both realizations stay finite (0 * Inf = NaN): a pair
  // with a non-finite value is handed to the range-robust instance, which
  // keeps separate columns per realization (D1 / D2 at 32 x, A at T_HA).
  static constexpr uint32_t T_HA_SH = 32, T_COLS_SH = 64;

  // Canonical no-swizzle layouts: 8 x 16-byte core matrices (128 contiguous bytes).
  // H: element (r, m); core (r / 8, m / 8); inside: row r % 8 (16 B), m % 8 (2 B).
  //   stage 1 B (K-major, N = r, K = m): LBO (K-group) 128, SBO (N-group) 16 M
  //   stage 2 A (MN-major, MN = m, K = r): LBO (K-group) 16 M, SBO (MN-group) 128
  static __device__ __forceinline__ int hoff(int r, int m) {
    return (r >> 3) * (16 * M) + (m >> 3) * 128 + (r & 7) * 16 + (m & 7) * 2;
  }
  // PAIR: realization x's stage-1 B operand alone, K-major: N-groups g = (hilo,
  // part) of its 8 users (rows kl), K-groups of 8 of its 64 antennas (ml):
  // LBO 128, SBO 1024 — the [hi p0 | hi p1 | lo p0 | lo p1] order of its chain.
  static __device__ __forceinline__ int hoffp(int x, int g, int kl, int ml) {
    return x * 4096 + g * 1024 + (ml >> 3) * 128 + kl * 16 + (ml & 7) * 2;
  }
  // W operand: element (q, m), MN-major (MN = q, K = m): core (q / 8, m / 8);
  // inside: row m % 8 (16 B), q % 8 (2 B). LBO (K-group) 16 Q, SBO 128.
  static __device__ __forceinline__ int woff(int q, int m) {
    return (m >> 3) * (16 * Q) + (q >> 3) * 128 + (m & 7) * 16 + (q & 7) * 2;
  }
  // Stage-1 operand row of (hilo, part, frame user k).
  static __device__ __forceinline__ int qrow(int hl, int part, int k) {
    if constexpr (DBS)
      return (k >> 2) * 16 + part * 8 + hl * 4 + (k & 3);
    else
      return hl * R + part * K + k;
  }
  // Bs builder chunk ch -> X' row k, columns c .. c + CWD - 1 (= Bs rows kk, column n = k).
  // CWD 4: each half-warp covers one 8 x 8 block of X' — rows k0 .. k0+7 (lanes
  // i & 7) x two 4-wide column halves (i >> 3) — so every Bs put of the half-warp
  // fills one whole 128-byte core matrix (conflict-free 8-byte stores), and each
  // quarter-warp reads 8 rows of one column chunk of the F / G exchange rows
  // (row stride FSTR = 4 mod 32 words: conflict-free 16-byte loads).
  // CWD 2 (the (16,128) shape, whose M = 64 stage-1 drain reads TMEM with the
  // 16x256b shape: thread i holds rows i / 4 and i / 4 + 8, column pairs
  // 2 (i % 4)): each warp covers one 8 x 8 block of X' — rows (i & 3) +
  // 4 (i >> 4) x four 2-wide column chunks ((i >> 2) & 3) — so every 4-byte Bs
  // put of the warp fills one whole core matrix, and each half-warp's 8-byte
  // F / G loads cover 4 rows x 8 consecutive words (FSTR = 8 mod 32), as do the
  // drain's 8-byte stores: all conflict-free.
  static __device__ __forceinline__ void chunk(int ch, int& k, int& c) {
    if constexpr (CWD == 4) {
      const int hw = ch >> 4, i = ch & 15;
      k = (hw / (K / 8)) * 8 + (i & 7);
      c = (hw % (K / 8)) * 8 + (i >> 3) * 4;
    } else {
      const int w = ch >> 5, i = ch & 31;
      k = (w / (K / 8)) * 8 + (i & 3) + 4 * (i >> 4);
      c = (w % (K / 8)) * 8 + ((i >> 2) & 3) * 2;
    }
  }
  // Bs: element (kk, n), K-major (K = kk, N = n): LBO (K-group) 128, SBO (N-group) BSBO.
  static __device__ __forceinline__ int boff(int kk, int n) {
    return (kk >> 3) * BLBO + (n >> 3) * BSBO + (n & 7) * 16 + (kk & 7) * 2;
  }
  // PAIR: stage 2 runs one K-step per realization x (the TMEM A operand's
  // K order is r' = (x, part, k_local)), so Bs is one tile per realization:
  // [16 K-rows (p_in, k'_local) x 32 N-columns ((p_out, k_local) hi | lo)],
  // K-major, N-group stride BSBOP, tile x at x * BST, lo after the 2 hi N-groups.
  static __device__ __forceinline__ int boffp(int kk, int n) {
    return (kk >> 3) * BLBO + (n >> 3) * BSBOP + (n & 7) * 16 + (kk & 7) * 2;
  }
  // Byte offset from OFF_BH of the (p_in, p_out) Bs entry of X'(k, c .. c+CWD-1)
  // (frame users k, c), and of its lo part from its hi part.
  static __device__ __forceinline__ int bpos(int pin, int pout, int k, int c) {
    if constexpr (PAIR)
      return (k / KX) * BST + boffp(pin * KX + c % KX, pout * KX + k % KX);
    else
      return boff(pin * K + c, pout * K + k);
  }
  static constexpr int BLO = PAIR ? 2 * BSBOP : (R / 8) * BSBO;
};

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Instruction descriptor, kind::f16: f16 A/B, f32 D, A MN-major, B K-major.
template <int MM, int NN>
__device__ __forceinline__ constexpr uint32_t idesc_f16_amn() {
  return (1u << 4) | (1u << 15) | (static_cast<uint32_t>(NN >> 3) << 17) | (static_cast<uint32_t>(MM >> 4) << 24);
}
// The same with A K-major (A from TMEM).
template <int MM, int NN>
__device__ __forceinline__ constexpr uint32_t idesc_f16_ak() {
  return (1u << 4) | (static_cast<uint32_t>(NN >> 3) << 17) | (static_cast<uint32_t>(MM >> 4) << 24);
}
// MMA issue, executed by a whole warp with warp-uniform operands; one lane
// (elect.sync) issues. Issued from a single thread inside a thread-divergent
// branch, ptxas moved every descriptor through R2UR and an ELECT loop: ~48
// clocks per MMA, against back-to-back UTCHMMAs from uniform registers here
// (tools/probe/stage_probe.cu: 4 MMAs issued in 40 clocks instead of 284, and an
// 8-MMA chain done at 618 instead of 680 clocks).
__device__ __forceinline__ void umma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// tcgen05 shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// umma_f16w: the descriptors passed as their two 32-bit words (used at
// (16,128); at (32,256) ptxas already keeps umma_f16's 64-bit descriptors in
// uniform registers across the layer loop, and the split form measured 1%
// slower there — it routed them through R2UR): the low word (start address
// >> 4 | LBO >> 4 << 16) is a per-layer base plus a compile-time K-step offset (the 14-bit address field
// never carries into LBO: shared addresses are < 256 KB), the high word (SBO >> 4,
// version bit 46) a constant — one uniform add per descriptor instead of the
// shifts and masks recomputed for each MMA (~70 uniform instructions between the
// barrier and the first stage-1 MMA at (16,128), on the per-layer critical path).
__device__ __forceinline__ void umma_f16w(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                          uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b64 da, db;\nmov.b64 da, {%1, %2};\nmov.b64 db, {%3, %4};\n"
      "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %6, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n}\n" ::"r"(d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc));
}
// A from TMEM (K-major, [a_tmem]), B from a shared-memory descriptor.
__device__ __forceinline__ void umma_f16_ta(uint32_t d, uint32_t a, uint32_t blo, uint32_t bhi, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b64 db;\nmov.b64 db, {%2, %3};\n"
      "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %5, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n}\n" ::"r"(d),
      "r"(a), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_f16_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint32_t sdesc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr >> 4) & 0x3FFFu) | (((lbo >> 4) & 0x3FFFu) << 16);
}
__host__ __device__ constexpr uint32_t sdesc_hi(uint32_t sbo) { return ((sbo >> 4) & 0x3FFFu) | (1u << 14); }
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// UNROLL 4: four try_waits per round of the guard counter, each followed only
// by its exit branch — the spin loop's own instructions take issue slots (at
// (32,256), one CTA per SM: -2% per launch); UNROLL 1 measured better at
// (16,128), where 4 CTAs share the SM.
template <int UNROLL>
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  static_assert(UNROLL == 1 || UNROLL == 4, "");
  for (uint32_t round = UNROLL == 4 ? (1u << 26) : (1u << 28);; --round) {
    uint32_t ok;
    if constexpr (UNROLL == 4) {
      asm volatile(
          "{\n.reg .pred p;\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "@p bra.uni MBW_DONE;\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "@p bra.uni MBW_DONE;\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "@p bra.uni MBW_DONE;\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "MBW_DONE:\n"
          "selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(bar), "r"(parity)
          : "memory");
    } else {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(bar), "r"(parity)
          : "memory");
    }
    if (ok) return;
    if (round == 0) __trap();  // never hang the GPU on a lost arrive
  }
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// 16 consecutive TMEM columns of this warp's 32 lanes -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
}
// 16 lanes x 32 columns (from the 16-lane group at taddr): thread i gets rows
// i / 4 (v[4 j], v[4 j + 1]) and i / 4 + 8 (v[4 j + 2], v[4 j + 3]) at columns
// 8 j + 2 (i % 4) + {0, 1}, j = 0..3 (layout measured: tools/probe/tmem_layout.cu).
__device__ __forceinline__ void tmem_ld16x256(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
}
// 8 consecutive TMEM columns of this warp's 32 lanes -> 8 registers per thread.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "r"(taddr));
}
// 8 registers per thread -> 8 consecutive TMEM columns of this warp's 32 lanes.
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
// 16 registers per thread -> 16 consecutive TMEM columns of this warp's 32 lanes.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// Waits for this thread's tcgen05.ld results; the laundering asm keeps every
// use of v after the wait.
template <int N>
__device__ __forceinline__ void tmem_wait(float* v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+f"(v[i]));
}
// f16 pair split of (a, b): hi = f16(x), lo = f16((x - hi) * 2^11).
// The residual hi - x comes from the mixed-precision add (add.f32.f16: one
// FHADD reading the f16 half in place, so hi is never converted back to FP32 —
// 5 instructions per pair instead of 6; the f16 splits were ~24% of the
// (16,128) kernel's instructions), scaled by -2^11 as one packed FMUL2. Both
// steps are exact (x - hi is representable), so the bits are those of the
// FP32 residual.
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const uint32_t hb = *reinterpret_cast<const uint32_t*>(&h);
  float d0, d1;
  asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(d0) : "h"(static_cast<unsigned short>(hb & 0xffffu)), "f"(-a));
  asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(d1) : "h"(static_cast<unsigned short>(hb >> 16)), "f"(-b));
  const float2 r = __fmul2_rn(make_float2(d0, d1), make_float2(-2048.f, -2048.f));
  const __half2 l = __floats2half2_rn(r.x, r.y);
  hi = hb;
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ uint16_t f16_bits(__half h) { return *reinterpret_cast<const uint16_t*>(&h); }

constexpr float kLoScale = 1.f / 2048.f;

// 2^e as a float, |e| <= 126 (exact).
__device__ __forceinline__ float pow2i(int e) { return __int_as_float((127 + e) << 23); }

// Fixed-step power iteration on H^T H^* (pgd.cpp:146-162 with the BASELINE
// 30-step rule), FP32 on the unscaled H, one thread per antenna:
// u = H^* v reduced over the CTA (shuffles, then per-warp partials in `scr`),
// w_m = sum_k H(k, m) u_k in-thread, Rayleigh quotient Re(v^H w) of the last step.
// PAIR: each realization over its own half of the CTA (its users, its warps).
template <class T>
__device__ float cta_power(const float4 (&hv)[T::KX / 2], const float2* v0, int steps, float* scr, float* red,
                           int warp, int lane, int hx) {
  constexpr int K = T::KX, NWX = T::PAIR ? T::NW / 2 : T::NW;
  const int m = threadIdx.x % T::MX;  // the antenna within the thread's realization
  float2 v = v0[m];
  float est = 0.f;
  bool zero = false;
  for (int st = 0; st < steps; ++st) {
    float u[2 * K];  // (Re, Im) of conj(H(k, m)) v_m, then of u_k
#pragma unroll
    for (int j = 0; j < K / 2; ++j) {
      u[4 * j + 0] = hv[j].x * v.x + hv[j].y * v.y;  // conj(h) v = (hr vr + hi vi, hr vi - hi vr)
      u[4 * j + 1] = hv[j].x * v.y - hv[j].y * v.x;
      u[4 * j + 2] = hv[j].z * v.x + hv[j].w * v.y;
      u[4 * j + 3] = hv[j].z * v.y - hv[j].w * v.x;
    }
#pragma unroll
    for (int i = 0; i < 2 * K; ++i)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) u[i] += __shfl_xor_sync(kFull, u[i], off);
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < 2 * K; ++i) scr[warp * 2 * K + i] = u[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) {
      float a = 0.f;
#pragma unroll
      for (int w = hx * NWX; w < (hx + 1) * NWX; ++w) a += scr[w * 2 * K + i];
      u[i] = a;
    }
    float2 wm = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < K / 2; ++j) {
      cmac(wm, make_float2(hv[j].x, hv[j].y), make_float2(u[4 * j], u[4 * j + 1]));
      cmac(wm, make_float2(hv[j].z, hv[j].w), make_float2(u[4 * j + 2], u[4 * j + 3]));
    }
    float dot = fmaf(v.x, wm.x, v.y * wm.y), wn2 = fmaf(wm.x, wm.x, wm.y * wm.y);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dot += __shfl_xor_sync(kFull, dot, off);
      wn2 += __shfl_xor_sync(kFull, wn2, off);
    }
    __syncthreads();  // scr reads done before the next step's writes
    if (lane == 0) {
      red[warp] = dot;
      red[16 + warp] = wn2;
    }
    __syncthreads();
    dot = 0.f;
    wn2 = 0.f;
#pragma unroll
    for (int w = hx * NWX; w < (hx + 1) * NWX; ++w) {
      dot += red[w];
      wn2 += red[16 + w];
    }
    __syncthreads();
    if (!zero) {
      if (wn2 == 0.f) {
        zero = true;
        est = 0.f;
      } else {
        est = dot;
        const float inv = 1.f / sqrtf(wn2);
        v = make_float2(wm.x * inv, wm.y * inv);
      }
    }
  }
  return est;
}

// RB = false (fast path): one CTA per realization; a realization that needs
// the range-robust path is appended to redo_list instead of writing its
// per-realization outputs. RB = true (range-robust path): a grid-stride loop
// over the redo_list entries (normally none). The body is written inline in
// the kernel (a device-function body taking the params by reference measured
// 3% slower at (16,128)).
// RESID (PGD pairs only): solve_pgd's residual_tol early stop per realization
// (pgd.cpp:246-260; see the layer loop).
template <class T, bool PGD, bool RB, bool RESID = false>
__global__ void __launch_bounds__(T::NT, RB ? 1 : T::MINB)
    mma_kernel(const __grid_constant__ FusedArgs p, int* redo_list, int* redo_count) {
  static_assert(!RESID || (PGD && T::PAIR), "the early stop is built for the (8,64) PGD pairs");
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int K = T::K, M = T::M, R = T::R, Q = T::Q, NW = T::NW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wu = __shfl_sync(kFull, warp, 0);  // warp index the compiler knows is warp-uniform
  const int n_real = RB ? *redo_count : 1;
  for (int it = RB ? static_cast<int>(blockIdx.x) : 0; it < n_real; it += RB ? static_cast<int>(gridDim.x) : 1) {
  const long long rid = RB ? static_cast<long long>(redo_list[it]) : static_cast<long long>(blockIdx.x);
  // the thread's realization (PAIR: 2 rid + tid / 64) and its antenna there
  constexpr int KT = T::KX;  // users per thread
  constexpr bool SH = T::PAIR && !RB;  // pair with shared accumulators (see MmaShape)
  constexpr uint32_t THA = SH ? T::T_HA_SH : T::T_HA, TCOLS = SH ? T::T_COLS_SH : T::T_COLS;
  const int hx = T::PAIR ? tid / T::MX : 0;
  const long long rx = T::PAIR ? 2 * rid + hx : rid;
  const bool xvalid = !T::PAIR || rx < p.B;  // PAIR: an odd batch's last CTA has one realization
  const int ml = T::PAIR ? tid % T::MX : tid;
#ifdef UFPGD_MMA_TIMING
  long long pst[7];  // prologue / epilogue stamps of the probe CTA (see tst below)
#define PSTAMP(i) pst[i] = clock64();
  PSTAMP(0)
#else
#define PSTAMP(i)
#endif
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar1 = sb + T::OFF_BAR;                // + 8 t: stage-1 part t done
  const uint32_t bar2 = sb + T::OFF_BAR + 8 * T::NTILE;  // + 8 t: stage-2 tile t done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + T::OFF_BAR + 48);
  float* red = reinterpret_cast<float*>(smem + T::OFF_BAR + 64);           // [2][16]
  long long* fbs = reinterpret_cast<long long*>(smem + T::OFF_BAR + 192);  // [16]
  float* redw = reinterpret_cast<float*>(smem + T::OFF_BAR + 320);         // [16]: robust-path maxima
  float* rsd = reinterpret_cast<float*>(smem + T::OFF_BAR + 384);          // [NW][2]: early-stop partials

  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < 2 * T::NTILE; ++b) mbar_init(bar1 + 8 * b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(TCOLS)
                 : "memory");
    // (the robust kernel allocates again for its next realization)
    if (!RB) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }

  // The realization that will most likely take this CTA slot next (blocks are
  // dispatched in order, one wave = prefetch_ahead CTAs) gets its H pulled into
  // L2 now, so its prologue loads hit L2 instead of waiting on HBM: with one
  // CTA per SM at (32,256) nothing else overlaps a prologue (the launch's
  // L-independent cost was ~15% of config 4 before).
  if (!RB && tid == 0 && p.prefetch_ahead > 0) {
    constexpr int RPC = T::PAIR ? 2 : 1;  // realizations per CTA
    const long long r0 = (rid + p.prefetch_ahead) * RPC, nr = min(static_cast<long long>(RPC), p.B - r0);
    if (nr > 0) {
      const float2* nh = p.H + r0 * T::MX * T::KX;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nh),
                   "r"(static_cast<uint32_t>(nr * T::MX * T::KX * 8))
                   : "memory");
    }
  }
  // ---- H row of antenna m = tid: registers, max |.| over the realization ----
  const int m = tid;
  float4 hv[KT / 2];  // hv[j] = (Re H(2j, m), Im H(2j, m), Re H(2j+1, m), Im H(2j+1, m)) of the thread's realization
  {
    const float4* hg = reinterpret_cast<const float4*>(p.H + (rx * T::MX + ml) * KT);
    // (16,128) and pairs: L1-allocating loads, so the staging items' re-read of
    // the same lines below hits L1 (config 5 -1.5%, config 2 -0.7%); at (32,256)
    // the 144 KB of shared memory leaves too little L1 (+0.4%): streaming loads
    constexpr bool L1 = T::K < 32;
#pragma unroll
    for (int j = 0; j < KT / 2; ++j)
      hv[j] = xvalid ? (L1 ? __ldg(hg + j) : ldg_stream(hg + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // The shared-memory H staging works on items (user pair j, group of 8
  // antennas G) instead of the thread's own antenna: 8 antennas of one row r
  // fill one 16-byte core-matrix row, so each item writes 16-byte rows
  // (STS.128) where the thread-per-antenna layout needed 2-byte stores that
  // four antenna groups of a warp sent to the same banks (~770 excess
  // wavefronts per realization at (16,128)). Its loads re-read H (L2 hits)
  // and are issued before the CTA barrier.
  constexpr int NJ = K / 2, NIT = NJ * (M / 8) / T::NT;
  static_assert(NJ * (M / 8) % T::NT == 0 && NJ % 8 == 0, "");
  float4 hs[NIT][8];  // hs[q][i] = (Re, Im) of H(2j, 8G + i), H(2j + 1, 8G + i)
#pragma unroll
  for (int q = 0; q < NIT; ++q) {
    const int it = tid + q * T::NT, j = it % NJ, G = it / NJ;
    if constexpr (T::PAIR) {
      // frame user pair j, antenna group G: realization G / 8 (= hx here); the
      // off-diagonal items (j / 4 != G / 8) are never read by stage 1: skipped
      const bool diag = (j / (T::KX / 2)) == (G / (T::MX / 8));
      const float4* hg = reinterpret_cast<const float4*>(p.H + (rx * T::MX + 8 * (G % (T::MX / 8))) * KT) +
                         j % (T::KX / 2);
#pragma unroll
      for (int i = 0; i < 8; ++i) hs[q][i] = diag && xvalid ? __ldg(hg + i * (KT / 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const float4* hg = reinterpret_cast<const float4*>(p.H + (rid * M + 8 * G) * K) + j;
#pragma unroll
      for (int i = 0; i < 8; ++i)  // (32,256): streaming, as the row loads (-0.3%)
        hs[q][i] = T::K < 32 ? __ldg(hg + i * (K / 2)) : ldg_stream(hg + i * (K / 2));
    }
  }
  float amax = 0.f;
  bool bad = false;  // fmaxf drops NaN: a non-finite channel keeps g = 1 (and diverges at layer 0)
#pragma unroll
  for (int j = 0; j < KT / 2; ++j) {
    const float a = fmaxf(fmaxf(fabsf(hv[j].x), fabsf(hv[j].y)), fmaxf(fabsf(hv[j].z), fabsf(hv[j].w)));
    amax = fmaxf(amax, a);
    bad |= !(fabsf(hv[j].x) + fabsf(hv[j].y) + fabsf(hv[j].z) + fabsf(hv[j].w) <= FLT_MAX);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(kFull, amax, off));
  const unsigned anybad = __ballot_sync(kFull, bad);
  if (lane == 0) {
    red[warp] = amax;
    red[16 + warp] = anybad ? 1.f : 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  PSTAMP(1)
  const uint32_t tmem = *tslot;
  float gmax = 0.f, gbad = 0.f;  // over the thread's realization (PAIR: its half of the warps)
  constexpr int NWX = T::PAIR ? NW / 2 : NW;
#pragma unroll
  for (int w = 0; w < NWX; ++w) {
    gmax = fmaxf(gmax, red[hx * NWX + w]);
    gbad = fmaxf(gbad, red[16 + hx * NWX + w]);
  }
  // g = 2^-e with gmax in [2^e, 2^(e+1)): g * gmax in [1, 2). Exact scaling.
  float g = 1.f;
  if (gbad == 0.f && gmax > 0.f) g = ldexpf(1.f, -ilogbf(gmax));
  const float ginv = 1.f / g;  // exact (power of two)

  // ---- stage H (hi / lo f16) in the shared core layout -------------------------
  // Item (j, G) writes rows Re 2j, Re 2j+1, Im 2j, Im 2j+1 over antennas 8G..8G+7.
  // Rows 2j and 2j + 1 go out in swapped order for j & 4, so the 8 lanes of a
  // quarter-warp (j = 8n .. 8n+7) hit the 8 distinct 16-byte rows of a core
  // matrix pair: conflict-free.
#pragma unroll
  for (int q = 0; q < NIT; ++q) {
    const int it = tid + q * T::NT, j = it % NJ, G = it / NJ;
    if (T::PAIR && (j / (T::KX / 2)) != (G / (T::MX / 8))) continue;  // off-diagonal item: not staged
    const bool swp = (j >> 2) & 1;
#pragma unroll
    for (int s = 0; s < 2; ++s) {      // user 2j + (s ^ swp)
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        uint32_t hh[4], hl[4];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float4 a = hs[q][i], b = hs[q][i + 1];
          const bool up = (s == 1) != swp;  // user 2j + 1
          const float va = part == 0 ? (up ? a.z : a.x) : (up ? a.w : a.y);
          const float vb = part == 0 ? (up ? b.z : b.x) : (up ? b.w : b.y);
          split2(va * g, vb * g, hh[i / 2], hl[i / 2]);
        }
        const int r = part * K + 2 * j + ((s == 1) != swp ? 1 : 0);
        if constexpr (T::PAIR) {
          const int x = G / (T::MX / 8), kl = r % T::KX, ml = 8 * (G % (T::MX / 8));
          *reinterpret_cast<uint4*>(smem + T::OFF_HH + T::hoffp(x, part, kl, ml)) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
          *reinterpret_cast<uint4*>(smem + T::OFF_HH + T::hoffp(x, 2 + part, kl, ml)) =
              make_uint4(hl[0], hl[1], hl[2], hl[3]);
        } else {
          *reinterpret_cast<uint4*>(smem + T::OFF_HH + T::hoff(r, 8 * G)) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
          *reinterpret_cast<uint4*>(smem + T::OFF_HL + T::hoff(r, 8 * G)) = make_uint4(hl[0], hl[1], hl[2], hl[3]);
        }
      }
    }
  }
  fence_async_smem();  // H is read by the tensor cores (async proxy)
  PSTAMP(2)
  // Stage 2's A operand in TMEM: antenna m's row (K-major, r = part K + k) in
  // TMEM lane m % 128 of its tile's H columns — the same f16 values (same
  // rounding) as the shared copy stage 1 reads. Ordered before the first
  // stage-2 MMA by tcgen05.wait::st and the fenced CTA barriers of layer 0.
  if constexpr (T::PAIR) {
    // K order r' = (x, part, k_local): the thread's realization fills K-step hx
    // (8 columns of hi, 8 of lo), the other K-step is zeros (both K-steps
    // accumulate into one D2)
    const uint32_t th = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + THA;
    uint32_t hh[16], hl[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // columns (part, users 2 c' .. 2 c' + 1), c' = c % 4
      const int part = c / 4, kl = 2 * (c % 4);
      const float4 hq = hv[kl / 2];
      uint32_t h, l;
      split2((part == 0 ? hq.x : hq.y) * g, (part == 0 ? hq.z : hq.w) * g, h, l);
      hh[c] = hx == 0 ? h : 0u;
      hh[8 + c] = hx == 1 ? h : 0u;
      hl[c] = hx == 0 ? l : 0u;
      hl[8 + c] = hx == 1 ? l : 0u;
    }
    tmem_st16(th, hh);
    tmem_st16(th + R / 2, hl);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else {
    const uint32_t th = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + T::T_HA + (m >> 7) * R;
#pragma unroll
    for (int half = 0; half < R / 32; ++half) {  // 16 columns = 32 rows r per store
      uint32_t hh[16], hl[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int r = half * 32 + 2 * c;  // rows r, r + 1: one part, users k, k + 1 (K even)
        const int part = r / K, k = r % K;
        const float4 hq = hv[k / 2];
        split2((part == 0 ? hq.x : hq.y) * g, (part == 0 ? hq.z : hq.w) * g, hh[c], hl[c]);
      }
      tmem_st16(th + half * 16, hh);
      tmem_st16(th + R / 2 + half * 16, hl);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  PSTAMP(3)

  // ---- W0 (scaled: W_s = W / g) in registers: wr[k], wi[k] for antenna m ------
  float wr[KT], wi[KT];
  if (p.w0_mode == UFPGD_W0_CONJ_H) {
#pragma unroll
    for (int j = 0; j < KT / 2; ++j) {
      wr[2 * j] = hv[j].x * ginv;
      wi[2 * j] = -hv[j].y * ginv;
      wr[2 * j + 1] = hv[j].z * ginv;
      wi[2 * j + 1] = -hv[j].w * ginv;
    }
  } else if (p.w0_mode == UFPGD_W0_GIVEN) {
    const float4* wg0 = reinterpret_cast<const float4*>(p.W0 + (rx * T::MX + ml) * KT);
#pragma unroll
    for (int j = 0; j < KT / 2; ++j) {
      const float4 v = xvalid ? wg0[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      wr[2 * j] = v.x * ginv;
      wi[2 * j] = v.y * ginv;
      wr[2 * j + 1] = v.z * ginv;
      wi[2 * j + 1] = v.w * ginv;
    }
  } else {
#pragma unroll
    for (int k = 0; k < KT; ++k) wr[k] = wi[k] = 0.f;
  }
  if constexpr (T::PAIR) {
    // zeros of the other realization's users at this antenna in the W operand,
    // written once (the split only rewrites the thread's own rows, F / G have
    // their own region): the other realization's stage-1 chain accumulates
    // exactly 0 onto this realization's D1 rows. Ordered before the first
    // stage-1 MMA by the split's fence and barrier.
    // (8-row chunks: DBS (quadrant, part) of the other realization's two
    // quadrants, else (hilo, part) of its 8 users)
#pragma unroll
    for (int hl = 0; hl < 2; ++hl)
#pragma unroll
      for (int part = 0; part < 2; ++part)
        *reinterpret_cast<uint4*>(smem + T::OFF_W +
                                  T::woff(T::DBS ? T::qrow(0, part, T::KX * (1 - hx) + 4 * hl)
                                                 : T::qrow(hl, part, T::KX * (1 - hx)), m)) =
            make_uint4(0u, 0u, 0u, 0u);
  }
  int aW = 0;        // robust path: the W registers hold W_s 2^-aW ...
  float wn2 = 0.f;   // ... and ||w_m||^2 in that domain
  if (RB) {
#pragma unroll
    for (int k = 0; k < KT; ++k) wn2 = fmaf(wr[k], wr[k], fmaf(wi[k], wi[k], wn2));
  }

  constexpr uint32_t IDESC1 = idesc_f16_amn<Q, 2 * R>();
  constexpr uint32_t IDESC1P = idesc_f16_amn<Q, R>();  // PAIR: per-realization N = 32
  constexpr uint32_t IDESC2W = idesc_f16_ak<128, 2 * R>();  // A = H from TMEM (K-major)
  constexpr uint32_t IDESC2 = idesc_f16_ak<128, R>();
  constexpr uint32_t IDESC2PW = idesc_f16_ak<128, 32>(), IDESC2P = idesc_f16_ak<128, 16>();  // PAIR
  static_assert(T::OFF_HL == T::OFF_HH + (R / 8) * 16 * M && T::OFF_BL == T::OFF_BH + (R / 8) * T::BSBO,
                "lo operands continue the hi ones along N");
  float* F = reinterpret_cast<float*>(smem + T::OFF_F);
  float* G = reinterpret_cast<float*>(smem + T::OFF_G);
  uint32_t ph1 = 0, ph2 = 0;  // stage-1 barrier (skipped at a W0 = 0 layer 0), stage-2 tile barriers
  bool nonfinite = false;
  long long first_bad = -1;
  float l21 = 0.f;
  int act = 0;
  const float g2inv = ginv * ginv;
  const int tile = m >> 7;
  const uint32_t lrow = static_cast<uint32_t>((warp & 3) * 32) << 16;  // this warp's TMEM lane quadrant

#ifdef UFPGD_MMA_TIMING
  // development probe: thread 0 of realization 5000 stamps the phases of layer 10
  // into its own W output (a timing-only build; W is garbage there)
  long long tst[10];
  const bool probe = (rid == 5000 && tid == 0);
#define TSTAMP(i) \
  if (probe && l == 10) tst[i] = clock64();
#else
#define TSTAMP(i)
#endif
  float eta_b = 0.f, thr_b = 0.f;  // PGD: the realization's fixed step 1/L and threshold lambda/L
  if constexpr (PGD) {
    if (p.eta_in) {
      eta_b = xvalid ? p.eta_in[rx] : 1.f;
    } else {
      eta_b = 1.f / cta_power<T>(hv, p.v0, p.power_steps, F, red, warp, lane, hx);  // F: free before stage 1
      if (!xvalid) eta_b = 1.f;  // phantom partner (zero channel: L = 0)
    }
    thr_b = p.lambda * eta_b;
    if (p.eta_out && tid == hx * (T::NT / (T::PAIR ? 2 : 1)) && xvalid) p.eta_out[rx] = eta_b;
  }
  PSTAMP(4)
  // RESID: a realization whose relative iterate change ||W_new - W|| / max(||W||,
  // 1e-12) fell below residual_tol after iteration l stops there (taken = l + 1;
  // its statistics are those of that iteration): from then on its step and
  // threshold are 0, so every further iteration is exactly the identity while
  // its partner runs on, and the CTA leaves once both have stopped. The
  // per-warp sums of |dW|^2 and |W|^2 of iteration l are read after the next
  // iteration's split barrier (no extra barrier per iteration); "stopped after
  // l" is just "the criterion held at l", since a stopped realization's dW is 0.
  bool stopped = false;
  long long taken = 0;
  float l21_prev = 0.f, l21_keep = 0.f;
  int act_prev = 0, act_keep = 0;
  const float tol2 = RESID ? p.residual_tol * p.residual_tol : 0.f;
  float wor[RESID ? KT : 1], woi[RESID ? KT : 1];  // W before the iteration's update
  (void)wor;
  (void)woi;
#ifndef UFPGD_MMA_CDIAG
#define UFPGD_MMA_CDIAG 1  // 0: the diagonal test and c[k] load inside the layer loop (A/B)
#endif
  // DBS fast path: the thread's share of diag(c) in its Bs chunk (see the Bs
  // build), fixed for the realization: c[k] where chunk column c + u is the
  // row's own user k (and the chunk holds Xr), else 0.
  float cdg[2] = {0.f, 0.f};
  // ... and the byte offsets of its Bs puts (PAIR: the hi-row lane stores the
  // (0,0) and (1,1) entries, the lo-row lane (1,0) and (0,1); full frame: the
  // other three entries are compile-time offsets from (0,0)).
  // Kept in registers across the layers where measured faster: the full frame
  // (config 5: 3.429 -> 3.397 ms per 65,536) and the PGD pairs (config 3:
  // 14.2 -> 13.65 ms); the unfolded pairs at their 72-register cap recompute
  // them per layer (0.965 vs 0.997 ms hoisted).
  constexpr bool HOIST_BO = UFPGD_MMA_CDIAG && (!T::PAIR || PGD);
  int bo1 = 0, bo2 = 0;
  if constexpr (T::DBS && UFPGD_MMA_CDIAG) {
    const int k = 4 * warp + ((lane >> 2) & 3);
    const int c = T::PAIR ? T::KX * (warp >> 1) + 2 * (lane & 3) : 2 * (lane & 3) + (lane >= 16 ? 8 : 0);
    if (!RB && (!T::PAIR || lane < 16)) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (c + u == k) cdg[u] = p.c[k];
    }
    if constexpr (HOIST_BO && T::PAIR) {
      bo1 = T::OFF_BH + (lane >= 16 ? T::bpos(1, 0, k, c) : T::bpos(0, 0, k, c));
      bo2 = T::OFF_BH + (lane >= 16 ? T::bpos(0, 1, k, c) : T::bpos(1, 1, k, c));
    } else if constexpr (HOIST_BO) {
      bo1 = T::OFF_BH + T::bpos(0, 0, k, c);
    }
  }
  (void)bo1;
  (void)bo2;
#ifndef UFPGD_MMA_CDQ
#define UFPGD_MMA_CDQ 1  // 0: (32,256) tests c + u == k and loads c[k] in every layer (A/B)
#endif
  // The exchange-path Bs build with one chunk per thread ((32,256)): the same
  // share of diag(c) for the thread's 4-wide chunk of X' row k.
  constexpr bool CDQ = UFPGD_MMA_CDQ && !T::DBS && !RB && !T::PAIR && (K * K / T::CWD == T::NT);
  float cdq[CDQ ? T::CWD : 1];
  if constexpr (CDQ) {
    int k, c;
    T::chunk(tid, k, c);
#pragma unroll
    for (int u = 0; u < T::CWD; ++u) cdq[u] = (c + u == k) ? p.c[k] : 0.f;
  }
  (void)cdq;
  for (long long l = 0; l < p.L; ++l) {
    TSTAMP(0)
    const bool xzero = (l == 0 && p.w0_mode == UFPGD_W0_ZERO);
    float ts = (PGD ? thr_b : p.thr[l]) * ginv;             // threshold in the scaled domain
    if constexpr (RB) {
      // exact max ||w_m|| of the register W over the CTA, brought to [2^12, 2^13)
      if (!xzero) {
        const float wm = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(wn2 >= 0.f ? wn2 : __int_as_float(0x7f800000))));
        if (lane == 0) redw[warp] = wm;
        __syncthreads();
        float mc2 = 0.f;
#pragma unroll
        for (int w = hx * NWX; w < (hx + 1) * NWX; ++w) mc2 = fmaxf(mc2, redw[w]);  // PAIR: own realization
        __syncthreads();  // redw is reused by the Bs maximum
        if (mc2 > 0.f && mc2 < FLT_MAX) {
          const int d = ilogbf(mc2) / 2 - 12;
          if (d != 0) {
            const float f = pow2i(-d);
#pragma unroll
            for (int k = 0; k < K; ++k) {
              wr[k] *= f;
              wi[k] *= f;
            }
            wn2 *= f * f;
            aW += d;
          }
        }
      }
      ts *= pow2i(-aW);
    }
    float fstep = -(PGD ? eta_b : p.eta[l]) * g2inv;  // -eta / g^2 folded into Bs
    // DBS: the thread's Bs chunk of X, straight from the stage-1 drain. Lane i
    // of warp w: X row k = 4w + (i / 4) % 4, hl = i / 16. Full frame: columns
    // c = 2 (i % 4) + 8 hl, dx = (Xr(k,c), Xr(k,c+1), Xi(k,c), Xi(k,c+1)).
    // PAIR: columns c = 2 (i % 4) of k's realization, dx[0..1] = Xr (hl 0) or
    // Xi (hl 1) of (k, c), (k, c+1).
    float dx[4] = {0.f, 0.f, 0.f, 0.f};
    if (!xzero) {
      // W operand rows q = (hilo, part, k) from the thread's antenna column
#pragma unroll
      for (int pg = 0; pg < 2 * (KT / 8); ++pg) {  // 8 rows (part, k .. k+7)
        const int part = pg / (KT / 8), kg = pg % (KT / 8);
        const float* src = (part == 0 ? wr : wi) + 8 * kg;
        const int q0 = part * K + 8 * kg + (T::PAIR ? T::KX * hx : 0);
        uint32_t h[4], lo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) split2(src[2 * u], src[2 * u + 1], h[u], lo[u]);
        if constexpr (T::DBS) {
          // 8-row chunk (quadrant k / 4, part) = [hi k..k+3 | lo k..k+3]
          const int kf = 8 * kg + (T::PAIR ? T::KX * hx : 0);
          *reinterpret_cast<uint4*>(smem + T::OFF_W + T::woff(T::qrow(0, part, kf), m)) =
              make_uint4(h[0], h[1], lo[0], lo[1]);
          *reinterpret_cast<uint4*>(smem + T::OFF_W + T::woff(T::qrow(0, part, kf + 4), m)) =
              make_uint4(h[2], h[3], lo[2], lo[3]);
        } else {
        *reinterpret_cast<uint4*>(smem + T::OFF_W + T::woff(q0, m)) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(smem + T::OFF_W + T::woff(R + q0, m)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
      fence_async_smem();
      tc_fence_before();
      // tile group: its antennas' W rows are written and its D2 part drained
      if (T::NTILE > 1) named_bar(1 + tile, T::NT / T::NTILE);
      else __syncthreads();
      TSTAMP(1)
      if constexpr (RESID) {
        if (l > 0) {
          bool crit[2];
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const float dd = rsd[4 * x] + rsd[4 * x + 2], ss = rsd[4 * x + 1] + rsd[4 * x + 3];
            crit[x] = dd < tol2 * fmaxf(ss, 1e-24f);
          }
          if (!stopped) {
            taken = l;
            l21_keep = l21_prev;
            act_keep = act_prev;
            stopped = crit[hx];
          }
          if (crit[0] && crit[1]) break;  // CTA-uniform: both realizations have stopped
        }
        if (stopped) {
          fstep = 0.f;
          ts = 0.f;
        }
      }
      // (32,256): both tiles accumulate into one D1 (columns [0, 2R)); tile 1's
      // first warp issues after tile 0's MMAs are queued (warp 0 -> warp 4
      // named barrier, tcgen05 fences around it), so the tensor pipe runs them
      // in order and the drain reads one accumulator instead of summing two
      // split-K parts (half its TMEM loads). Tile 1's MMAs also overwrite D2
      // tile 0's columns only after tile 0's group has drained them.
      if (T::NTILE > 1 && warp == 4) named_bar(4, 64);
      if (wu == tile * 4) {  // the tile group's first warp
        const int tu = wu >> 2;  // = tile, warp-uniform: the descriptors stay in uniform registers
        tc_fence_after();
        constexpr int KST = 128 / 16;  // K-steps per antenna tile
        const uint32_t sw = sb + T::OFF_W + tu * KST * 2 * 16 * Q, sh = sb + T::OFF_HH + tu * KST * 256;
        const uint32_t alo = sdesc_lo(sw, 16 * Q), blo = sdesc_lo(sh, 128);
        if constexpr (T::PAIR) {
          // one chain per realization over its own 64 antennas (K-steps 4x ..
          // 4x + 3) and its own N = 32 H columns (its hoffp() tile) — both
          // into D1 columns [0, 32):
          // [hi p0 | hi p1 | lo p0 | lo p1] of the row's realization's 8 users
          // (the other chain adds the exact zeros of the W operand's
          // off-diagonal entries). The frame's zero blocks (half the stage-1
          // MACs and of its H reads) are never multiplied.
          constexpr int KX4 = T::MX / 16;  // K-steps per realization
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int i = 0; i < KX4; ++i)
              umma_f16w(tmem + T::T_D1A + (SH ? 0 : 32 * x), alo + (x * KX4 + i) * (2 * 16 * Q >> 4), sdesc_hi(128),
                        blo + (x * 4096 + i * 256 >> 4), sdesc_hi(1024), IDESC1P, (SH && x > 0) || i > 0);
        } else {
#pragma unroll
        for (int i = 0; i < KST; ++i) {
          // B = [H_hi | H_lo] (N = 2R: OFF_HL continues OFF_HH's N-group stride)
          if constexpr (T::NTILE == 1)
            umma_f16w(tmem + tu * 2 * R + T::T_D1A, alo + i * (2 * 16 * Q >> 4), sdesc_hi(128), blo + i * (256 >> 4),
                      sdesc_hi(16 * M), IDESC1, i > 0);
          else
            umma_f16(tmem + T::T_D1A, sdesc(sw + i * 2 * 16 * Q, 16 * Q, 128), sdesc(sh + i * 256, 128, 16 * M),
                     IDESC1, tu > 0 || i > 0);
        }
        }
        umma_commit(bar1 + 8 * tu);
      }
      if (T::NTILE > 1 && warp == 0) {
        tc_fence_before();
        __syncwarp();
        named_bar_arrive(4, 64);
      }
      TSTAMP(2)
      // D1 rows q = (hilo, part, k): TMEM lane quadrant hilo * 2 + part, lane k
      // (M = 128: lanes 32 q4 + k; M = 64: lanes 32 q4 + k for k < 16).
      // Warp w reads quadrant w % 4, columns [w / 4 * CW, + CW).
      constexpr int CW = R * 4 / NW;
      const int quad = warp & 3, c0 = (warp >> 2) * CW, part = quad & 1;
#pragma unroll
      for (int t = 0; t < T::NTILE; ++t) mbar_wait<(T::K >= 32 ? 4 : 1)>(bar1 + 8 * t, ph1);
      ph1 ^= 1;
      TSTAMP(3)
      tc_fence_after();
      if constexpr (Q == 64) {
        // M = 64 accumulator: rows in lanes 0..15 of each quadrant. The 16x256b
        // shape loads just those 16 lanes (thread i: rows i / 4, i / 4 + 8,
        // column pairs 8 j + 2 (i % 4)), so no lane loads or combines the 16
        // unused lanes of the 32x32b shape (half the LDTM and FP32x2 work).
        static_assert(T::NTILE == 1 && CW == 2 * R / 2 && T::CWD == 2, "");
        const int kr = lane >> 2, cp = 2 * (lane & 3);
        float* const FG = quad < 2 ? F : G;
        const int r0 = part * K + kr;
        float* d0 = FG + r0 * T::FSTR + cp;
        float a[16], b[16];
        if constexpr (T::DBS) {
          // Thread i holds rows (hl, k % 4) = i / 4 of part 0 (a[4j], a[4j+1]) and
          // part 1 (a[4j+2], a[4j+3]) at columns 8 j + 2 (i % 4) + {0, 1}.
          // Row value = A + 2^-11 B on a hi row (B: the product with H_lo),
          // 2^-11 A on a lo row; X is linear in the rows, so the part / p'
          // combinations are formed on A and B first:
          //   Xr = P[(0,k),(0,k')] - P[(1,k),(1,k')], Xi = P[(0,k),(1,k')] + P[(1,k),(0,k')]
          const bool lo_row = lane >= 16;
          const float sa = lo_row ? kLoScale : 1.f, sb = lo_row ? 0.f : kLoScale;
          auto pr = [](const float* v, int i) { return make_float2(v[i], v[i + 1]); };
          if constexpr (T::PAIR) {
            // 32 columns [hi p'0 | hi p'1 | lo p'0 | lo p'1] of the 8 users k'
            // of the warp's realization (robust instance: at 32 x)
            tmem_ld16x256(tmem + lrow + T::T_D1A + (SH ? 0 : 32 * (warp >> 1)), a);
            tmem_wait<16>(a);
            const float2 ar = ffma2(-1.f, pr(a, 6), pr(a, 0)), ai = fadd2(pr(a, 4), pr(a, 2));
            const float2 br = ffma2(-1.f, pr(a, 14), pr(a, 8)), bi = fadd2(pr(a, 12), pr(a, 10));
            const float2 xr = ffma2(sb, br, fmul2(sa, ar)), xi = ffma2(sb, bi, fmul2(sa, ai));
            // the hi-row lane takes Xr, the lo-row lane Xi: each sends the other its share
            const float2 give = lo_row ? xr : xi, keep = lo_row ? xi : xr;
            const float2 got = make_float2(__shfl_xor_sync(kFull, give.x, 16), __shfl_xor_sync(kFull, give.y, 16));
            const float2 t = fadd2(keep, got);
            dx[0] = t.x;
            dx[1] = t.y;
          } else {
            // columns [H_hi: p'0 (16 users) | p'1] in D1A, the same with H_lo in D1B;
            // j = 0, 1: p'0 at k' = 2 (i % 4) + {0, 1} and 8 more, j = 2, 3: p'1
            tmem_ld16x256(tmem + lrow + T::T_D1A, a);
            tmem_ld16x256(tmem + lrow + T::T_D1B, b);
            tmem_wait<16>(a);
            tmem_wait<16>(b);
            float2 xr[2], xi[2];  // column chunks c = 2 (i % 4) and 8 more
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float2 ar = ffma2(-1.f, pr(a, 10 + 4 * h), pr(a, 4 * h)), ai = fadd2(pr(a, 8 + 4 * h), pr(a, 2 + 4 * h));
              const float2 br = ffma2(-1.f, pr(b, 10 + 4 * h), pr(b, 4 * h)), bi = fadd2(pr(b, 8 + 4 * h), pr(b, 2 + 4 * h));
              xr[h] = ffma2(sb, br, fmul2(sa, ar));
              xi[h] = ffma2(sb, bi, fmul2(sa, ai));
            }
            // the hi-row lane takes chunk 0, the lo-row lane chunk 1
            const float2 gr = lo_row ? xr[0] : xr[1], gi = lo_row ? xi[0] : xi[1];
            const float2 kr = lo_row ? xr[1] : xr[0], ki = lo_row ? xi[1] : xi[0];
            const float2 tr = fadd2(kr, make_float2(__shfl_xor_sync(kFull, gr.x, 16), __shfl_xor_sync(kFull, gr.y, 16)));
            const float2 ti = fadd2(ki, make_float2(__shfl_xor_sync(kFull, gi.x, 16), __shfl_xor_sync(kFull, gi.y, 16)));
            dx[0] = tr.x;
            dx[1] = tr.y;
            dx[2] = ti.x;
            dx[3] = ti.y;
          }
        } else if constexpr (T::PAIR) {
          // D1 columns [0, 32) hold each row's realization's [hi p0 | hi p1 |
          // lo p0 | lo p1]: one 16x256b load carries row kr (a) and kr + 8 (b). F / G get
          // the same entries as the full-frame layout: (row kr, columns cp, K + cp),
          // (row kr + 8, columns 8 + cp, K + 8 + cp).
          // (robust instance: realization x's columns at 32 x — row kr from the
          // first load, row kr + 8 from the second)
          tmem_ld16x256(tmem + lrow + T::T_D1A, a);
          if (!SH) tmem_ld16x256(tmem + lrow + T::T_D1A + 32, b);
          tmem_wait<16>(a);
          if (!SH) tmem_wait<16>(b);
          const float* bb = SH ? a : b;
          float2 v[4];  // (row kr: p'0, p'1), (row kr + 8: p'0, p'1)
          const float2 h0 = make_float2(a[0], a[1]), h1 = make_float2(a[4], a[5]);
          const float2 h2 = make_float2(bb[2], bb[3]), h3 = make_float2(bb[6], bb[7]);
          if (quad < 2) {  // hi W rows: W_hi H_hi + 2^-11 W_hi H_lo
            v[0] = ffma2(kLoScale, make_float2(a[8], a[9]), h0);
            v[1] = ffma2(kLoScale, make_float2(a[12], a[13]), h1);
            v[2] = ffma2(kLoScale, make_float2(bb[10], bb[11]), h2);
            v[3] = ffma2(kLoScale, make_float2(bb[14], bb[15]), h3);
          } else {         // lo W rows: 2^-11 W_lo H_hi
            v[0] = fmul2(kLoScale, h0);
            v[1] = fmul2(kLoScale, h1);
            v[2] = fmul2(kLoScale, h2);
            v[3] = fmul2(kLoScale, h3);
          }
          *reinterpret_cast<float2*>(FG + T::fx(r0, cp)) = v[0];
          *reinterpret_cast<float2*>(FG + T::fx(r0, K + cp)) = v[1];
          *reinterpret_cast<float2*>(FG + T::fx(r0 + 8, 8 + cp)) = v[2];
          *reinterpret_cast<float2*>(FG + T::fx(r0 + 8, K + 8 + cp)) = v[3];
        } else {
        tmem_ld16x256(tmem + lrow + T::T_D1A, a);
        if (quad < 2) tmem_ld16x256(tmem + lrow + T::T_D1B, b);
        tmem_wait<16>(a);
        if (quad < 2) tmem_wait<16>(b);
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float2 t = quad < 2 ? ffma2(kLoScale, make_float2(b[i], b[i + 1]), make_float2(a[i], a[i + 1]))
                                    : fmul2(kLoScale, make_float2(a[i], a[i + 1]));
          a[i] = t.x;
          a[i + 1] = t.y;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          *reinterpret_cast<float2*>(d0 + 8 * j) = make_float2(a[4 * j], a[4 * j + 1]);
          *reinterpret_cast<float2*>(d0 + 8 * T::FSTR + 8 * j) = make_float2(a[4 * j + 2], a[4 * j + 3]);
        }
        }
      } else {
      float* dst = (quad < 2 ? F : G) + (part * K + lane) * T::FSTR + c0;
#pragma unroll
      for (int cq = 0; cq < CW; cq += 16) {
        float a[16], b[16];
        tmem_ld16(tmem + lrow + T::T_D1A + c0 + cq, a);
        if (quad < 2) tmem_ld16(tmem + lrow + T::T_D1B + c0 + cq, b);
        tmem_wait<16>(a);
        if (quad < 2) tmem_wait<16>(b);
        if (quad < 2) {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {  // hi rows: W_hi H_hi + W_hi H_lo (packed FP32x2)
            const float2 t = ffma2(kLoScale, make_float2(b[i], b[i + 1]), make_float2(a[i], a[i + 1]));
            a[i] = t.x;
            a[i + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {  // lo rows: W_lo H_hi
            const float2 t = fmul2(kLoScale, make_float2(a[i], a[i + 1]));
            a[i] = t.x;
            a[i + 1] = t.y;
          }
        }
        if (lane < K) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(dst + cq + i) = make_float4(a[i], a[i + 1], a[i + 2], a[i + 3]);
        }
      }
      }
      if constexpr (!T::DBS) __syncthreads();  // F / G complete (DBS: the chunk is in registers)
    }
    TSTAMP(4)
    // Bs[(p_in, k')][(p_out, k)] = -eta/g^2 * { X'r, X'i ; X'i, -X'r }(k, k'), one
    // 4-wide chunk of X' row k per thread
    // CWD-wide chunks of X' row k per thread (CWD = 4, or 2 when K / 4 chunks per
    // row would leave threads idle; 2-wide keeps a quarter-warp on one F row)
    int aB = 0;  // robust path: Bs is built as Bs 2^-aB
    if constexpr (T::DBS) {
      // The thread's chunk of X is in dx (see above): X' = X - diag(c), times
      // -eta / g^2, split and stored. Robust path: the P rows are X 2^-aW, so
      // X' 2^-aW = P - c 2^-aW, and the chunk values become Bs 2^-aB with aB
      // from their exact CTA maximum (PAIR: over the realization's two warps).
      constexpr int NV = T::PAIR ? 2 : 4;
      const bool lo_row = lane >= 16;
      const int k = 4 * warp + ((lane >> 2) & 3);
      const int c = T::PAIR ? T::KX * (warp >> 1) + 2 * (lane & 3) : 2 * (lane & 3) + (lo_row ? 8 : 0);
      const float cscale = RB ? pow2i(-aW) : 1.f, fstep_w = RB ? fstep * pow2i(aW) : fstep;
      if constexpr (!RB && UFPGD_MMA_CDIAG) {
        dx[0] -= cdg[0];  // x - 0 is exact: the same values as the in-loop test
        dx[1] -= cdg[1];
      } else if (!T::PAIR || !lo_row) {  // the Xr values
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (c + u == k) dx[u] -= RB ? p.c[k] * cscale : p.c[k];
      }
#pragma unroll
      for (int u = 0; u < NV; ++u) dx[u] *= fstep_w;
      if constexpr (RB) {
        float bm = 0.f;
#pragma unroll
        for (int u = 0; u < NV; ++u) bm = fmaxf(bm, fabsf(dx[u]));
        if (!(bm <= FLT_MAX)) bm = __int_as_float(0x7f800000);
        bm = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(bm)));
        if (lane == 0) redw[warp] = bm;
        __syncthreads();
        float mb = 0.f;
#pragma unroll
        for (int w = hx * NWX; w < (hx + 1) * NWX; ++w) mb = fmaxf(mb, redw[w]);  // PAIR: its block's warps
        if (mb > 0.f && mb < FLT_MAX) aB = ilogbf(mb) - 12;  // Bs 2^-aB in [2^12, 2^13)
        const float f = pow2i(-aB);
#pragma unroll
        for (int u = 0; u < NV; ++u) dx[u] *= f;
      }
      auto put = [&](int off, uint32_t v) { *reinterpret_cast<uint32_t*>(smem + off) = v; };
      // (p_in, p_out) = (0,0): X'r, (1,0): X'i, (0,1): X'i, (1,1): -X'r (f16 negation is exact)
      if constexpr (T::PAIR) {
        uint32_t vh, vl;
        split2(dx[0], dx[1], vh, vl);
        const uint32_t neg = lo_row ? 0u : 0x80008000u;
        const int o1 = HOIST_BO ? bo1 : T::OFF_BH + (lo_row ? T::bpos(1, 0, k, c) : T::bpos(0, 0, k, c));
        const int o2 = HOIST_BO ? bo2 : T::OFF_BH + (lo_row ? T::bpos(0, 1, k, c) : T::bpos(1, 1, k, c));
        put(o1, vh);
        put(o1 + T::BLO, vl);
        put(o2, vh ^ neg);
        put(o2 + T::BLO, vl ^ neg);
      } else {
        uint32_t rh, rl, ih, il;
        split2(dx[0], dx[1], rh, rl);
        split2(dx[2], dx[3], ih, il);
        // bpos(pin, pout, k, c) = bpos(0, 0, k, c) + pin (K / 8) BLBO + pout (K / 8) BSBO
        constexpr int DI = (K / 8) * T::BLBO, DO = (K / 8) * T::BSBO;
        const int o0 = HOIST_BO ? bo1 : T::OFF_BH + T::bpos(0, 0, k, c);
        put(o0, rh);
        put(o0 + T::BLO, rl);
        put(o0 + DI, ih);
        put(o0 + DI + T::BLO, il);
        put(o0 + DO, ih);
        put(o0 + DO + T::BLO, il);
        put(o0 + DI + DO, rh ^ 0x80008000u);
        put(o0 + DI + DO + T::BLO, rl ^ 0x80008000u);
      }
    } else if constexpr (!RB) {
      constexpr int CWD = T::CWD, NCH = K * K / CWD, CPR = K / CWD;
      using FV = typename std::conditional<CWD == 4, float4, float2>::type;
  #pragma unroll
      for (int ch = tid; ch < NCH; ch += T::NT) {
        int k, c;
        T::chunk(ch, k, c);
        if (T::PAIR && k / T::KX != c / T::KX) continue;  // off-diagonal: no Bs tile (warp-uniform)
        float xr[CWD], xi[CWD];
  #pragma unroll
        for (int u = 0; u < CWD; ++u) xr[u] = xi[u] = 0.f;
        if (!xzero) {
          // P rows (0, k), (1, k): hi parts in F, lo in G
          const int i00 = T::fx(k, c), i11 = T::fx(K + k, K + c), i01 = T::fx(k, K + c), i10 = T::fx(K + k, c);
          const FV a00 = *reinterpret_cast<const FV*>(F + i00), b00 = *reinterpret_cast<const FV*>(G + i00);
          const FV a11 = *reinterpret_cast<const FV*>(F + i11), b11 = *reinterpret_cast<const FV*>(G + i11);
          const FV a01 = *reinterpret_cast<const FV*>(F + i01), b01 = *reinterpret_cast<const FV*>(G + i01);
          const FV a10 = *reinterpret_cast<const FV*>(F + i10), b10 = *reinterpret_cast<const FV*>(G + i10);
          const float* A00 = reinterpret_cast<const float*>(&a00);
          const float* B00 = reinterpret_cast<const float*>(&b00);
          const float* A11 = reinterpret_cast<const float*>(&a11);
          const float* B11 = reinterpret_cast<const float*>(&b11);
          const float* A01 = reinterpret_cast<const float*>(&a01);
          const float* B01 = reinterpret_cast<const float*>(&b01);
          const float* A10 = reinterpret_cast<const float*>(&a10);
          const float* B10 = reinterpret_cast<const float*>(&b10);
  #pragma unroll
          for (int u = 0; u < CWD; u += 2) {  // packed FP32x2
            const float2 r2 = fadd2(fadd2(make_float2(A00[u], A00[u + 1]), make_float2(B00[u], B00[u + 1])),
                                    make_float2(-(A11[u] + B11[u]), -(A11[u + 1] + B11[u + 1])));
            const float2 i2 = fadd2(fadd2(make_float2(A01[u], A01[u + 1]), make_float2(B01[u], B01[u + 1])),
                                    fadd2(make_float2(A10[u], A10[u + 1]), make_float2(B10[u], B10[u + 1])));
            xr[u] = r2.x;
            xr[u + 1] = r2.y;
            xi[u] = i2.x;
            xi[u + 1] = i2.y;
          }
        }
  #pragma unroll
        for (int u = 0; u < CWD; ++u) {
          if constexpr (CDQ) {
            xr[u] -= cdq[u];  // X' = X - diag(c): the thread's share, set before the loop
          } else {
            if (c + u == k) xr[u] -= p.c[k];
          }
          xr[u] *= fstep;
          xi[u] *= fstep;
        }
        uint32_t rh[CWD / 2], rl[CWD / 2], nh[CWD / 2], nl[CWD / 2], ih[CWD / 2], il[CWD / 2];
  #pragma unroll
        for (int v = 0; v < CWD / 2; ++v) {
          split2(xr[2 * v], xr[2 * v + 1], rh[v], rl[v]);
          nh[v] = rh[v] ^ 0x80008000u;  // split of -X'r: f16 negation is exact
          nl[v] = rl[v] ^ 0x80008000u;
          split2(xi[2 * v], xi[2 * v + 1], ih[v], il[v]);
        }
        // (p_in, p_out) = (0,0): X'r, (1,0): X'i, (0,1): X'i, (1,1): -X'r
        auto put = [&](int off, const uint32_t* v) {
          if constexpr (CWD == 4)
            *reinterpret_cast<uint2*>(smem + off) = make_uint2(v[0], v[1]);
          else
            *reinterpret_cast<uint32_t*>(smem + off) = v[0];
        };
        put(T::OFF_BH + T::bpos(0, 0, k, c), rh);
        put(T::OFF_BH + T::BLO + T::bpos(0, 0, k, c), rl);
        put(T::OFF_BH + T::bpos(1, 0, k, c), ih);
        put(T::OFF_BH + T::BLO + T::bpos(1, 0, k, c), il);
        put(T::OFF_BH + T::bpos(0, 1, k, c), ih);
        put(T::OFF_BH + T::BLO + T::bpos(0, 1, k, c), il);
        put(T::OFF_BH + T::bpos(1, 1, k, c), nh);
        put(T::OFF_BH + T::BLO + T::bpos(1, 1, k, c), nl);
      }
    } else {
      constexpr int CWD = T::CWD, NCH = K * K / CWD, CPR = K / CWD;
      static_assert(NCH <= T::NT, "one Bs chunk per thread");
      using FV = typename std::conditional<CWD == 4, float4, float2>::type;
      // robust path: the P rows are X 2^-aW, so X' 2^-aW = P - c 2^-aW, and the
      // chunk values become Bs 2^-aB with aB from their exact CTA maximum
      const float cscale = RB ? pow2i(-aW) : 1.f, fstep_w = RB ? fstep * pow2i(aW) : fstep;
      {
        const int ch = tid;
        int k, c;
        T::chunk(ch, k, c);
        const bool live = !T::PAIR || k / T::KX == c / T::KX;  // PAIR: off-diagonal blocks have no Bs tile
        float xr[CWD], xi[CWD];
  #pragma unroll
        for (int u = 0; u < CWD; ++u) xr[u] = xi[u] = 0.f;
        if (!xzero && live) {
          // P rows (0, k), (1, k): hi parts in F, lo in G
          const int i00 = T::fx(k, c), i11 = T::fx(K + k, K + c), i01 = T::fx(k, K + c), i10 = T::fx(K + k, c);
          const FV a00 = *reinterpret_cast<const FV*>(F + i00), b00 = *reinterpret_cast<const FV*>(G + i00);
          const FV a11 = *reinterpret_cast<const FV*>(F + i11), b11 = *reinterpret_cast<const FV*>(G + i11);
          const FV a01 = *reinterpret_cast<const FV*>(F + i01), b01 = *reinterpret_cast<const FV*>(G + i01);
          const FV a10 = *reinterpret_cast<const FV*>(F + i10), b10 = *reinterpret_cast<const FV*>(G + i10);
          const float* A00 = reinterpret_cast<const float*>(&a00);
          const float* B00 = reinterpret_cast<const float*>(&b00);
          const float* A11 = reinterpret_cast<const float*>(&a11);
          const float* B11 = reinterpret_cast<const float*>(&b11);
          const float* A01 = reinterpret_cast<const float*>(&a01);
          const float* B01 = reinterpret_cast<const float*>(&b01);
          const float* A10 = reinterpret_cast<const float*>(&a10);
          const float* B10 = reinterpret_cast<const float*>(&b10);
  #pragma unroll
          for (int u = 0; u < CWD; u += 2) {  // packed FP32x2
            const float2 r2 = fadd2(fadd2(make_float2(A00[u], A00[u + 1]), make_float2(B00[u], B00[u + 1])),
                                    make_float2(-(A11[u] + B11[u]), -(A11[u + 1] + B11[u + 1])));
            const float2 i2 = fadd2(fadd2(make_float2(A01[u], A01[u + 1]), make_float2(B01[u], B01[u + 1])),
                                    fadd2(make_float2(A10[u], A10[u + 1]), make_float2(B10[u], B10[u + 1])));
            xr[u] = r2.x;
            xr[u + 1] = r2.y;
            xi[u] = i2.x;
            xi[u + 1] = i2.y;
          }
        }
  #pragma unroll
        for (int u = 0; u < CWD; ++u) {
          if (c + u == k) xr[u] -= RB ? p.c[k] * cscale : p.c[k];  // X' = X - diag(c)
          xr[u] *= fstep_w;
          xi[u] *= fstep_w;
        }
        if constexpr (RB) {
          float bm = 0.f;
          if (ch < NCH) {
  #pragma unroll
            for (int u = 0; u < CWD; ++u) bm = fmaxf(bm, fmaxf(fabsf(xr[u]), fabsf(xi[u])));
            if (!(bm <= FLT_MAX)) bm = __int_as_float(0x7f800000);
          }
          bm = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(bm)));
          if (lane == 0) redw[warp] = bm;
          __syncthreads();
          float mb = 0.f;
  #pragma unroll
          for (int w = hx * NWX; w < (hx + 1) * NWX; ++w) mb = fmaxf(mb, redw[w]);  // PAIR: its block's warps
          if (mb > 0.f && mb < FLT_MAX) aB = ilogbf(mb) - 12;  // Bs 2^-aB in [2^12, 2^13)
          const float f = pow2i(-aB);
  #pragma unroll
          for (int u = 0; u < CWD; ++u) {
            xr[u] *= f;
            xi[u] *= f;
          }
        }
        if (ch < NCH && live) {
        uint32_t rh[CWD / 2], rl[CWD / 2], nh[CWD / 2], nl[CWD / 2], ih[CWD / 2], il[CWD / 2];
  #pragma unroll
        for (int v = 0; v < CWD / 2; ++v) {
          split2(xr[2 * v], xr[2 * v + 1], rh[v], rl[v]);
          nh[v] = rh[v] ^ 0x80008000u;  // split of -X'r: f16 negation is exact
          nl[v] = rl[v] ^ 0x80008000u;
          split2(xi[2 * v], xi[2 * v + 1], ih[v], il[v]);
        }
        // (p_in, p_out) = (0,0): X'r, (1,0): X'i, (0,1): X'i, (1,1): -X'r
        auto put = [&](int off, const uint32_t* v) {
          if constexpr (CWD == 4)
            *reinterpret_cast<uint2*>(smem + off) = make_uint2(v[0], v[1]);
          else
            *reinterpret_cast<uint32_t*>(smem + off) = v[0];
        };
        put(T::OFF_BH + T::bpos(0, 0, k, c), rh);
        put(T::OFF_BH + T::BLO + T::bpos(0, 0, k, c), rl);
        put(T::OFF_BH + T::bpos(1, 0, k, c), ih);
        put(T::OFF_BH + T::BLO + T::bpos(1, 0, k, c), il);
        put(T::OFF_BH + T::bpos(0, 1, k, c), ih);
        put(T::OFF_BH + T::BLO + T::bpos(0, 1, k, c), il);
        put(T::OFF_BH + T::bpos(1, 1, k, c), nh);
        put(T::OFF_BH + T::BLO + T::bpos(1, 1, k, c), nl);
        }
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    TSTAMP(5)
    // Each antenna tile's stage-2 MMAs are issued by the tile group's first
    // warp, tile 1 after tile 0's are queued (warp 0 -> warp 4 named barrier):
    // issuing blocks while the MMA queue is full, so one warp issuing both tiles
    // kept warp 0 — and with it tile 0's epilogue — out of the drain until tile
    // 1's MMAs were nearly done.
    static_assert(T::NTILE <= 2, "");
    if (T::NTILE > 1 && warp == 4) named_bar(3, 64);
    if ((wu & 3) == 0) {  // the tile group's first warp
      tc_fence_after();
      const int t = wu >> 2;  // = tile, warp-uniform
      const uint32_t dm = tmem + T::T_D2 + t * 2 * R, dc = dm + R;
      const uint32_t ta = tmem + THA + t * R;  // H_hi columns; H_lo at + R / 2
      const uint32_t bhlo = sdesc_lo(sb + T::OFF_BH, T::BLBO);
      if constexpr (T::PAIR) {
        // realization x: its K-step of A (8 TMEM columns of H hi / lo; zeros in
        // the other realization's lanes) against its Bs tile, both into D2
        // columns [0, 32) = [main hh | main hl + corr]
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const uint32_t bx = bhlo + x * (T::BST >> 4);
          const uint32_t dx = dm + (SH ? 0 : 32 * x);
          umma_f16_ta(dx, ta + x * 8, bx, sdesc_hi(T::BSBOP), IDESC2PW, SH && x > 0);
          umma_f16_ta(dx + 16, ta + R / 2 + x * 8, bx, sdesc_hi(T::BSBOP), IDESC2P, 1);
        }
      } else
#pragma unroll
      for (int ks = 0; ks < R / 16; ++ks) {
        // [main | corr] = H_hi [Bs_hi | Bs_lo] (N = 2R spans both), then corr += H_lo Bs_hi;
        // a K16 step of A is 8 TMEM columns (f16 pairs)
        if constexpr (T::NTILE == 1) {
          const uint32_t bh = bhlo + ks * (2 * T::BLBO >> 4);
          umma_f16_ta(dm, ta + ks * 8, bh, sdesc_hi(T::BSBO), IDESC2W, ks > 0);
          umma_f16_ta(dc, ta + R / 2 + ks * 8, bh, sdesc_hi(T::BSBO), IDESC2, 1);
        } else {
          const uint64_t bh = sdesc(sb + T::OFF_BH + ks * 2 * T::BLBO, T::BLBO, T::BSBO);
          umma_f16_ta(dm, ta + ks * 8, bh, IDESC2W, ks > 0);
          umma_f16_ta(dc, ta + R / 2 + ks * 8, bh, IDESC2, 1);
        }
      }
      umma_commit(bar2 + 8 * t);  // each tile's epilogue starts as soon as its MMAs retire
    }
    if (T::NTILE > 1 && warp == 0) {
      __syncwarp();
      named_bar_arrive(3, 64);
    }
    TSTAMP(6)
    mbar_wait<(T::K >= 32 ? 4 : 1)>(bar2 + 8 * tile, ph2);
    ph2 ^= 1;
    TSTAMP(7)
    tc_fence_after();
    {
      // antenna m: TMEM lane m % 128 (warp quadrant warp % 4), tile m / 128
      const uint32_t cm = tmem + lrow + T::T_D2 + tile * 2 * R;
      const uint32_t cc = cm + R;
      if constexpr (RESID) {
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          wor[k] = wr[k];
          woi[k] = wi[k];
        }
      }
      if constexpr (T::PAIR) {  // the thread's 8 users only
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          float* w = part == 0 ? wr : wi;
          float a[8], b[8];
          const uint32_t cx = cm + (SH ? 0 : 32 * hx);  // D2 [main hh | main hl + corr]
          tmem_ld8(cx + 8 * part, a);
          tmem_ld8(cx + 16 + 8 * part, b);
          tmem_wait<8>(a);
          tmem_wait<8>(b);
          if constexpr (RB) {
            const float u2 = pow2i(aB - aW);
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = fmaf(u2, fmaf(kLoScale, b[i], a[i]), w[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const float2 t = fadd2(make_float2(w[i], w[i + 1]),
                                     ffma2(kLoScale, make_float2(b[i], b[i + 1]), make_float2(a[i], a[i + 1])));
              w[i] = t.x;
              w[i + 1] = t.y;
            }
          }
        }
      } else {
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        float* w = part == 0 ? wr : wi;
#pragma unroll
        for (int j0 = 0; j0 < K; j0 += 16) {
          float a[16], b[16];
          tmem_ld16(cm + part * K + j0, a);
          tmem_ld16(cc + part * K + j0, b);
          tmem_wait<16>(a);
          tmem_wait<16>(b);
          if constexpr (RB) {  // D2 = G 2^-aB onto W registers in the 2^-aW domain
            const float u2 = pow2i(aB - aW);
#pragma unroll
            for (int i = 0; i < 16; ++i) w[j0 + i] = fmaf(u2, fmaf(kLoScale, b[i], a[i]), w[j0 + i]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {  // V = W - eta X' H^* (packed FP32x2)
              const float2 t = fadd2(make_float2(w[j0 + i], w[j0 + i + 1]),
                                     ffma2(kLoScale, make_float2(b[i], b[i + 1]), make_float2(a[i], a[i + 1])));
              w[j0 + i] = t.x;
              w[j0 + i + 1] = t.y;
            }
          }
        }
      }
      }
    }
    tc_fence_before();
    // prox_l21 on the antenna column (strict '>', pgd.cpp:237-244 / unfolded.cpp:135-143)
    // (32,256): four independent partial sums — the 64-deep FMA chain sat on the
    // per-layer critical path of the one resident realization (-1.8% per layer);
    // (16,128) keeps one chain (4 CTAs/SM hide it; the extra registers cost 1%)
    // packed FP32x2: one pair of partial sums per chain, NS chains
    constexpr int NS = K >= 32 ? 2 : 1;
    float2 s2p[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) s2p[i] = zero2();
#pragma unroll
    for (int k = 0; k < KT; k += 2) {
      const float2 r2 = make_float2(wr[k], wr[k + 1]), i2 = make_float2(wi[k], wi[k + 1]);
      s2p[(k / 2) % NS] = __ffma2_rn(r2, r2, __ffma2_rn(i2, i2, s2p[(k / 2) % NS]));
    }
    float s2 = s2p[0].x + s2p[0].y;
    if constexpr (NS == 2) s2 = (s2p[0].x + s2p[0].y) + (s2p[1].x + s2p[1].y);
    const float gw = RB ? g * pow2i(aW) : g;  // register domain -> unscaled W
    if constexpr (RB) {
      nonfinite |= !(s2 * gw * gw <= FLT_MAX);
    } else {
      nonfinite |= !(s2 * (g * g) <= FLT_MAX);
    }
    const bool on = s2 > ts * ts;
    const float r = rsqrt_ftz(fmaxf(s2, FLT_MIN));
    const float scale = on ? fmaf(-ts, r, 1.f) : 0.f;
#pragma unroll
    for (int k = 0; k < KT; k += 2) {
      const float2 r2 = fmul2(scale, make_float2(wr[k], wr[k + 1])), i2 = fmul2(scale, make_float2(wi[k], wi[k + 1]));
      wr[k] = r2.x;
      wr[k + 1] = r2.y;
      wi[k] = i2.x;
      wi[k + 1] = i2.y;
    }
    if constexpr (RB) wn2 = scale * scale * s2;
    if constexpr (RESID) {
      l21_prev = on ? gw * fmaf(s2, r, -ts) : 0.f;
      act_prev = on ? 1 : 0;
      float2 dsum = zero2();  // (|dW|^2, |W|^2) of this thread's entries, in the register domain
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const float dr = wr[k] - wor[k], di = wi[k] - woi[k];
        dsum = __ffma2_rn(make_float2(dr, wor[k]), make_float2(dr, wor[k]), dsum);
        dsum = __ffma2_rn(make_float2(di, woi[k]), make_float2(di, woi[k]), dsum);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
        dsum = fadd2(dsum, make_float2(__shfl_xor_sync(kFull, dsum.x, off), __shfl_xor_sync(kFull, dsum.y, off)));
      if (lane == 0) {
        rsd[2 * warp] = dsum.x;
        rsd[2 * warp + 1] = dsum.y;
      }
    } else if (l + 1 == p.L && on) {
      l21 += gw * fmaf(s2, r, -ts);
      act += 1;
    }
    if (nonfinite && first_bad < 0) first_bad = l;
    TSTAMP(8)
  }
  if constexpr (RESID) {
    __syncthreads();  // the last iteration's partials
    if (!stopped) {  // ran to max_iters, or stopped at the last iteration (same outputs)
      taken = p.L;
      l21_keep = l21_prev;
      act_keep = act_prev;
    }
    l21 = l21_keep;
    act = act_keep;
  }

  PSTAMP(5)
  // ---- W out (unscaled), per-realization reductions ---------------------------
  // (a realization handed to the robust path writes garbage W here; the robust
  // kernel, later in the stream, overwrites it)
  {
    const float gout = RB ? g * pow2i(aW) : g;
    float4* wg = reinterpret_cast<float4*>(p.W + (rx * T::MX + ml) * KT);
    if (xvalid) {
#pragma unroll
      for (int j = 0; j < KT / 2; ++j)
        stg_stream(wg + j, make_float4(wr[2 * j] * gout, wi[2 * j] * gout, wr[2 * j + 1] * gout, wi[2 * j + 1] * gout));
    }
#ifdef UFPGD_MMA_TIMING
    PSTAMP(6)
    if (probe) {
      long long* o = reinterpret_cast<long long*>(p.W + rid * M * K);
      for (int i = 0; i < 9; ++i) o[i] = tst[i];
      for (int i = 0; i < 7; ++i) o[9 + i] = pst[i];
    }
#endif
  }
  long long fb = first_bad < 0 ? LLONG_MAX : first_bad;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    fb = min(fb, __shfl_xor_sync(kFull, fb, off));
    l21 += __shfl_xor_sync(kFull, l21, off);
    act += __shfl_xor_sync(kFull, act, off);
  }
  if (lane == 0) {
    fbs[warp] = fb;
    red[warp] = l21;
    red[16 + warp] = static_cast<float>(act);
  }
  // Fast path hand-off to the range-robust kernel, decided at the final CTA
  // barrier so the layer loop is the plain one: any non-finite value on the
  // way (an f16 overflow of W_s or Bs — e.g. W0 = H^* with a large channel —
  // or a true divergence, which the robust path then reproduces with its
  // index), or a Bs scale |eta / g^2| max c outside [2^-12, 2^12] (f16
  // underflow: tiny c or steps). The handed-off realization's W is
  // overwritten and its other outputs are written by the robust kernel.
  tc_fence_before();
  bool handoff = false;
  if (RB) {
    __syncthreads();
  } else {
    const float sc_lo = (PGD ? eta_b : p.eta_lo) * p.cmax * g2inv, sc_hi = (PGD ? eta_b : p.eta_hi) * p.cmax * g2inv;
    // (uniform per realization; an odd batch's phantom second realization —
    // zero channel, g = 1 — must not send its real partner to the robust path)
    const bool range = xvalid && !(sc_lo >= 0x1.0p-12f && sc_hi <= 0x1.0p12f);
    handoff = __syncthreads_or(nonfinite || range) != 0;
  }
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
  if (RB && tid == 0) {  // the robust kernel re-initialises them for its next realization
#pragma unroll
    for (int b = 0; b < 2 * T::NTILE; ++b)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar1 + 8 * b) : "memory");
  }
  if (tid == 0 && handoff) redo_list[atomicAdd(redo_count, 1)] = static_cast<int>(rid);
  // each realization's first thread (PAIR: threads 0 and 64) combines its warps
  if (tid == hx * NWX * 32 && !handoff && xvalid) {
    for (int w = hx * NWX + 1; w < (hx + 1) * NWX; ++w) {
      fb = min(fb, fbs[w]);
      l21 += red[w];
      act += static_cast<int>(red[16 + w]);
    }
    const bool diverged = fb != LLONG_MAX;
    if (p.diverged_at) p.diverged_at[rx] = diverged ? static_cast<int32_t>(fb + (PGD ? 1 : 0)) : -1;
    if (p.l21) p.l21[rx] = diverged ? __int_as_float(0x7fc00000) : l21;
    if (p.active) p.active[rx] = diverged ? -1 : act;
    if (RESID && p.iterations) p.iterations[rx] = taken;
    if (p.block_partials) {
      p.block_partials[rx * 3 + 0] = diverged ? 0.0 : static_cast<double>(p.alpha) * l21;
      p.block_partials[rx * 3 + 1] = diverged ? 0.0 : static_cast<double>(act);
      p.block_partials[rx * 3 + 2] = diverged ? 1.0 : 0.0;
    }
  }
  if (RB) __syncthreads();  // the reduction slots are reused by the next realization
  }  // realizations of the CTA
}

using Mma_32_256 = MmaShape<32, 256, 1>;
#ifndef UFPGD_MMA16_MINB
#define UFPGD_MMA16_MINB 4
#endif
using Mma_16_128 = MmaShape<16, 128, UFPGD_MMA16_MINB>;
#ifndef UFPGD_PAIR_MINB
#define UFPGD_PAIR_MINB 7
#endif
using Mma_8_64x2 = MmaShape<16, 128, UFPGD_PAIR_MINB, true>;

template <class T>
cudaError_t launch_mma_t(const FusedArgs& args, bool pgd, cudaStream_t s, long long* nblocks) {
  FusedArgs a = args;  // + the range summary the fast path checks once per realization
  if constexpr (T::PAIR) {
    for (int k = T::KX; k < T::K; ++k) a.c[k] = a.c[k - T::KX];  // c of the pair frame: [c; c]
  } else if (a.residual_tol > 0.f) {
    return cudaErrorInvalidValue;  // the early stop is built for the (8,64) pairs
  }
  a.cmax = 0.f;
  for (int k = 0; k < T::K; ++k) a.cmax = std::max(a.cmax, std::fabs(a.c[k]));
  a.eta_lo = FLT_MAX;
  a.eta_hi = 0.f;
  for (long long l = 0; !pgd && l < a.L && l < UFPGD_MAX_LAYERS; ++l) {
    a.eta_lo = std::min(a.eta_lo, std::fabs(a.eta[l]));
    a.eta_hi = std::max(a.eta_hi, std::fabs(a.eta[l]));
  }
  auto kern = pgd ? mma_kernel<T, true, false> : mma_kernel<T, false, false>;
  auto robust = pgd ? mma_kernel<T, true, true> : mma_kernel<T, false, true>;
  if constexpr (T::PAIR) {
    if (pgd && a.residual_tol > 0.f) {
      kern = mma_kernel<T, true, false, true>;
      robust = mma_kernel<T, true, true, true>;
    }
  }
  const long long ncta = T::PAIR ? (a.B + 1) / 2 : a.B;  // CTAs (PAIR: two realizations each)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(robust, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
  if (e != cudaSuccess) return e;
  if (nblocks) *nblocks = a.B;
  if (a.B == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {
    int fast_per_sm = 1;  // one wave of the fast kernel = the L2 prefetch distance
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fast_per_sm, kern, T::NT, T::SMEM) != cudaSuccess ||
        fast_per_sm < 1)
      fast_per_sm = 1;
    a.prefetch_ahead = static_cast<long long>(sms) * fast_per_sm;
  }
  int* list = nullptr;
  if ((e = scratch_alloc_async(reinterpret_cast<void**>(&list), sizeof(int) * (ncta + 1), s)) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(list, 0, sizeof(int), s)) == cudaSuccess) {
    kern<<<static_cast<unsigned>(ncta), T::NT, T::SMEM, s>>>(a, list + 1, list);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    // one wave of the robust instance: enough CTAs for a batch that is handed
    // off entirely (e.g. every channel far outside the f16 range), and a few
    // hundred CTAs that read a zero count and exit in the usual case
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, robust, T::NT, T::SMEM) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    const long long grid = std::min<long long>(ncta, static_cast<long long>(sms) * per_sm);
    robust<<<static_cast<unsigned>(grid), T::NT, T::SMEM, s>>>(a, list + 1, list);
    e = cudaGetLastError();
  }
  cudaFreeAsync(list, s);
  return e;
}

}  // namespace

// Unfolded forward and fixed-step PGD at (16,128), (32,256);
// ufpgd_gpu_set_option(UFPGD_OPT_TENSOR_CORES, 0) selects the CUDA-core tile
// kernel for A/B runs.
// (8,64) (BASELINE configs 2 and 3): realization pairs in the (16,128) frame
// (solve_pgd's residual_tol early stop stays on the FFMA2 team kernel).
bool mma_supported(int K, int M, bool pgd) {
  (void)pgd;
  if (!((K == 32 && M == 256) || (K == 16 && M == 128) || (K == 8 && M == 64))) return false;
  return option(UFPGD_OPT_TENSOR_CORES) != 0;
}

cudaError_t launch_mma(const FusedArgs& a, bool pgd, int K, int M, cudaStream_t s, long long* nblocks) {
  if (K == 32 && M == 256) return launch_mma_t<Mma_32_256>(a, pgd, s, nblocks);
  if (K == 16 && M == 128) return launch_mma_t<Mma_16_128>(a, pgd, s, nblocks);
  if (K == 8 && M == 64) return launch_mma_t<Mma_8_64x2>(a, pgd, s, nblocks);
  return cudaErrorInvalidValue;
}

}  // namespace ufpgd_gpu_impl
