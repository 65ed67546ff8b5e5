// Internal interface between the C ABI (capi.cpp) and the kernels (csrc/*.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "ufpgd_gpu.h"

namespace ufpgd_gpu_impl {

// Arguments of the fused team kernel (one team of TK*TM threads per
// realization; see team.cu). Passed by value as a __grid_constant__.
struct FusedArgs {
  const float2* H;
  float2* W;
  const float2* W0;
  const float* eta_in;    // PGD: per-realization step (nullable -> power iteration)
  float* eta_out;         // PGD: step used (nullable)
  int32_t* diverged_at;   // nullable
  float* l21;             // nullable
  int32_t* active;        // nullable
  double* block_partials; // [gridDim.x][3], nullable
  long long B;
  long long L;            // layers (unfolded) or iterations (PGD)
  int w0_mode;
  int power_steps;        // PGD with eta_in == nullptr
  float lambda;           // PGD threshold factor (thr = lambda * eta)
  float alpha;            // PA constant for the consumed-power statistic
  float residual_tol;     // PGD: relative iterate-change stop (0 = run all iterations; team kernels)
  int64_t* iterations;    // PGD with residual_tol: iterations taken per realization (nullable)
  float cmax;             // tensor-core kernel: max |c_k| and the range of the
  float eta_lo, eta_hi;   //   per-layer steps (filled by launch_mma)
  long long prefetch_ahead;  // tensor-core kernel: L2 prefetch distance in realizations (0: none)
  // taped team kernel (launch_fused_taped; nullable): iterates[(L+1)][B][M][K],
  // step images tape_v[L][B][M][K], column norms / shrink factors [L][B][M]
  float2* iterates;
  float2* tape_v;
  float* tape_norms;
  float* tape_shrink;
  float c[UFPGD_MAX_USERS];
  float eta[UFPGD_MAX_LAYERS];
  float thr[UFPGD_MAX_LAYERS];
  float2 v0[256];         // power-iteration start vector (PGD)
};

// Vector type of a real type for the general kernel (FP32 and FP64 builds).
template <class T>
struct Vec2;
template <>
struct Vec2<float> {
  using type = float2;
};
template <>
struct Vec2<double> {
  using type = double2;
};

// Arguments of the general-shape kernel (one CTA per realization), in FP32
// (GeneralArgs) or FP64 (GeneralArgs64: the precision path of the
// per-channel C++ API and of oracle_solve).
template <class T>
struct GeneralArgsT {
  using V2 = typename Vec2<T>::type;
  const V2* H;
  V2* W;
  const V2* W0;
  int32_t* diverged_at;
  int64_t* iterations;
  T* l21;
  int32_t* active;
  double* block_partials;  // [B][3]
  V2* iterates;
  V2* tape_v;
  T* tape_norms;
  T* tape_shrink;
  long long B;
  int K, M, L;
  int w0_mode;
  int mode;         // 0 layers, 1 gradient only
  int pgd;          // 1: every layer uses the realization's own step (below)
  long long iters;  // layer / iteration count when pgd == 1
  const T* eta_b;   // pgd: per-realization step (nullable -> 1 / lip_b)
  const T* lip_b;   // pgd: per-realization Lipschitz estimate
  T* eta_out;       // pgd: step used (nullable)
  T lambda;         // pgd: thr = lambda * eta
  int index_base;   // 0: layer index, 1: 1-based iteration
  T residual_tol;
  T alpha;
  T c[UFPGD_MAX_USERS];
  T eta[UFPGD_MAX_LAYERS];
  T thr[UFPGD_MAX_LAYERS];
};
using GeneralArgs = GeneralArgsT<float>;
using GeneralArgs64 = GeneralArgsT<double>;

// Arguments of the training-gradient kernel (one CTA per realization).
template <class T>
struct GradArgsT {
  using V2 = typename Vec2<T>::type;
  const V2* H;
  const V2* labels;  // loss_kind 1: supervised loss targets
  const V2* W0;      // w0_mode UFPGD_W0_GIVEN: start point [B][M][K]
  const V2* dcost;   // loss_kind 2: given dC/dRe(W) + i dC/dIm(W) of the output [B][M][K]
  V2* tape;          // [B][2][L][M*K] workspace
  double* out_loss;  // [B] (0 for loss_kind 2)
  double* out_grads; // [B][2L]
  long long B;
  int K, M, L;
  int w0_mode;
  int loss_kind;  // 0 unsupervised (lagrangian, lambda_cost), 1 supervised, 2 given dC/dW (backward)
  T lambda_cost;
  T c[UFPGD_MAX_USERS];
  T eta[UFPGD_MAX_LAYERS];
  T thr[UFPGD_MAX_LAYERS];
  double lam[UFPGD_MAX_LAYERS];
  double eta64[UFPGD_MAX_LAYERS];
};
using GradArgs = GradArgsT<float>;
using GradArgs64 = GradArgsT<double>;

struct PowerArgs {
  const float2* H;
  float* Lout;
  long long B;
  int K, M, steps;
  float2 v0[1024];
};

// Library options (ufpgd_gpu_set_option; capi.cpp), read at launch time.
int64_t option(int id);
// Stream-ordered scratch from the library's private pool (kept mapped across
// calls); free with cudaFreeAsync.
cudaError_t scratch_alloc_async(void** p, size_t bytes, cudaStream_t s);

// Fused team kernel availability for (K, M); fills the launch geometry.
bool fused_supported(int K, int M);
int fused_realizations_per_block(int K, int M);
// *nblocks receives the grid size (= number of block partials written).
cudaError_t launch_fused(const FusedArgs& a, bool pgd, int K, int M, cudaStream_t s,
                         long long* nblocks);
// Unfolded layers with tapes / iterates (ForwardOptions, unfolded.hpp:40-62) on
// the fused team kernel, for the K <= 8 team shapes; raw per-layer eta / thr.
bool fused_taped_supported(int K, int M);
cudaError_t launch_fused_taped(const FusedArgs& a, int K, int M, cudaStream_t s);
// Tiled CTA kernels (tile.cu) for (16,128) and (32,256); launch_fused forwards there.
cudaError_t launch_tiled(const FusedArgs& a, bool pgd, int K, int M, cudaStream_t s, long long* nblocks);
// Tensor-core (tcgen05) unfolded forward / fixed-step PGD at (16,128), (32,256) (mma.cu);
// launch_tiled forwards there.
bool mma_supported(int K, int M, bool pgd);
cudaError_t launch_mma(const FusedArgs& a, bool pgd, int K, int M, cudaStream_t s, long long* nblocks);
size_t general_smem_bytes(int K, int M);
cudaError_t launch_general(const GeneralArgs& a, cudaStream_t s);
cudaError_t launch_general64(const GeneralArgs64& a, cudaStream_t s);
// FP64 warp-per-realization PGD for (8,64) and (4,32) (team64.cu); launch_general64
// dispatches there for plain batched PGD without tapes or iterates.
bool pgd64_team_supported(const GeneralArgs64& a);
cudaError_t launch_pgd64_team(const GeneralArgs64& a, cudaStream_t s);
size_t general64_smem_bytes(int K, int M);
cudaError_t launch_power(const PowerArgs& a, cudaStream_t s);
cudaError_t launch_lipschitz_exact(const double2* H, long long B, int K, int M, const double2* v0,
                                   double* Lout, int32_t* status, cudaStream_t s);
size_t metrics_smem_bytes(int K, int M);
cudaError_t launch_metrics(const float2* H, const float2* W, long long B, int K, int M, const double* c,
                           double sigma2, double alpha, double* out, float2* Wzf, cudaStream_t s);
size_t grad_smem_bytes(int K, int M);
cudaError_t launch_grad(const GradArgs& a, double* mean, cudaStream_t s);
size_t grad64_smem_bytes(int K, int M);
cudaError_t launch_grad64(const GradArgs64& a, double* mean, cudaStream_t s);
cudaError_t launch_channel_gen(unsigned long long seed_h, unsigned long long seed_g, double gain_range_db,
                               long long first_index, long long B, int K, int M, void* H, bool f64, cudaStream_t s);
cudaError_t launch_convert(const void* src, void* dst, long long B, int K, int M, bool to_c64, cudaStream_t s);
cudaError_t launch_repack_c64(const float2* src, int Ms, int Ks, float2* dst, int Md, int Kd, long long B,
                              cudaStream_t s);
cudaError_t measure_fp32_peak(double* tflops, double* sm_ghz);
cudaError_t launch_fill_i64(int64_t* p, long long n, int64_t value, cudaStream_t s);
cudaError_t launch_stats_finalize(const double* partials, long long n, double* stats,
                                  cudaStream_t s);

}  // namespace ufpgd_gpu_impl
