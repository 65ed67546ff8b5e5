/*
 * ufpgd_gpu.h — C ABI of the B200-native batched PA-aware precoder solver.
 *
 * This is the drop-in boundary for the reference's hot path: the precoder
 * entry points of /root/reference/proj/core (namespace ufpgd). Each function
 * below names the reference interface it replaces. The C++ API in
 * include/ufpgd/ (C++ headers) restores the reference signatures, validation and
 * exception types on top of this ABI; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Matrices are batches of K x M complex matrices in the reference's storage
 *    (Eigen col-major, column m = antenna m, types.hpp:14-20), i.e. row-major
 *    [B][M][K] arrays of ufpgd_c64 (layout-identical to CUDA float2 and to
 *    std::complex<float>).
 *  - Functions without a _host suffix take DEVICE pointers for the batch
 *    arrays, enqueue work on `stream` (a cudaStream_t, NULL = legacy default
 *    stream) of `device`, and return without synchronising. Small parameter
 *    arrays (lambda, eta, c, v0) are HOST pointers and are copied at the call.
 *  - _host functions take HOST pointers (pinned or pageable), run
 *    synchronously and pipeline the host<->device copies with the kernels.
 *  - No exceptions cross the ABI: 0 on success or a negative UFPGD_E* status,
 *    with ufpgd_gpu_last_error() giving the message of the calling thread's
 *    last failure.
 *  - One CUDA context per device; calls on a given device are serialised by
 *    the caller (the reference API is reentrant per realization; batches are
 *    the unit here).
 */
#ifndef UFPGD_GPU_H
#define UFPGD_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UFPGD_GPU_ABI_VERSION 2

typedef struct {
  float re, im;
} ufpgd_c64;

typedef void* ufpgd_stream_t; /* cudaStream_t */

enum ufpgd_status {
  UFPGD_OK = 0,
  UFPGD_EINVAL_SHAPE = -1, /* std::invalid_argument on shapes (pgd.cpp:19-24) */
  UFPGD_EINVAL_PARAM = -2, /* std::invalid_argument on lambda/eta/etc. */
  UFPGD_EDIVERGED = -3,    /* DivergenceError (errors.hpp:18-25) */
  UFPGD_ECONVERGENCE = -4, /* ConvergenceError (errors.hpp:27-31) */
  UFPGD_ECUDA = -5,
  UFPGD_ENCCL = -6,
  UFPGD_ENOTSUP = -7,
  UFPGD_EDATAFORMAT = -8 /* DataFormatError (errors.hpp:33-37) */
};

enum ufpgd_w0_mode {
  UFPGD_W0_ZERO = 0,   /* W0 = 0 (BASELINE configs 1, 2, 4, 5) */
  UFPGD_W0_CONJ_H = 1, /* W0 = H^* — the reference default (pgd.cpp:184, unfolded.cpp:96) */
  UFPGD_W0_GIVEN = 2   /* W0 from the caller (the `start` argument) */
};

/* Largest supported layer count of one unfolded launch and user count. */
#define UFPGD_MAX_LAYERS 256
#define UFPGD_MAX_USERS 64

int ufpgd_gpu_abi_version(void);
const char* ufpgd_gpu_last_error(void);

/*
 * Process-wide tuning / A-B options of the library. They are set only through
 * this call (never read from the environment), take effect at the next launch
 * and default to the measured-best choice. No reference counterpart: the
 * reference has one CPU code path.
 */
enum ufpgd_option {
  UFPGD_OPT_TENSOR_CORES = 0,   /* 1 (default): tcgen05 kernel at (16,128), (32,256); 0: FFMA2 tile kernel */
  UFPGD_OPT_FUSED_WARPS = 1,    /* 0 (default): warps per fused-kernel block chosen per launch; 1..8: forced */
  UFPGD_OPT_FP64_TEAM = 2,      /* 1 (default): warp-per-realization FP64 PGD at (8,64), (4,32); 0: general kernel */
  UFPGD_OPT_ZERO_PAD = 3,       /* 1 (default): unsupported shapes run zero-padded on a fused shape; 0: general */
  UFPGD_OPT_PAD_SUB_BYTES = 4,  /* padded-path sub-batch size in bytes of padded H (default 1 GiB) */
  UFPGD_OPT_HOST_PIPE = 5,      /* host-buffer pipeline: 0 (default) phased, 1 depth-first streams */
  UFPGD_OPT_HOST_CHUNK_BYTES = 6, /* host-buffer pipeline chunk in bytes of H (default 16 MiB) */
  UFPGD_OPT_HOST_TIMELINE = 7,  /* 1: per-chunk event timeline of the host pipeline on stderr */
  UFPGD_OPT_COUNT = 8
};
/* Returns UFPGD_EINVAL_PARAM for an unknown option or out-of-range value. */
int ufpgd_gpu_set_option(int option, int64_t value);
/* Current value, or INT64_MIN for an unknown option. */
int64_t ufpgd_gpu_get_option(int option);
int ufpgd_gpu_device_count(int* count);

/*
 * Batched unfolded forward pass — replaces ufpgd::forward / forward_infer
 * (unfolded.hpp:64-74, unfolded.cpp:83-156) applied to B independent
 * channels. Layer i uses step eta[i] and threshold lambda[i]*eta[i]
 * (computed in FP64 here, then rounded to FP32). c[k] = sigma_nu*sqrt(gamma_k)
 * (SystemConfig::constraint_diag, system_config.cpp:45-47). Parameters are NOT
 * projected or checked against the box here (the C++ layer does that exactly
 * like unfolded.cpp:19-35); only lambda >= 0 and eta > 0 are required.
 *
 * Outputs (device, any may be NULL):
 *   W[B][M][K]        final precoders
 *   diverged_at[B]    first 0-based layer whose step image was non-finite, -1 if none
 *                     (DivergenceError index semantics of unfolded.cpp:120-125)
 *   l21[B]            ||W_b||_{2,1} (metrics.cpp:10-16), NaN when diverged
 *   active[B]         #{m : ||w_m||^2 > 0} (pgd.cpp:23-29), -1 when diverged
 *   stats[3] (double) {sum_b alpha*||W_b||_{2,1}, sum_b active_b, #diverged},
 *                     sums over non-diverged realizations, deterministic order.
 *
 * Kernels: the fused FFMA2 kernels for (4,16), (4,32), (4,64), (8,32), (8,64),
 * (8,128); the tcgen05 tensor-core kernel (FP32-class 3-term f16 split, TMEM
 * accumulators) for (16,128), (32,256); any other (K, M) within 6x the flops
 * of one of them runs zero-padded on it (padded users / antennas stay exactly
 * zero); the rest run the general CTA-per-realization kernel.
 */
int ufpgd_gpu_unfolded_forward(const ufpgd_c64* H, int64_t B, int K, int M,
                               const double* lambda, const double* eta, int L,
                               const double* c, int w0_mode, const ufpgd_c64* W0,
                               ufpgd_c64* W, int32_t* diverged_at, float* l21,
                               int32_t* active, double* stats, double alpha,
                               int device, ufpgd_stream_t stream);

/*
 * Batched fixed-step power iteration on H^T H^* — replaces
 * ufpgd::lipschitz_bound's `exact` (pgd.hpp:85-89, pgd.cpp:120-169) with the
 * BASELINE rule: exactly `steps` applications from the reference's shared
 * start vector (Rng(0x1F2E3D4C5B6A7988), pgd.cpp:131-134; pass v0 = NULL) or
 * from a caller v0[M] (host). Lout[b] = Re(v^H w) of the last application;
 * 0 for an all-zero channel (pgd.cpp:150-153).
 */
int ufpgd_gpu_power_iteration(const ufpgd_c64* H, int64_t B, int K, int M,
                              const ufpgd_c64* v0, int steps, float* Lout, int device,
                              ufpgd_stream_t stream);

/*
 * Batched converged power iteration in FP64 — ufpgd::lipschitz_bound's
 * `exact` (pgd.cpp:120-169) with the reference's rule: relative change
 * <= 1e-8 marks convergence, refinement continues to 1e-13 or 1e4 iterations.
 * H is interleaved complex128 [B][M][K] (device); status[b] = 0 or
 * UFPGD_ECONVERGENCE. Synchronous on `stream`.
 */
int ufpgd_gpu_lipschitz_exact(const double* H, int64_t B, int K, int M, double* Lout,
                              int32_t* status, int device, ufpgd_stream_t stream);

/*
 * Batched plain PGD at a fixed step per realization — replaces
 * ufpgd::solve_pgd (pgd.hpp:102-110, pgd.cpp:178-268) with trace_every = 0 and
 * residual_tol = 0 over B channels. eta_in[B] (device) gives each
 * realization's step; with eta_in == NULL the kernel first runs `power_steps`
 * power iterations on its own channel and uses eta = 1/L (BASELINE config 3),
 * writing the step it used to eta_out[B] (nullable). Threshold = lambda*eta.
 * diverged_at holds the 1-based iteration of the first non-finite step image
 * (pgd.cpp:231-235 semantics), -1 if none. Other outputs as for
 * ufpgd_gpu_unfolded_forward.
 */
int ufpgd_gpu_pgd_fixed(const ufpgd_c64* H, int64_t B, int K, int M, const float* eta_in,
                        int power_steps, double lambda, int64_t iters, const double* c,
                        int w0_mode, const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at,
                        float* l21, int32_t* active, float* eta_out, double* stats,
                        double alpha, int device, ufpgd_stream_t stream);

/*
 * solve_pgd over B channels with solve_pgd's early stop — replaces
 * ufpgd::solve_pgd (pgd.hpp:102-110, pgd.cpp:178-268) with residual_tol > 0
 * (pgd.cpp:246-260): each realization stops after the first iteration whose
 * relative iterate change ||W_next - W||_F / max(||W||_F, 1e-12) is below
 * residual_tol; iterations[B] (device, nullable) receives the count taken
 * (result.iterations). residual_tol = 0 runs max_iters (= ufpgd_gpu_pgd_fixed).
 * K <= 8 shapes run the fused FFMA2 kernel with per-realization early exit; the
 * others the general kernel. Steps as for ufpgd_gpu_pgd_fixed.
 */
int ufpgd_gpu_solve_pgd_batch(const ufpgd_c64* H, int64_t B, int K, int M, const float* eta_in, int power_steps,
                              double lambda, int64_t max_iters, double residual_tol, const double* c, int w0_mode,
                              const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at, int64_t* iterations,
                              float* l21, int32_t* active, float* eta_out, double* stats, double alpha, int device,
                              ufpgd_stream_t stream);

/*
 * General layer sweep on any (K <= 64, M) shape — the per-realization
 * building blocks of pgd.hpp:41-72 (grad_f, prox_l21, pgd_step) and the taped
 * forward (ForwardOptions::with_tape / with_iterates, unfolded.hpp:40-62).
 * Runs L layers with raw per-layer (eta[i], thr[i]) — NO box check, thr given
 * directly (prox_l21 is eta = 0, thr = t; pgd_step is eta, lambda*eta).
 * mode 0: layers; mode 1: write grad_f(W0) to W and stop (W0 via w0_mode).
 * residual_tol > 0 enables solve_pgd's relative-change stop
 * (pgd.cpp:246-260) with iterations[B] receiving the steps taken.
 * Optional tapes (device, NULL skips): iterates[(L+1)][B][M][K],
 * tape_v[L][B][M][K] (step images), tape_norms / tape_shrink [L][B][M].
 * diverged_at: 0-based layer (index_base = 0) or 1-based iteration (1).
 * Mode 0 with index_base 0, no residual_tol and L >= 1 runs on the fused
 * kernels: with tapes on the team kernel's taped instance for the K <= 8
 * shapes ((4,16), (4,32), (4,64), (8,32), (8,64), (8,128); tapes written from
 * the registers of the layer sweep), without tapes on the unfolded forward's
 * kernel for every fused shape. The rest runs the general kernel (exact FP32
 * sqrt / division in the prox).
 */
int ufpgd_gpu_layers_general(const ufpgd_c64* H, int64_t B, int K, int M, const double* eta,
                             const double* thr, int L, const double* c, int w0_mode,
                             const ufpgd_c64* W0, int mode, double residual_tol, int index_base,
                             ufpgd_c64* W, int32_t* diverged_at, int64_t* iterations,
                             ufpgd_c64* iterates, ufpgd_c64* tape_v, float* tape_norms,
                             float* tape_shrink, int device, ufpgd_stream_t stream);

/*
 * FP64 twin of ufpgd_gpu_layers_general (all arrays interleaved complex128 /
 * double, device): the precision path behind the per-channel C++ API, so a
 * single-channel forward / solve_pgd / pgd_step / grad_f / prox_l21 on the
 * device reproduces the FP64 reference to rounding. K*M <= ~4500.
 */
int ufpgd_gpu_layers_general64(const double* H, int64_t B, int K, int M, const double* eta,
                               const double* thr, int L, const double* c, int w0_mode,
                               const double* W0, int mode, double residual_tol, int index_base,
                               double* W, int32_t* diverged_at, int64_t* iterations,
                               double* iterates, double* tape_v, double* tape_norms,
                               double* tape_shrink, int device, ufpgd_stream_t stream);

/*
 * solve_pgd in FP64 (pgd.cpp:178-268, trace off) over B channels with a
 * per-realization step eta[B] (device), shared lambda, max_iters and the
 * iterate-change stop residual_tol (0 disables); W0 (device, nullable ->
 * H^*). diverged_at[B]: 1-based iteration of the first non-finite step image
 * (the run stops there), -1 if none. Async on `stream`.
 */
int ufpgd_gpu_solve_pgd64(const double* H, int64_t B, int K, int M, const double* c, double lambda,
                          const double* eta, int64_t max_iters, double residual_tol, const double* W0,
                          double* W, int64_t* iterations, int32_t* diverged_at, int device,
                          ufpgd_stream_t stream);

/*
 * oracle_solve at scale (pgd.cpp:270-279) in FP64 over B
 * channels (complex128 [B][M][K], device): eta_b = 1 / the converged power
 * iteration (ufpgd_gpu_lipschitz_exact), PGD from H^* with lambda, at most
 * max_iters iterations and the per-realization iterate-change stop
 * residual_tol (the reference uses 1e5 and 1e-10). Outputs (device): W
 * complex128, eta_out[B] (nullable), iterations[B] (nullable), status[B] =
 * 0, UFPGD_ECONVERGENCE or UFPGD_EDIVERGED. Synchronous.
 */
int ufpgd_gpu_oracle_solve(const double* H, int64_t B, int K, int M, const double* c, double lambda,
                           int64_t max_iters, double residual_tol, double* W, double* eta_out,
                           int64_t* iterations, int32_t* status, int device, ufpgd_stream_t stream);

/*
 * Host-buffer (end-to-end) unfolded forward: H, W0, W, diverged_at and stats
 * are HOST pointers. The batch is streamed through the device in chunks with
 * H2D copy, kernel and D2H copy overlapped on separate streams; pageable
 * buffers are staged through pinned memory. Returns UFPGD_EDIVERGED (after
 * finishing the whole batch) when any realization diverged.
 */
int ufpgd_gpu_unfolded_forward_host(const ufpgd_c64* H, int64_t B, int K, int M,
                                    const double* lambda, const double* eta, int L,
                                    const double* c, int w0_mode, const ufpgd_c64* W0,
                                    ufpgd_c64* W, int32_t* diverged_at, double* stats,
                                    double alpha, int device);

/*
 * Asynchronous form of ufpgd_gpu_unfolded_forward_host, for streams of batches:
 * enqueues the batch's H2D copies, kernels, D2H copies and statistics on the
 * device's host pipeline and returns at once with a ticket; the pipeline of the
 * next call starts while this one drains, so back-to-back calls keep both PCIe
 * directions busy (no per-call fill / drain). H, W0 and W must stay valid (and
 * should be pinned) until ufpgd_gpu_host_wait(ticket), which also writes
 * diverged_at and stats and returns UFPGD_EDIVERGED like the synchronous call.
 * At most 3 calls per device may be in flight (UFPGD_ENOTSUP beyond).
 */
int ufpgd_gpu_unfolded_forward_host_async(const ufpgd_c64* H, int64_t B, int K, int M, const double* lambda,
                                          const double* eta, int L, const double* c, int w0_mode,
                                          const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at, double* stats,
                                          double alpha, int device, int64_t* ticket);
int ufpgd_gpu_host_wait(int64_t ticket);

/* Same for plain PGD with the in-kernel 1/L step (config 3 end to end). */
int ufpgd_gpu_pgd_fixed_host(const ufpgd_c64* H, int64_t B, int K, int M, int power_steps,
                             double lambda, int64_t iters, const double* c, int w0_mode,
                             const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at,
                             float* eta_out, double* stats, double alpha, int device);

/*
 * Single-process multi-GPU — replaces the reference's parallel_for over
 * channels (parallel.cpp:25-59, parallel.hpp:12-18) with devices
 * 0..ngpus-1 of this process and one ncclAllReduce of the three summary
 * statistics over the communicators built by ufpgd_gpu_init
 * (ncclCommInitAll). ufpgd_gpu_shutdown destroys the communicators and
 * releases the per-device workspaces of the host-buffer entry points and the
 * scratch pool of the zero-padded forward (they are re-created on demand).
 *
 * _sharded: host buffers, synchronous. Contiguous shards [g B/G, (g+1) B/G),
 * one host thread per device driving its pipelined host path; W0 (host,
 * [B][M][K]) for w0_mode = GIVEN. Returns UFPGD_EDIVERGED when any
 * realization diverged (per-realization indices in diverged_at).
 *
 * _sharded_device: every device's shard already resident (H[g], B[g]
 * realizations on device g; W0[g], W[g], diverged_at[g] likewise), outputs on
 * the same devices. stats[g] (device, 3 doubles) receives the GLOBAL sums
 * after the in-place all-reduce — no host round trip. Asynchronous on
 * streams[g] (NULL: the legacy default stream), like the single-device entry.
 */
int ufpgd_gpu_init(int ngpus);
int ufpgd_gpu_shutdown(void);
int ufpgd_gpu_unfolded_forward_sharded(const ufpgd_c64* H, int64_t B, int K, int M,
                                       const double* lambda, const double* eta, int L,
                                       const double* c, int w0_mode, const ufpgd_c64* W0, ufpgd_c64* W,
                                       int32_t* diverged_at, double* stats, double alpha);
int ufpgd_gpu_unfolded_forward_sharded_device(const ufpgd_c64* const* H, const int64_t* B, int K, int M,
                                              const double* lambda, const double* eta, int L, const double* c,
                                              int w0_mode, const ufpgd_c64* const* W0, ufpgd_c64* const* W,
                                              int32_t* const* diverged_at, double* const* stats, double alpha,
                                              const ufpgd_stream_t* streams);

/*
 * Training-step gradients — the per-sample body of
 * ufpgd::train (training.cpp:205-234) over B channels: taped forward from
 * W0 (H^* = the reference's default, or 0), the loss (loss_kind 0:
 * unsupervised_loss = lagrangian with lambda_cost; 1: supervised
 * ||W - labels||^2, training.cpp:59-95), its gradient, and backward
 * (unfolded.cpp:158-239). Device outputs: loss[B], grads[B][2L] in pack order
 * (d_lambda_0, d_eta_0, ...; training.hpp:50-51) and, if non-null,
 * mean[1 + 2L] = batch means (deterministic order) — what adam_update
 * consumes. FP32 compute, FP64 reductions. Async on `stream`.
 */
int ufpgd_gpu_unfolded_grad(const ufpgd_c64* H, int64_t B, int K, int M, const double* lambda,
                            const double* eta, int L, const double* c, int w0_mode, int loss_kind,
                            double lambda_cost, const ufpgd_c64* labels, double* loss, double* grads,
                            double* mean, int device, ufpgd_stream_t stream);

/*
 * backward (unfolded.hpp:80-89, unfolded.cpp:158-239) in FP64 over B channels:
 * the forward from W0 (w0_mode; UFPGD_W0_GIVEN reproduces a tape whose layer-0
 * input is W0) is re-run on the device with its tape, and the reverse sweep
 * starts from the given output gradient dcost_dw = dC/dRe(W) + i dC/dIm(W).
 * Device buffers, interleaved FP64 complex [B][M][K]; grads[B][2L] in pack
 * order (d_lambda_0, d_eta_0, ...). Async on `stream`.
 */
int ufpgd_gpu_unfolded_backward64(const double* H, int64_t B, int K, int M, const double* lambda,
                                  const double* eta, int L, const double* c, int w0_mode,
                                  const double* W0, const double* dcost_dw, double* grads, int device,
                                  ufpgd_stream_t stream);

/*
 * Batched metrics — compute_metrics (metrics.cpp:79-91)
 * with the ZF reference of zf_precoder (zf.cpp:9-30) for B (H, W) pairs,
 * the body of evaluate's parallel_for (training.cpp:324-357). FP64 on the
 * device. out[b][6 + K] = {tx_power, cons_power, sum_rate, pcg, residual,
 * zf_ok, sinr[0..K-1]}; zf_ok = 0 where zf_precoder would throw
 * SingularChannelError (pcg = NaN there). Wzf (nullable) receives the ZF
 * precoders. K <= 32. Synchronous on `stream`.
 */
int ufpgd_gpu_metrics(const ufpgd_c64* H, const ufpgd_c64* W, int64_t B, int K, int M, const double* c,
                      double sigma_nu, double alpha, double* out, ufpgd_c64* Wzf, int device,
                      ufpgd_stream_t stream);

/*
 * UFPD dataset files — the reference's binary format
 * (dataset.hpp:23-36, dataset.cpp:38-175): 36-byte little-endian header,
 * then N row-major K x M matrices of interleaved f64 (re, im), then N labels
 * when flagged. Errors are UFPGD_EDATAFORMAT (magic, version, dimensions,
 * truncation, trailing bytes, missing file) with ufpgd_dataset_last_error().
 *   read_header: host only.
 *   gpu_ufpd_load: samples [first, first + count) of the channels (which = 0)
 *     or labels (1) into a DEVICE complex64 batch [count][M][K]; the f64
 *     payload is streamed through pinned memory and transposed / rounded on
 *     the device. Synchronous.
 *   gpu_ufpd_store: write_dataset from DEVICE batches (labels nullable),
 *     atomically (temp file + rename).
 *   gpu_convert_f64_rowmajor: the device layout conversion alone
 *     (to_c64 = 1: f64 [B][K][M][2] -> c64 [B][M][K]; 0: the reverse, src is
 *     then the f64 destination). Async on `stream`.
 */
const char* ufpgd_dataset_last_error(void);
int ufpgd_ufpd_read_header(const char* path, int* K, int* M, int64_t* N, uint64_t* seed, int* has_labels);
int ufpgd_gpu_ufpd_load(const char* path, int64_t first, int64_t count, int which, ufpgd_c64* dst, int device);
int ufpgd_gpu_ufpd_store(const char* path, int K, int M, int64_t N, uint64_t seed, const ufpgd_c64* channels,
                         const ufpgd_c64* labels, int device);
int ufpgd_gpu_convert_f64_rowmajor(const double* src, int64_t B, int K, int M, ufpgd_c64* dst, int to_c64,
                                   int device, ufpgd_stream_t stream);

/*
 * Measurement helper (not a reference interface): FP32 FMA throughput of the
 * device with the kernel's own FFMA2 instruction form, and the SM clock read
 * in-kernel during the probe. The roofline denominator of bench.py.
 */
int ufpgd_gpu_fp32_peak(int device, double* tflops, double* sm_ghz);

/*
 * Seeded synthetic input generation (harness side of SURVEY §8d, not timed):
 * realization i = first_index + b is generate_channel(Rng::stream(seed_h, i))
 * (channel.cpp:7-16, rng.cpp:19-40), row k scaled in FP64 by
 * 10^(-u_k * gain_range_db / 20) with u_k = Rng::stream(seed_g, i).uniform()
 * (gain_range_db = 0 disables), then rounded once to complex64. Host output
 * [B][M][K]; `threads` host threads (<= 0: all).
 */
int ufpgd_generate_channels(uint64_t seed_h, uint64_t seed_g, double gain_range_db,
                            int64_t first_index, int64_t B, int K, int M, ufpgd_c64* H,
                            int threads);

/*
 * The same draw on the DEVICE (for million-realization
 * runs): DEVICE output [B][M][K], complex64 (out_f64 = 0; H is ufpgd_c64*) or
 * interleaved FP64 (out_f64 = 1; H is double*, the reference's precision
 * before rounding). The mt19937_64 integer streams are bit-identical to the
 * host's; FP64 entries agree to a few ulp (CUDA log/sincos/pow vs glibc).
 * K <= UFPGD_MAX_USERS. Async on `stream`.
 */
int ufpgd_gpu_generate_channels(uint64_t seed_h, uint64_t seed_g, double gain_range_db,
                                int64_t first_index, int64_t B, int K, int M, void* H, int out_f64,
                                int device, ufpgd_stream_t stream);

/* The reference's power-iteration start vector (pgd.cpp:131-134), FP64 -> c64,
 * and in FP64 (interleaved re, im). */
int ufpgd_power_v0(int M, ufpgd_c64* v0);
int ufpgd_power_v0_f64(int M, double* v0);

/*
 * BASELINE layer parameters: Rng::stream(seed_p, 0) draws in pack order
 * (lambda_0, mu_0, lambda_1, mu_1, ...) with lambda = 0.01 + 0.09u and
 * mu = (0.5 + u) / mp_bound(K, M). Raw (unprojected) FP64 values.
 */
int ufpgd_layer_params(uint64_t seed_p, int L, int K, int M, double* lambda, double* eta);

#ifdef __cplusplus
}
#endif

#endif /* UFPGD_GPU_H */
