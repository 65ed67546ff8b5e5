// C ABI of the B200 batched precoder solver (include/ufpgd_gpu.h).
// Validation, dispatch to the fused team kernel or the general-shape kernel,
// deterministic statistics, the pipelined host-buffer path and the
// single-process multi-GPU path with an NCCL all-reduce of the statistics.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ufpgd_gpu.h"
#include "ufpgd_internal.h"

using namespace ufpgd_gpu_impl;

// ---- library options (ufpgd_gpu_set_option) -----------------------------------
namespace {
std::atomic<int64_t> g_options[UFPGD_OPT_COUNT] = {
    1,           // UFPGD_OPT_TENSOR_CORES
    0,           // UFPGD_OPT_FUSED_WARPS (auto)
    1,           // UFPGD_OPT_FP64_TEAM
    1,           // UFPGD_OPT_ZERO_PAD
    1ll << 30,   // UFPGD_OPT_PAD_SUB_BYTES
    0,           // UFPGD_OPT_HOST_PIPE (phased)
    16ll << 20,  // UFPGD_OPT_HOST_CHUNK_BYTES
    0,           // UFPGD_OPT_HOST_TIMELINE
};
}  // namespace

namespace ufpgd_gpu_impl {
int64_t option(int id) { return g_options[id].load(std::memory_order_relaxed); }
}  // namespace ufpgd_gpu_impl

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(UFPGD_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define UFPGD_CUDA(call)                                      \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);       \
  } while (0)

// Sets the device for the duration of a call and restores the previous one.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Saves the caller's current device and restores it on scope exit.
struct DeviceRestore {
  int prev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceRestore() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int check_shape(int64_t B, int K, int M) {
  if (B < 0) return fail(UFPGD_EINVAL_SHAPE, "batch size must be >= 0");
  if (K < 1 || M < K) return fail(UFPGD_EINVAL_SHAPE, "need 1 <= K <= M (system_config.cpp:23-27)");
  if (K > UFPGD_MAX_USERS) return fail(UFPGD_ENOTSUP, "K exceeds UFPGD_MAX_USERS");
  return UFPGD_OK;
}

int check_c(const double* c, int K) {
  if (!c) return fail(UFPGD_EINVAL_PARAM, "c (constraint diagonal) is required");
  for (int k = 0; k < K; ++k)
    if (!std::isfinite(c[k])) return fail(UFPGD_EINVAL_PARAM, "c must be finite");
  return UFPGD_OK;
}

bool general_fits(int K, int M) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (optin <= 0) optin = 227 * 1024;
  return general_smem_bytes(K, M) + 1024 <= static_cast<size_t>(optin);
}

// Finalises block partials into stats (or just frees them).
int finish_stats(double* partials, long long n, double* stats, cudaStream_t s) {
  if (stats && partials) {
    cudaError_t e = launch_stats_finalize(partials, n, stats, s);
    if (e != cudaSuccess) return cuda_fail(e, "stats_finalize");
  }
  if (partials) cudaFreeAsync(partials, s);
  return UFPGD_OK;
}

// Fused-kernel shape a (K, M) batch can be zero-padded to: the cheapest
// supported (Kp >= K, Mp >= M) within 6x the flops (the fused kernels run
// 7-8x the general kernel's rate). Padded users (H row 0, c = 0) and antennas
// (H column 0) keep W exactly 0 through every layer and add exact zeros to
// every contraction and norm, so the cropped result is the (K, M) solve.
// Library-private stream-ordered pool for the padded path's scratch: keeps
// its memory across calls (release threshold unbounded) without changing the
// device's default pool that other code in the process may rely on.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    if (!g_pool[dev]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&g_pool[dev], &props);
      if (e != cudaSuccess) return e;
      // Keep up to 1 GiB mapped across calls (re-mapping the scratch of every
      // padded call made it 2x slower); memory above that goes back to the
      // device at the next synchronisation, so other users of HBM get it back.
      unsigned long long keep = 1ull << 30;
      cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return cudaMallocFromPoolAsync(p, bytes, g_pool[dev], s);
}

}  // namespace

namespace ufpgd_gpu_impl {
// Stream-ordered scratch that stays mapped across calls (the private pool
// above); during stream capture the graph's own allocator is used instead.
cudaError_t scratch_alloc_async(void** p, size_t bytes, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
    return cudaMallocAsync(p, bytes, s);
  return scratch_alloc(p, bytes, s);
}
}  // namespace ufpgd_gpu_impl

namespace {

void release_pool(int dev) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (g_pool[dev]) {
    cudaDeviceSynchronize();
    cudaMemPoolDestroy(g_pool[dev]);
    g_pool[dev] = nullptr;
  }
}

long long pad_sub_bytes() { return option(UFPGD_OPT_PAD_SUB_BYTES); }

bool padded_shape(int K, int M, int* Kp, int* Mp) {
  if (option(UFPGD_OPT_ZERO_PAD) == 0) return false;
  static const int shapes[][2] = {{4, 16}, {4, 32}, {4, 64}, {8, 32}, {8, 64}, {8, 128}, {16, 128}, {32, 256}};
  double best = 6.0 * K * K * M;
  bool found = false;
  for (const auto& sh : shapes) {
    const double cost = static_cast<double>(sh[0]) * sh[0] * sh[1];
    if (sh[0] >= K && sh[1] >= M && cost <= best && fused_supported(sh[0], sh[1])) {
      best = cost;
      *Kp = sh[0];
      *Mp = sh[1];
      found = true;
    }
  }
  return found;
}

// Runs `body` over zero-padded sub-batches: H (and W0 when given) repacked to
// [nb][Mp][Kp] scratch, `body(hp, w0p, wp, b0, nb, parts_at, &np)` enqueues
// the fused kernel, W cropped back. Returns the partial count in *nparts.
template <class Body>
int run_padded(const float2* H, const float2* W0, float2* W, int64_t B, int K, int M, int Kp, int Mp,
               double* partials, cudaStream_t s, long long* nparts, Body body) {
  // sub-batches of <= 1 GiB of padded H bound the scratch
  const int64_t sub = std::max<int64_t>(1, std::min<int64_t>(B, pad_sub_bytes() / (8ll * Kp * Mp)));
  const size_t bytes = static_cast<size_t>(sub) * Kp * Mp * sizeof(float2);
  float2 *hp = nullptr, *wp = nullptr, *w0p = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&hp), bytes, s);
  if (e == cudaSuccess) e = scratch_alloc(reinterpret_cast<void**>(&wp), bytes, s);
  if (e == cudaSuccess && W0) e = scratch_alloc(reinterpret_cast<void**>(&w0p), bytes, s);
  int rc = UFPGD_OK;
  long long parts = 0;
  for (int64_t b0 = 0; b0 < B && e == cudaSuccess && rc == UFPGD_OK; b0 += sub) {
    const int64_t nb = std::min<int64_t>(sub, B - b0);
    e = launch_repack_c64(H + b0 * K * M, M, K, hp, Mp, Kp, nb, s);
    if (e == cudaSuccess && w0p) e = launch_repack_c64(W0 + b0 * K * M, M, K, w0p, Mp, Kp, nb, s);
    if (e != cudaSuccess) break;
    long long np = 0;
    rc = body(hp, w0p, wp, b0, nb, partials ? partials + 3 * parts : nullptr, &np);
    parts += np;
    if (rc == UFPGD_OK) e = launch_repack_c64(wp, Mp, Kp, W + b0 * K * M, M, K, nb, s);
  }
  *nparts = parts;
  if (hp) cudaFreeAsync(hp, s);
  if (wp) cudaFreeAsync(wp, s);
  if (w0p) cudaFreeAsync(w0p, s);
  if (rc != UFPGD_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "zero-padded fused solve");
  return UFPGD_OK;
}

// Enqueues an unfolded forward on `s` (device buffers). Used by the public
// device API and by the chunked host path.
int enqueue_unfolded(const float2* H, int64_t B, int K, int M, const double* lambda,
                     const double* eta, int L, const double* c, int w0_mode, const float2* W0,
                     float2* W, int32_t* diverged_at, float* l21, int32_t* active,
                     double* partials, double alpha, cudaStream_t s, long long* nparts) {
  *nparts = B;
  if (fused_supported(K, M) && L >= 1) {
    FusedArgs a{};
    a.H = H;
    a.W = W;
    a.W0 = W0;
    a.diverged_at = diverged_at;
    a.l21 = l21;
    a.active = active;
    a.block_partials = partials;
    a.B = B;
    a.L = L;
    a.w0_mode = w0_mode;
    a.alpha = static_cast<float>(alpha);
    for (int k = 0; k < K; ++k) a.c[k] = static_cast<float>(c[k]);
    for (int l = 0; l < L; ++l) {
      a.eta[l] = static_cast<float>(eta[l]);
      a.thr[l] = static_cast<float>(lambda[l] * eta[l]);
    }
    cudaError_t e = launch_fused(a, false, K, M, s, nparts);
    if (e != cudaSuccess) return cuda_fail(e, "fused unfolded kernel");
    return UFPGD_OK;
  }
  int Kp = 0, Mp = 0;
  if (L >= 1 && padded_shape(K, M, &Kp, &Mp)) {
    double cp[UFPGD_MAX_USERS] = {};
    for (int k = 0; k < K; ++k) cp[k] = c[k];
    return run_padded(H, w0_mode == UFPGD_W0_GIVEN ? W0 : nullptr, W, B, K, M, Kp, Mp, partials, s, nparts,
                      [&](const float2* hp, const float2* w0p, float2* wp, int64_t b0, int64_t nb, double* parts,
                          long long* np) {
                        return enqueue_unfolded(hp, nb, Kp, Mp, lambda, eta, L, cp, w0_mode, w0p, wp,
                                                diverged_at ? diverged_at + b0 : nullptr, l21 ? l21 + b0 : nullptr,
                                                active ? active + b0 : nullptr, parts, alpha, s, np);
                      });
  }
  if (!general_fits(K, M)) return fail(UFPGD_ENOTSUP, "(K, M) too large for the general kernel");
  GeneralArgs g{};
  g.H = H;
  g.W = W;
  g.W0 = W0;
  g.diverged_at = diverged_at;
  g.l21 = l21;
  g.active = active;
  g.block_partials = partials;
  g.B = B;
  g.K = K;
  g.M = M;
  g.L = L;
  g.w0_mode = w0_mode;
  g.alpha = static_cast<float>(alpha);
  for (int k = 0; k < K; ++k) g.c[k] = static_cast<float>(c[k]);
  for (int l = 0; l < L; ++l) {
    g.eta[l] = static_cast<float>(eta[l]);
    g.thr[l] = static_cast<float>(lambda[l] * eta[l]);
  }
  cudaError_t e = launch_general(g, s);
  if (e != cudaSuccess) return cuda_fail(e, "general kernel");
  return UFPGD_OK;
}

long long partial_count(int64_t B, int K, int M, bool fused_path) {
  if (fused_path) {
    const int rpb = fused_realizations_per_block(K, M);
    return (B + rpb - 1) / rpb;
  }
  return B;
}

int check_layers(const double* lambda, const double* eta, int L) {
  if (L < 0 || L > UFPGD_MAX_LAYERS) return fail(UFPGD_EINVAL_PARAM, "layer count out of range");
  if (L > 0 && (!lambda || !eta)) return fail(UFPGD_EINVAL_PARAM, "lambda/eta required");
  for (int l = 0; l < L; ++l) {
    if (!(lambda[l] >= 0.0) || !std::isfinite(lambda[l]))
      return fail(UFPGD_EINVAL_PARAM, "layer " + std::to_string(l) + " lambda_i < 0");
    if (!(eta[l] > 0.0) || !std::isfinite(eta[l]))
      return fail(UFPGD_EINVAL_PARAM, "layer " + std::to_string(l) + " eta_i <= 0");
  }
  return UFPGD_OK;
}

int check_w0(int w0_mode, const void* W0) {
  if (w0_mode < 0 || w0_mode > 2) return fail(UFPGD_EINVAL_PARAM, "bad w0_mode");
  if (w0_mode == UFPGD_W0_GIVEN && !W0) return fail(UFPGD_EINVAL_PARAM, "W0 required");
  return UFPGD_OK;
}

// ---- NCCL, loaded lazily so the library never pins an NCCL build -----------
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
std::mutex g_nccl_mu;
Nccl g_nccl;
std::vector<ncclComm_t> g_comms;
constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclSum = 0;     // ncclSum

bool load_nccl() {
  if (g_nccl.h) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.h = h;
  g_nccl.CommInitAll = reinterpret_cast<decltype(g_nccl.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
  g_nccl.AllReduce = reinterpret_cast<decltype(g_nccl.AllReduce)>(dlsym(h, "ncclAllReduce"));
  g_nccl.GroupStart = reinterpret_cast<decltype(g_nccl.GroupStart)>(dlsym(h, "ncclGroupStart"));
  g_nccl.GroupEnd = reinterpret_cast<decltype(g_nccl.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
  g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.GetErrorString =
      reinterpret_cast<decltype(g_nccl.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  return g_nccl.CommInitAll && g_nccl.AllReduce && g_nccl.GroupStart && g_nccl.GroupEnd &&
         g_nccl.CommDestroy;
}

// In-place sum of a 3-double statistics buffer per device over the
// communicators of ufpgd_gpu_init (caller holds g_nccl_mu). Leaves the
// caller's current device unchanged.
int allreduce_stats(double* const* dstats, const cudaStream_t* streams, int G) {
  DeviceRestore keep;
  g_nccl.GroupStart();
  ncclResult_t first = 0;
  for (int gi = 0; gi < G; ++gi) {
    cudaSetDevice(gi);
    ncclResult_t r = g_nccl.AllReduce(dstats[gi], dstats[gi], 3, kNcclDouble, kNcclSum, g_comms[gi], streams[gi]);
    if (r != 0 && first == 0) first = r;
  }
  ncclResult_t end = g_nccl.GroupEnd();
  if (first == 0) first = end;
  if (first != 0)
    return fail(UFPGD_ENCCL, std::string("ncclAllReduce: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(first) : "?"));
  return UFPGD_OK;
}

// Per-device streams and 3-double statistics buffers of one sharded call,
// released on every exit path; the caller's current device is restored.
struct ShardSet {
  int G;
  bool ok = true;
  std::vector<cudaStream_t> streams;
  std::vector<double*> dstats;
  explicit ShardSet(int g) : G(g), streams(g, nullptr), dstats(g, nullptr) {
    DeviceRestore keep;
    for (int gi = 0; gi < G && ok; ++gi) {
      cudaSetDevice(gi);
      ok = cudaStreamCreateWithFlags(&streams[gi], cudaStreamNonBlocking) == cudaSuccess &&
           cudaMalloc(&dstats[gi], 3 * sizeof(double)) == cudaSuccess;
    }
  }
  ~ShardSet() {
    DeviceRestore keep;
    for (int gi = 0; gi < G; ++gi) {
      cudaSetDevice(gi);
      if (streams[gi]) cudaStreamSynchronize(streams[gi]);
      if (dstats[gi]) cudaFree(dstats[gi]);
      if (streams[gi]) cudaStreamDestroy(streams[gi]);
    }
  }
  int allreduce() { return allreduce_stats(dstats.data(), streams.data(), G); }
  int sync_and_read(double* out) {
    DeviceRestore keep;
    for (int gi = 0; gi < G; ++gi) {
      cudaSetDevice(gi);
      if (cudaStreamSynchronize(streams[gi]) != cudaSuccess) return fail(UFPGD_ECUDA, "sharded stream sync");
    }
    cudaSetDevice(0);
    if (cudaMemcpy(out, dstats[0], 3 * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(UFPGD_ECUDA, "statistics read");
    return UFPGD_OK;
  }
};

// Per-device workspace of the host-buffer path: NS chunk buffer sets, the
// pipeline streams and NC call slots, kept across calls so an end-to-end call
// costs only its copies and kernels. Enqueues on one device are serialised by
// its mutex; up to NC calls may be in flight (ufpgd_gpu_unfolded_forward_host_async).
struct HostWorkspace {
  std::mutex mu;
  std::condition_variable slot_free;  // signalled by host_finish
  bool init = false;
  static constexpr int NS = 4;  // chunk buffer sets
  static constexpr int NC = 3;  // host calls in flight
  cudaStream_t st[NS] = {};
  // phased pipeline: copy-in, two kernel and copy-out streams, chained per
  // buffer set by events (across calls too: set i's previous use may belong to
  // the previous call)
  cudaStream_t sx[4] = {};
  cudaEvent_t ev[NS][3] = {};
  void* buf[NS][5] = {};
  size_t cap[NS][5] = {};
  bool set_used[NS] = {};
  int next_set = 0;
  uint64_t chunk_seq = 0;
  // one in-flight call: its statistics partials (device), final statistics,
  // and pinned staging of the small per-realization outputs (a D2H copy into
  // pageable memory would block the host thread and serialise the pipeline)
  struct Call {
    bool busy = false;
    uint32_t gen = 0;
    cudaEvent_t done = nullptr;
    double* partials = nullptr;
    size_t partials_cap = 0;
    double* dstats = nullptr;
    void* pinned = nullptr;
    size_t pinned_cap = 0;
    int32_t* user_div = nullptr;
    float* user_eta = nullptr;
    double* user_stats = nullptr;
    int64_t B = 0;
    std::vector<cudaEvent_t> tev;  // UFPGD_OPT_HOST_TIMELINE = 2: printed by host_finish
  } calls[NC];
  cudaEvent_t tbase = nullptr;     // ... relative to the first such call's start
};
HostWorkspace g_ws[64];

cudaError_t ensure(void*& p, size_t& cap, size_t need) {
  if (need <= cap) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, need);
  if (e == cudaSuccess) cap = need;
  return e;
}

// Pipeline chunk size in bytes of H (UFPGD_OPT_HOST_CHUNK_BYTES).
long long host_chunk_bytes() { return option(UFPGD_OPT_HOST_CHUNK_BYTES); }

// Releases a device's host-path workspace (ufpgd_gpu_shutdown).
void release_workspace(HostWorkspace& ws) {
  std::lock_guard<std::mutex> lock(ws.mu);
  if (!ws.init) return;
  for (cudaStream_t x : ws.sx)
    if (x) cudaStreamSynchronize(x);
  for (int i = 0; i < HostWorkspace::NS; ++i) {
    cudaStreamSynchronize(ws.st[i]);
    for (int q = 0; q < 5; ++q) {
      if (ws.buf[i][q]) cudaFree(ws.buf[i][q]);
      ws.buf[i][q] = nullptr;
      ws.cap[i][q] = 0;
    }
    cudaStreamDestroy(ws.st[i]);
    ws.st[i] = nullptr;
    for (int q = 0; q < 3; ++q) {
      if (ws.ev[i][q]) cudaEventDestroy(ws.ev[i][q]);
      ws.ev[i][q] = nullptr;
    }
    ws.set_used[i] = false;
  }
  for (cudaStream_t& x : ws.sx) {
    if (x) cudaStreamDestroy(x);
    x = nullptr;
  }
  for (auto& c : ws.calls) {
    if (c.done) cudaEventDestroy(c.done);
    if (c.partials) cudaFree(c.partials);
    if (c.dstats) cudaFree(c.dstats);
    if (c.pinned) cudaFreeHost(c.pinned);
    const uint32_t gen = c.gen + 1;
    c = HostWorkspace::Call{};
    c.gen = gen;  // outstanding tickets of this device become invalid
  }
  ws.next_set = 0;
  ws.init = false;
}

// Host-call tickets: device (8 bits), slot (8 bits), generation (16 bits).
int64_t make_ticket(int device, int slot, uint32_t gen) {
  return (static_cast<int64_t>(gen & 0xFFFF) << 16) | (static_cast<int64_t>(slot) << 8) | device;
}

// Waits for an enqueued host call, copies its small outputs to the caller's
// pointers and frees its slot. Returns UFPGD_EDIVERGED when a realization diverged.
int host_finish(int64_t ticket) {
  const int device = static_cast<int>(ticket & 0xFF), slot = static_cast<int>((ticket >> 8) & 0xFF);
  const uint32_t gen = static_cast<uint32_t>((ticket >> 16) & 0xFFFF);
  if (ticket < 0 || device >= 64 || slot >= HostWorkspace::NC) return fail(UFPGD_EINVAL_PARAM, "bad host-call ticket");
  HostWorkspace& ws = g_ws[device];
  HostWorkspace::Call* c = nullptr;
  {
    std::lock_guard<std::mutex> lock(ws.mu);
    c = &ws.calls[slot];
    if (!c->busy || (c->gen & 0xFFFF) != gen) return fail(UFPGD_EINVAL_PARAM, "host-call ticket already completed");
  }
  cudaError_t e = cudaEventSynchronize(c->done);
  if (!c->tev.empty()) {  // deferred timeline (tuning aid): no synchronisation inside the enqueue
    const size_t nchunks = c->tev.size() / 4;
    for (size_t ci = 0; ci < nchunks; ++ci) {
      float t[4];
      for (int q = 0; q < 4; ++q) cudaEventElapsedTime(&t[q], ws.tbase, c->tev[4 * ci + q]);
      std::fprintf(stderr, "slot %d chunk %3zu  h2d %7.3f-%7.3f  kernel -%7.3f  d2h -%7.3f ms\n", slot, ci, t[0], t[1],
                   t[2], t[3]);
    }
    for (cudaEvent_t ev : c->tev)
      if (ev != ws.tbase) cudaEventDestroy(ev);
    c->tev.clear();
  }
  double host_stats[3] = {0.0, 0.0, 0.0};
  if (e == cudaSuccess) {
    const char* base = static_cast<const char*>(c->pinned);
    std::memcpy(host_stats, base, sizeof(host_stats));
    size_t off = 64;
    if (c->user_div) std::memcpy(c->user_div, base + off, sizeof(int32_t) * c->B);
    if (c->user_div) off += sizeof(int32_t) * c->B;
    if (c->user_eta) std::memcpy(c->user_eta, base + off, sizeof(float) * c->B);
    if (c->user_stats) std::memcpy(c->user_stats, host_stats, sizeof(host_stats));
  }
  {
    std::lock_guard<std::mutex> lock(ws.mu);
    c->busy = false;
    ++c->gen;
  }
  ws.slot_free.notify_all();
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline");
  if (host_stats[2] > 0.0) return fail(UFPGD_EDIVERGED, "non-finite iterate in at least one realization");
  return UFPGD_OK;
}

// Chunked host pipeline shared by the unfolded and PGD host entry points:
// enqueues every chunk's H2D, kernel and D2H plus the statistics finalisation,
// and returns a ticket for host_finish (the call itself does not wait).
// `run` enqueues the kernel for one chunk on stream s given device buffers.
// block_for_slot: the synchronous entry points wait for a free call slot
// (concurrent callers on one device); the asynchronous one reports UFPGD_ENOTSUP.
template <class Run>
int host_enqueue(int device, const ufpgd_c64* H, int64_t B, int K, int M, const ufpgd_c64* W0, ufpgd_c64* W,
                 int32_t* diverged_at, float* eta_out, long long parts_per_chunk_max, int64_t chunk, double* stats,
                 Run run, int64_t* ticket, bool block_for_slot) {
  if (device < 0 || device >= 64) return fail(UFPGD_EINVAL_PARAM, "device out of range");
  HostWorkspace& ws = g_ws[device];
  std::unique_lock<std::mutex> lock(ws.mu);
  constexpr int NS = HostWorkspace::NS;
  if (!ws.init) {
    for (int i = 0; i < NS; ++i) UFPGD_CUDA(cudaStreamCreateWithFlags(&ws.st[i], cudaStreamNonBlocking));
    for (cudaStream_t& x : ws.sx) UFPGD_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    for (int i = 0; i < NS; ++i)
      for (int q = 0; q < 3; ++q) UFPGD_CUDA(cudaEventCreateWithFlags(&ws.ev[i][q], cudaEventDisableTiming));
    for (auto& c : ws.calls) UFPGD_CUDA(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
    ws.init = true;
  }
  int slot = -1;
  for (;;) {
    for (int i = 0; i < HostWorkspace::NC && slot < 0; ++i)
      if (!ws.calls[i].busy) slot = i;
    if (slot >= 0) break;
    if (!block_for_slot)
      return fail(UFPGD_ENOTSUP, "too many host calls in flight on this device (wait for one first)");
    ws.slot_free.wait(lock);
  }
  HostWorkspace::Call& call = ws.calls[slot];
  const size_t per = static_cast<size_t>(K) * M * sizeof(float2);
  // Chunk boundaries (a geometric ramp of the first / last chunks was measured
  // and is no faster with the phased pipeline: the copy-out stream paces it).
  std::vector<int64_t> cs{0};
  for (int64_t b = chunk; b < B; b += chunk) cs.push_back(b);
  if (B > 0) cs.push_back(B);
  const int64_t nchunks = static_cast<int64_t>(cs.size()) - 1;
  const size_t need[5] = {per * chunk, per * chunk, W0 ? per * chunk : 0, sizeof(int32_t) * chunk,
                          eta_out ? sizeof(float) * chunk : 0};
  cudaError_t e = cudaSuccess;
  // a buffer set being regrown may still be in use by an earlier call
  bool regrow = false;
  for (int i = 0; i < NS; ++i)
    for (int q = 0; q < 5; ++q) regrow |= need[q] > ws.cap[i][q];
  if (regrow) {
    for (cudaStream_t x : ws.sx) cudaStreamSynchronize(x);
    for (cudaStream_t x : ws.st) cudaStreamSynchronize(x);
  }
  for (int i = 0; i < NS && e == cudaSuccess; ++i)
    for (int q = 0; q < 5 && e == cudaSuccess; ++q) e = ensure(ws.buf[i][q], ws.cap[i][q], need[q]);
  if (e == cudaSuccess) {
    void* pp = call.partials;
    e = ensure(pp, call.partials_cap, sizeof(double) * 3 * std::max<long long>(1, parts_per_chunk_max * nchunks));
    call.partials = static_cast<double*>(pp);
  }
  const size_t small_need = 64 + (diverged_at ? sizeof(int32_t) * B : 0) + (eta_out ? sizeof(float) * B : 0);
  if (e == cudaSuccess && small_need > call.pinned_cap) {
    if (call.pinned) cudaFreeHost(call.pinned);
    call.pinned = nullptr;
    call.pinned_cap = 0;
    // (default flags: under unified addressing every cudaHostAlloc allocation is
    // portable and device-addressable at its host address — the kernels store
    // diverged_at and the statistics into it)
    e = cudaHostAlloc(&call.pinned, small_need, cudaHostAllocDefault);
    if (e == cudaSuccess) call.pinned_cap = small_need;
  }
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline allocation");
  char* pin = static_cast<char*>(call.pinned);
  double* stats_stage = reinterpret_cast<double*>(pin);
  int32_t* div_stage = diverged_at ? reinterpret_cast<int32_t*>(pin + 64) : nullptr;
  float* eta_stage = eta_out ? reinterpret_cast<float*>(pin + 64 + (diverged_at ? sizeof(int32_t) * B : 0)) : nullptr;
  int rc = UFPGD_OK;
  std::vector<long long> part_off(nchunks + 1, 0);
  // Default pipeline ("phased"): one copy-in stream, two kernel streams, one
  // copy-out stream, chained per buffer set by events. The copy-out of chunk
  // k also waits for the copy-in of chunk k + 1, so every D2H starts together
  // with an H2D: PCIe then splits evenly between the directions (~48 GB/s
  // each), whereas a D2H started mid-way through an H2D takes the larger share
  // and slows the H2D stream that paces the pipeline (tools/pipe_probe2.py:
  // 88.8 vs 81.9 GB/s total). UFPGD_OPT_HOST_PIPE = 1 selects the earlier
  // depth-first pipeline over four streams, for A/B runs.
  const bool phased = option(UFPGD_OPT_HOST_PIPE) == 0;
  // UFPGD_OPT_HOST_TIMELINE = 1: per-chunk event timeline on stderr (tuning aid)
  // (= 2: deferred — printed by host_finish against the first call's start, so
  // the overlap of streamed calls shows)
  const bool timeline = option(UFPGD_OPT_HOST_TIMELINE) != 0;
  const bool timeline_deferred = option(UFPGD_OPT_HOST_TIMELINE) == 2;
  std::vector<cudaEvent_t> tev(timeline ? 4 * nchunks : 0);
  for (cudaEvent_t& ev : tev) cudaEventCreate(&ev);
  // Chunk ci uses buffer set set_of[ci] (a rotation that continues across
  // calls); events: 0 = copy-in done, 1 = kernel done, 2 = copy-out done. The
  // copy-in reuses the set's H buffer (waits for its previous kernel); the
  // kernel reuses its W buffer (waits for its previous copy-out).
  std::vector<int> set_of(nchunks);
  for (int64_t ci = 0; ci < nchunks; ++ci) set_of[ci] = (ws.next_set + static_cast<int>(ci % NS)) % NS;
  cudaStream_t sin = ws.sx[0], sout = ws.sx[3];
  if (phased)  // an earlier depth-first (A/B) call may still use the buffer sets
    for (int i = 1; i < NS; ++i) {
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, ws.st[i]);
      for (cudaStream_t x : ws.sx) cudaStreamWaitEvent(x, j, 0);
      cudaEventDestroy(j);
    }
  auto copy_out = [&](int64_t cj) -> int {
    const int j = set_of[cj];
    const int64_t b0 = cs[cj], nb = cs[cj + 1] - b0;
    cudaStreamWaitEvent(sout, ws.ev[j][1], 0);
    if (cj + 1 < nchunks) cudaStreamWaitEvent(sout, ws.ev[set_of[cj + 1]][0], 0);
    cudaError_t x = cudaMemcpyAsync(W + b0 * K * M, ws.buf[j][1], per * nb, cudaMemcpyDeviceToHost, sout);
    if (x == cudaSuccess && eta_out)
      x = cudaMemcpyAsync(eta_stage + b0, ws.buf[j][4], sizeof(float) * nb, cudaMemcpyDeviceToHost, sout);
    if (x != cudaSuccess) return cuda_fail(x, "D2H");
    if (timeline) cudaEventRecord(tev[4 * cj + 3], sout);
    cudaEventRecord(ws.ev[j][2], sout);
    return UFPGD_OK;
  };
  for (int64_t ci = 0; ci < nchunks && rc == UFPGD_OK && phased; ++ci) {
    const int i = set_of[ci];
    const int64_t b0 = cs[ci], nb = cs[ci + 1] - b0;
    cudaStream_t sk = ws.sx[1 + ((ws.chunk_seq + ci) & 1)];
    float2* dh = static_cast<float2*>(ws.buf[i][0]);
    float2* dw = static_cast<float2*>(ws.buf[i][1]);
    float2* dw0 = static_cast<float2*>(ws.buf[i][2]);
    int32_t* ddiv = static_cast<int32_t*>(ws.buf[i][3]);
    float* deta = static_cast<float*>(ws.buf[i][4]);
    if (ws.set_used[i]) cudaStreamWaitEvent(sin, ws.ev[i][1], 0);
    if (timeline) cudaEventRecord(tev[4 * ci], sin);
    e = cudaMemcpyAsync(dh, H + b0 * K * M, per * nb, cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess && W0) e = cudaMemcpyAsync(dw0, W0 + b0 * K * M, per * nb, cudaMemcpyHostToDevice, sin);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "H2D");
      break;
    }
    cudaEventRecord(ws.ev[i][0], sin);
    if (timeline) cudaEventRecord(tev[4 * ci + 1], sin);
    cudaStreamWaitEvent(sk, ws.ev[i][0], 0);
    if (ws.set_used[i]) cudaStreamWaitEvent(sk, ws.ev[i][2], 0);
    long long np = 0;
    // diverged_at: the kernels' only access is one coalesced 4-byte store per
    // realization, so they write the pinned stage directly (no 16 KB D2H copy
    // per chunk on the copy-out stream)
    rc = run(dh, nb, W0 ? dw0 : nullptr, dw, diverged_at ? div_stage + b0 : ddiv, eta_out ? deta : nullptr,
             call.partials + 3 * part_off[ci], &np, sk);
    if (rc != UFPGD_OK) break;
    part_off[ci + 1] = part_off[ci] + np;
    cudaEventRecord(ws.ev[i][1], sk);
    ws.set_used[i] = true;
    if (timeline) cudaEventRecord(tev[4 * ci + 2], sk);
    if (ci >= 1) rc = copy_out(ci - 1);
  }
  if (phased && rc == UFPGD_OK && nchunks > 0) rc = copy_out(nchunks - 1);
  if (phased) {
    ws.next_set = (ws.next_set + static_cast<int>(nchunks % NS)) % NS;
    ws.chunk_seq += static_cast<uint64_t>(nchunks);
  }
  for (int64_t ci = 0; ci < nchunks && rc == UFPGD_OK && !phased; ++ci) {
    // depth-first A/B pipeline (UFPGD_OPT_HOST_PIPE = 1): each chunk's copies
    // and kernel on one of the NS streams; it joins the call's tail below
    const int i = static_cast<int>(ci % NS);
    const int64_t b0 = cs[ci], nb = cs[ci + 1] - b0;
    cudaStream_t s = ws.st[i];
    for (cudaStream_t x : ws.sx) {  // the phased streams may hold an earlier call's use of set i
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, x);
      cudaStreamWaitEvent(s, j, 0);
      cudaEventDestroy(j);
    }
    float2* dh = static_cast<float2*>(ws.buf[i][0]);
    float2* dw = static_cast<float2*>(ws.buf[i][1]);
    float2* dw0 = static_cast<float2*>(ws.buf[i][2]);
    int32_t* ddiv = static_cast<int32_t*>(ws.buf[i][3]);
    float* deta = static_cast<float*>(ws.buf[i][4]);
    if (timeline) cudaEventRecord(tev[4 * ci], s);
    e = cudaMemcpyAsync(dh, H + b0 * K * M, per * nb, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && W0) e = cudaMemcpyAsync(dw0, W0 + b0 * K * M, per * nb, cudaMemcpyHostToDevice, s);
    if (timeline) cudaEventRecord(tev[4 * ci + 1], s);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "H2D");
      break;
    }
    long long np = 0;
    rc = run(dh, nb, W0 ? dw0 : nullptr, dw, ddiv, eta_out ? deta : nullptr, call.partials + 3 * part_off[ci], &np, s);
    if (rc != UFPGD_OK) break;
    part_off[ci + 1] = part_off[ci] + np;
    if (timeline) cudaEventRecord(tev[4 * ci + 2], s);
    e = cudaMemcpyAsync(W + b0 * K * M, dw, per * nb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && diverged_at)
      e = cudaMemcpyAsync(div_stage + b0, ddiv, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && eta_out)
      e = cudaMemcpyAsync(eta_stage + b0, deta, sizeof(float) * nb, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "D2H");
    if (timeline) cudaEventRecord(tev[4 * ci + 3], s);
  }
  // the call's tail on st[0]: after every stream that carried its chunks, the
  // statistics finalisation and their copy into the pinned slot, then `done`
  for (cudaStream_t x : ws.sx) {
    cudaEvent_t j;
    cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
    cudaEventRecord(j, x);
    cudaStreamWaitEvent(ws.st[0], j, 0);
    cudaEventDestroy(j);
  }
  if (!phased)
    for (int i = 1; i < NS; ++i) {
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, ws.st[i]);
      cudaStreamWaitEvent(ws.st[0], j, 0);
      cudaEventDestroy(j);
    }
  if (rc == UFPGD_OK) {
    // The finalisation kernel stores the three statistics straight into the
    // pinned slot (UVA: pinned host memory is device-addressable). A 24-byte
    // cudaMemcpyAsync here would sit in a copy-engine queue until this call's
    // last chunk is done, and the next streamed call's H2D copies queue up
    // behind it on the same engine: measured as every third streamed call
    // running ~7 ms instead of 5.6 (tools/e2e_periods.py, host_timeline2.py).
    e = launch_stats_finalize(call.partials, part_off[nchunks], stats_stage, ws.st[0]);
    if (e == cudaSuccess) e = cudaEventRecord(call.done, ws.st[0]);
    if (e != cudaSuccess) rc = cuda_fail(e, "host pipeline finalize");
  }
  if (timeline_deferred && rc == UFPGD_OK) {
    if (!ws.tbase && !tev.empty()) ws.tbase = tev[0];
    call.tev = std::move(tev);
  } else if (timeline) {
    cudaStreamSynchronize(ws.st[0]);
    for (int64_t ci = 0; ci < nchunks; ++ci) {
      float t[4];
      for (int q = 0; q < 4; ++q) cudaEventElapsedTime(&t[q], tev[0], tev[4 * ci + q]);
      std::fprintf(stderr, "chunk %3lld  h2d %7.3f-%7.3f  kernel -%7.3f  d2h -%7.3f ms\n", static_cast<long long>(ci),
                   t[0], t[1], t[2], t[3]);
    }
    for (cudaEvent_t ev : tev) cudaEventDestroy(ev);
  }
  if (rc != UFPGD_OK) {  // leave no work behind that still writes into the caller's buffers
    for (cudaStream_t x : ws.sx) cudaStreamSynchronize(x);
    for (int i = 0; i < NS; ++i) cudaStreamSynchronize(ws.st[i]);
    return rc;
  }
  call.busy = true;
  call.user_div = diverged_at;
  call.user_eta = eta_out;
  call.user_stats = stats;
  call.B = B;
  *ticket = make_ticket(device, slot, call.gen);
  return UFPGD_OK;
}

// Synchronous form: enqueue, then wait.
template <class Run>
int host_pipeline(int device, const ufpgd_c64* H, int64_t B, int K, int M, const ufpgd_c64* W0, ufpgd_c64* W,
                  int32_t* diverged_at, float* eta_out, long long parts_per_chunk_max, int64_t chunk, double* stats,
                  Run run) {
  int64_t ticket = -1;
  const int rc = host_enqueue(device, H, B, K, M, W0, W, diverged_at, eta_out, parts_per_chunk_max, chunk, stats,
                              run, &ticket, true);
  if (rc != UFPGD_OK) return rc;
  return host_finish(ticket);
}

}  // namespace

extern "C" {

int ufpgd_gpu_abi_version(void) { return UFPGD_GPU_ABI_VERSION; }

int ufpgd_gpu_set_option(int option, int64_t value) {
  bool ok = false;
  switch (option) {
    case UFPGD_OPT_TENSOR_CORES:
    case UFPGD_OPT_FP64_TEAM:
    case UFPGD_OPT_ZERO_PAD:
    case UFPGD_OPT_HOST_PIPE: ok = value == 0 || value == 1; break;
    case UFPGD_OPT_HOST_TIMELINE: ok = value >= 0 && value <= 2; break;
    case UFPGD_OPT_FUSED_WARPS: ok = value >= 0 && value <= 8; break;
    case UFPGD_OPT_PAD_SUB_BYTES:
    case UFPGD_OPT_HOST_CHUNK_BYTES: ok = value >= (1ll << 20) && value <= (1ll << 40); break;
    default: return fail(UFPGD_EINVAL_PARAM, "unknown option " + std::to_string(option));
  }
  if (!ok) return fail(UFPGD_EINVAL_PARAM, "option " + std::to_string(option) + ": value out of range");
  g_options[option].store(value, std::memory_order_relaxed);
  return UFPGD_OK;
}

int64_t ufpgd_gpu_get_option(int option) {
  if (option < 0 || option >= UFPGD_OPT_COUNT) return INT64_MIN;
  return g_options[option].load(std::memory_order_relaxed);
}

const char* ufpgd_gpu_last_error(void) { return g_last_error.c_str(); }

int ufpgd_gpu_device_count(int* count) {
  if (!count) return fail(UFPGD_EINVAL_PARAM, "count is null");
  UFPGD_CUDA(cudaGetDeviceCount(count));
  return UFPGD_OK;
}

int ufpgd_gpu_unfolded_forward(const ufpgd_c64* H, int64_t B, int K, int M, const double* lambda,
                               const double* eta, int L, const double* c, int w0_mode,
                               const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at, float* l21,
                               int32_t* active, double* stats, double alpha, int device,
                               ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_layers(lambda, eta, L)) || (rc = check_c(c, K)) ||
      (rc = check_w0(w0_mode, W0)))
    return rc;
  if (!(alpha > 0.0)) return fail(UFPGD_EINVAL_PARAM, "alpha must be > 0");
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    if (stats) UFPGD_CUDA(cudaMemsetAsync(stats, 0, 3 * sizeof(double), s));
    return UFPGD_OK;
  }
  const bool fused = fused_supported(K, M) && L >= 1;
  const long long np = partial_count(B, K, M, fused);
  double* partials = nullptr;
  if (stats) UFPGD_CUDA(scratch_alloc_async(reinterpret_cast<void**>(&partials), sizeof(double) * 3 * np, s));
  long long used = 0;
  rc = enqueue_unfolded(reinterpret_cast<const float2*>(H), B, K, M, lambda, eta, L, c, w0_mode,
                        reinterpret_cast<const float2*>(W0), reinterpret_cast<float2*>(W),
                        diverged_at, l21, active, partials, alpha, s, &used);
  int rc2 = finish_stats(partials, rc == UFPGD_OK ? used : 0, stats, s);
  return rc != UFPGD_OK ? rc : rc2;
}

int ufpgd_gpu_power_iteration(const ufpgd_c64* H, int64_t B, int K, int M, const ufpgd_c64* v0,
                              int steps, float* Lout, int device, ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M))) return rc;
  if (M > 1024) return fail(UFPGD_ENOTSUP, "power iteration supports M <= 1024");
  if (steps < 1) return fail(UFPGD_EINVAL_PARAM, "steps must be >= 1");
  if (B > 0 && (!H || !Lout)) return fail(UFPGD_EINVAL_PARAM, "H and Lout are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  PowerArgs a{};
  a.H = reinterpret_cast<const float2*>(H);
  a.Lout = Lout;
  a.B = B;
  a.K = K;
  a.M = M;
  a.steps = steps;
  if (v0) {
    std::memcpy(a.v0, v0, sizeof(float2) * M);
  } else {
    std::vector<ufpgd_c64> tmp(M);
    ufpgd_power_v0(M, tmp.data());
    std::memcpy(a.v0, tmp.data(), sizeof(float2) * M);
  }
  cudaError_t e = launch_power(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "power kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_lipschitz_exact(const double* H, int64_t B, int K, int M, double* Lout, int32_t* status,
                              int device, ufpgd_stream_t stream) {
  if (B < 0 || K < 1 || M < 1) return fail(UFPGD_EINVAL_SHAPE, "lipschitz_bound: empty channel");
  if (B > 0 && (!H || !Lout)) return fail(UFPGD_EINVAL_PARAM, "H and Lout are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Start vector Rng(0x1F2E3D4C5B6A7988), normalised, in FP64 (pgd.cpp:131-134).
  std::vector<double> v0(2 * static_cast<size_t>(M));
  ufpgd_power_v0_f64(M, v0.data());
  double2* dv0 = nullptr;
  UFPGD_CUDA(cudaMallocAsync(&dv0, sizeof(double2) * M, s));
  UFPGD_CUDA(cudaMemcpyAsync(dv0, v0.data(), sizeof(double2) * M, cudaMemcpyHostToDevice, s));
  cudaError_t e = launch_lipschitz_exact(reinterpret_cast<const double2*>(H), B, K, M, dv0, Lout, status, s);
  cudaFreeAsync(dv0, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // v0 host buffer lifetime
  if (e != cudaSuccess) return cuda_fail(e, "lipschitz_exact kernel");
  return UFPGD_OK;
}

}  // extern "C"

namespace {

// Enqueues a fixed-iteration PGD solve on `s` (device buffers): the fused
// kernel (power-iteration prologue), a zero-padded fused shape, or the power
// kernel + general kernel. Used by the device and host entry points.
int enqueue_pgd(const float2* H, int64_t B, int K, int M, const float* eta_in, int power_steps, double lambda,
                int64_t iters, const double* c, int w0_mode, const float2* W0, float2* W, int32_t* diverged_at,
                float* l21, int32_t* active, float* eta_out, double* partials, double alpha, int device,
                cudaStream_t s, long long* nparts, double residual_tol = 0.0, int64_t* iterations = nullptr) {
  // residual_tol > 0 (solve_pgd's early stop): the FFMA2 team kernels (K <= 8)
  // or the general kernel; the tensor-core and tile kernels run fixed counts
  const bool resid = residual_tol > 0.0;
  const bool fused = fused_supported(K, M) && iters >= 1 && (!resid || K <= 8);
  int rc = UFPGD_OK, Kp = 0, Mp = 0;
  long long used = B;
  std::vector<ufpgd_c64> v0(M);
  ufpgd_power_v0(M, v0.data());
  if (fused) {
    FusedArgs a{};
    a.H = H;
    a.W = W;
    a.W0 = W0;
    a.eta_in = eta_in;
    a.eta_out = eta_out;
    a.diverged_at = diverged_at;
    a.l21 = l21;
    a.active = active;
    a.block_partials = partials;
    a.B = B;
    a.L = iters;
    a.w0_mode = w0_mode;
    a.power_steps = power_steps;
    a.lambda = static_cast<float>(lambda);
    a.alpha = static_cast<float>(alpha);
    a.residual_tol = static_cast<float>(residual_tol);
    a.iterations = iterations;
    for (int k = 0; k < K; ++k) a.c[k] = static_cast<float>(c[k]);
    std::memcpy(a.v0, v0.data(), sizeof(float2) * M);
    cudaError_t e = launch_fused(a, true, K, M, s, &used);
    if (e != cudaSuccess) rc = cuda_fail(e, "fused PGD kernel");
    if (e == cudaSuccess && !resid && iterations) {  // fixed count: every realization ran `iters`
      e = launch_fill_i64(iterations, B, iters, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "iterations fill");
    }
  } else if (!resid && iters >= 1 && padded_shape(K, M, &Kp, &Mp)) {
    // zero-padded on a fused shape; the power-iteration start vector is padded
    // with zeros too, so the padded antennas stay 0 in every step
    rc = run_padded(H, w0_mode == UFPGD_W0_GIVEN ? W0 : nullptr, W, B, K, M, Kp, Mp, partials, s, &used,
                    [&](const float2* hp, const float2* w0p, float2* wp, int64_t b0, int64_t nb, double* parts,
                        long long* np) -> int {
                      FusedArgs a{};
                      a.H = hp;
                      a.W = wp;
                      a.W0 = w0p;
                      a.eta_in = eta_in ? eta_in + b0 : nullptr;
                      a.eta_out = eta_out ? eta_out + b0 : nullptr;
                      a.diverged_at = diverged_at ? diverged_at + b0 : nullptr;
                      a.l21 = l21 ? l21 + b0 : nullptr;
                      a.active = active ? active + b0 : nullptr;
                      a.block_partials = parts;
                      a.B = nb;
                      a.L = iters;
                      a.w0_mode = w0_mode;
                      a.power_steps = power_steps;
                      a.lambda = static_cast<float>(lambda);
                      a.alpha = static_cast<float>(alpha);
                      for (int k = 0; k < K; ++k) a.c[k] = static_cast<float>(c[k]);
                      std::memcpy(a.v0, v0.data(), sizeof(float2) * M);  // a.v0[M..Mp) stay 0
                      cudaError_t e = launch_fused(a, true, Kp, Mp, s, np);
                      return e == cudaSuccess ? UFPGD_OK : cuda_fail(e, "zero-padded fused PGD kernel");
                    });
    if (rc == UFPGD_OK && iterations) {
      cudaError_t e = launch_fill_i64(iterations, B, iters, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "iterations fill");
    }
  } else {
    if (!general_fits(K, M)) rc = fail(UFPGD_ENOTSUP, "(K, M) too large for the general kernel");
    float* lip = nullptr;
    if (rc == UFPGD_OK && !eta_in) {
      cudaError_t e = cudaMallocAsync(&lip, sizeof(float) * B, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "alloc");
      if (rc == UFPGD_OK) rc = ufpgd_gpu_power_iteration(reinterpret_cast<const ufpgd_c64*>(H), B, K, M, v0.data(), power_steps, lip, device, s);
    }
    if (rc == UFPGD_OK) {
      GeneralArgs gA{};
      gA.H = H;
      gA.W = W;
      gA.W0 = W0;
      gA.diverged_at = diverged_at;
      gA.l21 = l21;
      gA.active = active;
      gA.block_partials = partials;
      gA.B = B;
      gA.K = K;
      gA.M = M;
      gA.w0_mode = w0_mode;
      gA.pgd = 1;
      gA.iters = iters;
      gA.eta_b = eta_in;
      gA.lip_b = lip;
      gA.eta_out = eta_out;
      gA.lambda = static_cast<float>(lambda);
      gA.index_base = 1;
      gA.alpha = static_cast<float>(alpha);
      gA.residual_tol = static_cast<float>(residual_tol);
      gA.iterations = iterations;
      for (int k = 0; k < K; ++k) gA.c[k] = static_cast<float>(c[k]);
      cudaError_t e = launch_general(gA, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "general PGD kernel");
    }
    if (lip) cudaFreeAsync(lip, s);
  }
  *nparts = used;
  return rc;
}

}  // namespace

extern "C" {

int ufpgd_gpu_solve_pgd_batch(const ufpgd_c64* H, int64_t B, int K, int M, const float* eta_in, int power_steps,
                              double lambda, int64_t max_iters, double residual_tol, const double* c, int w0_mode,
                              const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at, int64_t* iterations,
                              float* l21, int32_t* active, float* eta_out, double* stats, double alpha, int device,
                              ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K)) || (rc = check_w0(w0_mode, W0))) return rc;
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(UFPGD_EINVAL_PARAM, "PgdParams: lambda must be >= 0");
  if (max_iters < 0) return fail(UFPGD_EINVAL_PARAM, "PgdParams: max_iters must be >= 0");
  if (!(residual_tol >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "PgdParams: residual_tol must be >= 0");
  if (!eta_in && power_steps < 1) return fail(UFPGD_EINVAL_PARAM, "need eta_in or power_steps >= 1");
  if (!(alpha > 0.0)) return fail(UFPGD_EINVAL_PARAM, "alpha must be > 0");
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    if (stats) UFPGD_CUDA(cudaMemsetAsync(stats, 0, 3 * sizeof(double), s));
    return UFPGD_OK;
  }
  const bool fused = fused_supported(K, M) && max_iters >= 1;
  const long long np = partial_count(B, K, M, fused);
  long long used = B;
  double* partials = nullptr;
  if (stats) UFPGD_CUDA(scratch_alloc_async(reinterpret_cast<void**>(&partials), sizeof(double) * 3 * np, s));
  rc = enqueue_pgd(reinterpret_cast<const float2*>(H), B, K, M, eta_in, power_steps, lambda, max_iters, c, w0_mode,
                   reinterpret_cast<const float2*>(W0), reinterpret_cast<float2*>(W), diverged_at, l21, active,
                   eta_out, partials, alpha, device, s, &used, residual_tol, iterations);
  int rc2 = finish_stats(partials, rc == UFPGD_OK ? used : 0, stats, s);
  return rc != UFPGD_OK ? rc : rc2;
}

int ufpgd_gpu_pgd_fixed(const ufpgd_c64* H, int64_t B, int K, int M, const float* eta_in,
                        int power_steps, double lambda, int64_t iters, const double* c, int w0_mode,
                        const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at, float* l21,
                        int32_t* active, float* eta_out, double* stats, double alpha, int device,
                        ufpgd_stream_t stream) {
  return ufpgd_gpu_solve_pgd_batch(H, B, K, M, eta_in, power_steps, lambda, iters, 0.0, c, w0_mode, W0, W,
                                   diverged_at, nullptr, l21, active, eta_out, stats, alpha, device, stream);
}

int ufpgd_gpu_layers_general(const ufpgd_c64* H, int64_t B, int K, int M, const double* eta,
                             const double* thr, int L, const double* c, int w0_mode,
                             const ufpgd_c64* W0, int mode, double residual_tol, int index_base,
                             ufpgd_c64* W, int32_t* diverged_at, int64_t* iterations,
                             ufpgd_c64* iterates, ufpgd_c64* tape_v, float* tape_norms,
                             float* tape_shrink, int device, ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K)) || (rc = check_w0(w0_mode, W0))) return rc;
  if (mode != 0 && mode != 1) return fail(UFPGD_EINVAL_PARAM, "bad mode");
  if (L < 0 || L > UFPGD_MAX_LAYERS) return fail(UFPGD_EINVAL_PARAM, "layer count out of range");
  if (mode == 1) L = 1;
  if (L > 0 && (!eta || !thr)) return fail(UFPGD_EINVAL_PARAM, "eta/thr required");
  for (int l = 0; l < L; ++l)
    if (!(eta[l] >= 0.0) || !(thr[l] >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "need eta >= 0, thr >= 0");
  if (!(residual_tol >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "residual_tol must be >= 0");
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  const bool taped = iterates || tape_v || tape_norms || tape_shrink;
  if (mode == 0 && residual_tol == 0.0 && index_base == 0 && L >= 1 &&
      (taped ? fused_taped_supported(K, M) : fused_supported(K, M))) {
    // the layer sweep on the fused kernels: same raw (eta, thr) per layer,
    // layer-indexed divergence, iterations = L. With tapes: the team kernel's
    // taped instance (K <= 8); without: the unfolded forward's own kernel
    // for the shape (tcgen05 / tiled / team, as ufpgd_gpu_unfolded_forward).
    FusedArgs f{};
    f.H = reinterpret_cast<const float2*>(H);
    f.W = reinterpret_cast<float2*>(W);
    f.W0 = reinterpret_cast<const float2*>(W0);
    f.diverged_at = diverged_at;
    f.iterations = iterations;
    f.iterates = reinterpret_cast<float2*>(iterates);
    f.tape_v = reinterpret_cast<float2*>(tape_v);
    f.tape_norms = tape_norms;
    f.tape_shrink = tape_shrink;
    f.B = B;
    f.L = L;
    f.w0_mode = w0_mode;
    f.alpha = 1.f;
    for (int k = 0; k < K; ++k) f.c[k] = static_cast<float>(c[k]);
    for (int l = 0; l < L; ++l) {
      f.eta[l] = static_cast<float>(eta[l]);
      f.thr[l] = static_cast<float>(thr[l]);
    }
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    long long nb = 0;
    cudaError_t e = taped ? launch_fused_taped(f, K, M, s) : launch_fused(f, false, K, M, s, &nb);
    if (e == cudaSuccess && !taped && iterations) e = launch_fill_i64(iterations, B, L, s);
    if (e != cudaSuccess) return cuda_fail(e, "fused layer sweep");
    return UFPGD_OK;
  }
  if (!general_fits(K, M)) return fail(UFPGD_ENOTSUP, "(K, M) too large for the general kernel");
  GeneralArgs a{};
  a.H = reinterpret_cast<const float2*>(H);
  a.W = reinterpret_cast<float2*>(W);
  a.W0 = reinterpret_cast<const float2*>(W0);
  a.diverged_at = diverged_at;
  a.iterations = iterations;
  a.iterates = reinterpret_cast<float2*>(iterates);
  a.tape_v = reinterpret_cast<float2*>(tape_v);
  a.tape_norms = tape_norms;
  a.tape_shrink = tape_shrink;
  a.B = B;
  a.K = K;
  a.M = M;
  a.L = L;
  a.w0_mode = w0_mode;
  a.mode = mode;
  a.index_base = index_base;
  a.residual_tol = static_cast<float>(residual_tol);
  a.alpha = 1.f;
  for (int k = 0; k < K; ++k) a.c[k] = static_cast<float>(c[k]);
  for (int l = 0; l < L; ++l) {
    a.eta[l] = static_cast<float>(eta[l]);
    a.thr[l] = static_cast<float>(thr[l]);
  }
  cudaError_t e = launch_general(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "general kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_layers_general64(const double* H, int64_t B, int K, int M, const double* eta, const double* thr, int L,
                               const double* c, int w0_mode, const double* W0, int mode, double residual_tol,
                               int index_base, double* W, int32_t* diverged_at, int64_t* iterations,
                               double* iterates, double* tape_v, double* tape_norms, double* tape_shrink, int device,
                               ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K)) || (rc = check_w0(w0_mode, W0))) return rc;
  if (mode != 0 && mode != 1) return fail(UFPGD_EINVAL_PARAM, "bad mode");
  if (L < 0 || L > UFPGD_MAX_LAYERS) return fail(UFPGD_EINVAL_PARAM, "layer count out of range");
  if (mode == 1) L = 1;
  if (L > 0 && (!eta || !thr)) return fail(UFPGD_EINVAL_PARAM, "eta/thr required");
  for (int l = 0; l < L; ++l)
    if (!(eta[l] >= 0.0) || !(thr[l] >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "need eta >= 0, thr >= 0");
  if (!(residual_tol >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "residual_tol must be >= 0");
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (general64_smem_bytes(K, M) > static_cast<size_t>(optin)) return fail(UFPGD_ENOTSUP, "(K, M) too large for FP64");
  GeneralArgs64 a{};
  a.H = reinterpret_cast<const double2*>(H);
  a.W = reinterpret_cast<double2*>(W);
  a.W0 = reinterpret_cast<const double2*>(W0);
  a.diverged_at = diverged_at;
  a.iterations = iterations;
  a.iterates = reinterpret_cast<double2*>(iterates);
  a.tape_v = reinterpret_cast<double2*>(tape_v);
  a.tape_norms = tape_norms;
  a.tape_shrink = tape_shrink;
  a.B = B;
  a.K = K;
  a.M = M;
  a.L = L;
  a.w0_mode = w0_mode;
  a.mode = mode;
  a.index_base = index_base;
  a.residual_tol = residual_tol;
  a.alpha = 1.0;
  for (int k = 0; k < K; ++k) a.c[k] = c[k];
  for (int l = 0; l < L; ++l) {
    a.eta[l] = eta[l];
    a.thr[l] = thr[l];
  }
  cudaError_t e = launch_general64(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "general FP64 kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_solve_pgd64(const double* H, int64_t B, int K, int M, const double* c, double lambda,
                          const double* eta, int64_t max_iters, double residual_tol, const double* W0, double* W,
                          int64_t* iterations, int32_t* diverged_at, int device, ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K))) return rc;
  if (!(lambda >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "PgdParams: lambda must be >= 0");
  if (max_iters < 0 || !(residual_tol >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "bad PGD parameters");
  if (B > 0 && (!H || !W || !eta)) return fail(UFPGD_EINVAL_PARAM, "H, eta and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (general64_smem_bytes(K, M) > static_cast<size_t>(optin)) return fail(UFPGD_ENOTSUP, "(K, M) too large for FP64");
  GeneralArgs64 a{};
  a.H = reinterpret_cast<const double2*>(H);
  a.W = reinterpret_cast<double2*>(W);
  a.W0 = reinterpret_cast<const double2*>(W0);
  a.diverged_at = diverged_at;
  a.iterations = iterations;
  a.B = B;
  a.K = K;
  a.M = M;
  a.w0_mode = W0 ? UFPGD_W0_GIVEN : UFPGD_W0_CONJ_H;
  a.pgd = 1;
  a.iters = max_iters;
  a.eta_b = eta;
  a.lambda = lambda;
  a.index_base = 1;
  a.residual_tol = residual_tol;
  a.alpha = 1.0;
  for (int k = 0; k < K; ++k) a.c[k] = c[k];
  cudaError_t e = launch_general64(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "solve_pgd FP64 kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_oracle_solve(const double* H, int64_t B, int K, int M, const double* c, double lambda,
                           int64_t max_iters, double residual_tol, double* W, double* eta_out, int64_t* iterations,
                           int32_t* status, int device, ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K))) return rc;
  if (!(lambda >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "PgdParams: lambda must be >= 0");
  if (max_iters < 0 || !(residual_tol >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "bad PGD parameters");
  if (B > 0 && (!H || !W || !status)) return fail(UFPGD_EINVAL_PARAM, "H, W and status are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (general64_smem_bytes(K, M) > static_cast<size_t>(optin)) return fail(UFPGD_ENOTSUP, "(K, M) too large for FP64");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* lip = nullptr;
  int32_t* div = nullptr;
  UFPGD_CUDA(cudaMallocAsync(&lip, sizeof(double) * B, s));
  UFPGD_CUDA(cudaMallocAsync(&div, sizeof(int32_t) * B, s));
  // pgd.cpp:270-279: eta = 1 / lipschitz_bound(H).exact (converged, FP64)
  rc = ufpgd_gpu_lipschitz_exact(H, B, K, M, lip, status, device, stream);
  if (rc == UFPGD_OK) {
    GeneralArgs64 a{};
    a.H = reinterpret_cast<const double2*>(H);
    a.W = reinterpret_cast<double2*>(W);
    a.diverged_at = div;
    a.iterations = iterations;
    a.B = B;
    a.K = K;
    a.M = M;
    a.w0_mode = UFPGD_W0_CONJ_H;
    a.pgd = 1;
    a.iters = max_iters;
    a.lip_b = lip;
    a.eta_out = eta_out;
    a.lambda = lambda;
    a.index_base = 1;
    a.residual_tol = residual_tol;
    a.alpha = 1.0;
    for (int k = 0; k < K; ++k) a.c[k] = c[k];
    cudaError_t e = launch_general64(a, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "oracle_solve kernel");
  }
  if (rc == UFPGD_OK) {
    // fold divergence into status (ECONVERGENCE from the power iteration wins)
    std::vector<int32_t> hs(static_cast<size_t>(B)), hd(static_cast<size_t>(B));
    cudaMemcpyAsync(hs.data(), status, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hd.data(), div, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "oracle_solve");
    for (int64_t b = 0; b < B && rc == UFPGD_OK; ++b)
      if (hs[b] == 0 && hd[b] >= 0) hs[b] = UFPGD_EDIVERGED;
    if (rc == UFPGD_OK) cudaMemcpy(status, hs.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice);
  }
  cudaFreeAsync(lip, s);
  cudaFreeAsync(div, s);
  cudaStreamSynchronize(s);
  return rc;
}

namespace {
int unfolded_host(const ufpgd_c64* H, int64_t B, int K, int M, const double* lambda, const double* eta, int L,
                  const double* c, int w0_mode, const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at,
                  double* stats, double alpha, int device, int64_t* ticket) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_layers(lambda, eta, L)) || (rc = check_c(c, K)) ||
      (rc = check_w0(w0_mode, W0)))
    return rc;
  if (!(alpha > 0.0)) return fail(UFPGD_EINVAL_PARAM, "alpha must be > 0");
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  const bool fused = fused_supported(K, M) && L >= 1;
  // 16 MiB of H per chunk: short pipeline fill, chunks still fill the GPU.
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, host_chunk_bytes() / (8ll * K * M)));
  const long long ppc = partial_count(chunk, K, M, fused);
  auto run = [&](float2* h, int64_t nb, float2* w0, float2* w, int32_t* div, float*, double* parts, long long* np,
                 cudaStream_t s) {
    return enqueue_unfolded(h, nb, K, M, lambda, eta, L, c, w0_mode, w0, w, div, nullptr, nullptr, parts, alpha, s,
                            np);
  };
  const ufpgd_c64* w0 = w0_mode == UFPGD_W0_GIVEN ? W0 : nullptr;
  if (ticket)
    return host_enqueue(device, H, B, K, M, w0, W, diverged_at, nullptr, ppc, chunk, stats, run, ticket, false);
  return host_pipeline(device, H, B, K, M, w0, W, diverged_at, nullptr, ppc, chunk, stats, run);
}
}  // namespace

int ufpgd_gpu_unfolded_forward_host(const ufpgd_c64* H, int64_t B, int K, int M,
                                    const double* lambda, const double* eta, int L, const double* c,
                                    int w0_mode, const ufpgd_c64* W0, ufpgd_c64* W,
                                    int32_t* diverged_at, double* stats, double alpha, int device) {
  return unfolded_host(H, B, K, M, lambda, eta, L, c, w0_mode, W0, W, diverged_at, stats, alpha, device, nullptr);
}

int ufpgd_gpu_unfolded_forward_host_async(const ufpgd_c64* H, int64_t B, int K, int M, const double* lambda,
                                          const double* eta, int L, const double* c, int w0_mode,
                                          const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at, double* stats,
                                          double alpha, int device, int64_t* ticket) {
  if (!ticket) return fail(UFPGD_EINVAL_PARAM, "ticket is required");
  *ticket = -1;
  return unfolded_host(H, B, K, M, lambda, eta, L, c, w0_mode, W0, W, diverged_at, stats, alpha, device, ticket);
}

int ufpgd_gpu_host_wait(int64_t ticket) { return host_finish(ticket); }

int ufpgd_gpu_pgd_fixed_host(const ufpgd_c64* H, int64_t B, int K, int M, int power_steps,
                             double lambda, int64_t iters, const double* c, int w0_mode,
                             const ufpgd_c64* W0, ufpgd_c64* W, int32_t* diverged_at,
                             float* eta_out, double* stats, double alpha, int device) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K)) || (rc = check_w0(w0_mode, W0))) return rc;
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(UFPGD_EINVAL_PARAM, "PgdParams: lambda must be >= 0");
  if (iters < 0) return fail(UFPGD_EINVAL_PARAM, "PgdParams: max_iters must be >= 0");
  if (power_steps < 1) return fail(UFPGD_EINVAL_PARAM, "power_steps must be >= 1");
  if (!(alpha > 0.0)) return fail(UFPGD_EINVAL_PARAM, "alpha must be > 0");
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  const bool fused = fused_supported(K, M) && iters >= 1;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, (8ll << 20) / (8ll * K * M)));
  const long long ppc = partial_count(chunk, K, M, fused);
  // The device entry point finalises its own stats per chunk; here the
  // pipeline collects block partials, so call the kernels with partials only.
  return host_pipeline(
      device, H, B, K, M, w0_mode == UFPGD_W0_GIVEN ? W0 : nullptr, W, diverged_at, eta_out, ppc, chunk,
      stats,
      [&](float2* h, int64_t nb, float2* w0, float2* w, int32_t* div, float* eo, double* parts,
          long long* np, cudaStream_t s) -> int {
        return enqueue_pgd(h, nb, K, M, nullptr, power_steps, lambda, iters, c, w0_mode, w0, w, div, nullptr,
                           nullptr, eo, parts, alpha, device, s, np);
      });
}

int ufpgd_gpu_metrics(const ufpgd_c64* H, const ufpgd_c64* W, int64_t B, int K, int M, const double* c,
                      double sigma_nu, double alpha, double* out, ufpgd_c64* Wzf, int device,
                      ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_c(c, K))) return rc;
  if (K > 32) return fail(UFPGD_ENOTSUP, "metrics support K <= 32");
  if (!(sigma_nu >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "SystemConfig: sigma_nu must be >= 0");
  if (!(alpha > 0.0)) return fail(UFPGD_EINVAL_PARAM, "alpha must be > 0");
  if (B > 0 && (!H || !W || !out)) return fail(UFPGD_EINVAL_PARAM, "H, W and out are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (metrics_smem_bytes(K, M) > static_cast<size_t>(optin)) return fail(UFPGD_ENOTSUP, "(K, M) too large for metrics");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* dc = nullptr;
  UFPGD_CUDA(cudaMallocAsync(&dc, sizeof(double) * K, s));
  UFPGD_CUDA(cudaMemcpyAsync(dc, c, sizeof(double) * K, cudaMemcpyHostToDevice, s));
  cudaError_t e = launch_metrics(reinterpret_cast<const float2*>(H), reinterpret_cast<const float2*>(W), B, K, M,
                                 dc, sigma_nu * sigma_nu, alpha, out, reinterpret_cast<float2*>(Wzf), s);
  cudaFreeAsync(dc, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // c is a host buffer of the caller
  if (e != cudaSuccess) return cuda_fail(e, "metrics kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_unfolded_grad(const ufpgd_c64* H, int64_t B, int K, int M, const double* lambda, const double* eta,
                            int L, const double* c, int w0_mode, int loss_kind, double lambda_cost,
                            const ufpgd_c64* labels, double* loss, double* grads, double* mean, int device,
                            ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_layers(lambda, eta, L)) || (rc = check_c(c, K))) return rc;
  if (L < 1) return fail(UFPGD_EINVAL_PARAM, "need at least one layer");
  if (w0_mode != UFPGD_W0_ZERO && w0_mode != UFPGD_W0_CONJ_H) return fail(UFPGD_EINVAL_PARAM, "W0 = 0 or H^* only");
  if (loss_kind != 0 && loss_kind != 1) return fail(UFPGD_EINVAL_PARAM, "bad loss kind");
  if (loss_kind == 1 && !labels) return fail(UFPGD_EINVAL_PARAM, "supervised mode requires labels");
  if (!(lambda_cost >= 0.0)) return fail(UFPGD_EINVAL_PARAM, "TrainConfig: lambda_cost must be >= 0");
  if (B > 0 && (!H || !loss || !grads)) return fail(UFPGD_EINVAL_PARAM, "H, loss and grads are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  if (!general_fits(K, M)) return fail(UFPGD_ENOTSUP, "(K, M) too large for the gradient kernel");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GradArgs a{};
  a.H = reinterpret_cast<const float2*>(H);
  a.labels = reinterpret_cast<const float2*>(labels);
  a.out_loss = loss;
  a.out_grads = grads;
  a.B = B;
  a.K = K;
  a.M = M;
  a.L = L;
  a.w0_mode = w0_mode;
  a.loss_kind = loss_kind;
  a.lambda_cost = static_cast<float>(lambda_cost);
  for (int k = 0; k < K; ++k) a.c[k] = static_cast<float>(c[k]);
  for (int l = 0; l < L; ++l) {
    a.eta[l] = static_cast<float>(eta[l]);
    a.thr[l] = static_cast<float>(lambda[l] * eta[l]);
    a.lam[l] = lambda[l];
    a.eta64[l] = eta[l];
  }
  UFPGD_CUDA(cudaMallocAsync(&a.tape, sizeof(float2) * 2ull * L * K * M * B, s));
  cudaError_t e = launch_grad(a, mean, s);
  cudaFreeAsync(a.tape, s);
  if (e != cudaSuccess) return cuda_fail(e, "gradient kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_generate_channels(uint64_t seed_h, uint64_t seed_g, double gain_range_db, int64_t first_index,
                                int64_t B, int K, int M, void* H, int out_f64, int device, ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M))) return rc;
  if (!(gain_range_db >= 0.0) || !std::isfinite(gain_range_db))
    return fail(UFPGD_EINVAL_PARAM, "gain_range_db must be finite and >= 0");
  if (first_index < 0) return fail(UFPGD_EINVAL_PARAM, "first_index must be >= 0");
  if (B > 0 && !H) return fail(UFPGD_EINVAL_PARAM, "H is required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  const cudaError_t e = launch_channel_gen(seed_h, seed_g, gain_range_db, first_index, B, K, M, H, out_f64 != 0,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "channel generation kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_unfolded_backward64(const double* H, int64_t B, int K, int M, const double* lambda,
                                  const double* eta, int L, const double* c, int w0_mode, const double* W0,
                                  const double* dcost_dw, double* grads, int device, ufpgd_stream_t stream) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_layers(lambda, eta, L)) || (rc = check_c(c, K)) ||
      (rc = check_w0(w0_mode, W0)))
    return rc;
  if (L < 1) return fail(UFPGD_EINVAL_PARAM, "need at least one layer");
  if (B > 0 && (!H || !dcost_dw || !grads)) return fail(UFPGD_EINVAL_PARAM, "H, dcost_dw and grads are required");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  if (B == 0) return UFPGD_OK;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (grad64_smem_bytes(K, M) + 1024 > static_cast<size_t>(optin))
    return fail(UFPGD_ENOTSUP, "(K, M) too large for the FP64 gradient kernel");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GradArgs64 a{};
  a.H = reinterpret_cast<const double2*>(H);
  a.W0 = reinterpret_cast<const double2*>(W0);
  a.dcost = reinterpret_cast<const double2*>(dcost_dw);
  a.out_grads = grads;
  a.B = B;
  a.K = K;
  a.M = M;
  a.L = L;
  a.w0_mode = w0_mode;
  a.loss_kind = 2;
  for (int k = 0; k < K; ++k) a.c[k] = c[k];
  for (int l = 0; l < L; ++l) {
    a.eta[l] = eta[l];
    a.thr[l] = lambda[l] * eta[l];
    a.lam[l] = lambda[l];
    a.eta64[l] = eta[l];
  }
  UFPGD_CUDA(cudaMallocAsync(&a.tape, sizeof(double2) * 2ull * L * K * M * B, s));
  UFPGD_CUDA(cudaMallocAsync(&a.out_loss, sizeof(double) * B, s));
  cudaError_t e = launch_grad64(a, nullptr, s);
  cudaFreeAsync(a.tape, s);
  cudaFreeAsync(a.out_loss, s);
  if (e != cudaSuccess) return cuda_fail(e, "FP64 backward kernel");
  return UFPGD_OK;
}

int ufpgd_gpu_fp32_peak(int device, double* tflops, double* sm_ghz) {
  if (!tflops || !sm_ghz) return fail(UFPGD_EINVAL_PARAM, "null output");
  DeviceGuard g(device);
  if (!g.ok) return fail(UFPGD_ECUDA, "cannot select device");
  cudaError_t e = measure_fp32_peak(tflops, sm_ghz);
  if (e != cudaSuccess) return cuda_fail(e, "fp32 peak probe");
  return UFPGD_OK;
}

int ufpgd_gpu_init(int ngpus) {
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  int count = 0;
  UFPGD_CUDA(cudaGetDeviceCount(&count));
  if (ngpus < 1 || ngpus > count) return fail(UFPGD_EINVAL_PARAM, "ngpus out of range");
  if (!g_comms.empty()) return UFPGD_OK;
  if (!load_nccl()) return fail(UFPGD_ENCCL, "libnccl.so.2 not loadable");
  std::vector<int> devs(ngpus);
  for (int i = 0; i < ngpus; ++i) devs[i] = i;
  g_comms.assign(ngpus, nullptr);
  ncclResult_t r = g_nccl.CommInitAll(g_comms.data(), ngpus, devs.data());
  if (r != 0) {
    g_comms.clear();
    return fail(UFPGD_ENCCL, std::string("ncclCommInitAll: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
  }
  return UFPGD_OK;
}

int ufpgd_gpu_shutdown(void) {
  {
    std::lock_guard<std::mutex> lock(g_nccl_mu);
    for (ncclComm_t c : g_comms)
      if (c) g_nccl.CommDestroy(c);
    g_comms.clear();
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
  for (int d = 0; d < count && d < 64; ++d) {
    if (!g_ws[d].init && !g_pool[d]) continue;
    DeviceGuard g(d);
    release_workspace(g_ws[d]);
    release_pool(d);
  }
  return UFPGD_OK;
}

int ufpgd_gpu_unfolded_forward_sharded(const ufpgd_c64* H, int64_t B, int K, int M,
                                       const double* lambda, const double* eta, int L,
                                       const double* c, int w0_mode, const ufpgd_c64* W0, ufpgd_c64* W,
                                       int32_t* diverged_at, double* stats, double alpha) {
  int rc;
  if ((rc = check_shape(B, K, M)) || (rc = check_layers(lambda, eta, L)) || (rc = check_c(c, K)) ||
      (rc = check_w0(w0_mode, W0)))
    return rc;
  if (B > 0 && (!H || !W)) return fail(UFPGD_EINVAL_PARAM, "H and W are required");
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  const int G = static_cast<int>(g_comms.size());
  if (G == 0) return fail(UFPGD_ENCCL, "call ufpgd_gpu_init first");
  ShardSet set(G);
  if (!set.ok) return fail(UFPGD_ECUDA, "cannot create per-device streams / statistics buffers");
  // Contiguous shards [g*B/G, (g+1)*B/G), each through its device's pipelined
  // host path on its own host thread (the H2D / D2H copies of all devices run
  // concurrently); the shard statistics land in device memory for the
  // all-reduce.
  std::vector<int> rcs(G, UFPGD_OK);
  std::vector<std::string> errs(G);
  std::vector<std::thread> th;
  for (int gi = 0; gi < G; ++gi) {
    th.emplace_back([&, gi] {
      const int64_t b0 = B * gi / G, b1 = B * (gi + 1) / G, nb = b1 - b0;
      DeviceGuard dg(gi);
      double part[3] = {0, 0, 0};
      const size_t off = static_cast<size_t>(b0) * K * M;
      int r = ufpgd_gpu_unfolded_forward_host(H + off, nb, K, M, lambda, eta, L, c, w0_mode,
                                              W0 ? W0 + off : nullptr, W + off,
                                              diverged_at ? diverged_at + b0 : nullptr, part, alpha, gi);
      if (r != UFPGD_OK && r != UFPGD_EDIVERGED) errs[gi] = g_last_error;
      rcs[gi] = r;
      if (cudaMemcpyAsync(set.dstats[gi], part, sizeof(part), cudaMemcpyHostToDevice, set.streams[gi]) !=
              cudaSuccess ||
          cudaStreamSynchronize(set.streams[gi]) != cudaSuccess) {
        if (rcs[gi] == UFPGD_OK || rcs[gi] == UFPGD_EDIVERGED) {
          rcs[gi] = UFPGD_ECUDA;
          errs[gi] = "statistics copy failed";
        }
      }
    });
  }
  for (auto& t : th) t.join();
  for (int gi = 0; gi < G; ++gi)
    if (rcs[gi] != UFPGD_OK && rcs[gi] != UFPGD_EDIVERGED) return fail(rcs[gi], errs[gi]);
  if ((rc = set.allreduce())) return rc;
  double out[3] = {0, 0, 0};
  if ((rc = set.sync_and_read(out))) return rc;
  if (stats) std::memcpy(stats, out, sizeof(out));
  if (out[2] > 0.0) return fail(UFPGD_EDIVERGED, "non-finite iterate in at least one realization");
  return UFPGD_OK;
}

int ufpgd_gpu_unfolded_forward_sharded_device(const ufpgd_c64* const* H, const int64_t* B, int K, int M,
                                              const double* lambda, const double* eta, int L, const double* c,
                                              int w0_mode, const ufpgd_c64* const* W0, ufpgd_c64* const* W,
                                              int32_t* const* diverged_at, double* const* stats, double alpha,
                                              const ufpgd_stream_t* streams) {
  int rc;
  if (!H || !B || !W || !stats) return fail(UFPGD_EINVAL_PARAM, "H, B, W and stats arrays are required");
  if ((rc = check_layers(lambda, eta, L)) || (rc = check_c(c, K))) return rc;
  if (w0_mode == UFPGD_W0_GIVEN && !W0) return fail(UFPGD_EINVAL_PARAM, "W0 required");
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  const int G = static_cast<int>(g_comms.size());
  if (G == 0) return fail(UFPGD_ENCCL, "call ufpgd_gpu_init first");
  for (int gi = 0; gi < G; ++gi) {
    if ((rc = check_shape(B[gi], K, M))) return rc;
    if (!stats[gi]) return fail(UFPGD_EINVAL_PARAM, "every device needs a stats buffer");
  }
  // Per device: the fused forward over its resident shard, its statistics
  // written to its own device buffer (no host round trip) ...
  for (int gi = 0; gi < G; ++gi) {
    const ufpgd_stream_t s = streams ? streams[gi] : nullptr;
    rc = ufpgd_gpu_unfolded_forward(H[gi], B[gi], K, M, lambda, eta, L, c, w0_mode, W0 ? W0[gi] : nullptr, W[gi],
                                    diverged_at ? diverged_at[gi] : nullptr, nullptr, nullptr, stats[gi], alpha, gi,
                                    s);
    if (rc != UFPGD_OK) return rc;
  }
  // ... then the only collective, in place on the device buffers, stream
  // ordered after each device's kernels. Asynchronous, like every device
  // entry point; divergence is reported in stats[g][2].
  std::vector<cudaStream_t> st(G);
  for (int gi = 0; gi < G; ++gi) st[gi] = static_cast<cudaStream_t>(streams ? streams[gi] : nullptr);
  return allreduce_stats(stats, st.data(), G);
}

}  // extern "C"
