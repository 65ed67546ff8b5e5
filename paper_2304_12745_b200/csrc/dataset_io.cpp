// UFPD dataset files: the reference's binary format
// (/root/reference/proj/core/include/ufpgd/dataset.hpp:23-36,
// dataset.cpp:38-175) read straight into device batches and written from
// them. The f64 row-major payload is streamed through pinned memory in chunks
// and transposed / rounded on the device (f64_rowmajor_to_c64_kernel), so a
// channel file feeds the solver without a host-side conversion pass.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "ufpgd_gpu.h"
#include "ufpgd_internal.h"

namespace {

constexpr std::uint32_t kMagic = 0x44504655;  // "UFPD" (dataset.hpp:34)
constexpr std::uint32_t kVersion = 1;
constexpr std::size_t kHeader = 36;

std::uint32_t get_u32(const unsigned char* p) {
  std::uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
std::uint64_t get_u64(const unsigned char* p) {
  std::uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
void put_u32(unsigned char* p, std::uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xFF);
}
void put_u64(unsigned char* p, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xFF);
}

struct Header {
  int K = 0, M = 0;
  std::uint64_t N = 0, seed = 0;
  bool labels = false;
};

thread_local std::string g_err;

int bad(const std::string& msg) {
  g_err = msg;
  return UFPGD_EDATAFORMAT;
}

// dataset.cpp:129-175 checks, plus the exact file size (which covers a
// truncated payload and trailing bytes before any payload is read).
int read_header(const char* path, Header& h) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return bad(std::string("cannot open dataset: ") + path);
  unsigned char hdr[kHeader];
  in.read(reinterpret_cast<char*>(hdr), kHeader);
  if (in.gcount() != static_cast<std::streamsize>(kHeader)) return bad(std::string("dataset header truncated: ") + path);
  if (get_u32(hdr) != kMagic) return bad(std::string("dataset magic mismatch: ") + path);
  if (get_u32(hdr + 4) != kVersion) return bad(std::string("dataset version unsupported: ") + path);
  h.K = static_cast<int>(get_u32(hdr + 8));
  h.M = static_cast<int>(get_u32(hdr + 12));
  h.N = get_u64(hdr + 16);
  h.seed = get_u64(hdr + 24);
  h.labels = (get_u32(hdr + 32) & 1u) != 0;
  if (h.K < 1 || h.M < h.K) return bad(std::string("dataset dimensions invalid: ") + path);
  const std::uintmax_t want =
      kHeader + static_cast<std::uintmax_t>(h.N) * 16ull * h.K * h.M * (h.labels ? 2ull : 1ull);
  std::error_code ec;
  const std::uintmax_t have = std::filesystem::file_size(path, ec);
  if (ec) return bad(std::string("cannot stat dataset: ") + path);
  if (have < want) return bad(std::string("dataset truncated: ") + path);
  if (have > want) return bad(std::string("dataset has trailing bytes: ") + path);
  return UFPGD_OK;
}

}  // namespace

extern "C" {

const char* ufpgd_dataset_last_error(void) { return g_err.c_str(); }

int ufpgd_ufpd_read_header(const char* path, int* K, int* M, int64_t* N, uint64_t* seed, int* has_labels) {
  if (!path) return bad("null path");
  Header h;
  const int rc = read_header(path, h);
  if (rc != UFPGD_OK) return rc;
  if (K) *K = h.K;
  if (M) *M = h.M;
  if (N) *N = static_cast<int64_t>(h.N);
  if (seed) *seed = h.seed;
  if (has_labels) *has_labels = h.labels ? 1 : 0;
  return UFPGD_OK;
}

int ufpgd_gpu_ufpd_load(const char* path, int64_t first, int64_t count, int which, ufpgd_c64* dst, int device) {
  Header h;
  int rc = read_header(path, h);
  if (rc != UFPGD_OK) return rc;
  if (which != 0 && which != 1) return bad("which must be 0 (channels) or 1 (labels)");
  if (which == 1 && !h.labels) return bad("dataset has no labels");
  if (first < 0 || count < 0 || static_cast<std::uint64_t>(first + count) > h.N) return bad("sample range out of bounds");
  if (count > 0 && !dst) return bad("null destination");
  if (cudaSetDevice(device) != cudaSuccess) return bad("cannot select device");
  const std::size_t per = 16ull * h.K * h.M;  // f64 bytes per matrix
  const std::uint64_t base = kHeader + (which == 1 ? h.N * per : 0) + static_cast<std::uint64_t>(first) * per;
  std::ifstream in(path, std::ios::binary);
  in.seekg(static_cast<std::streamoff>(base));
  const int64_t chunk = std::max<int64_t>(1, (32ll << 20) / static_cast<int64_t>(per));
  void* pinned = nullptr;
  void* draw = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t e = cudaHostAlloc(&pinned, per * std::min<int64_t>(chunk, std::max<int64_t>(count, 1)), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaMalloc(&draw, per * std::min<int64_t>(chunk, std::max<int64_t>(count, 1)));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  rc = UFPGD_OK;
  for (int64_t b0 = 0; b0 < count && e == cudaSuccess && rc == UFPGD_OK; b0 += chunk) {
    const int64_t nb = std::min(chunk, count - b0);
    in.read(static_cast<char*>(pinned), static_cast<std::streamsize>(per * nb));
    if (in.gcount() != static_cast<std::streamsize>(per * nb)) {
      rc = bad("dataset truncated while reading");
      break;
    }
    e = cudaMemcpyAsync(draw, pinned, per * nb, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = ufpgd_gpu_impl::launch_convert(draw, dst + b0 * h.K * h.M, nb, h.K, h.M, true, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // pinned staging is reused
  }
  if (s) cudaStreamDestroy(s);
  cudaFree(draw);
  cudaFreeHost(pinned);
  if (rc != UFPGD_OK) return rc;
  if (e != cudaSuccess) {
    g_err = std::string("ufpd load: ") + cudaGetErrorString(e);
    return UFPGD_ECUDA;
  }
  return UFPGD_OK;
}

// write_dataset (dataset.cpp:71-127) from device batches: atomic (temp file
// + rename), f64 payload produced on the device.
int ufpgd_gpu_ufpd_store(const char* path, int K, int M, int64_t N, uint64_t seed, const ufpgd_c64* channels,
                         const ufpgd_c64* labels, int device) {
  if (!path) return bad("null path");
  if (K < 1 || M < 1 || N < 0) {
    g_err = "write_dataset: bad dimensions";
    return UFPGD_EINVAL_SHAPE;
  }
  if (N > 0 && !channels) {
    g_err = "write_dataset: channels required";
    return UFPGD_EINVAL_PARAM;
  }
  if (cudaSetDevice(device) != cudaSuccess) return bad("cannot select device");
  const std::size_t per = 16ull * K * M;
  const std::string tmp = std::string(path) + ".tmp";
  std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
  if (!out) return bad("cannot open for writing: " + tmp);
  unsigned char hdr[kHeader];
  put_u32(hdr, kMagic);
  put_u32(hdr + 4, kVersion);
  put_u32(hdr + 8, static_cast<std::uint32_t>(K));
  put_u32(hdr + 12, static_cast<std::uint32_t>(M));
  put_u64(hdr + 16, static_cast<std::uint64_t>(N));
  put_u64(hdr + 24, seed);
  put_u32(hdr + 32, labels ? 1u : 0u);
  out.write(reinterpret_cast<const char*>(hdr), kHeader);
  const int64_t chunk = std::max<int64_t>(1, (32ll << 20) / static_cast<int64_t>(per));
  void* pinned = nullptr;
  void* draw = nullptr;
  cudaStream_t s = nullptr;
  const int64_t cap = std::min<int64_t>(chunk, std::max<int64_t>(N, 1));
  cudaError_t e = cudaHostAlloc(&pinned, per * cap, cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaMalloc(&draw, per * cap);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int part = 0; part < (labels ? 2 : 1) && e == cudaSuccess; ++part) {
    const ufpgd_c64* src = part == 0 ? channels : labels;
    for (int64_t b0 = 0; b0 < N && e == cudaSuccess; b0 += chunk) {
      const int64_t nb = std::min(chunk, N - b0);
      e = ufpgd_gpu_impl::launch_convert(src + b0 * K * M, draw, nb, K, M, false, s);
      if (e == cudaSuccess) e = cudaMemcpyAsync(pinned, draw, per * nb, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e == cudaSuccess) out.write(static_cast<const char*>(pinned), static_cast<std::streamsize>(per * nb));
    }
  }
  if (s) cudaStreamDestroy(s);
  cudaFree(draw);
  cudaFreeHost(pinned);
  out.flush();
  const bool ok = static_cast<bool>(out);
  out.close();
  if (e != cudaSuccess || !ok) {
    std::remove(tmp.c_str());
    g_err = e != cudaSuccess ? std::string("ufpd store: ") + cudaGetErrorString(e) : "write failed: " + tmp;
    return e != cudaSuccess ? UFPGD_ECUDA : UFPGD_EDATAFORMAT;
  }
  std::error_code ec;
  std::filesystem::rename(tmp, path, ec);
  if (ec) return bad("rename failed: " + tmp);
  return UFPGD_OK;
}

int ufpgd_gpu_convert_f64_rowmajor(const double* src, int64_t B, int K, int M, ufpgd_c64* dst, int to_c64,
                                   int device, ufpgd_stream_t stream) {
  if (B < 0 || K < 1 || M < 1) {
    g_err = "convert: bad shape";
    return UFPGD_EINVAL_SHAPE;
  }
  if (cudaSetDevice(device) != cudaSuccess) return bad("cannot select device");
  const cudaError_t e = to_c64 ? ufpgd_gpu_impl::launch_convert(src, dst, B, K, M, true, static_cast<cudaStream_t>(stream))
                               : ufpgd_gpu_impl::launch_convert(dst, const_cast<double*>(src), B, K, M, false,
                                                                static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    g_err = std::string("convert: ") + cudaGetErrorString(e);
    return UFPGD_ECUDA;
  }
  return UFPGD_OK;
}

}  // extern "C"
