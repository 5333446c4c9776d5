// pald_io.cu -- the input step before the hot path:
// the reference's binary distance-matrix format read straight into HBM and
// validated / symmetrized on the device, so an n = 32768 matrix never needs
// the reference's 8 GiB host `std::vector<double>`.
//
// Format (ingest.hpp:214-216): magic "PALD", version u8 = 1, element width
// u8 (4 or 8), u64 n, then n*n little-endian row-major elements.
// Semantics of read_distance_binary (ingest.hpp:280-283) = read_matrix_binary
// (:243-278) + validate_distances (:116-149), evaluated in double exactly as
// the reference does, then rounded to fp32 like to_real<float>
// (blocked.hpp:91-96):
//   pass 1, row-major: entries must be finite and >= 0; then the row's
//           diagonal must be 0;
//   pass 2, x < y:     |a - b| <= 1e-9 * max(|a|, |b|), else "asymmetry";
//                      avg = 0.5 * (a + b) must be > 0 (duplicate points);
//                      both entries become avg.
// The first violation in the reference's scan order is reported with the
// reference's message; status 2 (ValidationError) or 4 (IoError).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/pald_gpu.h"
#include "pald_internal.h"

namespace {

struct IoCheck {
  unsigned long long pass1;  // min key of a pass-1 violation (x*(n+1) + y, diag: x*(n+1) + n)
  unsigned long long pass2;  // min key of a pass-2 violation (2*(x*n + y) + kind)
  int pass1_kind;            // unused (derived on the host)
};

template <typename T>
__device__ __forceinline__ double val(const T* __restrict__ v, uint64_t ld, int r, int c) {
  return (double)v[(size_t)r * ld + c];
}

// Pass 1 and pass 2 checks of validate_distances; keys order violations as
// the reference's loops meet them.
template <typename T>
__global__ void check_kernel(const T* __restrict__ v, uint64_t ldv, int n, IoCheck* out) {
  unsigned long long k1 = ~0ull, k2 = ~0ull;
  for (int x = blockIdx.x; x < n; x += gridDim.x) {
    for (int y = threadIdx.x; y < n; y += blockDim.x) {
      const double d = val(v, ldv, x, y);
      if (!isfinite(d) || d < 0) k1 = min(k1, (unsigned long long)x * (n + 1) + y);
      if (y == x && d != 0.0) k1 = min(k1, (unsigned long long)x * (n + 1) + n);
      if (y > x) {
        const double a = d, b = val(v, ldv, y, x);
        const double scale = fmax(fabs(a), fabs(b));
        if (fabs(a - b) > 1e-9 * scale) {
          k2 = min(k2, 2ull * ((unsigned long long)x * n + y));
        } else {
          const double avg = 0.5 * (a + b);
          if (!(avg > 0)) k2 = min(k2, 2ull * ((unsigned long long)x * n + y) + 1);
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    k1 = min(k1, __shfl_xor_sync(0xffffffffu, k1, o));
    k2 = min(k2, __shfl_xor_sync(0xffffffffu, k2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out->pass1, k1);
    atomicMin(&out->pass2, k2);
  }
}

// Symmetrize (avg in double) and round to fp32 into dD (ld).
template <typename T>
__global__ void symmetrize_kernel(const T* __restrict__ v, uint64_t ldv, int n, float* __restrict__ d,
                                  uint64_t ldd) {
  for (int x = blockIdx.x; x < n; x += gridDim.x) {
    for (int y = threadIdx.x; y < n; y += blockDim.x) {
      double out;
      if (x == y) {
        out = val(v, ldv, x, x);  // 0 or -0, kept as the reference keeps it
      } else {
        const double a = val(v, ldv, min(x, y), max(x, y)), b = val(v, ldv, max(x, y), min(x, y));
        out = 0.5 * (a + b);
      }
      d[(size_t)x * ldd + y] = (float)out;
    }
  }
}

int io_error(int code, const std::string& msg) { return pald_gpu_set_error(code, msg.c_str()); }

#define IO_CUDA(expr)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return io_error(PALD_GPU_ERR_CUDA, std::string(#expr) + ": " + \
                                                            cudaGetErrorString(e_));      \
  } while (0)

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

int read_header(FILE* f, const std::string& path, int* width, uint64_t* n) {
  char magic[4];
  uint8_t ver = 0, w = 0;
  uint64_t n64 = 0;
  if (fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "PALD", 4) != 0)
    return io_error(PALD_GPU_ERR_VALIDATION, path + ": bad magic (not a PALD binary matrix)");
  if (fread(&ver, 1, 1, f) != 1 || ver != 1)
    return io_error(PALD_GPU_ERR_VALIDATION,
                    path + ": unsupported format version " + std::to_string((int)ver));
  if (fread(&w, 1, 1, f) != 1 || (w != 4 && w != 8))
    return io_error(PALD_GPU_ERR_VALIDATION,
                    path + ": unsupported element width " + std::to_string((int)w));
  if (fread(&n64, 8, 1, f) != 1) return io_error(PALD_GPU_ERR_VALIDATION, path + ": truncated header");
  *width = w;
  *n = n64;
  return PALD_GPU_OK;
}

// A corrupt header must not wrap n * n * width or truncate (int)n: check the
// payload against the file before anything is allocated. A file too short
// for its header is the reference's "truncated payload" (ingest.hpp:243-278
// fails on the read); a complete file beyond the engine's limit (n > 2^24:
// counts no longer exact in fp32) is refused. Leaves the file position
// unchanged.
int check_payload(FILE* f, const std::string& path, uint64_t n, int width) {
  const long pos = ftell(f);
  if (pos < 0 || fseek(f, 0, SEEK_END) != 0) return io_error(PALD_GPU_ERR_IO, path + ": cannot seek");
  const long end = ftell(f);
  if (end < 0 || fseek(f, pos, SEEK_SET) != 0) return io_error(PALD_GPU_ERR_IO, path + ": cannot seek");
  const unsigned __int128 need = (unsigned __int128)n * n * (unsigned)width;
  if (need > (unsigned __int128)(uint64_t)(end - pos))
    return io_error(PALD_GPU_ERR_VALIDATION, path + ": truncated payload");
  if (n > (1ull << 24))
    return io_error(PALD_GPU_ERR_UNSUPPORTED,
                    path + ": n = " + std::to_string(n) + " exceeds the engine limit 2^24");
  return PALD_GPU_OK;
}

}  // namespace

extern "C" {

int pald_gpu_read_binary_header(const char* path, uint64_t* n_out, int32_t* width_out) {
  if (!path || !n_out) return io_error(PALD_GPU_ERR_VALIDATION, "null argument");
  File file;
  file.f = fopen(path, "rb");
  if (!file.f) return io_error(PALD_GPU_ERR_IO, std::string("cannot open ") + path);
  int w = 0;
  int rc = read_header(file.f, path, &w, n_out);
  // callers size their buffers from n: refuse a header the payload cannot back
  if (rc == PALD_GPU_OK && *n_out >= 2) rc = check_payload(file.f, path, *n_out, w);
  if (rc == PALD_GPU_OK && width_out) *width_out = w;
  return rc;
}

int pald_gpu_read_distance_binary(const char* path, float* dD, uint64_t ldd, void* stream) {
  if (!path || !dD) return io_error(PALD_GPU_ERR_VALIDATION, "null argument");
  File file;
  file.f = fopen(path, "rb");
  if (!file.f) return io_error(PALD_GPU_ERR_IO, std::string("cannot open ") + path);
  int width = 0;
  uint64_t n = 0;
  int rc = read_header(file.f, path, &width, &n);
  if (rc) return rc;
  if (ldd < n) return io_error(PALD_GPU_ERR_VALIDATION, "ldd < n");
  if (n < 2) {  // read_matrix_binary reads (and may reject) the payload first
    const size_t need = (size_t)n * n * width;
    char tmp[8];
    if (need && fread(tmp, 1, need, file.f) != need)
      return io_error(PALD_GPU_ERR_VALIDATION, std::string(path) + ": truncated payload");
    return io_error(PALD_GPU_ERR_VALIDATION, std::string(path) + ": need at least 2 points");
  }
  if ((rc = check_payload(file.f, path, n, width))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Raw payload on the device (row-major, dense), streamed through a pinned
  // double buffer.
  const size_t bytes = (size_t)n * n * width;
  void* raw = nullptr;
  IO_CUDA(cudaMallocAsync(&raw, bytes, s));
  struct Free {
    void* p;
    cudaStream_t s;
    ~Free() { cudaFreeAsync(p, s); }
  } free_raw{raw, s};
  constexpr size_t kChunk = 64ull << 20;
  void* pin[2] = {nullptr, nullptr};
  IO_CUDA(cudaMallocHost(&pin[0], kChunk));
  IO_CUDA(cudaMallocHost(&pin[1], kChunk));
  cudaEvent_t done[2];
  IO_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  IO_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  struct Pinned {
    void** p;
    cudaEvent_t* e;
    ~Pinned() {
      cudaEventSynchronize(e[0]);
      cudaEventSynchronize(e[1]);
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
      cudaFreeHost(p[0]);
      cudaFreeHost(p[1]);
    }
  } pinned{pin, done};
  IO_CUDA(cudaEventRecord(done[0], s));
  IO_CUDA(cudaEventRecord(done[1], s));
  size_t off = 0;
  for (int b = 0; off < bytes; b ^= 1) {
    const size_t len = std::min(kChunk, bytes - off);
    IO_CUDA(cudaEventSynchronize(done[b]));  // the buffer's previous copy finished
    if (fread(pin[b], 1, len, file.f) != len)
      return io_error(PALD_GPU_ERR_VALIDATION, std::string(path) + ": truncated payload");
    IO_CUDA(cudaMemcpyAsync(static_cast<char*>(raw) + off, pin[b], len, cudaMemcpyHostToDevice, s));
    IO_CUDA(cudaEventRecord(done[b], s));
    off += len;
  }
  // Checks, then the first violation in the reference's order.
  IoCheck* chk = nullptr;
  IO_CUDA(cudaMallocAsync(&chk, sizeof(IoCheck), s));
  IO_CUDA(cudaMemsetAsync(chk, 0xff, sizeof(IoCheck), s));
  const int grid = (int)std::min<uint64_t>(n, 148ull * 16);
  if (width == 4)
    check_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(raw), n, (int)n, chk);
  else
    check_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(raw), n, (int)n, chk);
  IO_CUDA(cudaGetLastError());
  IoCheck h;
  IO_CUDA(cudaMemcpyAsync(&h, chk, sizeof(IoCheck), cudaMemcpyDeviceToHost, s));
  IO_CUDA(cudaFreeAsync(chk, s));
  IO_CUDA(cudaStreamSynchronize(s));
  const std::string origin(path);
  if (h.pass1 != ~0ull) {
    const uint64_t x = h.pass1 / (n + 1), y = h.pass1 % (n + 1);
    if (y == n)
      return io_error(PALD_GPU_ERR_VALIDATION, origin + ": nonzero diagonal at (" + std::to_string(x) +
                                                   "," + std::to_string(x) + ")");
    // re-read the offending element to tell non-finite from negative
    double d = 0.0;
    if (width == 4) {
      float fv;
      IO_CUDA(cudaMemcpy(&fv, static_cast<const float*>(raw) + x * n + y, 4, cudaMemcpyDeviceToHost));
      d = fv;
    } else {
      IO_CUDA(cudaMemcpy(&d, static_cast<const double*>(raw) + x * n + y, 8, cudaMemcpyDeviceToHost));
    }
    const std::string at = "(" + std::to_string(x) + "," + std::to_string(y) + ")";
    if (!std::isfinite(d)) return io_error(PALD_GPU_ERR_VALIDATION, origin + ": non-finite entry at " + at);
    return io_error(PALD_GPU_ERR_VALIDATION, origin + ": negative distance at " + at);
  }
  if (h.pass2 != ~0ull) {
    const uint64_t lin = h.pass2 / 2, kind = h.pass2 % 2, x = lin / n, y = lin % n;
    const std::string at = "(" + std::to_string(x) + "," + std::to_string(y) + ")";
    if (kind == 0) {
      double ab[2];
      for (int k = 0; k < 2; ++k) {
        const uint64_t idx = k == 0 ? x * n + y : y * n + x;
        if (width == 4) {
          float fv;
          IO_CUDA(cudaMemcpy(&fv, static_cast<const float*>(raw) + idx, 4, cudaMemcpyDeviceToHost));
          ab[k] = fv;
        } else {
          IO_CUDA(cudaMemcpy(&ab[k], static_cast<const double*>(raw) + idx, 8, cudaMemcpyDeviceToHost));
        }
      }
      return io_error(PALD_GPU_ERR_VALIDATION, origin + ": asymmetry beyond tolerance at " + at + ": " +
                                                   std::to_string(ab[0]) + " vs " + std::to_string(ab[1]));
    }
    return io_error(PALD_GPU_ERR_VALIDATION,
                    origin + ": zero off-diagonal distance at " + at + " (duplicate points)");
  }
  if (width == 4)
    symmetrize_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(raw), n, (int)n, dD, ldd);
  else
    symmetrize_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(raw), n, (int)n, dD, ldd);
  IO_CUDA(cudaGetLastError());
  return PALD_GPU_OK;
}

}  // extern "C"
