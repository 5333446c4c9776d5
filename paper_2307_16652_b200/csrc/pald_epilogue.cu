// pald_epilogue.cu -- O(n^2) epilogue of the PaLD path on the GPU (SURVEY
// 8(f) rank 1 and 4): normalization, local depths, the universal strong-tie
// threshold and the strong-tie edge list, computed straight from the fp32
// cohesion matrix the tile kernels leave in HBM (no double copy of C).
//
// Every quantity reproduces the reference's double arithmetic and summation
// order exactly:
//   normalize        c' = double(c) * (1.0 / (n - 1))       reference.hpp:223-228
//   local_depths     sum_z c'_xz, z ascending                 reference.hpp:231-241
//   threshold        0.5 * (sum_x c'_xx, x ascending) / n     analyze.hpp:34-39
//   strong_ties      x < y with min(c'_xy, c'_yx) >= thr,     analyze.hpp:43-53
//                    in (x, y) row-major order
// An optional double diagonal (the triplet's fill_diagonal, reference.hpp:
// 213-220) replaces c_xx before normalization, as the CLI does (pald.cpp:
// 159-160).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/pald_gpu.h"
#include "pald_internal.h"

namespace {

__device__ __forceinline__ double cval(const float* __restrict__ c, uint64_t ld, int x, int z,
                                       const double* __restrict__ diag, double scale) {
  const double v = (diag && x == z) ? diag[x] : (double)c[(size_t)x * ld + z];
  return __dmul_rn(v, scale);
}

// One warp per 32 rows: a 32 x 32 tile is staged through shared memory with
// coalesced loads, then each lane adds its own row's 32 values in ascending
// z, so each depth is the sequential double sum of the reference.
__global__ void depths_kernel(const float* __restrict__ c, uint64_t ld, int n,
                              const double* __restrict__ diag, double scale,
                              double* __restrict__ depths) {
  __shared__ float tile[32][33];
  const int lane = threadIdx.x;
  const int x0 = blockIdx.x * 32;
  const int x = x0 + lane;
  double s = 0.0;
  for (int z0 = 0; z0 < n; z0 += 32) {
    for (int r = 0; r < 32; ++r) {
      const int xr = x0 + r, z = z0 + lane;
      tile[r][lane] = (xr < n && z < n) ? c[(size_t)xr * ld + z] : 0.f;
    }
    __syncwarp();
    if (x < n) {
      const int zmax = min(32, n - z0);
      for (int j = 0; j < zmax; ++j) {
        const int z = z0 + j;
        const double v = (diag && z == x) ? diag[x] : (double)tile[lane][j];
        s = __dadd_rn(s, __dmul_rn(v, scale));
      }
    }
    __syncwarp();
  }
  if (x < n) depths[x] = s;
}

__global__ void threshold_kernel(const float* __restrict__ c, uint64_t ld, int n,
                                 const double* __restrict__ diag, double scale, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int x = 0; x < n; ++x) s = __dadd_rn(s, cval(c, ld, x, x, diag, scale));
  *out = __dmul_rn(0.5, s) / (double)n;
}

// Strong ties, pass A: count per row (one warp per row).
__global__ void ties_count_kernel(const float* __restrict__ c, uint64_t ld, int n,
                                  const double* __restrict__ diag, double scale,
                                  const double* __restrict__ thr, uint32_t* __restrict__ counts) {
  const int x = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (x >= n) return;
  const double t = *thr;
  uint32_t cnt = 0;
  for (int y0 = x + 1; y0 < n; y0 += 32) {
    const int y = y0 + lane;
    bool hit = false;
    if (y < n) hit = fmin(cval(c, ld, x, y, diag, scale), cval(c, ld, y, x, diag, scale)) >= t;
    cnt += __popc(__ballot_sync(0xffffffffu, hit));
  }
  if (lane == 0) counts[x] = cnt;
}

// Pass B: write the edges of row x at offsets[x] in ascending y.
__global__ void ties_write_kernel(const float* __restrict__ c, uint64_t ld, int n,
                                  const double* __restrict__ diag, double scale,
                                  const double* __restrict__ thr,
                                  const uint64_t* __restrict__ offsets, uint64_t capacity,
                                  uint32_t* __restrict__ xs, uint32_t* __restrict__ ys,
                                  double* __restrict__ strength) {
  const int x = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (x >= n) return;
  const double t = *thr;
  uint64_t pos = offsets[x];
  for (int y0 = x + 1; y0 < n; y0 += 32) {
    const int y = y0 + lane;
    double s = 0.0;
    bool hit = false;
    if (y < n) {
      s = fmin(cval(c, ld, x, y, diag, scale), cval(c, ld, y, x, diag, scale));
      hit = s >= t;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const uint64_t o = pos + __popc(m & ((1u << lane) - 1u));
      if (o < capacity) {
        xs[o] = (uint32_t)x;
        ys[o] = (uint32_t)y;
        strength[o] = s;
      }
    }
    pos += __popc(m);
  }
}

__global__ void exclusive_scan_kernel(const uint32_t* __restrict__ counts, int n,
                                      uint64_t* __restrict__ offsets, uint64_t* __restrict__ total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t s = 0;
  for (int x = 0; x < n; ++x) {
    offsets[x] = s;
    s += counts[x];
  }
  *total = s;
}

// Double-matrix epilogue of the Python mirror (its CohesionMatrix holds
// doubles, like the reference's): normalize in place, sequential row sums.
__global__ void normalize_f64_kernel(double* __restrict__ c, uint64_t ld, int n, double scale) {
  for (int r = blockIdx.x; r < n; r += gridDim.x)
    for (int z = threadIdx.x; z < n; z += blockDim.x) c[(size_t)r * ld + z] = __dmul_rn(c[(size_t)r * ld + z], scale);
}

__global__ void row_sums_f64_kernel(const double* __restrict__ c, uint64_t ld, int n, double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int lane = threadIdx.x, x0 = blockIdx.x * 32, x = x0 + lane;
  double s = 0.0;
  for (int z0 = 0; z0 < n; z0 += 32) {
    for (int r = 0; r < 32; ++r) {
      const int xr = x0 + r, z = z0 + lane;
      tile[r][lane] = (xr < n && z < n) ? c[(size_t)xr * ld + z] : 0.0;
    }
    __syncwarp();
    if (x < n) {
      const int zmax = min(32, n - z0);
      for (int j = 0; j < zmax; ++j) s = __dadd_rn(s, tile[lane][j]);
    }
    __syncwarp();
  }
  if (x < n) out[x] = s;
}

// nearest_neighbors (analyze.hpp:60-75), pass 1: for every z != focus the
// normalized strength min(c'_fz, c'_zf), as the key of a stable descending
// radix sort (non-negative doubles order as their bit patterns; equal
// strengths keep ascending z, the reference's std::stable_sort order).
__global__ void neighbor_keys_kernel(const float* __restrict__ c, uint64_t ld, int n, const double* __restrict__ diag,
                                     double scale, int focus, unsigned long long* __restrict__ keys,
                                     uint32_t* __restrict__ idx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
    const int z = i < focus ? i : i + 1;
    const double s = fmin(cval(c, ld, focus, z, diag, scale), cval(c, ld, z, focus, diag, scale));
    keys[i] = (unsigned long long)__double_as_longlong(s);
    idx[i] = (uint32_t)z;
  }
}

__global__ void neighbor_out_kernel(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ idx,
                                    int k, uint32_t* __restrict__ zs, double* __restrict__ strength) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    zs[i] = idx[i];
    strength[i] = __longlong_as_double((long long)keys[i]);
  }
}

int fail(cudaError_t e, const char* what) {
  return pald_gpu_set_error(PALD_GPU_ERR_CUDA, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

}  // namespace

extern "C" {

int pald_gpu_local_depths(const float* dC, uint64_t ldc, uint64_t n, const double* diag,
                          double* depths_out, void* stream) {
  if (!dC || !depths_out || n < 2 || ldc < n)
    return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "local_depths: invalid arguments");
  const double scale = 1.0 / (double)(n - 1);
  depths_kernel<<<(unsigned)((n + 31) / 32), 32, 0, static_cast<cudaStream_t>(stream)>>>(
      dC, ldc, (int)n, diag, scale, depths_out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PALD_GPU_OK : fail(e, "depths_kernel");
}

int pald_gpu_strong_ties(const float* dC, uint64_t ldc, uint64_t n, const double* diag,
                         const double* threshold_in, double* threshold_out, uint64_t capacity,
                         uint32_t* xs, uint32_t* ys, double* strength, uint64_t* count_out,
                         void* stream) {
  if (!dC || !threshold_out || !count_out || n < 2 || ldc < n)
    return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "strong_ties: invalid arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const double scale = 1.0 / (double)(n - 1);
  if (threshold_in) {
    cudaError_t e = cudaMemcpyAsync(threshold_out, threshold_in, sizeof(double),
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return fail(e, "threshold copy");
  } else {
    threshold_kernel<<<1, 32, 0, s>>>(dC, ldc, (int)n, diag, scale, threshold_out);
  }
  uint32_t* counts = nullptr;
  uint64_t* offsets = nullptr;
  cudaError_t e = cudaMallocAsync(&counts, n * sizeof(uint32_t), s);
  if (e != cudaSuccess) return fail(e, "alloc");
  e = cudaMallocAsync(&offsets, n * sizeof(uint64_t), s);
  if (e != cudaSuccess) return fail(e, "alloc");
  const unsigned blocks = (unsigned)((n + 7) / 8);
  ties_count_kernel<<<blocks, 256, 0, s>>>(dC, ldc, (int)n, diag, scale, threshold_out, counts);
  exclusive_scan_kernel<<<1, 32, 0, s>>>(counts, (int)n, offsets, count_out);
  if (xs && ys && strength && capacity)
    ties_write_kernel<<<blocks, 256, 0, s>>>(dC, ldc, (int)n, diag, scale, threshold_out, offsets,
                                             capacity, xs, ys, strength);
  cudaFreeAsync(counts, s);
  cudaFreeAsync(offsets, s);
  e = cudaGetLastError();
  return e == cudaSuccess ? PALD_GPU_OK : fail(e, "strong ties");
}

int pald_gpu_normalize_f64(double* dC, uint64_t ldc, uint64_t n, void* stream) {
  if (!dC || n < 2 || ldc < n) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "normalize: invalid arguments");
  normalize_f64_kernel<<<(unsigned)std::min<uint64_t>(n, 148 * 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dC, ldc, (int)n, 1.0 / (double)(n - 1));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PALD_GPU_OK : fail(e, "normalize_f64_kernel");
}

int pald_gpu_row_sums_f64(const double* dC, uint64_t ldc, uint64_t n, double* out, void* stream) {
  if (!dC || !out || n < 1 || ldc < n) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "row_sums: invalid arguments");
  row_sums_f64_kernel<<<(unsigned)((n + 31) / 32), 32, 0, static_cast<cudaStream_t>(stream)>>>(dC, ldc, (int)n, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PALD_GPU_OK : fail(e, "row_sums_f64_kernel");
}

int pald_gpu_nearest_neighbors(const float* dC, uint64_t ldc, uint64_t n, const double* diag, uint64_t focus,
                               uint64_t k, uint32_t* zs, double* strength, void* stream) {
  // analyze.hpp:64-65: the reference's checks and messages, in its order
  if (focus >= n) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "focus point out of range");
  if (k >= n) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "k must be smaller than the point count");
  if (!dC || ldc < n || (k && (!zs || !strength)))
    return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "nearest_neighbors: invalid arguments");
  if (k == 0) return PALD_GPU_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int m = (int)n - 1;
  unsigned long long *keys = nullptr, *keys_out = nullptr;
  uint32_t *idx = nullptr, *idx_out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, keys, keys_out, idx, idx_out, m, 0, 64, s);
  cudaError_t e = cudaMallocAsync(&keys, (size_t)m * 8 * 2 + (size_t)m * 4 * 2 + tmp_bytes, s);
  if (e != cudaSuccess) return fail(e, "alloc");
  keys_out = keys + m;
  idx = reinterpret_cast<uint32_t*>(keys_out + m);
  idx_out = idx + m;
  tmp = idx_out + m;
  neighbor_keys_kernel<<<(unsigned)std::min<int>((m + 255) / 256, 148 * 8), 256, 0, s>>>(
      dC, ldc, (int)n, diag, 1.0 / (double)(n - 1), (int)focus, keys, idx);
  // stable: equal strengths keep ascending z
  cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, keys, keys_out, idx, idx_out, m, 0, 64, s);
  neighbor_out_kernel<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(keys_out, idx_out, (int)k, zs, strength);
  cudaFreeAsync(keys, s);
  e = cudaGetLastError();
  return e == cudaSuccess ? PALD_GPU_OK : fail(e, "nearest_neighbors");
}

}  // extern "C"
