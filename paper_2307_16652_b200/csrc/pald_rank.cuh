// pald_rank.cuh -- per-row rank codes of D for the packed pass-1 kernel.
//
// Pairwise focus (blocked.hpp:101-122, reference.hpp:31-45) only ever
// compares two entries of the SAME row of D: [d_xz < d_xy] (row x) and
// [d_yz < d_xy] (row y). Replacing every entry of row r by its rank in that
// row,
//
//   Rk[r][k] = #{ j : d_rj < d_rk }          (ties share the lowest rank),
//
// preserves every such comparison exactly: d_rk < d_rc <=> Rk[r][k] <
// Rk[r][c], and d_rk <= d_rc <=> Rk[r][k] < Rk[r][c] + 1. Ranks of an
// n <= 32768 row fit in 15 bits, so the focus kernel can compare two output
// columns per 32-bit integer instruction (16-bit lanes with a borrow-free
// flag bit, pald_kernels.cuh k_step_rank). The codes are built once per load:
//
//   row_rank_kernel:    one CTA per row; CUB block radix sort of (key,
//                       index) pairs (rows > 16384: two sorted segments
//                       merged by merge path), then a max-scan over the
//                       sorted keys gives each element the position of the
//                       first element of its tie group; ranks scattered to
//                       Rk[r][*].
//   rank_layout_kernel: transposes Rk into the two panels the focus kernel
//                       streams by TMA: RA[k][r] = (0x8000 | Rk[r][k]) * 0x10001
//                       (the 16-bit code with its flag bit, broadcast to both
//                       halves) and RB[k][c] = 0x8000 | Rk[c][k] (uint16).
//
// Keys are the raw fp32 bits of D with the sign bit masked (the diagonal may
// be -0.0), or the plan's layout of D (scaled fp32 bits or the exact path's
// integer keys 2*bits(d)): all are monotone in d as unsigned integers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/block/block_radix_sort.cuh>

#include "pald_sym.cuh"  // tie masks of the tile-pair kernel (pair_index, kSymBK)

namespace pald_gpu {

constexpr int kRankMaxN = 32768;  // ranks < 2^15: one flag bit per 16-bit lane
constexpr int kRankRadixBits = 6;   // 5 digit passes over 30-bit fast-path keys, 6 over 32
constexpr int kRankBins = 16384;    // value-linear bins of the fast row path
constexpr int kRankMaxBin = 64;     // larger bins: the row takes the sort path
// packed u16 counts + cursors, and the keys of multi-key bins (their
// indices, read only on a tie, go to a per-CTA global scratch)
__host__ __device__ constexpr int rank_bin_smem(int keys) { return kRankBins * 2 * 2 + keys * 4; }

// Per-row sort configuration: THREADS x ITEMS keys per CUB block radix sort
// (one "segment"); rows longer than one segment (n > 16384) are sorted as two
// segments and merged.
template <int THREADS, int ITEMS>
struct RankCfg {
  static constexpr int kSeg = THREADS * ITEMS;
  using Sort = cub::BlockRadixSort<uint32_t, THREADS, ITEMS, uint16_t, kRankRadixBits>;
  static constexpr int kTempBytes = (int)((sizeof(typename Sort::TempStorage) + 127) / 128 * 128);
  // the two-segment merge keeps both sorted key runs in shared memory
  static constexpr int smem_bytes(int n) { return kTempBytes + (n > kSeg ? 2 * kSeg * 4 : 0); }
};

// Block-wide exclusive max-scan of one value per thread (tid order).
template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_max(uint32_t v, uint32_t* warp_buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = max(incl, u);
  }
  if (lane == 31) warp_buf[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < THREADS / 32 ? warp_buf[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = max(w, u);
    }
    if (lane < THREADS / 32) warp_buf[lane] = w;
  }
  __syncthreads();
  uint32_t ex = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) ex = 0u;
  if (warp > 0) ex = max(ex, warp_buf[warp - 1]);
  __syncthreads();  // warp_buf reused by the caller's next scan
  return ex;
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_reduce_max(uint32_t v, uint32_t* warp_buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) warp_buf[warp] = v;
  __syncthreads();
  uint32_t r = 0;
#pragma unroll
  for (int w = 0; w < THREADS / 32; ++w) r = max(r, warp_buf[w]);
  __syncthreads();
  return r;
}

// Block-wide exclusive sum of one value per thread (tid order); *total set.
template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* warp_buf, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) warp_buf[warp] = incl;
  __syncthreads();
  uint32_t before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < THREADS / 32; ++w) {
    const uint32_t x = warp_buf[w];
    if (w < warp) before += x;
    all += x;
  }
  __syncthreads();
  *total = all;
  return before + incl - v;
}

// Fast path of one row (fp32 layout keys, all finite): counting sort on
// NB value-linear bins, bin = floor(v * (NB-1)/vmax) (monotone in v), so
//   rank(x) = #{keys in lower bins} + #{keys < x in x's bin}.
// Bins hold ~n/NB keys; multi-key bins are resolved by scanning the bin's
// keys, scattered into shared memory. The row stays in registers (thread t
// holds elements t + e*THREADS). Returns false (row left to the sort path)
// when a bin holds more than kRankMaxBin keys.
//
// Equal keys meet in one bin, so the bin scan also finds every key of row j
// (= column j of the symmetric D) that occurs more than once. With tie masks
// given, those keys and their indices are collected (kTieList entries per
// row; more flag the whole tile, like tie_scan_kernel's overflow), and for
// every duplicate pair (a, b) third point k = b is marked in tile pair
// {tile(j), tile(a)} and k = a in {tile(j), tile(b)}: the marks of
// tie_scan_kernel (pald_sym.cuh) for this row.
struct TieMarks {
  uint32_t* masks;       // nullptr: no marking
  uint32_t* tile_flags;  // [nb]: the whole tile marked
  int nb, nch;
};
constexpr int kTieList = 1024;

template <int THREADS, int E>
__device__ bool rank_row_bins(const uint32_t* __restrict__ row, int j, int n, uint32_t key_mask, uint16_t* __restrict__ out,
                              uint32_t* hist, uint32_t* curs, uint32_t* kscr, uint2* tie_list, uint32_t* tie_count,
                              uint32_t* warp_buf, const TieMarks& tm) {
  constexpr int NB = kRankBins, W = NB / 2, PER = W / THREADS;  // E * THREADS >= n keys
  const int tid = threadIdx.x;
  uint32_t key[E];
  uint32_t mx = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * THREADS + tid;
    key[e] = i < n ? (__ldg(row + i) & key_mask) : 0u;
    mx = max(mx, key[e]);
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) hist[q * THREADS + tid] = 0u;
  mx = block_reduce_max<THREADS>(mx, warp_buf);  // (syncs: hist zeroed)
  const float scale = (float)(NB - 1) / __uint_as_float(mx);
  auto bin_of = [&](uint32_t k) { return min(NB - 1, (int)(__uint_as_float(k) * scale)); };
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (e * THREADS + tid < n) {
      const int b = bin_of(key[e]);
      atomicAdd(&hist[b >> 1], 1u << ((b & 1) * 16));
    }
  }
  __syncthreads();
  // exclusive scan of the NB counts (thread tid: words [tid*PER, (tid+1)*PER))
  uint32_t local = 0, cmax = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const uint32_t w = hist[tid * PER + q];
    local += (w & 0xffffu) + (w >> 16);
    cmax = max(cmax, max(w & 0xffffu, w >> 16));
  }
  uint32_t total;
  uint32_t run = block_excl_sum<THREADS>(local, warp_buf, &total);
  cmax = block_reduce_max<THREADS>(cmax, warp_buf);
  if (cmax > (uint32_t)kRankMaxBin) return false;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const uint32_t w = hist[tid * PER + q];
    const uint32_t lo = run, hi = run + (w & 0xffffu);
    run = hi + (w >> 16);
    const uint32_t pw = lo | (hi << 16);
    hist[tid * PER + q] = pw;  // bin starts
    curs[tid * PER + q] = pw;
  }
  __syncthreads();
  auto start = [&](int b) { return (hist[b >> 1] >> ((b & 1) * 16)) & 0xffffu; };
  auto next = [&](int b) { return b + 1 < NB ? start(b + 1) : (uint32_t)n; };
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (e * THREADS + tid < n) {
      const int b = bin_of(key[e]);
      if (next(b) - start(b) > 1u) {
        const uint32_t old = atomicAdd(&curs[b >> 1], 1u << ((b & 1) * 16));
        const uint32_t slot = (old >> ((b & 1) * 16)) & 0xffffu;
        kscr[slot] = key[e];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * THREADS + tid;
    if (i < n) {
      const int b = bin_of(key[e]);
      const uint32_t base = start(b), end = next(b);
      uint32_t cnt = 0, eq = 0;
      if (end - base > 1u) {
        for (uint32_t q = base; q < end; ++q) {
          const uint32_t kq = kscr[q];
          cnt += kq < key[e];
          eq += kq == key[e];
        }
      }
      out[i] = (uint16_t)(base + cnt);
      if (eq > 1u && tm.masks) {  // a duplicated value: collect (key, index)
        const uint32_t o = atomicAdd(tie_count, 1u);
        if (o < (uint32_t)kTieList) tie_list[o] = make_uint2(key[e], (uint32_t)i);
      }
    }
  }
  __syncthreads();
  if (tm.masks) {
    const uint32_t m = *tie_count;
    const int tj = j / kTile;
    if (m > (uint32_t)kTieList) {
      if (tid == 0) atomicOr(&tm.tile_flags[tj], 1u);
    } else {
      for (uint32_t a = tid; a < m; a += THREADS) {
        const uint2 ea = tie_list[a];
        const int ta = (int)ea.y / kTile;
        uint32_t* mrow = tm.masks + pair_index(min(tj, ta), max(tj, ta), tm.nb) * tm.nch;
        for (uint32_t b = 0; b < m; ++b) {
          const uint2 eb = tie_list[b];
          if (b != a && eb.x == ea.x) atomicOr(&mrow[eb.y / kSymBK], 1u << (eb.y % kSymBK));
        }
      }
    }
    __syncthreads();
    if (tid == 0) *tie_count = 0u;
  }
  __syncthreads();
  return true;
}

// Rk (uint16, n x ld, row-major) of the layout keys ds (n x ld). Rank of a
// sorted position = the last tie-group start at or before it (a max-scan of
// the positions where the key changes). idx_scratch: 2 * kSeg uint16 per
// CTA (two-segment rows only).
// Fast-layout rows through rank_row_bins (THREADS threads, E keys each, per
// row; several rows per SM for small n); rows it declines are appended to
// (fail_rows, *fail_count) for row_rank_kernel.
template <int THREADS, int E>
__global__ void __launch_bounds__(THREADS)
    row_rank_bins_kernel(const uint32_t* __restrict__ ds, int n, int ld, uint16_t* __restrict__ rk,
                         int* __restrict__ fail_rows, int* __restrict__ fail_count, TieMarks tm, int r_begin,
                         int r_end, uint32_t key_mask, size_t key_ld) {
  extern __shared__ __align__(128) uint8_t rank_smem[];
  __shared__ uint32_t warp_buf[THREADS / 32];
  uint32_t* hist = reinterpret_cast<uint32_t*>(rank_smem);
  uint32_t* kscr = hist + kRankBins;  // after counts and cursors
  __shared__ uint2 tie_list[kTieList];
  __shared__ uint32_t tie_count;
  if (threadIdx.x == 0) tie_count = 0u;
  __syncthreads();
  for (int r = r_begin + blockIdx.x; r < r_end; r += gridDim.x) {
    if (!rank_row_bins<THREADS, E>(ds + (size_t)r * key_ld, r, n, key_mask, rk + (size_t)r * ld, hist, hist + kRankBins / 2,
                                   kscr, tie_list, &tie_count, warp_buf, tm)) {
      if (threadIdx.x == 0) fail_rows[atomicAdd(fail_count, 1)] = r;
      __syncthreads();
    }
  }
}

// Sort path: all rows (rows == nullptr) or the listed rows.
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
    row_rank_kernel(const uint32_t* __restrict__ ds, int n, int ld, int end_bit, const int* __restrict__ rows,
                    const int* __restrict__ row_count, uint16_t* __restrict__ rk, uint32_t* __restrict__ scratch,
                    uint32_t key_mask, size_t key_ld) {
  using Cfg = RankCfg<THREADS, ITEMS>;
  constexpr int S = Cfg::kSeg;
  extern __shared__ __align__(128) uint8_t rank_smem[];
  auto& temp = *reinterpret_cast<typename Cfg::Sort::TempStorage*>(rank_smem);
  uint32_t* sk = reinterpret_cast<uint32_t*>(rank_smem + Cfg::kTempBytes);  // two-segment rows
  __shared__ uint32_t warp_buf[THREADS / 32];
  __shared__ uint32_t last_key[THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nseg = n > S ? 2 : 1;
  // per-CTA scratch: max(n, S) words (bin keys, or the two-segment indices)
  uint32_t* kscr = scratch + (size_t)blockIdx.x * max(n, S);
  uint16_t* scr = reinterpret_cast<uint16_t*>(kscr);

  const int nrows = rows ? *row_count : n;
  for (int ri = blockIdx.x; ri < nrows; ri += gridDim.x) {
    const int r = rows ? rows[ri] : ri;
    const uint32_t* row = ds + (size_t)r * key_ld;
    uint16_t* out = rk + (size_t)r * ld;
    for (int h = 0; h < nseg; ++h) {
      uint32_t keys[ITEMS];
      uint16_t vals[ITEMS];
#pragma unroll
      for (int e = 0; e < ITEMS; ++e) {  // striped (coalesced) load; order is irrelevant
        const int i = h * S + e * THREADS + tid;
        keys[e] = i < n ? (__ldg(row + i) & key_mask) : 0xffffffffu;  // never a key: sorts last
        vals[e] = (uint16_t)i;
      }
      Cfg::Sort(temp).Sort(keys, vals, 0, end_bit);  // blocked: positions tid*ITEMS + e
      if (nseg == 1) {
        // previous key of position tid*ITEMS: the last key of thread tid - 1
        uint32_t prev = __shfl_up_sync(0xffffffffu, keys[ITEMS - 1], 1);
        if (lane == 31) last_key[warp] = keys[ITEMS - 1];
        __syncthreads();
        if (lane == 0) prev = warp > 0 ? last_key[warp - 1] : ~keys[0];
        uint32_t m = 0, pk = prev;
#pragma unroll
        for (int e = 0; e < ITEMS; ++e) {
          if (keys[e] != pk) m = (uint32_t)(tid * ITEMS + e);
          pk = keys[e];
        }
        uint32_t run = block_excl_max<THREADS>(m, warp_buf);
        pk = prev;
#pragma unroll
        for (int e = 0; e < ITEMS; ++e) {
          if (keys[e] != pk) run = (uint32_t)(tid * ITEMS + e);
          pk = keys[e];
          if (vals[e] < n) out[vals[e]] = (uint16_t)run;
        }
      } else {
#pragma unroll
        for (int e = 0; e < ITEMS; ++e) {
          sk[h * S + tid * ITEMS + e] = keys[e];
          scr[h * S + tid * ITEMS + e] = vals[e];
        }
      }
      __syncthreads();  // TempStorage / last_key reuse
    }
    if (nseg == 1) continue;
    // Two sorted runs A = sk[0, S), B = sk[S, 2S): thread tid emits merged
    // positions [d, d + 2*ITEMS) (merge path; A first on equal keys).
    const uint32_t* A = sk;
    const uint32_t* B = sk + S;
    const int d = tid * 2 * ITEMS;
    int lo = max(0, d - S), hi = min(d, S);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (A[mid] <= B[d - mid - 1]) lo = mid + 1; else hi = mid;
    }
    const int i0 = lo, j0 = d - lo;
    uint32_t prev;  // merged key at position d - 1
    if (d == 0) prev = (A[0] <= B[0] ? A[0] : B[0]) ^ 1u;  // differs from the first merged key
    else prev = max(i0 > 0 ? A[i0 - 1] : 0u, j0 > 0 ? B[j0 - 1] : 0u);
    uint32_t m = 0;
    {
      int i = i0, j = j0;
      uint32_t pk = prev;
      for (int q = 0; q < 2 * ITEMS; ++q) {
        const bool ta = j >= S || (i < S && A[i] <= B[j]);
        const uint32_t k = ta ? A[i] : B[j];
        if (ta) ++i; else ++j;
        if (k != pk) m = (uint32_t)(d + q);
        pk = k;
      }
    }
    uint32_t run = block_excl_max<THREADS>(m, warp_buf);
    {
      int i = i0, j = j0;
      uint32_t pk = prev;
      for (int q = 0; q < 2 * ITEMS; ++q) {
        const bool ta = j >= S || (i < S && A[i] <= B[j]);
        const uint32_t k = ta ? A[i] : B[j];
        const int v = ta ? scr[i] : scr[S + j];
        if (ta) ++i; else ++j;
        if (k != pk) run = (uint32_t)(d + q);
        pk = k;
        if (v < n) out[v] = (uint16_t)run;
      }
    }
    __syncthreads();  // sk reused by the next row
  }
}

// RA[k][r] = (0x8000 | Rk[r][k]) * 0x10001, RB[k][r] = 0x8000 | Rk[r][k] for
// k < n, r in [r_begin, ld) covered by the grid; padding rows/columns
// (r >= n) get code 0.
__global__ void __launch_bounds__(256)
    rank_layout_kernel(const uint16_t* __restrict__ rk, int n, int ld, uint32_t* __restrict__ ra,
                       uint16_t* __restrict__ rb, int r_begin) {
  __shared__ uint16_t t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int r0 = r_begin + blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int yy = ty; yy < 32; yy += 8) {
    const int r = r0 + yy, k = k0 + tx;
    t[yy][tx] = (r < n && k < n) ? rk[(size_t)r * ld + k] : (uint16_t)0;
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int k = k0 + yy, r = r0 + tx;
    if (k < n && r < ld) {
      const uint32_t v = 0x8000u | t[tx][yy];
      ra[(size_t)k * ld + r] = v * 0x10001u;
      rb[(size_t)k * ld + r] = (uint16_t)v;
    }
  }
}

}  // namespace pald_gpu
