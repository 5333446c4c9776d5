// pald_sym.cuh -- pass 2 (cohesion) over tile PAIRS: one min + one compare
// per (r, c, k) feeds both C[r][c] and C[c][r].
//
// Gather form (pald_kernels.cuh): C[r][c] = sum_k W_rk [T_rc < min(A'_rk, B'_kc)]
// with A = D[k][r], B = D[k][c], T = D[r][c]. The transposed output reads
// T_cr = T_rc and the same two distances with the roles of A and B swapped:
//
//   C[c][r] = sum_k W_ck [T_rc < min(B''_kc, A''_rk)]
//
// so without the nu() transforms both indicators are the same number
// [T_rc < min(d_kr, d_kc)]. The transforms only change a comparison when
// the two compared values are EQUAL (T < nu(x) <=> T <= x), so:
//
//   * pairwise Strict (B' = nu(B) iff k < r; for the transposed output
//     nu(d_kr) iff k < c): both outputs equal the shared strict indicator
//     unless T_rc == d_kc or T_rc == d_kr for some k not in {r, c}, i.e.
//     unless column c of D holds d_rc twice (rows r and k) or column r holds
//     d_cr twice (rows c and k). A per-column duplicate scan at load time
//     (tie_scan_kernel) marks every third point k that can meet such a tie
//     in a tile pair (one 32-bit mask per (tile pair, 32-wide k chunk)); the
//     marked k steps take the per-element exact step (two mins, the nu() of
//     each output), all others the shared step. k in {r, c} needs no mark:
//     the min then contains d_rr = 0 or d_cc = 0 and both indicators are 0
//     (T > 0: the fast path requires positive off-diagonal distances),
//     unless the nu'd zero is compared with T = 0, which is itself a
//     duplicate of column c (d_rc = d_cc = 0) and marked.
//   * triplet (A' = nu(d_kr) iff k < c, B' = nu(d_kc) iff k < r; for the
//     transposed output nu(d_kc) iff k < r and nu(d_kr) iff k < c): the
//     same two transformed values, so the shared indicator is exact with
//     no tie scan. Chunks wholly below a tile take the nu'd layout through
//     the TMA map choice, chunks inside it the per-element step (like the
//     one-sided kernel); the diagonal of C is forced to 0.
//
// Every C entry is still one fp32 sum over k ascending of the same terms as
// the one-sided kernel (bit-identical to the reference); only the number of
// FMNMX / FFMA.SAT instructions per output halves: 4.75 instead of 7
// register-operand reads per output combo, the resource that bounds these
// loops (tools/microbench3.cu: 50 vs 36 output combos
// per SM-cycle).
#pragma once

#include "pald_kernels.cuh"

namespace pald_gpu {

#ifndef PALD_SYM_UNROLL  // unroll of the shared k loop (scheduling knob)
#define PALD_SYM_UNROLL 1
#endif
#ifndef PALD_SYM_ORDER  // shared-step instruction order: 0 row-major, 1 per-row batches, 2 column-pair outer
#define PALD_SYM_ORDER 2
#endif
#ifndef PALD_SYM_SCALAR_DIRECT  // 1: C[r][c] accumulated with scalar FFMA
#define PALD_SYM_SCALAR_DIRECT 0
#endif
constexpr int kSymUnroll = PALD_SYM_UNROLL;
constexpr int kSymBK = 32;                         // k chunk per stage
constexpr int kSymStages = 3;
constexpr int kSymBox = kSymBK * kTile * 4;        // one 32 x 128 fp32 box (16 KB)
constexpr int kSymStageBytes = 4 * kSymBox;        // A, B, W rows, W cols
constexpr int kSymSmem = kSymStages * kSymStageBytes + 1024;

// Tie scan: buckets and capacity of one pass over a column in shared memory.
constexpr int kTieBuckets = 4096;
constexpr int kTieCap = 16384;
constexpr int kTieThreads = 1024;
constexpr int kTieMaxBucket = 64;  // larger buckets flag the whole tile
constexpr int kTieSmem = kTieCap * 8 + kTieBuckets * 8;

struct SymArgs {
  const uint32_t* d;          // scaled fp32 layout of D (n x ld)
  float* c;                   // cohesion (n x ld)
  const int2* tiles;          // tile pairs (P <= Q), grouped order
  const uint32_t* masks;      // [pair_index(P, Q)][nch]: k bits of each 32-wide chunk
  const uint32_t* tile_flags; // [nb]: every k of every pair of this tile is marked
  int n, ld, nb, nch;
  int tile_begin, tile_end;   // share of the tile-pair list
  PeerBufs peers;             // PEERS: every C entry is stored to every rank's C
  unsigned int* round_bar;    // SYNC kernels: all CTAs start each full round together
  // SPLIT kernels (triplet): work items (tile row, tile col, chunk_begin |
  // chunk_end << 16, slot) replace whole pairs; slot >= 0 items write their
  // partial tiles to partial[slot] (2 x 128 x 128 floats) for sym_combine_kernel.
  const int4* items;
  float* partial;
  double* c64;                // ACC kernels: double sums of the fp32 block partials (n x ld)
  int acc_chunks;             // ACC kernels: k chunks (of kSymBK) per fp32 block partial
  int tri_marks;              // TRI: masks hold the tie marks (chunks inside the tiles
                              // run the shared step for unmarked k)
};

// Full-avalanche mix (murmur3 finalizer): the bucket takes the low bits and
// the partition the high bits, and quantized inputs (values on a coarse
// grid have zero low mantissa bits) must still spread over both.
__device__ __forceinline__ uint32_t tie_hash(uint32_t key) {
  key ^= key >> 16;
  key *= 0x85ebca6bu;
  key ^= key >> 13;
  key *= 0xc2b2ae35u;
  key ^= key >> 16;
  return key;
}
// Index of tile pair (P, Q), P <= Q, in row-major upper-triangular order.
__host__ __device__ __forceinline__ size_t pair_index(int P, int Q, int nb) {
  return (size_t)P * (2 * nb - P + 1) / 2 + (Q - P);
}

// Flags for the duplicate pairs of column j. One CTA per column (row j of
// the symmetric layout, read coalesced); `passes` hash partitions of the
// column are bucketed in shared memory in turn and compared within buckets.
__global__ void __launch_bounds__(kTieThreads)
    tie_scan_kernel(const uint32_t* __restrict__ d, int n, int ld, int nb, int nch, int passes,
                    uint32_t* __restrict__ masks, uint32_t* __restrict__ tile_flags,
                    const int* __restrict__ rows = nullptr, const int* __restrict__ row_count = nullptr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* idx = keys + kTieCap;
  uint32_t* cnt = idx + kTieCap;
  uint32_t* pos = cnt + kTieBuckets;
  __shared__ uint32_t warp_sums[kTieThreads / 32];
  __shared__ int overflow;
  const int tid = threadIdx.x;
  // all columns, or only the listed ones (rows the rank-code build left
  // unmarked: pald_rank.cuh)
  const int ncols = rows ? *row_count : n;
  for (int jj = blockIdx.x; jj < ncols; jj += gridDim.x) {
    const int j = rows ? rows[jj] : jj;
    const uint32_t* row = d + (size_t)j * ld;
    const int tj = j / kTile;
    for (int pass = 0; pass < passes; ++pass) {
      for (int b = tid; b < kTieBuckets; b += kTieThreads) cnt[b] = 0;
      if (tid == 0) overflow = 0;
      __syncthreads();
      for (int i = tid; i < n; i += kTieThreads) {
        const uint32_t h = tie_hash(row[i]);
        if ((int)(((uint64_t)h * (uint32_t)passes) >> 32) != pass) continue;
        atomicAdd(&cnt[h & (kTieBuckets - 1)], 1u);
      }
      __syncthreads();
      // exclusive scan of cnt -> pos (4 buckets per thread)
      uint32_t loc[4], s = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        loc[q] = s;
        s += cnt[tid * 4 + q];
      }
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= o) incl += v;
      }
      if ((tid & 31) == 31) warp_sums[tid >> 5] = incl;
      __syncthreads();
      if (tid < 32) {
        uint32_t ws = warp_sums[tid], wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
          if (tid >= o) wi += v;
        }
        warp_sums[tid] = wi - ws;  // exclusive prefix of the warps
      }
      __syncthreads();
      const uint32_t base = warp_sums[tid >> 5] + incl - s;
#pragma unroll
      for (int q = 0; q < 4; ++q) pos[tid * 4 + q] = base + loc[q];
      if (tid == kTieThreads - 1 && base + s > (uint32_t)kTieCap) overflow = 1;
      __syncthreads();
      if (overflow) {  // too many values in this partition: flag the tile
#ifdef PALD_TIE_DEBUG
        if (tid == 0 && j < 4) printf("tie_scan col %d pass %d overflow\n", j, pass);
#endif
        if (tid == 0) atomicOr(&tile_flags[tj], 1u);
        __syncthreads();
        break;
      }
      for (int i = tid; i < n; i += kTieThreads) {
        const uint32_t key = row[i], h = tie_hash(key);
        if ((int)(((uint64_t)h * (uint32_t)passes) >> 32) != pass) continue;
        const uint32_t o = atomicAdd(&pos[h & (kTieBuckets - 1)], 1u);
        keys[o] = key;
        idx[o] = (uint32_t)i;
      }
      __syncthreads();
      for (int b = tid; b < kTieBuckets; b += kTieThreads) {
        const uint32_t hi = pos[b], lo = hi - cnt[b];
        if (hi - lo > (uint32_t)kTieMaxBucket) {
#ifdef PALD_TIE_DEBUG
          if (j < 4) printf("tie_scan col %d pass %d bucket %d size %u\n", j, pass, b, hi - lo);
#endif
          atomicOr(&tile_flags[tj], 1u);
          continue;
        }
        for (uint32_t e1 = lo; e1 < hi; ++e1) {
          const uint32_t k1 = keys[e1];
          for (uint32_t e2 = e1 + 1; e2 < hi; ++e2) {
            if (keys[e2] != k1) continue;
            // column j holds the same value at rows a and b: mark k = b
            // in pair {tile(j), tile(a)} and k = a in pair {tile(j), tile(b)}
            const int a = (int)idx[e1], bb = (int)idx[e2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int x = h ? bb : a, k = h ? a : bb;
              const int tx = x / kTile, P = min(tj, tx), Q = max(tj, tx);
              atomicOr(&masks[pair_index(P, Q, nb) * nch + k / kSymBK], 1u << (k % kSymBK));
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

// Number of marked (pair, k) steps, for the cost model of the launcher.
__global__ void tie_count_kernel(const uint32_t* __restrict__ masks, size_t words,
                                 unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (size_t)gridDim.x * blockDim.x)
    c += __popc(masks[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Shared step: one min + one compare per (r, c) pair, two accumulates.
__device__ __forceinline__ void sym_step(const float* __restrict__ sa, const float* __restrict__ sb,
                                         const float* __restrict__ sw, const float* __restrict__ sv,
                                         int kk, int ty, int tx, const float2 (&thr)[8][4],
                                         float2 (&acc)[8][4], float2 (&act)[8][4]) {
  float a[8], b[8], w[8], v[8];
  {
    const float4 a0 = reinterpret_cast<const float4*>(sa + kk * kTile)[ty];
    const float4 a1 = reinterpret_cast<const float4*>(sa + kk * kTile)[16 + ty];
    const float4 b0 = reinterpret_cast<const float4*>(sb + kk * kTile)[tx];
    const float4 b1 = reinterpret_cast<const float4*>(sb + kk * kTile)[16 + tx];
    const float4 w0 = reinterpret_cast<const float4*>(sw + kk * kTile)[ty];
    const float4 w1 = reinterpret_cast<const float4*>(sw + kk * kTile)[16 + ty];
    const float4 v0 = reinterpret_cast<const float4*>(sv + kk * kTile)[tx];
    const float4 v1 = reinterpret_cast<const float4*>(sv + kk * kTile)[16 + tx];
    a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
    a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
    b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
    b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
    w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
    w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
    v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w;
    v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
  }
#if PALD_SYM_ORDER == 1
  // per row: the 8 mins, the 8 compares, then the two accumulate groups
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = fminf(a[i], b[j]);
    float2 kv[4];
#pragma unroll
    for (int jp = 0; jp < 4; ++jp)
      kv[jp] = make_float2(__saturatef(__fmaf_rn(m[2 * jp], kCmpScale, thr[i][jp].x)),
                           __saturatef(__fmaf_rn(m[2 * jp + 1], kCmpScale, thr[i][jp].y)));
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) acc[i][jp] = __ffma2_rn(kv[jp], make_float2(w[i], w[i]), acc[i][jp]);
#pragma unroll
    for (int jp = 0; jp < 4; ++jp)
      act[i][jp] = __ffma2_rn(kv[jp], make_float2(v[2 * jp], v[2 * jp + 1]), act[i][jp]);
  }
  return;
#endif
#if PALD_SYM_ORDER == 2
#pragma unroll
  for (int jp = 0; jp < 4; ++jp) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#else
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
#endif
      const float m0 = fminf(a[i], b[2 * jp]);
      const float m1 = fminf(a[i], b[2 * jp + 1]);
      const float2 kv = make_float2(__saturatef(__fmaf_rn(m0, kCmpScale, thr[i][jp].x)),
                                    __saturatef(__fmaf_rn(m1, kCmpScale, thr[i][jp].y)));
#if PALD_SYM_SCALAR_DIRECT
      acc[i][jp].x = __fmaf_rn(kv.x, w[i], acc[i][jp].x);
      acc[i][jp].y = __fmaf_rn(kv.y, w[i], acc[i][jp].y);
#else
      acc[i][jp] = __ffma2_rn(kv, make_float2(w[i], w[i]), acc[i][jp]);
#endif
      act[i][jp] = __ffma2_rn(kv, make_float2(v[2 * jp], v[2 * jp + 1]), act[i][jp]);
    }
  }
}

// Exact step (flagged blocks, ragged last chunk): each output with its own
// nu(): C[r][c] uses min(d_kr, nu(d_kc) iff k < r), C[c][r] uses
// min(d_kc, nu(d_kr) iff k < c) -- pairwise Strict, blocked.hpp:126-186.
__device__ __forceinline__ void sym_step_exact(const float* __restrict__ sa,
                                               const float* __restrict__ sb,
                                               const float* __restrict__ sw,
                                               const float* __restrict__ sv, int kk, int kg,
                                               int ty, int tx, int r0, int c0,
                                               const float2 (&thr)[8][4], float2 (&acc)[8][4],
                                               float2 (&act)[8][4]) {
  float a[8], b[8], w[8], v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = sa[kk * kTile + row_off<kTile>(ty, i)];
    w[i] = sw[kk * kTile + row_off<kTile>(ty, i)];
    b[i] = sb[kk * kTile + row_off<kTile>(tx, i)];
    v[i] = sv[kk * kTile + row_off<kTile>(tx, i)];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool below_r = kg < r0 + row_off<kTile>(ty, i);
    const float an = nu_f(a[i]);
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      float kd[2], kt[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jp + h;
        const bool below_c = kg < c0 + row_off<kTile>(tx, j);
        const float t = h ? thr[i][jp].y : thr[i][jp].x;
        const float md = fminf(a[i], below_r ? nu_f(b[j]) : b[j]);
        const float mt = fminf(b[j], below_c ? an : a[i]);
        kd[h] = __saturatef(__fmaf_rn(md, kCmpScale, t));
        kt[h] = __saturatef(__fmaf_rn(mt, kCmpScale, t));
      }
      acc[i][jp] = __ffma2_rn(make_float2(kd[0], kd[1]), make_float2(w[i], w[i]), acc[i][jp]);
      act[i][jp] = __ffma2_rn(make_float2(kt[0], kt[1]), make_float2(v[2 * jp], v[2 * jp + 1]),
                              act[i][jp]);
    }
  }
}

// Triplet step for chunks inside the row (b_in) or column (a_in) tile:
// per-element nu() of the shared indicator [T < min(A', B')].
__device__ __forceinline__ void sym_step_tri_sel(const float* __restrict__ sa,
                                                 const float* __restrict__ sb,
                                                 const float* __restrict__ sw,
                                                 const float* __restrict__ sv, int kk, int kg,
                                                 int ty, int tx, int r0, int c0, bool a_in,
                                                 bool b_in, const float2 (&thr)[8][4],
                                                 float2 (&acc)[8][4], float2 (&act)[8][4]) {
  float a[8], b[8], w[8], v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = sa[kk * kTile + row_off<kTile>(ty, i)];
    w[i] = sw[kk * kTile + row_off<kTile>(ty, i)];
    b[i] = sb[kk * kTile + row_off<kTile>(tx, i)];
    v[i] = sv[kk * kTile + row_off<kTile>(tx, i)];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool nub = b_in && kg < r0 + row_off<kTile>(ty, i);
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      float kv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jp + h;
        const bool nua = a_in && kg < c0 + row_off<kTile>(tx, j);
        const float m = fminf(nua ? nu_f(a[i]) : a[i], nub ? nu_f(b[j]) : b[j]);
        kv[h] = __saturatef(__fmaf_rn(m, kCmpScale, h ? thr[i][jp].y : thr[i][jp].x));
      }
      const float2 k2 = make_float2(kv[0], kv[1]);
      acc[i][jp] = __ffma2_rn(k2, make_float2(w[i], w[i]), acc[i][jp]);
      act[i][jp] = __ffma2_rn(k2, make_float2(v[2 * jp], v[2 * jp + 1]), act[i][jp]);
    }
  }
}

// C store of the pair kernel: the local buffer, or (PEERS) every rank's
// buffer over NVLink, so that no collective is needed after pass 2.
template <bool PEERS>
__device__ __forceinline__ void store_c4(const SymArgs& a, size_t off, float4 v) {
  if constexpr (PEERS) {
    for (int q = 0; q < a.peers.count; ++q) *reinterpret_cast<float4*>(a.peers.ptr[q] + off) = v;
  } else {
    *reinterpret_cast<float4*>(a.c + off) = v;
  }
}


// Persistent pass-2 kernel over the tile pairs [tile_begin, tile_end) of the
// grouped upper-triangular order (P <= Q). CTA g takes pairs
// tile_begin + g, + G, ...; each pair streams all k chunks through a
// 3-stage TMA/mbarrier pipeline (four 32 x 128 boxes per stage) and writes
// C[P rows][Q cols] and, for P < Q, C[Q rows][P cols]. Pairwise Strict
// (TRI = false) or triplet cohesion on the fast (scaled fp32) layout.
template <bool TRI, bool PEERS = false, bool SYNC = false, bool SPLIT = false, bool ACC = false>
__global__ void __launch_bounds__(kThreads, 1)
    pald_sym_cohesion_kernel(const __grid_constant__ CUtensorMap tm_d,
                             const __grid_constant__ CUtensorMap tm_dnu,
                             const __grid_constant__ CUtensorMap tm_w, const SymArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kSymStages];
  __shared__ uint32_t done_cnt[kSymStages];
  const int tid = threadIdx.x;
  const int n = args.n, ld = args.ld;
  const int nch = args.nch;
  const int G = gridDim.x, g = blockIdx.x;
  const int first = args.tile_begin + g;
  // ACC (accurate mode): whole pairs flush their fp32 sums into the double
  // sums every acc_chunks chunks inside the (uniform) chunk loop; SPLIT item
  // lists (the triplet's split last round) are cut into k blocks by the host
  // and flush at the end of each item.
  const int R = first < args.tile_end ? (args.tile_end - 1 - first) / G + 1 : 0;
  // item ri of this CTA: tile pair and chunk range [cb, ce) (whole pairs
  // unless SPLIT). SPLIT items come from the host's list: (tile row, tile
  // col, cb | ce << 15, slot); empty items (cb == ce) pad per-CTA queues.
  auto item = [&](int ri, int2& tp, int& cb, int& ce, int& slot) {
    if constexpr (SPLIT) {
      const int4 it = args.items[first + ri * G];
      tp = make_int2(it.x, it.y);
      cb = it.z & 0x7fff;
      ce = (it.z >> 15) & 0x7fff;
      slot = it.w;
    } else {
      tp = args.tiles[first + ri * G];
      cb = 0;
      ce = nch;
      slot = -1;
    }
  };
  int P = R * nch;
  if constexpr (SPLIT) {
    P = 0;
    for (int ri = 0; ri < R; ++ri) {
      int2 tp;
      int cb, ce, sl;
      item(ri, tp, cb, ce, sl);
      P += ce - cb;
    }
  }
  if (P <= 0) return;
  if (tid == 0) {
    for (int s = 0; s < kSymStages; ++s) {
      mbar_init(&full_bar[s], 1);
      done_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int ri, int ch, int s) {
    int2 tp;
    int cb_, ce_, sl_;
    item(ri, tp, cb_, ce_, sl_);
    const int r0 = tp.x * kTile, c0 = tp.y * kTile, k0 = ch * kSymBK;
    uint8_t* st = smem + s * kSymStageBytes;
    const int k1 = min(k0 + kSymBK, n);
    // triplet: a chunk wholly below the column (row) tile takes nu() on A (B)
    const CUtensorMap* ma = (TRI && k1 <= c0) ? &tm_dnu : &tm_d;
    const CUtensorMap* mb = (TRI && k1 <= r0) ? &tm_dnu : &tm_d;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // stage reads -> TMA refill
    mbar_expect_tx(&full_bar[s], kSymStageBytes);
    tma_load_2d(st, ma, r0, k0, &full_bar[s]);
    tma_load_2d(st + kSymBox, mb, c0, k0, &full_bar[s]);
    tma_load_2d(st + 2 * kSymBox, &tm_w, r0, k0, &full_bar[s]);
    tma_load_2d(st + 3 * kSymBox, &tm_w, c0, k0, &full_bar[s]);
  };
  constexpr bool ITEMS = SPLIT;  // items other than whole pairs
  int pr_ri = 0, pr_ch = 0, pr_end = nch;
  auto pr_load = [&]() {  // the next non-empty item at or after pr_ri
    for (; pr_ri < R; ++pr_ri) {
      int2 tp;
      int sl;
      item(pr_ri, tp, pr_ch, pr_end, sl);
      if (pr_ch < pr_end) break;
    }
  };
  if constexpr (ITEMS) pr_load();
  auto pr_advance = [&]() {
    if (++pr_ch == pr_end) {
      ++pr_ri;
      if constexpr (ITEMS) {
        pr_load();
      } else {
        pr_ch = 0;
      }
    }
  };
  for (int p = 0; p < kSymStages && p < P; ++p) {
    if (tid == 0) issue(pr_ri, pr_ch, p);
    pr_advance();
  }

  const int warp = tid >> 5, lane = tid & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);
  const int tx = (warp & 1) * 8 + (lane & 7);

  // Accurate mode: the thread's fp32 partial sums of both output tiles added
  // into the double sums with red.global.add.f64 (exact, order-independent,
  // no result to wait for). Measured alternatives at n = 32768 (pass 2, plain
  // kernel 2479 ms): these reductions 2637 ms; a plain vectorised load / add /
  // store (a whole pair owns its tiles) 2701 ms -- the loads' latency shows as
  // long-scoreboard stalls; sector-coalesced reductions after a 4 x 4 shuffle
  // transpose 2685 ms.
  auto add4 = [&](double* p4, float a, float b, float c, float d) { acc_red4(p4, a, b, c, d); };
  auto flush64 = [&](float2 (&acc)[8][4], float2 (&act)[8][4], int r0, int c0, bool diag) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + row_off<kTile>(ty, i);
      if (r >= n) continue;
      double* prow = args.c64 + (size_t)r * ld;
      const int ca = c0 + tx * 4, cb = c0 + 64 + tx * 4;
      if (ca < n) add4(prow + ca, acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
      if (cb < n) add4(prow + cb, acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y);
    }
    if (!diag) {  // the diagonal pair's direct tile holds every entry
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + row_off<kTile>(tx, j);
        if (c >= n) continue;
        double* prow = args.c64 + (size_t)c * ld;
        const int ra = r0 + ty * 4, rb = r0 + 64 + ty * 4;
        const int jp = j >> 1;
        const bool hi = (j & 1) != 0;
        if (ra < n)
          add4(prow + ra, hi ? act[0][jp].y : act[0][jp].x, hi ? act[1][jp].y : act[1][jp].x,
               hi ? act[2][jp].y : act[2][jp].x, hi ? act[3][jp].y : act[3][jp].x);
        if (rb < n)
          add4(prow + rb, hi ? act[4][jp].y : act[4][jp].x, hi ? act[5][jp].y : act[5][jp].x,
               hi ? act[6][jp].y : act[6][jp].x, hi ? act[7][jp].y : act[7][jp].x);
      }
    }
  };

  int p = 0;
  for (int ri = 0; ri < R; ++ri) {
    int2 tp;
    int ch_b, ch_e, slot;
    item(ri, tp, ch_b, ch_e, slot);
    if (SPLIT && ch_b >= ch_e) continue;  // queue padding
    const int r0 = tp.x * kTile, c0 = tp.y * kTile;
    const bool diag = tp.x == tp.y;
    const bool marks = !TRI || args.tri_marks;
    const uint32_t* mk = marks ? args.masks + pair_index(tp.x, tp.y, args.nb) * nch : nullptr;
    const bool all_marked = !marks || (__ldg(args.tile_flags + tp.x) | __ldg(args.tile_flags + tp.y)) != 0u;
    float2 thr[8][4], acc[8][4], act[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        float t2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + row_off<kTile>(ty, i), c = c0 + row_off<kTile>(tx, 2 * jp + h);
          const uint32_t tv = (r < n && c < n) ? __ldg(args.d + (size_t)r * ld + c) : 0u;
          t2[h] = __uint_as_float(tv) * -kCmpScale;
        }
        thr[i][jp] = make_float2(t2[0], t2[1]);
        acc[i][jp] = make_float2(0.f, 0.f);
        act[i][jp] = make_float2(0.f, 0.f);
      }
    }
    for (int ch = ch_b; ch < ch_e; ++ch, ++p) {
      const int s = p % kSymStages;
      mbar_wait(&full_bar[s], (p / kSymStages) & 1);
      const uint8_t* st = smem + s * kSymStageBytes;
      const float* sa = reinterpret_cast<const float*>(st);
      const float* sb = reinterpret_cast<const float*>(st + kSymBox);
      const float* sw = reinterpret_cast<const float*>(st + 2 * kSymBox);
      const float* sv = reinterpret_cast<const float*>(st + 3 * kSymBox);
      const int k0 = ch * kSymBK;
      const int kmax = min(kSymBK, n - k0);
      if constexpr (TRI) {
        const bool a_in = k0 >= c0 && k0 < c0 + kTile;
        const bool b_in = k0 >= r0 && k0 < r0 + kTile;
        if (!a_in && !b_in && kmax == kSymBK) {
#pragma unroll kSymUnroll
          for (int kk = 0; kk < kSymBK; ++kk) sym_step(sa, sb, sw, sv, kk, ty, tx, thr, acc, act);
        } else {
          // inside the row / column tile: per-element nu() only where a tie
          // is possible (marked k); without marks every k
          const uint32_t m = all_marked ? 0xffffffffu : __ldg(mk + ch);
          for (int kk = 0; kk < kmax; ++kk) {
            if ((m >> kk) & 1u)
              sym_step_tri_sel(sa, sb, sw, sv, kk, k0 + kk, ty, tx, r0, c0, a_in, b_in, thr, acc, act);
            else
              sym_step(sa, sb, sw, sv, kk, ty, tx, thr, acc, act);
          }
        }
      } else {
      const uint32_t m = all_marked ? 0xffffffffu : __ldg(mk + ch);
      if (m == 0u && kmax == kSymBK) {
#pragma unroll kSymUnroll
        for (int kk = 0; kk < kSymBK; ++kk) sym_step(sa, sb, sw, sv, kk, ty, tx, thr, acc, act);
      } else {
        for (int kk = 0; kk < kmax; ++kk) {
          if ((m >> kk) & 1u)
            sym_step_exact(sa, sb, sw, sv, kk, k0 + kk, ty, tx, r0, c0, thr, acc, act);
          else
            sym_step(sa, sb, sw, sv, kk, ty, tx, thr, acc, act);
        }
      }
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t old = stage_arrive(&done_cnt[s]);
        if (old == (uint32_t)(p / kSymStages + 1) * (kThreads / 32) - 1u && p + kSymStages < P)
          issue(pr_ri, pr_ch, s);
        pr_advance();
      }
      if constexpr (ACC && !SPLIT) {  // k block done (not the last: that is the flush below)
        if ((ch + 1) % args.acc_chunks == 0 && ch + 1 < ch_e) {
          flush64(acc, act, r0, c0, diag);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) {
              acc[i][jp] = make_float2(0.f, 0.f);
              act[i][jp] = make_float2(0.f, 0.f);
            }
        }
      }
    }
    if constexpr (ACC) {  // into the double sums (rounded by acc_round_*_kernel)
      flush64(acc, act, r0, c0, diag);
      continue;
    }
    if (SPLIT && !ACC && slot >= 0) {  // partial tiles: [0] rows of P x cols of Q, [1] rows of Q x cols of P
      float* pt = args.partial + (size_t)slot * 2 * kTile * kTile;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rl = row_off<kTile>(ty, i);
        if (TRI && diag) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (row_off<kTile>(tx, j) != rl) continue;
            if (j & 1)
              acc[i][j >> 1].y = 0.f;
            else
              acc[i][j >> 1].x = 0.f;
          }
        }
        *reinterpret_cast<float4*>(pt + rl * kTile + tx * 4) =
            make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
        *reinterpret_cast<float4*>(pt + rl * kTile + 64 + tx * 4) =
            make_float4(acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y);
      }
      if (!diag) {
        float* pq = pt + kTile * kTile;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int cl = row_off<kTile>(tx, j), jp = j >> 1;
          float v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = (j & 1) ? act[i][jp].y : act[i][jp].x;
          *reinterpret_cast<float4*>(pq + cl * kTile + ty * 4) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(pq + cl * kTile + 64 + ty * 4) = make_float4(v[4], v[5], v[6], v[7]);
        }
      }
      continue;
    }
    // ---- flush: C[r][c] (rows of P, columns of Q) ------------------------
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + row_off<kTile>(ty, i);
      if (r >= n) continue;
      if (TRI && diag) {  // the triplet leaves the diagonal of C at 0
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (c0 + row_off<kTile>(tx, j) != r) continue;
          if (j & 1)
            acc[i][j >> 1].y = 0.f;
          else
            acc[i][j >> 1].x = 0.f;
        }
      }
      const size_t rowo = (size_t)r * ld;
      const int ca = c0 + tx * 4, cb = c0 + 64 + tx * 4;
      if (ca < n)
        store_c4<PEERS>(args, rowo + ca, make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y));
      if (cb < n)
        store_c4<PEERS>(args, rowo + cb, make_float4(acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y));
    }
    // ---- C[c][r] (rows of Q, columns of P); the diagonal pair already
    // wrote every entry of its tile above.
    if (!diag) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + row_off<kTile>(tx, j);
        if (c >= n) continue;
        const size_t rowo = (size_t)c * ld;
        const int ra = r0 + ty * 4, rb = r0 + 64 + ty * 4;
        const int jp = j >> 1;
        if ((j & 1) == 0) {
          if (ra < n)
            store_c4<PEERS>(args, rowo + ra, make_float4(act[0][jp].x, act[1][jp].x, act[2][jp].x, act[3][jp].x));
          if (rb < n)
            store_c4<PEERS>(args, rowo + rb, make_float4(act[4][jp].x, act[5][jp].x, act[6][jp].x, act[7][jp].x));
        } else {
          if (ra < n)
            store_c4<PEERS>(args, rowo + ra, make_float4(act[0][jp].y, act[1][jp].y, act[2][jp].y, act[3][jp].y));
          if (rb < n)
            store_c4<PEERS>(args, rowo + rb, make_float4(act[4][jp].y, act[5][jp].y, act[6][jp].y, act[7][jp].y));
        }
      }
    }
    // Round barrier (cooperative launch): the CTAs of one round work on
    // pairs that share row and column panels chunk by chunk; starting every
    // full round together keeps them at the same k so that those panels
    // are read from DRAM once per round, not once per CTA.
    if (SYNC && ri + 1 < (args.tile_end - args.tile_begin) / G) {
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(args.round_bar, 1u);
        const unsigned int target = (unsigned int)(ri + 1) * (unsigned int)G;
        while (true) {
          unsigned int v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(args.round_bar) : "memory");
          if (v >= target) break;
          __nanosleep(200);
        }
      }
      __syncthreads();
    }
  }
}

// Sum of the split items' partial tiles, in slot order (deterministic), into
// C. One CTA per (split pair, tile half, 8 rows): pairs[q] = (tile row,
// tile col, first slot, parts).
__global__ void __launch_bounds__(256)
    sym_combine_kernel(const int4* __restrict__ pairs, const float* __restrict__ partial, float* __restrict__ c,
                       int n, int ld) {
  const int q = blockIdx.x, half = blockIdx.y;
  const int4 pr = pairs[q];
  if (half == 1 && pr.x == pr.y) return;  // diagonal pair: one tile
  const int rl = blockIdx.z * 8 + (threadIdx.x >> 5), cl = (threadIdx.x & 31) * 4;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int t = 0; t < pr.w; ++t) {
    const float4 v = *reinterpret_cast<const float4*>(partial + ((size_t)(pr.z + t) * 2 + half) * kTile * kTile +
                                                      rl * kTile + cl);
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  const int row = (half ? pr.y : pr.x) * kTile + rl, col = (half ? pr.x : pr.y) * kTile + cl;
  if (row >= n) return;
  float* dst = c + (size_t)row * ld + col;
  if (col + 3 < n) {
    *reinterpret_cast<float4*>(dst) = s;
  } else {
    if (col < n) dst[0] = s.x;
    if (col + 1 < n) dst[1] = s.y;
    if (col + 2 < n) dst[2] = s.z;
  }
}

}  // namespace pald_gpu
