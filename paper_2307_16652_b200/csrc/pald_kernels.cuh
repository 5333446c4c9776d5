// pald_kernels.cuh -- sm_100a kernels for the PaLD focus/cohesion hot path.
//
// Both O(n^3) passes are written as "semiring GEMMs" over the pair grid
// (hard part 2). With A = D[k][row-tile], B = D[k][col-tile]
// (D is symmetric, so both panels are row-major TMA boxes), per output
// (r, c) and third point k:
//
//   focus    (pass 1): U[r][c] = sum_k [ min(A'_rk, B'_kc) <  T'_rc ]
//   cohesion (pass 2): C[r][c] = sum_k W_rk * [ T_rc < min(A'_rk, B'_kc) ]
//
// where X' is either X or nu(X) = the next representable value above X
// (fp32 bits + 1), chosen per (k, r, c) so that each strict/non-strict
// comparison of the reference is reproduced exactly:
//
//   pairwise focus     (blocked.hpp:101-122): no transforms.
//   pairwise cohesion  (blocked.hpp:126-186, reference.hpp:121-129):
//                      output (x, z), k = partner y, A = d_xy, B = d_yz,
//                      B' = nu(B) iff y < x (the tie of pair (y, x) goes to
//                      its second point x: d_xz <= d_yz <=> d_xz < nu(d_yz)).
//   triplet focus      (reference.hpp:160-183, blocked.hpp:195-238): output
//                      (x, y), k = z, A' = nu(d_xz) iff z < y,
//                      B' = nu(d_yz) iff z < x, T' = nu(d_xy); the z = x and
//                      z = y terms supply the initial 2.
//   triplet cohesion   (reference.hpp:187-206, blocked.hpp:248-335): output
//                      (p, q), k = third point o, A = d_po, B = d_qo,
//                      A' = nu(A) iff o < q, B' = nu(B) iff o < p, W = 1/u_po;
//                      diagonal forced to 0.
//
// The derivations are restated and brute-force checked on CPU in
// tests/test_formulation.py. Summation in pass 2 runs over k ascending in
// fp32 in one register per output, which is exactly the order of the
// reference's fp32 pairwise C (blocked.hpp:384-411): bit-identical output.
//
// Compare instruction: when D's dynamic range allows (checked on the
// device), D is scaled by an exact power of two
// into [2^-102, 1) and [a < b] is computed on the FMA pipe as
// sat(fma(b, 2^125, -a*2^125)) in {0, 1} (exact: every nonzero |b - a| is
// >= 2^-125). Otherwise ("exact path") D is stored as integer keys
// 2*bits(d) (nu = key + 1) and compared with integer min/compare.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pald_gpu {

constexpr int kTile = 128;      // pair-tile edge (rows and columns)
#ifndef PALD_BK
#define PALD_BK 64
#endif
#ifndef PALD_KUNROLL  // unroll of the fast k loop (scheduling knob)
#define PALD_KUNROLL 2
#endif
constexpr int kKUnroll = PALD_KUNROLL;
#ifndef PALD_RANK_UNROLL  // unroll of the rank-coded k loop: the bare loop prefers 8
#define PALD_RANK_UNROLL 2  // (tools/microbench4.cu), the 255-register kernel 2-4 (8: -1.2 %)
#endif
constexpr int kRankUnroll = PALD_RANK_UNROLL;
#ifndef PALD_RANK_BUMP  // 1: the k loop bumps the two operand pointers instead of indexing by kk
#define PALD_RANK_BUMP 1  // n = 32768 pass 1: 1236 -> 1202 ms (unroll 4: 1218, 4 + bump: 1273;
#endif                    // profiles/rank_loop_variants_r02.txt)
#ifndef PALD_K_ORDER  // k-step instruction order: 0 rows outer, 1 column pairs outer
#define PALD_K_ORDER 0
#endif
#ifndef PALD_COH_ACC  // cohesion accumulate: 0 = packed FFMA2 (default), 1 = scalar FFMA
#define PALD_COH_ACC 0
#endif

constexpr int kBK = PALD_BK;    // third-point chunk per pipeline stage
constexpr int kThreads = 256;   // 8 warps, 16 x 16 threads (8 x 8 outputs each on 128-wide tiles)
__host__ __device__ constexpr int box_bytes(int tile) { return kBK * tile * 4; }
__host__ __device__ constexpr int stage_bytes(int pass, int tile, bool rank = false) {
  // rank-coded pass 1: a 4-byte RA box and a 2-byte RB box (pald_rank.cuh)
  return rank ? box_bytes(tile) + box_bytes(tile) / 2 : (pass == 0 ? 2 : 3) * box_bytes(tile);
}
// CTAs per SM: 1 for 128-wide tiles (8 x 8 outputs per thread, ~230
// registers), 2 for the 64-wide small-n tiles (4 x 4 per thread).
#ifndef PALD_RANK_CTAS  // CTAs per SM of the rank-coded pass 1 (A/B knob; 2 CTAs at 128
#define PALD_RANK_CTAS 1   // registers with 2 stages: 44.1 vs 48.5 combos/SM-cycle)
#endif
__host__ __device__ constexpr int ctas_per_sm(int tile, bool rank = false) {
  return rank ? PALD_RANK_CTAS : tile == 128 ? 1 : tile == 64 ? 2 : 4;
}
// Pipeline depth so that stages x stage_bytes fits the shared memory of
// ctas_per_sm CTAs (227 KB per SM).
#ifndef PALD_SMEM_BUDGET_KB
#define PALD_SMEM_BUDGET_KB 200
#endif
__host__ __device__ constexpr int stages_for(int pass, int tile, bool rank = false) {
  return stage_bytes(pass, tile, rank) * 4 <= PALD_SMEM_BUDGET_KB * 1024 / ctas_per_sm(tile, rank) ? 4
         : stage_bytes(pass, tile, rank) * 3 <= PALD_SMEM_BUDGET_KB * 1024 / ctas_per_sm(tile, rank) ? 3 : 2;
}
constexpr int kBoxBytes = kBK * kTile * 4;  // one TMA box of a 128-wide panel (32 KB)
constexpr float kCmpScale = 0x1p125f;       // S of the FFMA.SAT compare

__host__ __device__ constexpr int smem_bytes(int pass, int tile, bool rank = false) {
  return stages_for(pass, tile, rank) * stage_bytes(pass, tile, rank) + 1024;
}

// Multi-GPU exchange over peer memory: the same buffer (W or C) of every
// rank of one node, mapped into this process (CUDA IPC over NVLink; the
// calling rank's own buffer included).
constexpr int kMaxPeers = 8;
struct PeerBufs {
  float* ptr[kMaxPeers];
  int count;
};

struct KernelArgs {
  const uint32_t* d;     // layout of D (scaled fp32 bits or integer keys), n x ld
  int32_t* u;            // focus sizes
  float* w;              // 1/u
  float* c;              // cohesion
  int n;
  int ld;
  int nb;                // tiles per dimension
  int tile_row_begin;    // cohesion: first tile row of this launch
  int tile_row_end;
  long long total_tiles; // cohesion: tiles covered by this launch
  long long unit_begin;  // work units [unit_begin, unit_end), u = tile*nchunks + chunk, tile
  long long unit_end;    // index in the launch's tile order (focus: the whole upper triangle)
  const int2* focus_tiles;  // focus tile order: (tile row, tile col), grouped raster;
                            // pass 2: optional explicit tile list (else the raster)
  int group_rows;           // cohesion raster group height (tile rows)
  PeerBufs peers;           // PEERS kernels: pass-1 counts go to every rank's W
  double* c64;              // ACC kernels: double sums of the fp32 block partials (n x ld)
  int acc_chunks;           // ACC kernels: k chunks per fp32 block partial
  // rank-coded triplet pass 1: tie marks per (tile pair, 32-point chunk)
  // (pald_sym.cuh); chunks inside the tiles without a marked k run the fast
  // step (strict and non-strict tests agree without a tie). NULL: none.
  const uint32_t* tie_masks;
  const uint32_t* tie_tile_flags;
  int tie_nch;
};

constexpr int kGroupRows = 16;  // tile rows per raster group (L2 reuse of the panels)

// ---------------------------------------------------------------------------
// mbarrier / TMA primitives (PTX).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Stage release of the pipelines: each warp's lane 0 adds one arrival
// after __syncwarp (which orders the warp's shared-memory reads of the
// stage before it); the arrival that completes the count refills the stage
// with TMA. acq_rel: every warp's reads happen-before the refill issued by
// the last arriver, which then crosses to the async proxy
// (fence.proxy.async in issue()) for the write of the next TMA load.
__device__ __forceinline__ uint32_t stage_arrive(uint32_t* cnt) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
               : "=r"(old)
               : "r"(smem_u32(cnt))
               : "memory");
  return old;
}

// Accurate mode (PALD_GPU_FLAG_ACCURATE): the fp32 register sums of an
// output are flushed every `acc_chunks` k chunks (one k block) into a
// zeroed double buffer with red.global.add.f64 and restarted from 0. Adding
// a partial fp32 sum of positive terms 1/u (u in [2, 2^24]) to a double sum
// of such partials is exact (all values are multiples of 2^-38 below 2^14,
// 52 bits), so the result is the exact sum of the fp32 block partials --
// independent of the order of the additions, hence deterministic however
// the blocks are spread over CTAs -- and only the blocks' own fp32 rounding
// remains (<= acc_chunks * BK-term chains instead of one n-term chain). The
// reductions need no result (RED, no scoreboard wait); acc_round_*_kernel
// rounds the double sums to the fp32 C afterwards.
__device__ __forceinline__ void acc_red4(double* p, float a, float b, float c, float d) {
  atomicAdd(p, (double)a);
  atomicAdd(p + 1, (double)b);
  atomicAdd(p + 2, (double)c);
  atomicAdd(p + 3, (double)d);
}
__device__ __forceinline__ void acc_red2(double* p, float a, float b) {
  atomicAdd(p, (double)a);
  atomicAdd(p + 1, (double)b);
}

__device__ __forceinline__ uint32_t nu_bits(uint32_t v) { return v + 1u; }
__device__ __forceinline__ float nu_f(float v) { return __uint_as_float(__float_as_uint(v) + 1u); }

// ---------------------------------------------------------------------------
// Thread layout: 8 warps as a 4 x 2 grid of 4 x 8-thread warp tiles; thread
// (ty, tx) in 16 x 16 owns TT = TILE/16 rows {h*TILE/2 + ty*4 + i} and TT
// columns {h*TILE/2 + tx*4 + j} (h < TT/4, i, j < 4) of the TILE x TILE
// tile: 8 x 8 outputs for TILE 128, 4 x 4 for TILE 64 (small n). A-panel
// LDS.128 of a warp touch 4 distinct 16-byte words (broadcast), B-panel
// loads 8 consecutive words: one wavefront each.
template <int TILE>
__device__ __forceinline__ int row_off(int ty, int i) {
  if constexpr (TILE == 128) return i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
  if constexpr (TILE == 32) return ty * 2 + i;  // 2 x 2 outputs per thread (tail tiles)
  return (i >> 2) * (TILE / 2) + ty * 4 + (i & 3);
}

template <int TILE, int N>
__device__ __forceinline__ void lds_vec(const float* __restrict__ row, int t, float (&v)[N]) {
  if constexpr (N == 2) {
    const float2 q = reinterpret_cast<const float2*>(row)[t];
    v[0] = q.x;
    v[1] = q.y;
    return;
  }
#pragma unroll
  for (int h = 0; h < N / 4; ++h) {
    const float4 q = reinterpret_cast<const float4*>(row)[h * (TILE / 8) + t];
    v[4 * h + 0] = q.x;
    v[4 * h + 1] = q.y;
    v[4 * h + 2] = q.z;
    v[4 * h + 3] = q.w;
  }
}

// One k step of the uniform (no per-element transform) fast path.
template <int PASS, bool FAST, int TILE, int TT = TILE / 16>
__device__ __forceinline__ void k_step(const float* __restrict__ sa, const float* __restrict__ sb,
                                       const float* __restrict__ sw, int kk, int ty, int tx,
                                       const float2 (&thr)[TT][TT / 2], float2 (&acc)[TT][TT / 2]) {
  float a[TT], b[TT], w[TT];
  if constexpr (TILE == 128) {
    const float4 a0 = reinterpret_cast<const float4*>(sa + kk * TILE)[ty];
    const float4 a1 = reinterpret_cast<const float4*>(sa + kk * TILE)[16 + ty];
    const float4 b0 = reinterpret_cast<const float4*>(sb + kk * TILE)[tx];
    const float4 b1 = reinterpret_cast<const float4*>(sb + kk * TILE)[16 + tx];
    a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
    a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
    b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
    b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
    if (PASS == 1) {
      const float4 w0 = reinterpret_cast<const float4*>(sw + kk * TILE)[ty];
      const float4 w1 = reinterpret_cast<const float4*>(sw + kk * TILE)[16 + ty];
      w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
      w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
    }
  } else {
    lds_vec<TILE>(sa + kk * TILE, ty, a);
    lds_vec<TILE>(sb + kk * TILE, tx, b);
    if (PASS == 1) lds_vec<TILE>(sw + kk * TILE, ty, w);
  }
#if PALD_K_ORDER == 1
#pragma unroll
  for (int jp = 0; jp < TT / 2; ++jp) {
#pragma unroll
    for (int i = 0; i < TT; ++i) {
#else
#pragma unroll
  for (int i = 0; i < TT; ++i) {
#pragma unroll
    for (int jp = 0; jp < TT / 2; ++jp) {
#endif
      if (FAST) {
        const float m0 = fminf(a[i], b[2 * jp]);
        const float m1 = fminf(a[i], b[2 * jp + 1]);
        if (PASS == 0) {
          const float k0f = __saturatef(__fmaf_rn(m0, -kCmpScale, thr[i][jp].x));
          const float k1f = __saturatef(__fmaf_rn(m1, -kCmpScale, thr[i][jp].y));
          acc[i][jp] = __fadd2_rn(acc[i][jp], make_float2(k0f, k1f));
        } else {
          const float k0f = __saturatef(__fmaf_rn(m0, kCmpScale, thr[i][jp].x));
          const float k1f = __saturatef(__fmaf_rn(m1, kCmpScale, thr[i][jp].y));
#if PALD_COH_ACC == 1
          acc[i][jp].x = __fmaf_rn(k0f, w[i], acc[i][jp].x);
          acc[i][jp].y = __fmaf_rn(k1f, w[i], acc[i][jp].y);
#else
          acc[i][jp] = __ffma2_rn(make_float2(k0f, k1f), make_float2(w[i], w[i]), acc[i][jp]);
#endif
        }
      } else {
        const uint32_t ai = __float_as_uint(a[i]);
        const uint32_t m0 = min(ai, __float_as_uint(b[2 * jp]));
        const uint32_t m1 = min(ai, __float_as_uint(b[2 * jp + 1]));
        const uint32_t t0 = __float_as_uint(thr[i][jp].x), t1 = __float_as_uint(thr[i][jp].y);
        if (PASS == 0) {
          acc[i][jp].x += (m0 < t0) ? 1.f : 0.f;
          acc[i][jp].y += (m1 < t1) ? 1.f : 0.f;
        } else {
          // fma(k, w, acc) as on the fast path: exact for finite w, and
          // 0 * inf = NaN like the reference's masked update when u = 0
          const float2 k2 = make_float2((t0 < m0) ? 1.f : 0.f, (t1 < m1) ? 1.f : 0.f);
          acc[i][jp] = __ffma2_rn(k2, make_float2(w[i], w[i]), acc[i][jp]);
        }
      }
    }
  }
}

// One k step with per-element transforms (chunks that cross the row or
// column tile, and the ragged last chunk).
template <int PASS, bool FAST, int TILE, int TT = TILE / 16>
__device__ __forceinline__ void k_step_sel(const float* __restrict__ sa, const float* __restrict__ sb,
                                           const float* __restrict__ sw, int kk, int kg, int ty,
                                           int tx, int r0, int c0, bool a_in, bool b_in,
                                           const float2 (&thr)[TT][TT / 2], float2 (&acc)[TT][TT / 2]) {
  float a[TT], b[TT], w[TT];
  if constexpr (TILE == 128) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = sa[kk * TILE + row_off<TILE>(ty, i)];
      if (PASS == 1) w[i] = sw[kk * TILE + row_off<TILE>(ty, i)];
      b[i] = sb[kk * TILE + row_off<TILE>(tx, i)];
    }
  } else {
    lds_vec<TILE>(sa + kk * TILE, ty, a);
    lds_vec<TILE>(sb + kk * TILE, tx, b);
    if (PASS == 1) lds_vec<TILE>(sw + kk * TILE, ty, w);
  }
#pragma unroll
  for (int i = 0; i < TT; ++i) {
#pragma unroll
    for (int jp = 0; jp < TT / 2; ++jp) {
      float kv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jp + h;
        const bool nua = a_in && (kg < c0 + row_off<TILE>(tx, j));
        const bool nub = b_in && (kg < r0 + row_off<TILE>(ty, i));
        const uint32_t av = nua ? nu_bits(__float_as_uint(a[i])) : __float_as_uint(a[i]);
        const uint32_t bv = nub ? nu_bits(__float_as_uint(b[j])) : __float_as_uint(b[j]);
        const float t = (h == 0) ? thr[i][jp].x : thr[i][jp].y;
        if (FAST) {
          const float m = fminf(__uint_as_float(av), __uint_as_float(bv));
          kv[h] = (PASS == 0) ? __saturatef(__fmaf_rn(m, -kCmpScale, t))
                              : __saturatef(__fmaf_rn(m, kCmpScale, t));
        } else {
          const uint32_t m = min(av, bv), tu = __float_as_uint(t);
          kv[h] = (PASS == 0) ? ((m < tu) ? 1.f : 0.f) : ((tu < m) ? 1.f : 0.f);
        }
      }
      if (PASS == 0) {
        acc[i][jp] = __fadd2_rn(acc[i][jp], make_float2(kv[0], kv[1]));
      } else {
        acc[i][jp] = __ffma2_rn(make_float2(kv[0], kv[1]), make_float2(w[i], w[i]), acc[i][jp]);
      }
    }
  }
}

// One k step of the InclusiveSplit cohesion pass (pairwise, blocked.hpp:
// 150-158). With A' = nu(d_xy) (the A panel comes from nu(D)), B = d_yz and
// T = d_xz, the reference's r*sx*w (r = [min(d_xz,d_yz) <= d_xy],
// sx = [d_xz < d_yz] + 0.5 [d_xz == d_yz]) equals, for either order of the
// pair, (w/2) * ([T < min(A', B)] + [T < min(A', nu(B))]); the sum of the
// two indicators (0, 1, 2) times w/2 is one exact product, so each pair still
// adds a single correctly rounded term, in ascending y.
template <bool FAST, int TILE, int TT = TILE / 16>
__device__ __forceinline__ void k_step_split(const float* __restrict__ sa, const float* __restrict__ sb,
                                             const float* __restrict__ sw, int kk, int ty, int tx,
                                             const float2 (&thr)[TT][TT / 2], float2 (&acc)[TT][TT / 2]) {
  float a[TT], b[TT], bn[TT], wh[TT];
  lds_vec<TILE>(sa + kk * TILE, ty, a);
  lds_vec<TILE>(sb + kk * TILE, tx, b);
  lds_vec<TILE>(sw + kk * TILE, ty, wh);
#pragma unroll
  for (int i = 0; i < TT; ++i) {
    wh[i] *= 0.5f;
    bn[i] = nu_f(b[i]);
  }
#pragma unroll
  for (int i = 0; i < TT; ++i) {
#pragma unroll
    for (int jp = 0; jp < TT / 2; ++jp) {
      float k1[2], k2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * jp + h;
        const float t = (h == 0) ? thr[i][jp].x : thr[i][jp].y;
        if (FAST) {
          k1[h] = __saturatef(__fmaf_rn(fminf(a[i], b[j]), kCmpScale, t));
          k2[h] = __saturatef(__fmaf_rn(fminf(a[i], bn[j]), kCmpScale, t));
        } else {
          const uint32_t ai = __float_as_uint(a[i]), tu = __float_as_uint(t);
          k1[h] = (tu < min(ai, __float_as_uint(b[j]))) ? 1.f : 0.f;
          k2[h] = (tu < min(ai, __float_as_uint(bn[j]))) ? 1.f : 0.f;
        }
      }
      const float2 kk2 = __fadd2_rn(make_float2(k1[0], k1[1]), make_float2(k2[0], k2[1]));
      acc[i][jp] = __ffma2_rn(kk2, make_float2(wh[i], wh[i]), acc[i][jp]);
    }
  }
}

// One k step of the rank-coded pairwise focus pass (pald_rank.cuh). Per
// output (r, c) the focus test [d_rk < d_rc] | [d_ck < d_rc] becomes
// [Rk[r][k] < RR] | [Rk[c][k] < CR] with RR = Rk[r][c], CR = Rk[c][r]
// (+1 each for InclusiveSplit's <=). Two columns share one 32-bit word in
// 16-bit lanes: X = (0x8000 | code) - threshold never borrows across lanes
// and its bit 15 is [code >= threshold], so
//   F = ~(X1 & X2) & 0x80008000   (focus flags of both columns)
//   acc += F >> 15                (LEA.HI: the two counts in the two halves)
// = 4 integer instructions per 2 output combos (vs 5 on the fp32 path).
// thr[i][jp] holds -RR (.x) and -CR (.y) packed per column pair, acc .x the
// packed counts.
// (pa, pb: the thread's first A / B words of the chunk, i.e. the stage's
// RA rows + ty and RB rows + tx: the k loop then only adds constants to two
// pointers -- the stage base is not a uniform value in the stream-K kernel)
template <int TT = 8>
__device__ __forceinline__ void k_step_rank(const uint4* __restrict__ pa, const uint2* __restrict__ pb,
                                            int kk, const float2 (&thr)[TT][TT / 2],
                                            float2 (&acc)[TT][TT / 2]) {
  const uint4 a0 = pa[kk * (kTile / 4)];
  const uint4 a1 = pa[kk * (kTile / 4) + 16];
  const uint2 b0 = pb[kk * (kTile / 4)];
  const uint2 b1 = pb[kk * (kTile / 4) + 16];
  const uint32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  const uint32_t b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      const uint32_t x1 = a[i] + __float_as_uint(thr[i][jp].x);
      const uint32_t x2 = b[jp] + __float_as_uint(thr[i][jp].y);
      const uint32_t f = ~(x1 & x2) & 0x80008000u;
      // hi32(f * 2^17) + acc = (f >> 15) + acc: ptxas emits one LEA.HI (a plain
      // shift + add compiles to SHF + IADD3, tools/microbench4.cu)
      uint32_t sum;
      asm("mad.hi.u32 %0, %1, 0x20000, %2;" : "=r"(sum) : "r"(f), "r"(__float_as_uint(acc[i][jp].x)));
      acc[i][jp].x = __uint_as_float(sum);
    }
  }
}

// Rank-coded k step with per-element strictness (triplet focus, chunks
// inside the row or column tile): output (r, c), third point z = kg. With
// T' = nu(d_rc), [nu(A) < T'] = [A < T] (strict) and [A < T'] = [A <= T], so
// the A test is strict iff z < c (A' = nu(A)) and <= otherwise; the B test
// strict iff z < r (reference.hpp:171-180). thr holds the strict thresholds
// for the per-element side(s); a <= test subtracts one more from its lane.
template <int TT = 8>
__device__ __forceinline__ void k_step_rank_sel(const uint32_t* __restrict__ sa, const uint16_t* __restrict__ sb,
                                                int kk, int kg, int ty, int tx, int r0, int c0, bool a_in, bool b_in,
                                                const float2 (&thr)[TT][TT / 2], float2 (&acc)[TT][TT / 2]) {
  const uint4 a0 = reinterpret_cast<const uint4*>(sa + kk * kTile)[ty];
  const uint4 a1 = reinterpret_cast<const uint4*>(sa + kk * kTile)[16 + ty];
  const uint2 b0 = reinterpret_cast<const uint2*>(sb + kk * kTile)[tx];
  const uint2 b1 = reinterpret_cast<const uint2*>(sb + kk * kTile)[16 + tx];
  const uint32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  const uint32_t b[4] = {b0.x, b0.y, b1.x, b1.y};
  uint32_t ma[4], mb[8];
#pragma unroll
  for (int jp = 0; jp < 4; ++jp)
    ma[jp] = a_in ? ((kg >= c0 + row_off<kTile>(tx, 2 * jp) ? 1u : 0u) |
                     (kg >= c0 + row_off<kTile>(tx, 2 * jp + 1) ? 0x10000u : 0u))
                  : 0u;
#pragma unroll
  for (int i = 0; i < 8; ++i) mb[i] = (b_in && kg >= r0 + row_off<kTile>(ty, i)) ? 0x10001u : 0u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      const uint32_t x1 = a[i] + __float_as_uint(thr[i][jp].x) - ma[jp];
      const uint32_t x2 = b[jp] + __float_as_uint(thr[i][jp].y) - mb[i];
      const uint32_t f = ~(x1 & x2) & 0x80008000u;
      uint32_t sum;
      asm("mad.hi.u32 %0, %1, 0x20000, %2;" : "=r"(sum) : "r"(f), "r"(__float_as_uint(acc[i][jp].x)));
      acc[i][jp].x = __uint_as_float(sum);
    }
  }
}

// Focus-finish tile index -> (tile row, tile col): upper-triangular tiles in
// row-major order.
__device__ __forceinline__ void tri_coords(int t, int nb, int& tr, int& tc) {
  const double bb = 2.0 * nb + 1.0;
  int r = (int)((bb - sqrt(bb * bb - 8.0 * (double)t)) * 0.5);
  r = max(0, min(r, nb - 1));
  auto S = [&](int rr) { return rr * nb - rr * (rr - 1) / 2; };
  while (r > 0 && S(r) > t) --r;
  while (r + 1 < nb && S(r + 1) <= t) ++r;
  tr = r;
  tc = r + (t - S(r));
}

// Launch tile index -> (tile row, tile col).
//   focus:    the plan's grouped upper-triangular order (args.focus_tiles);
//   cohesion: grouped raster over tile rows [tile_row_begin, tile_row_end) x
//             all tile columns: groups of kGroupRows rows, column-major inside
//             a group, so the ~148 concurrently resident tiles share a few
//             row panels and column panels in L2.
template <int PASS, bool LIST = false>
__device__ __forceinline__ void tile_coords(const KernelArgs& a, int t, int& tr, int& tc) {
  if (PASS == 0 || LIST) {  // pass 1 order, or an explicit pass-2 tile list
    const int2 v = a.focus_tiles[t];
    tr = v.x;
    tc = v.y;
  } else {
    const int nrows = a.tile_row_end - a.tile_row_begin, gr = a.group_rows;
    const int grp = t / (gr * a.nb);
    const int rows_in = min(gr, nrows - grp * gr);
    const int local = t - grp * gr * a.nb;
    tc = local / rows_in;
    tr = a.tile_row_begin + grp * gr + (local - tc * rows_in);
  }
}

// Work split of a launch over its G CTAs (hybrid data-parallel + stream-K):
// whole tiles in rounds of G (CTA g takes tiles t_a + j*G + g), then the
// remainder -- the partial head tile, the leftover tiles and the partial
// tail tile -- split into equal contiguous unit shares (focus) or one whole
// leftover tile per CTA (cohesion, whose tiles are never split).
struct WorkSplit {
  int C;          // chunks per tile
  int t_a;        // first whole tile
  int full;       // rounds of whole tiles
  int head_len;   // remainder part 1: units [ub, ub + head_len)
  long long ub;
  long long mid;  // remainder part 2 starts at unit `mid`
  int rs, re;     // this CTA's remainder share [rs, re)
  __device__ __forceinline__ long long rem_unit(int q) const {
    return q < head_len ? ub + q : mid + (q - head_len);
  }
  __device__ __forceinline__ long long unit_of(int p, int g, int G) const {
    if (p < full * C) {
      const int j = p / C;
      return (long long)(t_a + j * G + g) * C + (p - j * C);
    }
    return rem_unit(rs + (p - full * C));
  }
};

template <int PASS>
__device__ __forceinline__ WorkSplit make_split(const KernelArgs& a, int C, int g, int G) {
  WorkSplit w;
  w.C = C;
  w.ub = a.unit_begin;
  const long long ue = a.unit_end;
  long long ta = (w.ub + C - 1) / C, tb = ue / C;
  if (ta > tb) {  // the range lies inside one tile
    ta = tb = w.ub / C;
    w.t_a = (int)ta;
    w.full = 0;
    w.head_len = (int)(ue - w.ub);
    w.mid = ue;
  } else {
    w.t_a = (int)ta;
    const int M = (int)(tb - ta);
    w.full = M / G;
    w.head_len = (int)(ta * C - w.ub);
    w.mid = (ta + (long long)w.full * G) * C;
  }
  const int rem = w.head_len + (int)(ue - w.mid);
  if (PASS == 0) {
    w.rs = (int)((long long)rem * g / G);
    w.re = (int)((long long)rem * (g + 1) / G);
  } else {  // whole leftover tiles, one per CTA
    const int left = rem / C;
    w.rs = g < left ? g * C : 0;
    w.re = g < left ? (g + 1) * C : 0;
  }
  return w;
}

// ---------------------------------------------------------------------------
// The persistent tile kernel. Each CTA (one per SM) owns a contiguous range
// of work units u = tile * nchunks + chunk:
//   focus    (PASS 0): an equal share of the launch's unit range
//            ("stream-K"); partial tiles are combined exactly with
//            red.global.add.f32 of integer counts (< 2^24) into the count
//            buffer (W), converted to U and W = 1/U by focus_finish_kernel.
//            Ranks of a multi-GPU run take equal unit ranges and SUM the
//            count buffers before the finish;
//   cohesion (PASS 1): whole tiles only, so every C entry is one in-order
//            fp32 sum (bit-identical to the reference).
// TMA streams 64-row chunks of the A/B(/W) panels through a 2-4 stage
// mbarrier pipeline that runs across tile boundaries. A stage is refilled by
// the last warp to finish with it (shared-memory arrival counter), so no
// block-wide barrier sits in the main loop.
template <int PASS, bool A_NU, bool B_NU, bool T_NU, bool ZERO_DIAG, bool FAST, bool SPLIT = false,
          int TILE = kTile, bool LIST = false, bool PEERS = false, bool RANK = false, bool ACC = false>
__global__ void __launch_bounds__(kThreads, ctas_per_sm(TILE, RANK))
    pald_tile_kernel(const __grid_constant__ CUtensorMap tm_d,
                     const __grid_constant__ CUtensorMap tm_dnu,
                     const __grid_constant__ CUtensorMap tm_w, const KernelArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Align the pipeline buffers to 1 KB with an offset into the same array,
  // so the compiler keeps the shared address space (LDS, not generic LD).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  static_assert(!RANK || (PASS == 0 && TILE == kTile), "rank codes: 128-wide pass 1 only");
  static_assert(!ACC || PASS == 1, "accurate mode: cohesion pass only");
  constexpr int kStages = stages_for(PASS, TILE, RANK);
  constexpr int TT = TILE / 16;  // outputs per thread per dimension
  constexpr int BOX = box_bytes(TILE);
  __shared__ uint64_t full_bar[kStages];
  __shared__ uint32_t done_cnt[kStages];

  const int tid = threadIdx.x;
  const int n = args.n, ld = args.ld, nb = args.nb;
  const int nchunks = (n + kBK - 1) / kBK;
  const int G = gridDim.x, g = blockIdx.x;
  const WorkSplit ws = make_split<PASS>(args, nchunks, g, G);
  const int P = ws.full * nchunks + (ws.re - ws.rs);
  if (P <= 0) return;

  // Run table: run ri < full is whole tile t_a + ri*G + g; the (at most
  // kMaxRem) remainder runs are built once by thread 0.
  constexpr int kMaxRem = 6;
  __shared__ int s_rem[kMaxRem][3];
  __shared__ int s_nrem;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      done_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int nr = 0;
    for (int q = ws.rs; q < ws.re && nr < kMaxRem;) {
      const long long u = ws.rem_unit(q);
      const int t = (int)(u / nchunks), ch = (int)(u - (long long)t * nchunks);
      int len = min(nchunks - ch, ws.re - q);
      if (q < ws.head_len) len = min(len, ws.head_len - q);
      s_rem[nr][0] = t;
      s_rem[nr][1] = ch;
      s_rem[nr][2] = ch + len;
      ++nr;
      q += len;
    }
    s_nrem = nr;
  }
  __syncthreads();
  // ACC (whole cohesion tiles): each tile is walked as nsub consecutive
  // runs of acc_chunks chunks (k blocks), flushed to the double sums in order
  const int nsub = ACC ? (nchunks + args.acc_chunks - 1) / args.acc_chunks : 1;
  const int R = (ws.full + s_nrem) * nsub;
  auto run_t = [&](int ri) {
    if constexpr (ACC) ri /= nsub;
    return ri < ws.full ? ws.t_a + ri * G + g : s_rem[ri - ws.full][0];
  };
  auto run_c0 = [&](int ri) {
    if constexpr (ACC) return (ri % nsub) * args.acc_chunks;
    return ri < ws.full ? 0 : s_rem[ri - ws.full][1];
  };
  auto run_c1 = [&](int ri) {
    if constexpr (ACC) return min(nchunks, (ri % nsub + 1) * args.acc_chunks);
    return ri < ws.full ? nchunks : s_rem[ri - ws.full][2];
  };

  constexpr int SB = stage_bytes(PASS, TILE, RANK);
  auto issue = [&](int t, int ch, int s) {
    int tr, tc;
    tile_coords<PASS, LIST>(args, t, tr, tc);
    const int r0 = tr * TILE, c0 = tc * TILE;
    const int k0 = ch * kBK, k1 = min(k0 + kBK, n);
    // Uniform per-chunk transform choice: the whole chunk lies below the
    // column (A) / row (B) tile => every element takes nu().
    const CUtensorMap* ma = ((PASS == 1 && SPLIT) || (A_NU && k1 <= c0)) ? &tm_dnu : &tm_d;
    const CUtensorMap* mb = (B_NU && k1 <= r0) ? &tm_dnu : &tm_d;
    uint8_t* st = smem + s * SB;
    // generic-proxy reads of the stage (ordered before this point by the
    // acq_rel arrivals) -> async-proxy write of the refill
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&full_bar[s], SB);
    if (RANK) {  // tm_d: RA (uint32 codes, rows R), tm_dnu: RB (uint16 codes, columns Q)
      tma_load_2d(st, &tm_d, r0, k0, &full_bar[s]);
      tma_load_2d(st + BOX, &tm_dnu, c0, k0, &full_bar[s]);
      return;
    }
    tma_load_2d(st, ma, r0, k0, &full_bar[s]);
    tma_load_2d(st + BOX, mb, c0, k0, &full_bar[s]);
    if (PASS == 1) tma_load_2d(st + 2 * BOX, &tm_w, r0, k0, &full_bar[s]);
  };
  // Producer iterator (run index, chunk) of unit p + kStages, kept by every
  // warp's lane 0 so that whichever warp releases a stage can refill it.
  int pr_ri = 0, pr_ch = R > 0 ? run_c0(0) : 0;
  auto pr_advance = [&]() {
    if (++pr_ch >= run_c1(pr_ri)) {
      ++pr_ri;
      if (pr_ri < R) pr_ch = run_c0(pr_ri);
    }
  };
  for (int p = 0; p < kStages && p < P; ++p) {
    if (tid == 0) issue(run_t(pr_ri), pr_ch, p);
    pr_advance();
  }

  const int warp = tid >> 5, lane = tid & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);  // 0..15
  const int tx = (warp & 1) * 8 + (lane & 7);    // 0..15

  int p = 0;
  for (int ri = 0; ri < R; ++ri) {
    const int t = run_t(ri), ch_begin = run_c0(ri), ch_end = run_c1(ri);
    int tr, tc;
    tile_coords<PASS, LIST>(args, t, tr, tc);
    const int r0 = tr * TILE, c0 = tc * TILE;
    float2 thr[TT][TT / 2];
    float2 acc[TT][TT / 2];
#pragma unroll
    for (int i = 0; i < TT; ++i) {
#pragma unroll
      for (int jp = 0; jp < TT / 2; ++jp) {
        uint32_t t2[2];
        if constexpr (RANK) {  // args.d = RA: Rk[r][c] = RA[c][r] & 0x7fff
          // pairwise: T_NU (InclusiveSplit) tests <= everywhere; triplet
          // (A_NU, B_NU): strict base thresholds, <= chosen per chunk below
          constexpr uint32_t plus = (T_NU && !A_NU) ? 1u : 0u;
          uint32_t rr = 0, cr = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = r0 + row_off<TILE>(ty, i), c = c0 + row_off<TILE>(tx, 2 * jp + h);
            if (r < n && c < n) {
              const uint32_t t_rc = (__ldg(args.d + (size_t)c * ld + r) & 0x7fffu) + plus;
              const uint32_t t_cr = (__ldg(args.d + (size_t)r * ld + c) & 0x7fffu) + plus;
              rr |= t_rc << (16 * h);
              cr |= t_cr << (16 * h);
            }
          }
          thr[i][jp] = make_float2(__uint_as_float(0u - rr), __uint_as_float(0u - cr));
          acc[i][jp] = make_float2(0.f, 0.f);
          continue;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + row_off<TILE>(ty, i), c = c0 + row_off<TILE>(tx, 2 * jp + h);
          uint32_t tv = (r < n && c < n) ? __ldg(args.d + (size_t)r * ld + c) : 0u;
          if (T_NU) tv = nu_bits(tv);
          t2[h] = tv;
        }
        if (FAST) {
          const float sc = (PASS == 0) ? kCmpScale : -kCmpScale;
          thr[i][jp] = make_float2(__uint_as_float(t2[0]) * sc, __uint_as_float(t2[1]) * sc);
        } else {
          thr[i][jp] = make_float2(__uint_as_float(t2[0]), __uint_as_float(t2[1]));
        }
        acc[i][jp] = make_float2(0.f, 0.f);
      }
    }

    int le_a = 0, le_b = 0;  // rank-coded triplet: thresholds currently shifted for <=
    for (int ch = ch_begin; ch < ch_end; ++ch, ++p) {
      const int s = p % kStages;
      mbar_wait(&full_bar[s], (p / kStages) & 1);
      const uint8_t* st = smem + s * SB;
      const float* sa = reinterpret_cast<const float*>(st);
      const float* sb = reinterpret_cast<const float*>(st + BOX);
      const float* sw = reinterpret_cast<const float*>(st + 2 * BOX);
      const int k0 = ch * kBK;
      // the chunk overlaps the column (row) tile: per-element transforms
      // (TILE >= kBK: the chunk lies inside the tile; 32-wide tail tiles sit
      // inside a 64-point chunk)
      const bool a_in = A_NU && (k0 < c0 + TILE) && (k0 + kBK > c0);
      const bool b_in = B_NU && (k0 < r0 + TILE) && (k0 + kBK > r0);
      const int kmax = min(kBK, n - k0);
      if constexpr (RANK) {
        const uint32_t* ra = reinterpret_cast<const uint32_t*>(st);
        const uint16_t* rb = reinterpret_cast<const uint16_t*>(st + BOX);
        if constexpr (A_NU) {  // triplet: strictness by the chunk's place (see k_step_rank_sel)
          const int k1 = k0 + kBK;
          const int want_a = (!a_in && k1 > c0) ? 1 : 0, want_b = (!b_in && k1 > r0) ? 1 : 0;
          if (want_a != le_a || want_b != le_b) {
            const uint32_t da = (uint32_t)(le_a - want_a) * 0x10001u, db = (uint32_t)(le_b - want_b) * 0x10001u;
#pragma unroll
            for (int i = 0; i < TT; ++i)
#pragma unroll
              for (int jp = 0; jp < TT / 2; ++jp)
                thr[i][jp] = make_float2(__uint_as_float(__float_as_uint(thr[i][jp].x) + da),
                                         __uint_as_float(__float_as_uint(thr[i][jp].y) + db));
            le_a = want_a;
            le_b = want_b;
          }
        }
        bool sel = a_in || b_in;
        if (sel && args.tie_masks) {  // triplet: no marked k in the chunk -> the fast step is exact
          static_assert(kBK == 64, "two 32-point mask words per chunk");
          const size_t pi = ((size_t)tr * (2 * nb - tr + 1) / 2 + (tc - tr)) * args.tie_nch + k0 / 32;
          const uint32_t flagged = __ldg(args.tie_tile_flags + tr) | __ldg(args.tie_tile_flags + tc);
          const uint32_t m = __ldg(args.tie_masks + pi) | (k0 / 32 + 1 < args.tie_nch ? __ldg(args.tie_masks + pi + 1) : 0u);
          sel = flagged || m;
        }
        if (sel) {
          for (int kk = 0; kk < kmax; ++kk) k_step_rank_sel(ra, rb, kk, k0 + kk, ty, tx, r0, c0, a_in, b_in, thr, acc);
        } else {
          const uint4* pa = reinterpret_cast<const uint4*>(ra) + ty;
          const uint2* pb = reinterpret_cast<const uint2*>(rb) + tx;
          if (kmax == kBK) {
#if PALD_RANK_BUMP
#pragma unroll 1
            for (int it = 0; it < kBK / kRankUnroll; ++it) {
#pragma unroll
              for (int u = 0; u < kRankUnroll; ++u) k_step_rank(pa, pb, u, thr, acc);
              pa += kRankUnroll * (kTile / 4);
              pb += kRankUnroll * (kTile / 4);
            }
#else
#pragma unroll kRankUnroll
            for (int kk = 0; kk < kBK; ++kk) k_step_rank(pa, pb, kk, thr, acc);
#endif
          } else {
            for (int kk = 0; kk < kmax; ++kk) k_step_rank(pa, pb, kk, thr, acc);
          }
        }
      } else if (PASS == 1 && SPLIT) {
        for (int kk = 0; kk < kmax; ++kk) k_step_split<FAST, TILE>(sa, sb, sw, kk, ty, tx, thr, acc);
      } else if (!a_in && !b_in && kmax == kBK) {
#pragma unroll kKUnroll
        for (int kk = 0; kk < kBK; ++kk) k_step<PASS, FAST, TILE>(sa, sb, sw, kk, ty, tx, thr, acc);
      } else {
        for (int kk = 0; kk < kmax; ++kk)
          k_step_sel<PASS, FAST, TILE>(sa, sb, sw, kk, k0 + kk, ty, tx, r0, c0, a_in, b_in, thr, acc);
      }
      // Release the stage: the last warp to arrive refills it.
      __syncwarp();
      if (lane == 0) {
        const uint32_t old = stage_arrive(&done_cnt[s]);
        if (old == (uint32_t)(p / kStages + 1) * (kThreads / 32) - 1u && p + kStages < P)
          issue(run_t(pr_ri), pr_ch, s);
        pr_advance();
      }
    }

    // ---- flush ------------------------------------------------------------
    if (PASS == 0) {
#pragma unroll
      for (int i = 0; i < TT; ++i) {
        const int r = r0 + row_off<TILE>(ty, i);
        if (r >= n) continue;
#pragma unroll
        for (int j = 0; j < TT; ++j) {
          const int c = c0 + row_off<TILE>(tx, j);
          float v;
          if constexpr (RANK) {
            const uint32_t packed = __float_as_uint(acc[i][j >> 1].x);
            v = (float)((j & 1) ? (packed >> 16) : (packed & 0xffffu));
          } else {
            v = (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
          }
          if constexpr (PEERS) {  // fused exchange: the partial count to every rank
            if (c < n && v != 0.f)
              for (int q = 0; q < args.peers.count; ++q)
                atomicAdd(args.peers.ptr[q] + (size_t)r * ld + c, v);
          } else {
            if (c < n) atomicAdd(args.w + (size_t)r * ld + c, v);  // RED.ADD.F32, exact
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < TT; ++i) {
        const int r = r0 + row_off<TILE>(ty, i);
        if (r >= n) continue;
        float v[TT];
#pragma unroll
        for (int jp = 0; jp < TT / 2; ++jp) {
          v[2 * jp] = acc[i][jp].x;
          v[2 * jp + 1] = acc[i][jp].y;
        }
        if constexpr (ACC) {  // k block done: into the double sums (rounded by acc_round_rows_kernel)
          double* prow = args.c64 + (size_t)r * ld;
          if constexpr (TILE == 32) {
            const int cc = c0 + tx * 2;
            if (cc < n) acc_red2(prow + cc, v[0], v[1]);
          } else {
#pragma unroll
            for (int h = 0; h < TT / 4; ++h) {
              const int cc = c0 + h * (TILE / 2) + tx * 4;
              if (cc < n) acc_red4(prow + cc, v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
            }
          }
          continue;
        }
        if (ZERO_DIAG) {
#pragma unroll
          for (int j = 0; j < TT; ++j)
            if (c0 + row_off<TILE>(tx, j) == r) v[j] = 0.f;
        }
        float* crow = args.c + (size_t)r * ld;
        // Columns past n land in the row padding (ld >= round_up(n, 32)).
        if constexpr (TILE == 128) {
          const int ca = c0 + tx * 4, cb = c0 + 64 + tx * 4;
          if (ca < n) *reinterpret_cast<float4*>(crow + ca) = make_float4(v[0], v[1], v[2], v[3]);
          if (cb < n) *reinterpret_cast<float4*>(crow + cb) = make_float4(v[4], v[5], v[6], v[7]);
        } else if constexpr (TILE == 32) {
          const int cc = c0 + tx * 2;
          if (cc < n) *reinterpret_cast<float2*>(crow + cc) = make_float2(v[0], v[1]);
        } else {
#pragma unroll
          for (int h = 0; h < TT / 4; ++h) {
            const int cc = c0 + h * (TILE / 2) + tx * 4;
            if (cc < n)
              *reinterpret_cast<float4*>(crow + cc) =
                  make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
          }
        }
      }
    }
  }
}

// Focus epilogue: counts (accumulated in the W buffer, upper-triangular
// tiles t_begin + blockIdx.x / 4 of the row-major tile list) -> U[r][c] =
// U[c][r] = count and W[r][c] = W[c][r] = 1/count (IEEE division,
// Real(1)/Real(cnt), blocked.hpp:401); diagonal 0. One CTA per 64 x 64
// quadrant of a tile; the quadrant is staged in shared memory so that both
// the direct and the mirrored writes coalesce.
//
// PEERS (multi-GPU exchange of pass 1, "peer pull"): the count of an entry
// is the SUM of the partial counts in every device's W (read over peer
// memory, integers < 2^24: exact in any order), and U / W are stored into
// every device's buffers (peer stores). Each device finishes a disjoint
// range of tiles, so the reads (upper tiles of its range, in every W) and
// the writes (the same tiles and their mirrors) of different devices never
// touch the same entries. u_all / w_all hold every device's buffers; the
// calling device's own are u / w.
struct FinishPeers {
  int32_t* u[kMaxPeers];
  float* w[kMaxPeers];
  int count;
  // where U goes: 0 own U only; 1 every device; 2 the device that owns the
  // entry's row in the tile-row band split (bands [nb*i/count, nb*(i+1)/count)
  // of tile rows: the devices that download U by row bands)
  int u_mode;
};

template <bool PEERS>
__global__ void __launch_bounds__(256)
    focus_finish_kernel(int32_t* __restrict__ u, float* __restrict__ w, int n, int ld, int nb,
                        int t_begin, FinishPeers peers) {
  constexpr int Q = kTile / 2;
  __shared__ float tile[Q][Q + 1];
  int tr, tc;
  tri_coords(t_begin + (int)(blockIdx.x >> 2), nb, tr, tc);
  const int qr = (blockIdx.x >> 1) & 1, qc = blockIdx.x & 1;
  if (tr == tc && qr > qc) return;  // below the diagonal: the mirror of (0,1)
  const int r0 = tr * kTile + qr * Q, c0 = tc * kTile + qc * Q;
  const bool diag = (r0 == c0);
  for (int idx = threadIdx.x; idx < Q * Q; idx += 256) {
    const int rl = idx / Q, cl = idx % Q;
    const int r = r0 + rl, c = c0 + cl;
    float v = 0.f;
    if (r < n && c < n) {
      const size_t o = (size_t)r * ld + c;
      if constexpr (PEERS) {
        for (int q = 0; q < peers.count; ++q) v += peers.w[q][o];
      } else {
        v = w[o];
      }
    }
    tile[rl][cl] = v;
  }
  __syncthreads();
  const int nw = PEERS ? peers.count : 1;
  auto put = [&](size_t o, int row, int32_t uv, float wv) {
    if constexpr (PEERS) {
      for (int q = 0; q < nw; ++q) peers.w[q][o] = wv;
      if (peers.u_mode == 0) {
        u[o] = uv;
      } else if (peers.u_mode == 1) {
        for (int q = 0; q < nw; ++q) peers.u[q][o] = uv;
      } else {
        const int t = row / kTile;
        int q = 0;
        while (q + 1 < nw && nb * (q + 1) / nw <= t) ++q;
        peers.u[q][o] = uv;
      }
    } else {
      (void)row;
      u[o] = uv;
      w[o] = wv;
    }
  };
  for (int idx = threadIdx.x; idx < Q * Q; idx += 256) {
    {  // direct (r, c), r <= c
      const int rl = idx / Q, cl = idx % Q;
      const int r = r0 + rl, c = c0 + cl;
      if (r < n && c < n && (!diag || rl <= cl)) {
        const size_t o = (size_t)r * ld + c;
        if (r == c) {
          put(o, r, 0, 0.f);
        } else {
          const float v = tile[rl][cl];
          put(o, r, static_cast<int32_t>(v), 1.0f / v);
        }
      }
    }
    {  // mirror (c, r), r < c
      const int rl = idx % Q, cl = idx / Q;
      const int r = r0 + rl, c = c0 + cl;
      if (r < n && c < n && r < c) {
        const float v = tile[rl][cl];
        put((size_t)c * ld + r, c, static_cast<int32_t>(v), 1.0f / v);
      }
    }
  }
}

// Accurate mode: the double sums of rows [row0, row1) rounded to the fp32
// C (triplet: diagonal 0, in the double sums too).
__global__ void __launch_bounds__(256)
    acc_round_rows_kernel(double* __restrict__ c64, float* __restrict__ c, int n, int ld, int row0,
                          int row1, int zero_diag) {
  for (int r = row0 + blockIdx.x; r < row1; r += gridDim.x)
    for (int z = threadIdx.x; z < n; z += blockDim.x) {
      const size_t o = (size_t)r * ld + z;
      if (zero_diag && z == r) {
        c64[o] = 0.0;
        c[o] = 0.f;
      } else {
        c[o] = __double2float_rn(c64[o]);
      }
    }
}

// Accurate mode, tile pairs [t0, t1) of a pair list (both C[P][Q] and
// C[Q][P]): rounded to fp32 into every buffer of `out` (the devices of a
// multi-GPU exchange, or just the local C).
__global__ void __launch_bounds__(256)
    acc_round_pairs_kernel(const int2* __restrict__ tiles, int t0, double* __restrict__ c64, PeerBufs out,
                           int n, int ld, int zero_diag) {
  const int2 tp = tiles[t0 + blockIdx.x];
  const int half = blockIdx.y;
  if (half == 1 && tp.x == tp.y) return;
  const int R = half ? tp.y : tp.x, Q = half ? tp.x : tp.y;
  for (int e = threadIdx.x; e < kTile * kTile / 4; e += blockDim.x) {
    const int rl = e / (kTile / 4), cl = (e % (kTile / 4)) * 4;
    const int r = R * kTile + rl, c = Q * kTile + cl;
    if (r >= n || c >= n) continue;
    const size_t o = (size_t)r * ld + c;
    const double2 a = *reinterpret_cast<const double2*>(c64 + o);
    const double2 b = *reinterpret_cast<const double2*>(c64 + o + 2);
    float4 f = make_float4(__double2float_rn(a.x), __double2float_rn(a.y), __double2float_rn(b.x),
                           __double2float_rn(b.y));
    if (zero_diag && r >= c && r < c + 4) {
      (&f.x)[r - c] = 0.f;
      c64[(size_t)r * ld + r] = 0.0;
    }
    for (int q = 0; q < out.count; ++q) *reinterpret_cast<float4*>(out.ptr[q] + o) = f;
  }
}

}  // namespace pald_gpu
