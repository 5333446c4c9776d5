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
constexpr int kBK = 32;         // third-point chunk per pipeline stage
constexpr int kThreads = 256;   // 8 warps, 16 x 16 threads, 8 x 8 outputs each
constexpr int kStages = 4;
constexpr int kBoxBytes = kBK * kTile * 4;  // one TMA box (16 KB)
constexpr float kCmpScale = 0x1p125f;       // S of the FFMA.SAT compare

__host__ __device__ constexpr int stage_bytes(int pass) { return (pass == 0 ? 2 : 3) * kBoxBytes; }
__host__ __device__ constexpr int smem_bytes(int pass) { return kStages * stage_bytes(pass) + 1024; }

struct KernelArgs {
  const uint32_t* d;     // layout of D (scaled fp32 bits or integer keys), n x ld
  int32_t* u;            // focus sizes
  float* w;              // 1/u
  float* c;              // cohesion
  int n;
  int ld;
  int nb;                // tiles per dimension
  int tile_row_begin;    // first tile row of this launch
  int tile_row_end;
};

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

__device__ __forceinline__ uint32_t nu_bits(uint32_t v) { return v + 1u; }
__device__ __forceinline__ float nu_f(float v) { return __uint_as_float(__float_as_uint(v) + 1u); }

// ---------------------------------------------------------------------------
// The tile kernel. One CTA computes one 128 x 128 output tile over all n
// third points; TMA streams 32-row chunks of the A/B(/W) panels through a
// 4-stage mbarrier pipeline. Thread (ty, tx) owns rows {ty*4+i, 64+ty*4+i}
// and columns {tx*4+j, 64+tx*4+j}; pairs of adjacent columns share one
// packed FADD2/FFMA2 accumulate.
//
// PASS 0 = focus, 1 = cohesion. A_NU / B_NU / T_NU select the nu()
// transforms above; ZERO_DIAG zeroes the cohesion diagonal (triplet).
template <int PASS, bool A_NU, bool B_NU, bool T_NU, bool ZERO_DIAG, bool FAST>
__global__ void __launch_bounds__(kThreads, 1)
    pald_tile_kernel(const __grid_constant__ CUtensorMap tm_d,
                     const __grid_constant__ CUtensorMap tm_dnu,
                     const __grid_constant__ CUtensorMap tm_w, const KernelArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t full_bar[kStages];
  __shared__ int s_tile[2];

  const int tid = threadIdx.x;
  const int n = args.n, ld = args.ld, nb = args.nb;

  // ---- tile coordinates -------------------------------------------------
  if (tid == 0) {
    int b = blockIdx.x, tr = args.tile_row_begin, tc;
    if (PASS == 0) {  // upper-triangular tiles of rows [begin, end)
      while (b >= nb - tr) { b -= nb - tr; ++tr; }
      tc = tr + b;
    } else {          // all tiles of rows [begin, end)
      tr += b / nb;
      tc = b % nb;
    }
    s_tile[0] = tr;
    s_tile[1] = tc;
    for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int r0 = s_tile[0] * kTile, c0 = s_tile[1] * kTile;

  const int warp = tid >> 5, lane = tid & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);  // 0..15
  const int tx = (warp & 1) * 8 + (lane & 7);    // 0..15
  int rows[8], cols[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    rows[i] = r0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    cols[i] = c0 + (i < 4 ? tx * 4 + i : 64 + tx * 4 + (i - 4));
  }

  const int nchunks = (n + kBK - 1) / kBK;
  constexpr int SB = stage_bytes(PASS);
  auto issue = [&](int ch) {
    const int s = ch % kStages;
    const int k0 = ch * kBK, k1 = min(k0 + kBK, n);
    // Uniform per-chunk transform choice: the whole chunk lies below the
    // column (A) / row (B) tile => every element takes nu().
    const CUtensorMap* ma = (A_NU && k1 <= c0) ? &tm_dnu : &tm_d;
    const CUtensorMap* mb = (B_NU && k1 <= r0) ? &tm_dnu : &tm_d;
    uint8_t* st = smem + s * SB;
    mbar_expect_tx(&full_bar[s], SB);
    tma_load_2d(st, ma, r0, k0, &full_bar[s]);
    tma_load_2d(st + kBoxBytes, mb, c0, k0, &full_bar[s]);
    if (PASS == 1) tma_load_2d(st + 2 * kBoxBytes, &tm_w, r0, k0, &full_bar[s]);
  };
  if (tid == 0) {
    for (int ch = 0; ch < kStages && ch < nchunks; ++ch) issue(ch);
  }

  // ---- per-output thresholds (hoisted out of the k loop) -----------------
  // thr[i][jp] holds columns (2jp, 2jp+1) of row i.
  float2 thr[8][4];
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      uint32_t t2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = rows[i], c = cols[2 * jp + h];
        uint32_t t = (r < n && c < n) ? __ldg(args.d + (size_t)r * ld + c) : 0u;
        if (T_NU) t = nu_bits(t);
        t2[h] = t;
      }
      if (FAST) {
        const float s = (PASS == 0) ? kCmpScale : -kCmpScale;
        thr[i][jp] = make_float2(__uint_as_float(t2[0]) * s, __uint_as_float(t2[1]) * s);
      } else {
        thr[i][jp] = make_float2(__uint_as_float(t2[0]), __uint_as_float(t2[1]));
      }
      acc[i][jp] = make_float2(0.f, 0.f);
    }
  }

  // ---- main loop ----------------------------------------------------------
  for (int ch = 0; ch < nchunks; ++ch) {
    const int s = ch % kStages;
    mbar_wait(&full_bar[s], (ch / kStages) & 1);
    const uint8_t* st = smem + s * SB;
    const float* sa = reinterpret_cast<const float*>(st);
    const float* sb = reinterpret_cast<const float*>(st + kBoxBytes);
    const float* sw = reinterpret_cast<const float*>(st + 2 * kBoxBytes);
    const int k0 = ch * kBK;
    const bool a_in = A_NU && (k0 >= c0) && (k0 < c0 + kTile);
    const bool b_in = B_NU && (k0 >= r0) && (k0 < r0 + kTile);
    const int kmax = min(kBK, n - k0);

    if (!a_in && !b_in && kmax == kBK) {
      // Fast, uniform chunk.
#pragma unroll 2
      for (int kk = 0; kk < kBK; ++kk) {
        const float4 a0 = reinterpret_cast<const float4*>(sa + kk * kTile)[ty];
        const float4 a1 = reinterpret_cast<const float4*>(sa + kk * kTile)[16 + ty];
        const float4 b0 = reinterpret_cast<const float4*>(sb + kk * kTile)[tx];
        const float4 b1 = reinterpret_cast<const float4*>(sb + kk * kTile)[16 + tx];
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        float w[8];
        if (PASS == 1) {
          const float4 w0 = reinterpret_cast<const float4*>(sw + kk * kTile)[ty];
          const float4 w1 = reinterpret_cast<const float4*>(sw + kk * kTile)[16 + ty];
          w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
          w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {
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
                acc[i][jp] = __ffma2_rn(make_float2(k0f, k1f), make_float2(w[i], w[i]), acc[i][jp]);
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
                acc[i][jp].x = __fadd_rn(acc[i][jp].x, (t0 < m0) ? w[i] : 0.f);
                acc[i][jp].y = __fadd_rn(acc[i][jp].y, (t1 < m1) ? w[i] : 0.f);
              }
            }
          }
        }
      }
    } else {
      // Chunk that crosses the row/column tile (per-element nu choice) or
      // the ragged last chunk.
      for (int kk = 0; kk < kmax; ++kk) {
        const int kg = k0 + kk;
        float a[8], b[8], w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int off = (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
          a[i] = sa[kk * kTile + off];
          if (PASS == 1) w[i] = sw[kk * kTile + off];
          const int offc = (i < 4 ? tx * 4 + i : 64 + tx * 4 + (i - 4));
          b[i] = sb[kk * kTile + offc];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {
            float kv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = 2 * jp + h;
              const bool nua = a_in && (kg < cols[j]);
              const bool nub = b_in && (kg < rows[i]);
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
    }
    __syncthreads();  // every warp is done with stage s
    if (tid == 0 && ch + kStages < nchunks) issue(ch + kStages);
  }

  // ---- epilogue -----------------------------------------------------------
  if (PASS == 0) {
    // Stage the count tile in shared memory, then write U and W = 1/U for
    // the tile (coalesced rows) and its mirror image (coalesced columns).
    float* tile = reinterpret_cast<float*>(smem);
    constexpr int TS = kTile + 1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rl = rows[i] - r0;
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        tile[rl * TS + (cols[2 * jp] - c0)] = acc[i][jp].x;
        tile[rl * TS + (cols[2 * jp + 1] - c0)] = acc[i][jp].y;
      }
    }
    __syncthreads();
    const bool diag = (r0 == c0);
    for (int idx = tid; idx < kTile * kTile; idx += kThreads) {
      {  // direct: (r, c) with r < c (r == c -> 0)
        const int rl = idx / kTile, cl = idx % kTile;
        const int r = r0 + rl, c = c0 + cl;
        if (r < n && c < n && (!diag || rl <= cl)) {
          const float v = tile[rl * TS + cl];
          const size_t o = (size_t)r * ld + c;
          if (r == c) {
            args.u[o] = 0;
            args.w[o] = 0.f;
          } else {
            args.u[o] = static_cast<int32_t>(v);
            args.w[o] = 1.0f / v;  // IEEE division: Real(1)/Real(cnt), blocked.hpp:401
          }
        }
      }
      {  // mirror: (c, r) for r < c
        const int rl = idx % kTile, cl = idx / kTile;
        const int r = r0 + rl, c = c0 + cl;
        if (r < n && c < n && r < c) {
          const float v = tile[rl * TS + cl];
          const size_t o = (size_t)c * ld + r;
          args.u[o] = static_cast<int32_t>(v);
          args.w[o] = 1.0f / v;
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = rows[i];
      if (r >= n) continue;
      float v[8];
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        v[2 * jp] = acc[i][jp].x;
        v[2 * jp + 1] = acc[i][jp].y;
      }
      if (ZERO_DIAG) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (cols[j] == r) v[j] = 0.f;
      }
      float* crow = args.c + (size_t)r * ld;
      // Columns past n land in the row padding (ld >= round_up(n, 32)).
      if (cols[0] < n) *reinterpret_cast<float4*>(crow + cols[0]) = make_float4(v[0], v[1], v[2], v[3]);
      if (cols[4] < n) *reinterpret_cast<float4*>(crow + cols[4]) = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

}  // namespace pald_gpu
