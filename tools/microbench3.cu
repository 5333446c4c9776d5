// Symmetric-pair cohesion inner loop: one min + one compare per (r, c, k)
// feeds both C[r][c] (weight w_rk, broadcast) and C[c][r] (weight w_ck,
// packed per column pair). Compared against the one-sided loop.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ unsigned long long g_cyc[4096];

template <int TM, int TN, bool SYM, int NSET = 0, int PRED = 0, int ORD = 0>
__global__ void __launch_bounds__(128 * 128 / (TM * TN), 1) tile_kernel(float* out, int reps, const float* thr_in) {
  constexpr int NT = 128 * 128 / (TM * TN), BK = 16;
  __shared__ __align__(16) float sA[BK][128];
  __shared__ __align__(16) float sW[BK][128];
  __shared__ __align__(16) float sB[BK][128];
  __shared__ __align__(16) float sV[BK][128];
  for (int i = threadIdx.x; i < BK * 128; i += NT) {
    (&sA[0][0])[i] = (i * 2654435761u % 1000) * 1e-3f;
    (&sW[0][0])[i] = (i * 40503u % 977) * 1e-4f;
    (&sB[0][0])[i] = (i * 2246822519u % 1013) * 1e-3f;
    (&sV[0][0])[i] = (i * 7919u % 983) * 1e-4f;
  }
  __syncthreads();
  constexpr int NTX = 128 / TN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int WX = NTX / 8;
  const int ty = (warp / WX) * 4 + (lane >> 3), tx = (warp % WX) * 8 + (lane & 7);
  float2 acc[TM][TN / 2], act[SYM ? TM : 1][TN / 2], thr[TM][TN / 2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int p = 0; p < TN / 2; ++p) {
      acc[i][p] = make_float2(0.f, 0.f);
      if (SYM) act[i][p] = make_float2(0.f, 0.f);
      thr[i][p] = make_float2(thr_in[((i * 8 + p) * 2) * 512 + threadIdx.x], thr_in[((i * 8 + p) * 2 + 1) * 512 + threadIdx.x]);
    }
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int k = 0; k < BK; ++k) {
      float a[TM], w[TM], b[TN], v[TN];
#pragma unroll
      for (int h = 0; h < TM / 4; ++h) {
        const float4 av = *reinterpret_cast<const float4*>(&sA[k][h * 64 + ty * 4]);
        a[h * 4 + 0] = av.x; a[h * 4 + 1] = av.y; a[h * 4 + 2] = av.z; a[h * 4 + 3] = av.w;
        const float4 wv = *reinterpret_cast<const float4*>(&sW[k][h * 64 + ty * 4]);
        w[h * 4 + 0] = wv.x; w[h * 4 + 1] = wv.y; w[h * 4 + 2] = wv.z; w[h * 4 + 3] = wv.w;
      }
#pragma unroll
      for (int h = 0; h < TN / 4; ++h) {
        const float4 bv = *reinterpret_cast<const float4*>(&sB[k][h * 64 + tx * 4]);
        b[h * 4 + 0] = bv.x; b[h * 4 + 1] = bv.y; b[h * 4 + 2] = bv.z; b[h * 4 + 3] = bv.w;
        if (SYM) {
          const float4 vv = *reinterpret_cast<const float4*>(&sV[k][h * 64 + tx * 4]);
          v[h * 4 + 0] = vv.x; v[h * 4 + 1] = vv.y; v[h * 4 + 2] = vv.z; v[h * 4 + 3] = vv.w;
        }
      }
      if (ORD == 1) {  // per row: all mins, then compares, then direct, then transposed
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          float m[TN];
#pragma unroll
          for (int j = 0; j < TN; ++j) m[j] = fminf(a[i], b[j]);
          float2 kv[TN / 2];
#pragma unroll
          for (int p = 0; p < TN / 2; ++p)
            kv[p] = make_float2(__saturatef(__fmaf_rn(m[2 * p], 0x1p20f, thr[i][p].x)),
                                __saturatef(__fmaf_rn(m[2 * p + 1], 0x1p20f, thr[i][p].y)));
#pragma unroll
          for (int p = 0; p < TN / 2; ++p) acc[i][p] = __ffma2_rn(kv[p], make_float2(w[i], w[i]), acc[i][p]);
#pragma unroll
          for (int p = 0; p < TN / 2; ++p)
            act[i][p] = __ffma2_rn(kv[p], make_float2(v[2 * p], v[2 * p + 1]), act[i][p]);
        }
        continue;
      }
      if (ORD == 3 || ORD == 4) {  // column-pair outer; the 8 transposed-output FFMA2s of a column pair in ONE asm block
        float2 kv[TM][TN / 2];
#pragma unroll
        for (int p = 0; p < TN / 2; ++p) {
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float m0 = fminf(a[i], b[2 * p]), m1 = fminf(a[i], b[2 * p + 1]);
            kv[i][p] = make_float2(__saturatef(__fmaf_rn(m0, 0x1p20f, thr[i][p].x)),
                                   __saturatef(__fmaf_rn(m1, 0x1p20f, thr[i][p].y)));
          }
          unsigned long long vv = (unsigned long long)__float_as_uint(v[2 * p]) | ((unsigned long long)__float_as_uint(v[2 * p + 1]) << 32);
          unsigned long long* A = reinterpret_cast<unsigned long long*>(&act[0][0]);
          unsigned long long* K = reinterpret_cast<unsigned long long*>(&kv[0][0]);
          asm volatile(
              "fma.rn.f32x2 %0, %8, %16, %0;\n\tfma.rn.f32x2 %1, %9, %16, %1;\n\t"
              "fma.rn.f32x2 %2, %10, %16, %2;\n\tfma.rn.f32x2 %3, %11, %16, %3;\n\t"
              "fma.rn.f32x2 %4, %12, %16, %4;\n\tfma.rn.f32x2 %5, %13, %16, %5;\n\t"
              "fma.rn.f32x2 %6, %14, %16, %6;\n\tfma.rn.f32x2 %7, %15, %16, %7;"
              : "+l"(A[0 * (TN / 2) + p]), "+l"(A[1 * (TN / 2) + p]), "+l"(A[2 * (TN / 2) + p]), "+l"(A[3 * (TN / 2) + p]),
                "+l"(A[4 * (TN / 2) + p]), "+l"(A[5 * (TN / 2) + p]), "+l"(A[6 * (TN / 2) + p]), "+l"(A[7 * (TN / 2) + p])
              : "l"(K[0 * (TN / 2) + p]), "l"(K[1 * (TN / 2) + p]), "l"(K[2 * (TN / 2) + p]), "l"(K[3 * (TN / 2) + p]),
                "l"(K[4 * (TN / 2) + p]), "l"(K[5 * (TN / 2) + p]), "l"(K[6 * (TN / 2) + p]), "l"(K[7 * (TN / 2) + p]), "l"(vv));
          if (ORD == 3) {
#pragma unroll
            for (int i = 0; i < TM; ++i) acc[i][p] = __ffma2_rn(kv[i][p], make_float2(w[i], w[i]), acc[i][p]);
          }
        }
        if (ORD == 4) {
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int p = 0; p < TN / 2; ++p) acc[i][p] = __ffma2_rn(kv[i][p], make_float2(w[i], w[i]), acc[i][p]);
        }
        continue;
      }
      if (ORD == 2) {  // column-pair outer, rows inner
#pragma unroll
        for (int p = 0; p < TN / 2; ++p)
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float m0 = fminf(a[i], b[2 * p]), m1 = fminf(a[i], b[2 * p + 1]);
            const float2 kv = make_float2(__saturatef(__fmaf_rn(m0, 0x1p20f, thr[i][p].x)),
                                          __saturatef(__fmaf_rn(m1, 0x1p20f, thr[i][p].y)));
            acc[i][p] = __ffma2_rn(kv, make_float2(w[i], w[i]), acc[i][p]);
            act[i][p] = __ffma2_rn(kv, make_float2(v[2 * p], v[2 * p + 1]), act[i][p]);
          }
        continue;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int p = 0; p < TN / 2; ++p) {
          const float m0 = fminf(a[i], b[2 * p]), m1 = fminf(a[i], b[2 * p + 1]);
          if (PRED) {
            const bool p0 = m0 > thr[i][p].x, p1 = m1 > thr[i][p].y;
            if (PRED == 1) {
              if (p0) { acc[i][p].x += w[i]; act[i][p].x += v[2 * p]; }
              if (p1) { acc[i][p].y += w[i]; act[i][p].y += v[2 * p + 1]; }
            } else {
              acc[i][p].x += p0 ? w[i] : 0.f; act[i][p].x += p0 ? v[2 * p] : 0.f;
              acc[i][p].y += p1 ? w[i] : 0.f; act[i][p].y += p1 ? v[2 * p + 1] : 0.f;
            }
            continue;
          }
          float k0, k1;
          if (p < NSET) {
            k0 = (m0 > thr[i][p].x) ? 1.f : 0.f;
            k1 = (m1 > thr[i][p].y) ? 1.f : 0.f;
          } else {
            k0 = __saturatef(__fmaf_rn(m0, 0x1p20f, thr[i][p].x));
            k1 = __saturatef(__fmaf_rn(m1, 0x1p20f, thr[i][p].y));
          }
          const float2 kk = make_float2(k0, k1);
          acc[i][p] = __ffma2_rn(kk, make_float2(w[i], w[i]), acc[i][p]);
          if (SYM) act[i][p] = __ffma2_rn(kk, make_float2(v[2 * p], v[2 * p + 1]), act[i][p]);
        }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int p = 0; p < TN / 2; ++p) {
      s += acc[i][p].x + acc[i][p].y;
      if (SYM) s += act[i][p].x * 3.f + act[i][p].y;
    }
  out[blockIdx.x * 1024 + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int TM, int TN, bool SYM, int NSET = 0, int PRED = 0, int ORD = 0>
void run(const char* name, float* out, const float* thr, int nsm) {
  constexpr int NT = 128 * 128 / (TM * TN);
  const int reps = 1024;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    tile_kernel<TM, TN, SYM, NSET, PRED, ORD><<<nsm, NT>>>(out, reps, thr);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    cudaEventElapsedTime(&ms, e0, e1);
  }
  static unsigned long long h[4096];
  CK(cudaMemcpyFromSymbol(h, g_cyc, sizeof(unsigned long long) * nsm));
  double cyc = 0; for (int i = 0; i < nsm; ++i) cyc += h[i]; cyc /= nsm;
  const double outputs = (SYM ? 2.0 : 1.0) * 128.0 * 128 * 16 * reps;  // (output, k) combos
  printf("{\"bench\": \"%s\", \"threads\": %d, \"output_combos_per_sm_cycle\": %.2f, \"ms\": %.3f, \"mhz_est\": %.0f}\n", name, NT, outputs / cyc, ms, cyc / (ms * 1e3));
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int nsm = prop.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, sizeof(float) * 4096 * 1024));
  float* thr; CK(cudaMalloc(&thr, sizeof(float) * 256 * 512)); CK(cudaMemset(thr, 0, sizeof(float) * 256 * 512));
  run<8, 8, false>("cohesion_8x8_onesided", out, thr, nsm);
  run<8, 8, false, 1>("cohesion_8x8_onesided_fset1", out, thr, nsm);
  run<8, 8, false, 2>("cohesion_8x8_onesided_fset2", out, thr, nsm);
  run<8, 8, true>("cohesion_8x8_sym", out, thr, nsm);
  run<8, 8, true, 1>("cohesion_8x8_sym_fset1", out, thr, nsm);
  run<8, 8, true, 2>("cohesion_8x8_sym_fset2", out, thr, nsm);
  run<8, 8, true, 3>("cohesion_8x8_sym_fset3", out, thr, nsm);
  run<8, 8, true, 4>("cohesion_8x8_sym_fset4", out, thr, nsm);
  run<8, 8, true, 0, 1>("cohesion_8x8_sym_pred_branch", out, thr, nsm);
  run<8, 8, true, 0, 0, 1>("cohesion_8x8_sym_rowbatch", out, thr, nsm);
  run<8, 8, true, 0, 0, 2>("cohesion_8x8_sym_colouter", out, thr, nsm);
  run<8, 8, true, 0, 2>("cohesion_8x8_sym_pred_select", out, thr, nsm);
  run<8, 8, true, 0, 0, 3>("cohesion_8x8_sym_colblock", out, thr, nsm);
  run<8, 8, true, 0, 0, 4>("cohesion_8x8_sym_colblock_rowbcast", out, thr, nsm);
  return 0;
}
