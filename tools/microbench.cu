// Pipe-rate microbenchmarks for the PaLD inner loops on sm_100a.
// Measures per-SM lane-ops/cycle of the candidate instruction mixes
// (FMNMX, FFMA(.SAT), FFMA2, FADD2, FMNMX3) and of full 8x8 register-tile
// inner loops for the focus (pass 1) and cohesion (pass 2) kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ unsigned long long g_cyc[4096];

template <int OP>
__global__ void chain_kernel(float* out, int iters, float seed) {
  float v[16];
  float2 w[8];
  unsigned u[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { v[i] = seed + i * 0.001f + threadIdx.x * 1e-6f; u[i] = i * 7 + threadIdx.x; }
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = make_float2(v[2 * i], v[2 * i + 1]);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) v[i] = fminf(v[i], v[(i + 1) & 15]);                                  // FMNMX
      if (OP == 1) v[i] = __fmaf_rn(v[i], v[(i + 1) & 15], v[(i + 2) & 15]);             // FFMA 3-reg
      if (OP == 2) v[i] = __saturatef(__fmaf_rn(v[i], 0x1p20f, v[(i + 1) & 15]));        // FFMA.SAT imm
      if (OP == 3 && i < 8) w[i] = __ffma2_rn(w[i], w[(i + 1) & 7], w[(i + 2) & 7]);     // FFMA2
      if (OP == 4 && i < 8) w[i] = __fadd2_rn(w[i], w[(i + 1) & 7]);                     // FADD2
      if (OP == 5) v[i] = __fadd_rn(v[i], v[(i + 1) & 15]);                              // FADD
      if (OP == 6) u[i] = (u[i] + u[(i + 1) & 15]) ^ u[(i + 3) & 15];                    // IADD3/LOP3
      if (OP == 7) { float r; asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(v[i]), "f"(v[(i + 1) & 15]), "f"(v[(i + 2) & 15])); v[i] = r; }  // FMNMX3
      if (OP == 8) v[i] = __fmul_rn(v[i], 1.0001f);                                       // FMUL imm
    }
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i] + (float)u[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += w[i].x + w[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// 8x8 register-tile inner loops with shared-memory operands, as in the real kernels.
// MODE 0: cohesion scalar   (FMNMX, FFMA.SAT, FFMA)           per ordered combo
// MODE 1: cohesion packed   (2 FMNMX, 2 FFMA.SAT, 1 FFMA2)     per 2 combos
// MODE 2: focus scalar      (FMNMX, FFMA.SAT, FADD)
// MODE 3: focus packed      (2 FMNMX, 2 FFMA.SAT, 1 FADD2)
// MODE 4: cohesion predicated (FMNMX, FSETP, @P FADD)
template <int MODE>
__global__ void __launch_bounds__(256, 1) tile_kernel(float* out, int reps, const float* thr_in) {
  constexpr int BK = 32;
  __shared__ __align__(16) float sA[BK][128];
  __shared__ __align__(16) float sW[BK][128];
  __shared__ __align__(16) float sB[BK][128];
  for (int i = threadIdx.x; i < BK * 128; i += 256) {
    (&sA[0][0])[i] = (i * 2654435761u % 1000) * 1e-3f;
    (&sW[0][0])[i] = (i * 40503u % 977) * 1e-4f;
    (&sB[0][0])[i] = (i * 2246822519u % 1013) * 1e-3f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3), tx = (warp & 1) * 8 + (lane & 7);
  float2 acc[8][4];
  float2 thr[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int p = 0; p < 4; ++p) { acc[j][p] = make_float2(0.f, 0.f); thr[j][p] = make_float2(thr_in[(j * 8 + p * 2) * 256 + threadIdx.x], thr_in[(j * 8 + p * 2 + 1) * 256 + threadIdx.x]); }
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&sA[k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&sA[k][64 + ty * 4]);
      const float4 w0 = *reinterpret_cast<const float4*>(&sW[k][ty * 4]);
      const float4 w1 = *reinterpret_cast<const float4*>(&sW[k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&sB[k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&sB[k][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 w[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y), make_float2(w1.z, w1.w)};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
if (MODE >= 5) {
        // x-outer / z-inner: the x operand (a, w) is reused across the inner loop.
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float wi = (i & 1) ? w[i >> 1].y : w[i >> 1].x;
          if (MODE == 5 || MODE == 7) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float m = fminf(a[i], b[j]);
              float& t = (i & 1) ? thr[j][i >> 1].y : thr[j][i >> 1].x;
              float& c = (i & 1) ? acc[j][i >> 1].y : acc[j][i >> 1].x;
              if (MODE == 5) { const float kk = __saturatef(__fmaf_rn(m, 0x1p20f, t)); c = __fmaf_rn(kk, wi, c); }
              else { const float kk = __saturatef(__fmaf_rn(m, -0x1p20f, t)); c = __fadd_rn(c, kk); }
            }
          } else {
            const float2 w2 = make_float2(wi, wi);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              // pairs along z: acc2[i][jj] held in acc[2jj..2jj+1][i>>1] halves
              const float m0 = fminf(a[i], b[2 * jj]), m1 = fminf(a[i], b[2 * jj + 1]);
              float& t0 = (i & 1) ? thr[2 * jj][i >> 1].y : thr[2 * jj][i >> 1].x;
              float& t1 = (i & 1) ? thr[2 * jj + 1][i >> 1].y : thr[2 * jj + 1][i >> 1].x;
              float& c0 = (i & 1) ? acc[2 * jj][i >> 1].y : acc[2 * jj][i >> 1].x;
              float& c1 = (i & 1) ? acc[2 * jj + 1][i >> 1].y : acc[2 * jj + 1][i >> 1].x;
              if (MODE == 6) {
                const float k0 = __saturatef(__fmaf_rn(m0, 0x1p20f, t0)), k1 = __saturatef(__fmaf_rn(m1, 0x1p20f, t1));
                float2 cc = __ffma2_rn(make_float2(k0, k1), w2, make_float2(c0, c1)); c0 = cc.x; c1 = cc.y;
              } else {
                const float k0 = __saturatef(__fmaf_rn(m0, -0x1p20f, t0)), k1 = __saturatef(__fmaf_rn(m1, -0x1p20f, t1));
                float2 cc = __fadd2_rn(make_float2(c0, c1), make_float2(k0, k1)); c0 = cc.x; c1 = cc.y;
              }
            }
          }
        }
      } else
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const float m0 = fminf(a[2 * p], b[j]);
          const float m1 = fminf(a[2 * p + 1], b[j]);
          if (MODE == 4) {
            if (__fmaf_rn(m0, 1.f, thr[j][p].x) > 0.f) acc[j][p].x = __fadd_rn(acc[j][p].x, w[p].x);
            if (__fmaf_rn(m1, 1.f, thr[j][p].y) > 0.f) acc[j][p].y = __fadd_rn(acc[j][p].y, w[p].y);
          } else {
            const float sgn = (MODE >= 2) ? -0x1p20f : 0x1p20f;
            const float k0 = __saturatef(__fmaf_rn(m0, sgn, thr[j][p].x));
            const float k1 = __saturatef(__fmaf_rn(m1, sgn, thr[j][p].y));
            if (MODE == 0) {
              acc[j][p].x = __fmaf_rn(k0, w[p].x, acc[j][p].x);
              acc[j][p].y = __fmaf_rn(k1, w[p].y, acc[j][p].y);
            } else if (MODE == 1) {
              acc[j][p] = __ffma2_rn(make_float2(k0, k1), w[p], acc[j][p]);
            } else if (MODE == 2) {
              acc[j][p].x = __fadd_rn(acc[j][p].x, k0);
              acc[j][p].y = __fadd_rn(acc[j][p].y, k1);
            } else {
              acc[j][p] = __fadd2_rn(acc[j][p], make_float2(k0, k1));
            }
          }
        }
      }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int p = 0; p < 4; ++p) s += acc[j][p].x + acc[j][p].y;
  out[blockIdx.x * 256 + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

static double mean_cycles(int nblocks) {
  static unsigned long long h[4096];
  CK(cudaMemcpyFromSymbol(h, g_cyc, sizeof(unsigned long long) * nblocks));
  double s = 0;
  for (int i = 0; i < nblocks; ++i) s += (double)h[i];
  return s / nblocks;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  const int nsm = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d}\n", prop.name, nsm);
  float* out; CK(cudaMalloc(&out, sizeof(float) * 4096 * 1024));
  float* thr; CK(cudaMalloc(&thr, sizeof(float) * 64 * 256)); CK(cudaMemset(thr, 0, sizeof(float) * 64 * 256));
  const char* names[] = {"FMNMX", "FFMA_3reg", "FFMA_SAT_imm", "FFMA2", "FADD2", "FADD", "IADD_LOP", "FMNMX3", "FMUL_imm"};
  // lane-ops per thread per iteration (packed ops count both halves)
  const double ops_per_iter[] = {16, 16, 16, 16, 16, 16, 32, 16, 16};
  const double instr_per_iter[] = {16, 16, 16, 8, 8, 16, 32, 16, 16};
  const int bpsm = 4, threads = 256, iters = 65536;
  auto run_chain = [&](int op) {
    const int grid = nsm * bpsm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      switch (op) {
        case 0: chain_kernel<0><<<grid, threads>>>(out, iters, 1.f); break;
        case 1: chain_kernel<1><<<grid, threads>>>(out, iters, 1.f); break;
        case 2: chain_kernel<2><<<grid, threads>>>(out, iters, 1.f); break;
        case 3: chain_kernel<3><<<grid, threads>>>(out, iters, 1.f); break;
        case 4: chain_kernel<4><<<grid, threads>>>(out, iters, 1.f); break;
        case 5: chain_kernel<5><<<grid, threads>>>(out, iters, 1.f); break;
        case 6: chain_kernel<6><<<grid, threads>>>(out, iters, 1.f); break;
        case 7: chain_kernel<7><<<grid, threads>>>(out, iters, 1.f); break;
        case 8: chain_kernel<8><<<grid, threads>>>(out, iters, 1.f); break;
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = mean_cycles(grid);
    const double lane_ops = ops_per_iter[op] * iters * threads * bpsm;  // per SM
    const double warp_instr = instr_per_iter[op] * iters * (threads / 32) * bpsm;  // per SM
    printf("{\"bench\": \"%s\", \"lane_ops_per_sm_cycle\": %.2f, \"warp_instr_per_sm_cycle\": %.3f, \"ms\": %.3f, \"mhz_est\": %.0f, \"lane_ops_per_sm_ns\": %.2f}\n",
           names[op], lane_ops / cyc, warp_instr / cyc, ms, cyc / (ms * 1e3), lane_ops / (ms * 1e6));
  };
  if (getenv("MB_CHAIN")) for (int op = 0; op < 9; ++op) run_chain(op);
  const char* tnames[] = {"tile_cohesion_scalar", "tile_cohesion_ffma2", "tile_focus_scalar", "tile_focus_fadd2", "tile_cohesion_pred",
                          "tile_cohesion_scalar_xouter", "tile_cohesion_ffma2_zpairs", "tile_focus_scalar_xouter", "tile_focus_fadd2_zpairs"};
  for (int mode = 0; mode < 9; ++mode) {
    if (getenv("MB_MODE") && atoi(getenv("MB_MODE")) != mode) continue;
    const int reps = 1024, grid = nsm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      switch (mode) {
        case 0: tile_kernel<0><<<grid, 256>>>(out, reps, thr); break;
        case 1: tile_kernel<1><<<grid, 256>>>(out, reps, thr); break;
        case 2: tile_kernel<2><<<grid, 256>>>(out, reps, thr); break;
        case 3: tile_kernel<3><<<grid, 256>>>(out, reps, thr); break;
        case 4: tile_kernel<4><<<grid, 256>>>(out, reps, thr); break;
        case 5: tile_kernel<5><<<grid, 256>>>(out, reps, thr); break;
        case 6: tile_kernel<6><<<grid, 256>>>(out, reps, thr); break;
        case 7: tile_kernel<7><<<grid, 256>>>(out, reps, thr); break;
        case 8: tile_kernel<8><<<grid, 256>>>(out, reps, thr); break;
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = mean_cycles(grid);
    const double combos = 64.0 * 256 * 32 * reps;  // per SM (one CTA per SM)
    printf("{\"bench\": \"%s\", \"combos_per_sm_cycle\": %.2f, \"ms\": %.3f, \"mhz_est\": %.0f, \"combos_per_sm_ns\": %.2f}\n", tnames[mode], combos / cyc, ms, cyc / (ms * 1e3), combos / (ms * 1e6));
  }
  return 0;
}
