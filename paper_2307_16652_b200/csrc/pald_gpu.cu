// pald_gpu.cu -- host side of the C ABI declared in include/pald_gpu.h.
//
// Owns device workspaces ("plans"), the input range check / layout kernels,
// the launch schedule over the pair-tile grid, CUDA-event phase timing and
// the error mapping of the reference (types.hpp:14-25 -> status codes).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pald_gpu.h"
#include "pald_internal.h"
#include "pald_kernels.cuh"
#include "pald_rank.cuh"
#include "pald_sym.cuh"

using namespace pald_gpu;

namespace {

thread_local std::string g_last_error;

// Hooks of the f64io entry points (pald_internal.h), per calling thread.
thread_local pald_gpu_host_hooks t_hooks{nullptr, nullptr, nullptr, nullptr};
inline void hook_rows_needed(uint64_t r0, uint64_t r1) {
  if (t_hooks.rows_needed) t_hooks.rows_needed(t_hooks.ctx, r0, r1);
}
// Host callbacks queued behind the D2H copies (payloads live in the plan-independent
// static pool below: one call at a time per thread, <= 64 bands).
struct LandedMsg {
  pald_gpu_host_hooks hooks;
  uint64_t r1;
};
void CUDART_CB cb_c_rows_landed(void* m) {
  auto* msg = static_cast<LandedMsg*>(m);
  msg->hooks.c_rows_landed(msg->hooks.ctx, msg->r1);
}
void CUDART_CB cb_u_landed(void* m) {
  auto* msg = static_cast<LandedMsg*>(m);
  msg->hooks.u_landed(msg->hooks.ctx);
}
thread_local LandedMsg t_msgs[80];
thread_local int t_msg_next = 0;
// Queue "rows [0, r1) of C_out landed" (r1 > 0) or "U_out landed" (r1 == 0)
// behind the copies already on `sc`.
int queue_landed(cudaStream_t sc, uint64_t r1) {
  if (r1 ? !t_hooks.c_rows_landed : !t_hooks.u_landed) return PALD_GPU_OK;
  LandedMsg* m = &t_msgs[t_msg_next++ % 80];
  m->hooks = t_hooks;
  m->r1 = r1;
  if (cudaLaunchHostFunc(sc, r1 ? cb_c_rows_landed : cb_u_landed, m) != cudaSuccess) {
    cudaGetLastError();  // hooks are an optimisation: the caller converts the rest at the end
  }
  return PALD_GPU_OK;
}

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define PALD_CUDA(expr)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_error(PALD_GPU_ERR_CUDA, "CUDA error %s at %s:%d (%s)",                 \
                       cudaGetErrorString(e_), __FILE__, __LINE__, #expr);               \
  } while (0)

// ---------------------------------------------------------------------------
// Range check / validation of the fp32 input (types.hpp:45-65 semantics,
// evaluated on the fp32 values).
struct Stats {
  uint32_t min_pos_bits;   // smallest positive off-diagonal value (bits)
  uint32_t max_bits;       // largest off-diagonal value (bits, non-NaN)
  uint32_t diag_nonzero;
  uint32_t offdiag_not_positive;  // 0, negative or NaN
  uint32_t offdiag_zero;
  uint32_t has_inf;
  uint32_t has_nan;
  uint32_t asymmetric;
  // first violation of each kind in the reference's scan order
  // (types.hpp:50-62: row by row, (x, x) then (x, y > x)); key = x * n + y
  unsigned long long key_diag, key_notpos, key_asym;
};

__global__ void stats_kernel(const float* __restrict__ d, uint64_t ldd, int n, int check_sym,
                             Stats* out, int r_begin, int r_end) {
  uint32_t mn = 0xffffffffu, mx = 0u, flags = 0u;
  unsigned long long kd = ~0ull, knp = ~0ull, kas = ~0ull;
  // rows [r_begin, r_end); symmetry is checked against the rows above
  // (c < r), so a banded H2D can check each band as it arrives
  for (int r = r_begin + blockIdx.x; r < r_end; r += gridDim.x) {
    const float* row = d + (size_t)r * ldd;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      const float v = row[c];
      const uint32_t bits = __float_as_uint(v);
      if (r == c) {
        if ((bits & 0x7fffffffu) != 0u) {
          flags |= 1u;
          kd = min(kd, (unsigned long long)r * n + r);
        }
        continue;
      }
      if (!(v > 0.f)) {
        flags |= 2u;
        // the reference tests positivity on the upper entry (x, y > x); a
        // bad lower entry shows up there as an asymmetry (below)
        if (c > r) knp = min(knp, (unsigned long long)r * n + c);
      }
      if (v == 0.f) flags |= 4u;
      if (isinf(v)) flags |= 8u;
      if (isnan(v)) flags |= 16u;
      if (v > 0.f) {
        mn = min(mn, bits);
        mx = max(mx, bits);
      }
      if (check_sym && c < r) {
        const float t = d[(size_t)c * ldd + r];
        if (__float_as_uint(t) != bits) {
          flags |= 32u;
          kas = min(kas, (unsigned long long)c * n + r);
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    kd = min(kd, __shfl_xor_sync(0xffffffffu, kd, o));
    knp = min(knp, __shfl_xor_sync(0xffffffffu, knp, o));
    kas = min(kas, __shfl_xor_sync(0xffffffffu, kas, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (kd != ~0ull) atomicMin(&out->key_diag, kd);
    if (knp != ~0ull) atomicMin(&out->key_notpos, knp);
    if (kas != ~0ull) atomicMin(&out->key_asym, kas);
    atomicMin(&out->min_pos_bits, mn);
    atomicMax(&out->max_bits, mx);
    if (flags & 1u) atomicOr(&out->diag_nonzero, 1u);
    if (flags & 2u) atomicOr(&out->offdiag_not_positive, 1u);
    if (flags & 4u) atomicOr(&out->offdiag_zero, 1u);
    if (flags & 8u) atomicOr(&out->has_inf, 1u);
    if (flags & 16u) atomicOr(&out->has_nan, 1u);
    if (flags & 32u) atomicOr(&out->asymmetric, 1u);
  }
}

// Lays D out for the tile kernels: fast path -> fp32 scaled by 2^p (exact)
// and its successor nu; exact path -> keys 2*bits and key+1. Diagonal is
// canonicalised to +0 (types.hpp:51 accepts -0.0).
__global__ void layout_kernel(const float* __restrict__ d, uint64_t ldd, int n, uint64_t ld,
                              int fast, int p2, uint32_t* __restrict__ ds,
                              uint32_t* __restrict__ dnu) {
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      float v = d[(size_t)r * ldd + c];
      if (r == c) v = 0.f;
      const uint32_t out = fast ? __float_as_uint(scalbnf(v, p2)) : 2u * (__float_as_uint(v) & 0x7fffffffu);
      ds[(size_t)r * ld + c] = out;
      dnu[(size_t)r * ld + c] = out + 1u;
    }
  }
}

__global__ void fill_diagonal_kernel(const int32_t* __restrict__ u, uint64_t ldu, int n,
                                     double* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  double s = 0.0;
  const int32_t* row = u + (size_t)x * ldu;
  for (int y = 0; y < n; ++y)
    if (y != x) s = __dadd_rn(s, __ddiv_rn(1.0, (double)row[y]));
  out[x] = s;
}

// points_to_distances (ingest.hpp:303-322): each unordered pair evaluated in
// the same (min, max) order so D is exactly symmetric; sum = fma(diff, diff,
// sum) in coordinate order, which is the reference's `sum += diff * diff` as
// its own build compiles it (-O3 -march=native: contracted to an FMA; checked
// bit-exact against oracle/_ref in tests/test_gpu_analyze.py). A zero
// distance records the pair's row-major key (the reference throws on the
// first duplicate pair of its x < y loop).
__global__ void points_kernel(const double* __restrict__ p, int n, int dim, float* __restrict__ d,
                              uint64_t ldd, unsigned long long* __restrict__ dup_key) {
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      float out = 0.f;
      if (r != c) {
        const int a = min(r, c), b = max(r, c);
        double s = 0.0;
        for (int k = 0; k < dim; ++k) {
          const double diff = __dsub_rn(p[(size_t)a * dim + k], p[(size_t)b * dim + k]);
          s = __fma_rn(diff, diff, s);
        }
        const double dist = __dsqrt_rn(s);
        if (dist == 0.0 && r < c) atomicMin(dup_key, (unsigned long long)r * n + c);
        out = __double2float_rn(dist);
      }
      d[(size_t)r * ldd + c] = out;
    }
  }
}

// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_map(CUtensorMap* map, const void* base, uint64_t n, uint64_t ld, int box_cols = kTile,
             int box_rows = kBK, CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
             int elem_bytes = 4) {
  auto encode = get_encode();
  if (!encode) return set_error(PALD_GPU_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {n, n};
  cuuint64_t strides[1] = {ld * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, dtype, 2, const_cast<void*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PALD_GPU_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PALD_GPU_OK;
}

template <int PASS, bool A_NU, bool B_NU, bool T_NU, bool ZD, bool FAST, bool SPLIT = false,
          int TILE = kTile, bool LIST = false, bool PEERS = false, bool RANK = false, bool ACC = false>
int launch_tile(const CUtensorMap& md, const CUtensorMap& mnu, const CUtensorMap& mw,
                const KernelArgs& a, int grid, cudaStream_t s) {
  auto k = pald_tile_kernel<PASS, A_NU, B_NU, T_NU, ZD, FAST, SPLIT, TILE, LIST, PEERS, RANK, ACC>;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    PALD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(PASS, TILE, RANK)));
    attr_done[dev & 63] = true;
  }
  k<<<grid, kThreads, smem_bytes(PASS, TILE, RANK), s>>>(md, mnu, mw, a);
  PALD_CUDA(cudaGetLastError());
  return PALD_GPU_OK;
}

uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

// Options of the caller's ABI version (v3: no device list) -> a full v4
// struct with the defaults for the fields the caller does not have.
int read_opts(const pald_gpu_opts* in, pald_gpu_opts* o) {
  if (!in) return set_error(PALD_GPU_ERR_VALIDATION, "null options");
  if (in->struct_size != sizeof(pald_gpu_opts) && in->struct_size != PALD_GPU_OPTS_V3_SIZE)
    return set_error(PALD_GPU_ERR_VALIDATION, "pald_gpu_opts.struct_size mismatch (%u: expected %zu or %u)",
                     in->struct_size, sizeof(pald_gpu_opts), PALD_GPU_OPTS_V3_SIZE);
  std::memset(o, 0, sizeof(*o));
  std::memcpy(o, in, in->struct_size);
  o->struct_size = sizeof(pald_gpu_opts);
  if (o->num_devices < 0 || o->num_devices > PALD_GPU_MAX_DEVICES)
    return set_error(PALD_GPU_ERR_VALIDATION, "num_devices %d out of range [0, %d]", o->num_devices,
                     PALD_GPU_MAX_DEVICES);
  for (int e : {o->exchange_focus, o->exchange_cohesion})
    if (e < PALD_GPU_EXCHANGE_AUTO || e > PALD_GPU_EXCHANGE_RED)
      return set_error(PALD_GPU_ERR_VALIDATION, "unknown exchange transport %d", e);
  if (o->exchange_cohesion == PALD_GPU_EXCHANGE_RED)
    return set_error(PALD_GPU_ERR_VALIDATION, "the RED exchange applies to pass 1 only");
  if (o->num_devices > 1) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    for (int i = 0; i < o->num_devices; ++i)
      if (o->devices[i] < 0 || o->devices[i] >= count)
        return set_error(PALD_GPU_ERR_VALIDATION, "devices[%d] = %d is not a visible device (%d visible)", i,
                         o->devices[i], count);
  }
  return PALD_GPU_OK;
}

int check_opts(const pald_gpu_opts* o) {
  if (!o) return set_error(PALD_GPU_ERR_VALIDATION, "null options");
  if (o->struct_size != sizeof(pald_gpu_opts))
    return set_error(PALD_GPU_ERR_VALIDATION, "pald_gpu_opts.struct_size mismatch (%u != %zu)",
                     o->struct_size, sizeof(pald_gpu_opts));
  if (o->algorithm != PALD_GPU_PAIRWISE && o->algorithm != PALD_GPU_TRIPLET)
    return set_error(PALD_GPU_ERR_VALIDATION, "unknown algorithm %d", o->algorithm);
  if (o->policy != PALD_GPU_STRICT && o->policy != PALD_GPU_INCLUSIVE_SPLIT)
    return set_error(PALD_GPU_ERR_VALIDATION, "unknown policy %d", o->policy);
  // blocked.hpp:429-431, parallel.hpp:262-265 check policy before sizes.
  if (o->algorithm == PALD_GPU_TRIPLET) {
    if (o->policy != PALD_GPU_STRICT)
      return set_error(PALD_GPU_ERR_UNSUPPORTED, "the triplet algorithm supports the strict policy only");
    if (o->block_focus < 1 || o->block_cohesion < 1)
      return set_error(PALD_GPU_ERR_VALIDATION, "triplet block sizes must be >= 1");
  } else {
    if (o->block < 1) return set_error(PALD_GPU_ERR_VALIDATION, "pairwise block size must be >= 1");
  }
  return PALD_GPU_OK;
}

}  // namespace

#ifndef PALD_HOST_BANDS  // pass-2 bands of the host API (the last band's D2H is exposed)
#define PALD_HOST_BANDS 16  // one raster group per band at n = 32768: e2e 3.790 -> 3.773 s
#endif
#define PALD_HOST_BANDS_MAX PALD_HOST_BANDS

// ---------------------------------------------------------------------------
struct pald_gpu_plan {
  int device = 0;
  uint64_t n = 0, ld = 0, nb = 0;
  int algorithm = 0;
  int policy = 0;
  uint32_t flags = 0;
  uint32_t* ds = nullptr;
  uint32_t* dnu = nullptr;
  int32_t* u = nullptr;
  float* w = nullptr;
  float* c = nullptr;
  Stats* stats = nullptr;
  Stats* stats_host = nullptr;
  CUtensorMap tm_d, tm_dnu, tm_w;        // 128-wide boxes
  CUtensorMap tm_d64, tm_dnu64, tm_w64;  // 64-wide boxes (small-n cohesion tiles)
  CUtensorMap tm_d32, tm_dnu32, tm_w32;  // 128 x 32 boxes (tile-pair cohesion)
  CUtensorMap tm_dt32, tm_dnut32, tm_wt32;  // 32-wide boxes (tail tiles)
  uint32_t* sym_masks = nullptr;         // tie k-masks per (tile pair, 32-wide k chunk)
  uint32_t* sym_tile_flags = nullptr;
  unsigned long long* sym_count = nullptr;
  unsigned int* round_bar = nullptr;     // round barrier counter of the pair kernel
  // Rank-coded pass 1 (pairwise, n <= 32768; pald_rank.cuh): RA / RB panels.
  uint32_t* rank_a = nullptr;
  uint16_t* rank_b = nullptr;
  uint32_t* rank_scratch = nullptr;      // per-CTA scratch of the rank kernels
  int* rank_fail = nullptr;              // [count, rows...] declined by the bins kernel
  int2* band_tiles = nullptr;            // pass-1 tiles by the band of their column tile (host API)
  std::vector<long long> band_units;     // unit offsets of the bands in band_tiles
  size_t rank_fail_ints = 0;
  cudaStream_t aux = nullptr;            // load: rank codes beside the range check / layout;
                                         // pass 2: tail tiles beside the pair launch
  cudaEvent_t ev_in = nullptr, ev_ranks = nullptr;
  size_t rank_scratch_words = 0;
  CUtensorMap tm_ra, tm_rb;
  bool rank_ready = false;               // RA / RB built for the loaded D
  int sym_nch = 0;
  double sym_marked = 0;                 // share of (pair, k) steps on the exact step
  int last_kernel = PALD_GPU_KERNEL_NONE;
  // Fused multi-GPU exchange: every rank's W and C mapped through CUDA IPC.
  PeerBufs peer_w{}, peer_c{};
  PeerBufs peer_u{};                 // U of every rank (int32, stored as float*): peer-pull finish
  bool peer_mapped[kMaxPeers] = {};  // opened by this plan (to be closed)
  bool peer_u_mapped[kMaxPeers] = {};
  int peer_rank = -1;
  bool sym_ready = false;                // tie scan done for the loaded D
  bool tri_marks = false;                // triplet: tie marks built with the rank codes
  bool loaded = false;
  bool exact = false;
  bool focus_dirty = false;
  int sms = 148;
  int2* focus_tiles = nullptr;  // grouped upper-triangular tile order
  std::vector<int2> pair_order;  // host copy of it (tile pairs of pass 2)
  int2* tail = nullptr;          // 64- (or 32-) wide one-sided tiles of the last partial pair round
  int tail_count = 0;
  int tail_tile = 64;            // width of the tail tiles
  int sym_main_pairs = 0;        // pairs of the full-range pair launch (rest: tail tiles)
  // Triplet pass 2 with the last partial round of pairs split along k
  // (pald_sym.cuh SPLIT items + sym_combine_kernel); built on first use.
  // [0]: fp32 partial tiles; [1]: accurate mode (double partial tiles, the
  // item list in per-CTA queues of k blocks)
  struct SplitPlan {
    int4* items = nullptr;
    int4* pairs = nullptr;
    void* partial = nullptr;
    int item_count = -1;  // -1: not built; 0: no split
    int pair_count = 0;
  } split[2];
  // Accurate mode (PALD_GPU_FLAG_ACCURATE): double sums of the fp32 block
  // partials of pass 2 (n x ld doubles, allocated on first use).
  double* c64 = nullptr;
  // One-shot host API (pald_gpu_cohesion_f32): its streams and events,
  // created on first use and kept with the cached plan.
  cudaStream_t os_s = nullptr, os_sc = nullptr, os_s2 = nullptr;
  cudaEvent_t os_ev[4 + PALD_HOST_BANDS_MAX] = {};
  std::vector<cudaEvent_t> band_ev;  // banded load: one per H2D band + the layout's
  uint64_t launches = 0;

  void close_peers() {
    for (int q = 0; q < peer_w.count; ++q) {
      if (!peer_mapped[q]) continue;
      cudaIpcCloseMemHandle(peer_w.ptr[q]);
      cudaIpcCloseMemHandle(peer_c.ptr[q]);
      peer_mapped[q] = false;
    }
    close_peer_u();
    peer_w = PeerBufs{};
    peer_c = PeerBufs{};
    peer_rank = -1;
  }
  void close_peer_u() {
    for (int q = 0; q < peer_u.count; ++q) {
      if (!peer_u_mapped[q]) continue;
      cudaIpcCloseMemHandle(peer_u.ptr[q]);
      peer_u_mapped[q] = false;
    }
    peer_u = PeerBufs{};
  }

  ~pald_gpu_plan() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(ds);
    cudaFree(dnu);
    cudaFree(u);
    cudaFree(w);
    cudaFree(c);
    cudaFree(stats);
    cudaFreeHost(stats_host);
    cudaFree(focus_tiles);
    cudaFree(tail);
    close_peers();
    cudaFree(sym_masks);
    cudaFree(sym_tile_flags);
    cudaFree(sym_count);
    cudaFree(round_bar);
    cudaFree(rank_a);
    cudaFree(rank_b);
    cudaFree(rank_scratch);
    cudaFree(rank_fail);
    cudaFree(band_tiles);
    if (aux) cudaStreamDestroy(aux);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_ranks) cudaEventDestroy(ev_ranks);
    for (auto& sp : split) {
      cudaFree(sp.items);
      cudaFree(sp.pairs);
      cudaFree(sp.partial);
    }
    cudaFree(c64);
    for (cudaStream_t st : {os_s, os_sc, os_s2})
      if (st) cudaStreamDestroy(st);
    for (cudaEvent_t e : os_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : band_ev) cudaEventDestroy(e);
    cudaSetDevice(prev);
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Tile-pair cohesion (pald_sym.cuh): PALD_GPU_SYM=0 selects the one-sided
// kernel everywhere, 2 the pair kernel wherever it applies (A/B and tests),
// default 1 = by the cost model (sym_preferred).
int sym_mode() {
  static const int m = [] {
    const char* e = getenv("PALD_GPU_SYM");
    return e ? atoi(e) : 1;
  }();
  return m;
}
bool sym_enabled() { return sym_mode() != 0; }
// PALD_GPU_SPLIT=0 keeps the triplet pass 2 on whole pairs (A/B, tests).
bool split_enabled() {
  static const int m = [] {
    const char* e = getenv("PALD_GPU_SPLIT");
    return e ? atoi(e) : 1;
  }();
  return m != 0;
}

// Accurate mode: pass-2 terms per fp32 block partial (PALD_GPU_ACC_BLOCK,
// default 1024; rounded to whole k chunks of each kernel). Measured on
// configs 3 / 2 (tools/acc_sweep.py, profiles/acc_sweep_r02.jsonl): 256-term
// blocks 2.1e-7 / 3.9e-7 max rel_diff vs fp64, 1024 7.4e-7 / 1.4e-6, 4096
// 2.8e-6 / 1.0e-5 (the plain fp32 chain: 5.4e-6 / 1.3e-5); the flush of a
// block costs one reduction per output, outside the inner loop.
// Longer blocks were measured at n = 32768 (profiles/acc_block_cfg5_r02.txt):
// 4096-term blocks save 1.5 % of pass 2 but triple the error (1.3e-6) and
// lose the 1e-7 conservation of sum(C); the default stays 1024 for every n.
int acc_block_terms(const pald_gpu_plan* p);
// Triplet C is a tolerance result (the reference's own fp32 triplet C
// depends on b_cohesion), so the triplet always accumulates accurately: one
// 4096-term fp32 chain already drifts by 1.3e-5 on config 2 (full matrix vs
// parallel_triplet<double>). PALD_GPU_TRIPLET_FP32=1 restores the plain
// fp32 chains (A/B).
bool accurate(const pald_gpu_plan* p) {
  static const bool tri_fp32 = [] {
    const char* e = getenv("PALD_GPU_TRIPLET_FP32");
    return e && atoi(e) != 0;
  }();
  return (p->flags & PALD_GPU_FLAG_ACCURATE) != 0 || (p->algorithm == PALD_GPU_TRIPLET && !tri_fp32);
}

int acc_block_terms(const pald_gpu_plan* p) {
  static const int env = [] {
    const char* e = getenv("PALD_GPU_ACC_BLOCK");
    return e ? atoi(e) : 0;
  }();
  (void)p;
  return env >= kSymBK ? env : 1024;
}

int ensure_c64(pald_gpu_plan* p) {
  if (p->c64) return PALD_GPU_OK;
  PALD_CUDA(cudaMalloc(&p->c64, p->n * p->ld * sizeof(double)));
  return PALD_GPU_OK;
}

int acc_zero_rows(pald_gpu_plan* p, uint64_t r0, uint64_t r1, cudaStream_t s);
int acc_round_rows(pald_gpu_plan* p, uint64_t r0, uint64_t r1, cudaStream_t s);

size_t sym_mask_words(const pald_gpu_plan* p) { return p->nb * (p->nb + 1) / 2 * p->sym_nch; }

// Width of the tail tiles of the pair launch (PALD_GPU_TAIL: 0 none, 32, 64;
// default -1: the cheaper of 32 and 64 by tail_rounds).
int tail_width() {
  static const int w = [] {
    const char* e = getenv("PALD_GPU_TAIL");
    const int v = e ? atoi(e) : -1;
    return (v == 0 || v == 32 || v == 64) ? v : -1;
  }();
  return w;
}
// Time of `count` W-wide tail tiles in pair-round units (64: 0.52 / 1.44 per
// round of 2 CTAs/SM; 32: 0.29 per round of 4 CTAs/SM, measured on config 3:
// pass 2 39.87 ms with 64-wide, 39.66 ms with 32-wide tail tiles).
double tail_rounds_w(const pald_gpu_plan* p, int width, int count) {
  if (count <= 0) return 0.0;
  const double sms = p->sms;
  return width == 32 ? std::ceil(count / (4.0 * sms)) * 0.29 : std::ceil(count / (2.0 * sms)) * 0.52 / 1.44;
}
double tail_rounds(const pald_gpu_plan* p, int count) { return tail_rounds_w(p, p->tail_tile, count); }

// The W-wide one-sided tiles covering pairs [first, end) of the pair order:
// direct tiles (P, Q), then (Q, P).
std::vector<int2> make_tail_list(const pald_gpu_plan* p, int first, int end, int W) {
  std::vector<int2> t;
  const int f = kTile / W, nbw = (int)((p->n + W - 1) / W);
  for (int i = first; i < end; ++i) {
    const int P = p->pair_order[i].x, Q = p->pair_order[i].y;
    for (int h = 0; h < (P == Q ? 1 : 2); ++h) {
      const int R = h ? Q : P, Cc = h ? P : Q;
      for (int a = 0; a < f; ++a)
        for (int b = 0; b < f; ++b)
          if (f * R + a < nbw && f * Cc + b < nbw) t.push_back(make_int2(f * R + a, f * Cc + b));
    }
  }
  return t;
}

int plan_alloc(pald_gpu_plan* p) {
  const size_t bytes = p->n * p->ld * 4;
  PALD_CUDA(cudaMalloc(&p->ds, bytes));
  PALD_CUDA(cudaMalloc(&p->dnu, bytes));
  PALD_CUDA(cudaMalloc(&p->u, bytes));
  PALD_CUDA(cudaMalloc(&p->w, bytes));
  PALD_CUDA(cudaMalloc(&p->c, bytes));
  PALD_CUDA(cudaMemset(p->ds, 0, bytes));
  PALD_CUDA(cudaMemset(p->dnu, 0, bytes));
  PALD_CUDA(cudaMemset(p->c, 0, bytes));
  PALD_CUDA(cudaMalloc(&p->stats, sizeof(Stats)));
  {
    // Focus tile order: groups of kGroupRows tile rows; inside a group,
    // column by column, the group's rows r <= c. Concurrently resident CTAs
    // then share few row and column panels in L2.
    std::vector<int2> order;
    const int nb = (int)p->nb;
    order.reserve((size_t)nb * (nb + 1) / 2);
    for (int g0 = 0; g0 < nb; g0 += kGroupRows)
      for (int c = g0; c < nb; ++c)
        for (int r = g0; r < std::min(nb, g0 + kGroupRows) && r <= c; ++r) order.push_back(make_int2(r, c));
    PALD_CUDA(cudaMalloc(&p->focus_tiles, order.size() * sizeof(int2)));
    PALD_CUDA(cudaMemcpy(p->focus_tiles, order.data(), order.size() * sizeof(int2), cudaMemcpyHostToDevice));
    p->pair_order = order;
  }
  {
    // Tail of the full-range pair launch: the last partial round of L < 148
    // pairs keeps L SMs busy for a whole pair time. When it is cheaper, those
    // pairs run instead as W-wide one-sided tiles (W = 64: 2 CTAs/SM, ~0.36
    // of a pair time per round; W = 32: 4 CTAs/SM; identical in-order sums).
    const std::vector<int2>& order = p->pair_order;
    const int G = p->sms, pairs = (int)order.size(), L = pairs > G ? pairs % G : 0;
    p->sym_main_pairs = pairs;
    int W = tail_width();
    if (W < 0)
      W = tail_rounds_w(p, 32, (int)make_tail_list(p, pairs - L, pairs, 32).size()) <
                  tail_rounds_w(p, 64, (int)make_tail_list(p, pairs - L, pairs, 64).size())
              ? 32
              : 64;
    p->tail_tile = W;
    if (L > 0 && W > 0) {
      const std::vector<int2> tl = make_tail_list(p, pairs - L, pairs, W);
      if (tail_rounds(p, (int)tl.size()) < 1.0) {
        PALD_CUDA(cudaMalloc(&p->tail, tl.size() * sizeof(int2)));
        PALD_CUDA(cudaMemcpy(p->tail, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice));
        p->tail_count = (int)tl.size();
        p->sym_main_pairs = pairs - L;
      }
    }
  }
  PALD_CUDA(cudaMallocHost(&p->stats_host, sizeof(Stats)));
  int rc;
  if ((rc = make_map(&p->tm_d, p->ds, p->n, p->ld))) return rc;
  if ((rc = make_map(&p->tm_dnu, p->dnu, p->n, p->ld))) return rc;
  if ((rc = make_map(&p->tm_w, p->w, p->n, p->ld))) return rc;
  if ((rc = make_map(&p->tm_d64, p->ds, p->n, p->ld, 64))) return rc;
  if ((rc = make_map(&p->tm_dnu64, p->dnu, p->n, p->ld, 64))) return rc;
  if ((rc = make_map(&p->tm_w64, p->w, p->n, p->ld, 64))) return rc;
  if ((rc = make_map(&p->tm_dt32, p->ds, p->n, p->ld, 32))) return rc;
  if ((rc = make_map(&p->tm_dnut32, p->dnu, p->n, p->ld, 32))) return rc;
  if ((rc = make_map(&p->tm_wt32, p->w, p->n, p->ld, 32))) return rc;
  // Pair-kernel state for every algorithm / policy: the one-shot APIs
  // reuse a cached plan across calls with other options (same n).
  if ((rc = make_map(&p->tm_d32, p->ds, p->n, p->ld, kTile, kSymBK))) return rc;
  if ((rc = make_map(&p->tm_dnu32, p->dnu, p->n, p->ld, kTile, kSymBK))) return rc;
  if ((rc = make_map(&p->tm_w32, p->w, p->n, p->ld, kTile, kSymBK))) return rc;
  p->sym_nch = (int)((p->n + kSymBK - 1) / kSymBK);
  PALD_CUDA(cudaMalloc(&p->round_bar, sizeof(unsigned int)));
  PALD_CUDA(cudaMalloc(&p->sym_masks, sym_mask_words(p) * sizeof(uint32_t)));
  PALD_CUDA(cudaMalloc(&p->sym_tile_flags, p->nb * sizeof(uint32_t)));
  PALD_CUDA(cudaMalloc(&p->sym_count, sizeof(unsigned long long)));
  // The memsets above run on the legacy default stream; callers may use
  // non-blocking streams, so finish them before the plan is handed out.
  PALD_CUDA(cudaDeviceSynchronize());
  return PALD_GPU_OK;
}

int grid_rows(uint64_t n) { return (int)std::min<uint64_t>(n, 148ull * 16); }


// Rank-coded pass 1 (pald_rank.cuh): pairwise and triplet focus with
// 2048 < n <= 32768 (below that the code build costs more than the faster
// pass 1 saves).
// PALD_GPU_RANK=0 keeps the fp32 / integer-key compare path everywhere, 2
// forces the rank path for every n <= 32768 (A/B, tests).
bool rank_wanted(const pald_gpu_plan* p) {
  static const int m = [] {
    const char* e = getenv("PALD_GPU_RANK");
    return e ? atoi(e) : 1;
  }();
  if (m == 0 || p->n < 2 || p->n > (uint64_t)kRankMaxN) return false;
  if (p->algorithm == PALD_GPU_TRIPLET && p->policy != PALD_GPU_STRICT) return false;
  return m == 2 || p->n > 2048;
}

int ensure_rank_scratch(pald_gpu_plan* p, size_t words) {
  if (words <= p->rank_scratch_words) return PALD_GPU_OK;
  cudaFree(p->rank_scratch);
  p->rank_scratch = nullptr;
  p->rank_scratch_words = 0;
  PALD_CUDA(cudaMalloc(&p->rank_scratch, words * 4));
  p->rank_scratch_words = words;
  return PALD_GPU_OK;
}

// Source keys of the rank codes: the plan's layout of D (scaled fp32 bits
// or exact-path keys 2*bits), or the raw fp32 D with the sign bit masked
// (the banded host path, before the range check; positive floats order as
// their bits, and scaling by 2^p is exact, so the ranks are the same).
struct RankSrc {
  const uint32_t* keys;
  uint32_t mask;
  int end_bit;    // CUB sort: significant key bits
  bool bins;      // value-linear bins apply (finite fp32 keys, or raw fp32)
  size_t key_ld;  // row stride of keys
};

RankSrc rank_src_layout(const pald_gpu_plan* p) {
  return {p->ds, 0xffffffffu, p->exact ? 32 : 30, !p->exact, p->ld};  // fast layout: scaled values < 1.0
}
RankSrc rank_src_raw(const float* d, uint64_t ldd) {
  return {reinterpret_cast<const uint32_t*>(d), 0x7fffffffu, 31, true, ldd};
}

// Bins path of the rank codes: THREADS x E keys per row, rows [r0, r1);
// declined rows appended to (fail_rows, *fail_count).
template <int THREADS, int E>
int launch_rank_bins(pald_gpu_plan* p, const RankSrc& src, uint16_t* rk, const TieMarks& tm, int r0, int r1,
                     int* fail_rows, int* fail_count, cudaStream_t s) {
  auto k = row_rank_bins_kernel<THREADS, E>;
  const int n = (int)p->n, smem = rank_bin_smem(THREADS * E);
  PALD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 1;
  PALD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  const int grid = std::min(r1 - r0, p->sms * std::max(1, per_sm));
  if (grid <= 0) return PALD_GPU_OK;
  k<<<grid, THREADS, smem, s>>>(src.keys, n, (int)p->ld, rk, fail_rows, fail_count, tm, r0, r1, src.mask,
                                src.key_ld);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}

int launch_rank_bins_n(pald_gpu_plan* p, const RankSrc& src, uint16_t* rk, const TieMarks& tm, int r0, int r1,
                       int* fail_rows, int* fail_count, cudaStream_t s) {
  const int n = (int)p->n;
  return n <= 4096    ? launch_rank_bins<256, 16>(p, src, rk, tm, r0, r1, fail_rows, fail_count, s)
         : n <= 8192  ? launch_rank_bins<512, 16>(p, src, rk, tm, r0, r1, fail_rows, fail_count, s)
         : n <= 16384 ? launch_rank_bins<1024, 16>(p, src, rk, tm, r0, r1, fail_rows, fail_count, s)
                      : launch_rank_bins<1024, 32>(p, src, rk, tm, r0, r1, fail_rows, fail_count, s);
}

// Sort path of the rank codes over all rows (rows == nullptr) or over the
// rows listed by the bins kernel (count on the device).
template <int THREADS, int ITEMS>
int launch_row_rank(pald_gpu_plan* p, const RankSrc& src, uint16_t* rk, const int* rows, const int* count,
                    cudaStream_t s) {
  using Cfg = RankCfg<THREADS, ITEMS>;
  auto k = row_rank_kernel<THREADS, ITEMS>;
  const int n = (int)p->n, smem = Cfg::smem_bytes(n);
  PALD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 1;
  PALD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  const int grid = std::min(n, p->sms * std::max(1, per_sm));
  int rc = ensure_rank_scratch(p, (size_t)grid * std::max(n, Cfg::kSeg));
  if (rc) return rc;
  k<<<grid, THREADS, smem, s>>>(src.keys, n, (int)p->ld, src.end_bit, rows, count, rk, p->rank_scratch, src.mask,
                                src.key_ld);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}

int launch_row_rank_n(pald_gpu_plan* p, const RankSrc& src, uint16_t* rk, const int* rows, const int* count,
                      cudaStream_t s) {
  const int n = (int)p->n;
  return n <= 2048   ? launch_row_rank<256, 8>(p, src, rk, rows, count, s)
         : n <= 4096 ? launch_row_rank<256, 16>(p, src, rk, rows, count, s)
         : n <= 8192 ? launch_row_rank<256, 32>(p, src, rk, rows, count, s)
                     : launch_row_rank<512, 32>(p, src, rk, rows, count, s);
}

// RA / RB columns [r0, r1) (r1 = n: through the padding columns up to ld).
int launch_rank_layout(pald_gpu_plan* p, const uint16_t* rk, int r0, int r1, cudaStream_t s) {
  const int n = (int)p->n, ld = (int)p->ld;
  const int rc1 = r1 >= n ? ld : r1;
  if (rc1 <= r0) return PALD_GPU_OK;
  rank_layout_kernel<<<dim3((unsigned)((rc1 - r0 + 31) / 32), (unsigned)((p->n + 31) / 32)), 256, 0, s>>>(
      rk, n, ld, p->rank_a, p->rank_b, r0);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}

int ensure_rank_buffers(pald_gpu_plan* p, size_t fail_ints) {
  if (!p->rank_a) {
    PALD_CUDA(cudaMalloc(&p->rank_a, p->n * p->ld * 4));
    PALD_CUDA(cudaMalloc(&p->rank_b, p->n * p->ld * 2));
    int rc;
    if ((rc = make_map(&p->tm_ra, p->rank_a, p->n, p->ld, kTile, kBK, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4))) return rc;
    if ((rc = make_map(&p->tm_rb, p->rank_b, p->n, p->ld, kTile, kBK, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2))) return rc;
  }
  if (fail_ints > p->rank_fail_ints) {
    cudaFree(p->rank_fail);
    p->rank_fail = nullptr;
    p->rank_fail_ints = 0;
    PALD_CUDA(cudaMalloc(&p->rank_fail, fail_ints * sizeof(int)));
    p->rank_fail_ints = fail_ints;
  }
  return PALD_GPU_OK;
}

// Builds RA / RB from src (n rows), using W as the Rk scratch (W is zeroed
// afterwards by the caller). With mark_ties, the bins kernel marks the pair
// kernel's ties of its rows and tie_scan_kernel those of the rows it
// declined (the masks must be zeroed before).
int launch_tie_scan(pald_gpu_plan* p, const uint32_t* keys, const int* rows, const int* count, cudaStream_t s,
                    uint64_t key_ld);

int build_rank_codes(pald_gpu_plan* p, const RankSrc& src, bool mark_ties, cudaStream_t s) {
  int rc = ensure_rank_buffers(p, p->n + 1);
  if (rc) return rc;
  const int n = (int)p->n;
  uint16_t* rk = reinterpret_cast<uint16_t*>(p->w);  // W[0, n*ld*2 B)
  const int* rows = nullptr;
  const int* count = nullptr;
  if (src.bins) {  // value-linear bins; declined rows -> sort path
    PALD_CUDA(cudaMemsetAsync(p->rank_fail, 0, sizeof(int), s));
    const TieMarks tm{mark_ties ? p->sym_masks : nullptr, p->sym_tile_flags, (int)p->nb, p->sym_nch};
    if ((rc = launch_rank_bins_n(p, src, rk, tm, 0, n, p->rank_fail + 1, p->rank_fail, s))) return rc;
    rows = p->rank_fail + 1;
    count = p->rank_fail;
  }
  if ((rc = launch_row_rank_n(p, src, rk, rows, count, s))) return rc;
  if (mark_ties && (rc = launch_tie_scan(p, src.keys, rows, count, s, src.key_ld))) return rc;
  if ((rc = launch_rank_layout(p, rk, 0, n, s))) return rc;
  p->rank_ready = true;
  return PALD_GPU_OK;
}

bool sym_wins(const pald_gpu_plan* p, double marked);

// Duplicate scan of the columns (all, or the listed rows) of keys (n x ld).
int launch_tie_scan(pald_gpu_plan* p, const uint32_t* keys, const int* rows, const int* count, cudaStream_t s,
                    uint64_t key_ld) {
  static bool attr_done[64] = {};
  if (!attr_done[p->device & 63]) {
    PALD_CUDA(cudaFuncSetAttribute(tie_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTieSmem));
    attr_done[p->device & 63] = true;
  }
  const int passes = (int)((p->n + kTieCap * 3 / 4 - 1) / (kTieCap * 3 / 4));
  tie_scan_kernel<<<(unsigned)std::min<uint64_t>(p->n, (uint64_t)p->sms), kTieThreads, kTieSmem, s>>>(
      keys, (int)p->n, (int)(key_ld ? key_ld : p->ld), (int)p->nb, p->sym_nch, passes, p->sym_masks,
      p->sym_tile_flags, rows, count);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}

int check_stats(const pald_gpu_plan* p, const Stats& st, bool validate, bool* fast_out, int* p2_out,
                const float* d, uint64_t ldd);
int tie_summary(pald_gpu_plan* p, cudaStream_t s);

int ensure_aux(pald_gpu_plan* p) {
  if (p->aux) return PALD_GPU_OK;
  PALD_CUDA(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking));
  PALD_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
  PALD_CUDA(cudaEventCreateWithFlags(&p->ev_ranks, cudaEventDisableTiming));
  return PALD_GPU_OK;
}

int ensure_oneshot(pald_gpu_plan* p) {
  if (p->os_s) return PALD_GPU_OK;
  PALD_CUDA(cudaStreamCreateWithFlags(&p->os_s, cudaStreamNonBlocking));
  PALD_CUDA(cudaStreamCreateWithFlags(&p->os_sc, cudaStreamNonBlocking));
  PALD_CUDA(cudaStreamCreateWithFlags(&p->os_s2, cudaStreamNonBlocking));
  for (int i = 0; i < 4 + PALD_HOST_BANDS_MAX; ++i)
    PALD_CUDA(cudaEventCreateWithFlags(&p->os_ev[i], i < 4 ? cudaEventDefault : cudaEventDisableTiming));
  return PALD_GPU_OK;
}

// Tie marks (duplicate values per row, pald_sym.cuh) built with the rank
// codes: the pairwise Strict pair kernel needs them to share its compares;
// the triplet uses them to run the chunks inside the row / column tiles on
// the fast steps (an unmarked k cannot meet the tie the nu() transforms
// decide, in either pass).
bool tie_marks_wanted(const pald_gpu_plan* p) {
  static const int m = [] {
    const char* e = getenv("PALD_GPU_TRI_MARKS");  // 0: triplet without marks (A/B)
    return e ? atoi(e) : 1;
  }();
  if (!p->sym_masks || !sym_enabled()) return false;
  if (p->algorithm == PALD_GPU_PAIRWISE) return p->policy == PALD_GPU_STRICT;
  return m != 0;
}

int plan_load_impl(pald_gpu_plan* p, const float* dD, uint64_t ldd, cudaStream_t s) {
  const int n = (int)p->n;
  Stats init{};
  init.min_pos_bits = 0xffffffffu;
  init.key_diag = init.key_notpos = init.key_asym = ~0ull;
  *p->stats_host = init;
  int rc;
  p->rank_ready = false;
  p->sym_ready = false;
  p->sym_marked = 0;
  // Rank codes (pald_rank.cuh) from the raw fp32 bits of D on the aux
  // stream, concurrent with the range check and the layout (ranks need no
  // range check: positive floats order as their bits, and the scaling of the
  // fast layout is exact). The bins kernel also marks the pair kernel's ties.
  const bool ranks = rank_wanted(p);
  const bool mark = ranks && tie_marks_wanted(p);
  p->tri_marks = false;
  if (ranks) {
    if ((rc = ensure_aux(p))) return rc;
    PALD_CUDA(cudaEventRecord(p->ev_in, s));  // D is ready in stream order of s
    PALD_CUDA(cudaStreamWaitEvent(p->aux, p->ev_in, 0));
    if (mark) {
      PALD_CUDA(cudaMemsetAsync(p->sym_masks, 0, sym_mask_words(p) * sizeof(uint32_t), p->aux));
      PALD_CUDA(cudaMemsetAsync(p->sym_tile_flags, 0, p->nb * sizeof(uint32_t), p->aux));
    }
    if ((rc = build_rank_codes(p, rank_src_raw(dD, ldd), mark, p->aux))) return rc;
    PALD_CUDA(cudaEventRecord(p->ev_ranks, p->aux));
  }
  PALD_CUDA(cudaMemcpyAsync(p->stats, p->stats_host, sizeof(Stats), cudaMemcpyHostToDevice, s));
  const bool validate = !(p->flags & PALD_GPU_FLAG_SKIP_VALIDATION);
  stats_kernel<<<grid_rows(p->n), 256, 0, s>>>(dD, ldd, n, validate ? 1 : 0, p->stats, 0, n);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  PALD_CUDA(cudaMemcpyAsync(p->stats_host, p->stats, sizeof(Stats), cudaMemcpyDeviceToHost, s));
  PALD_CUDA(cudaStreamSynchronize(s));
  bool fast = false;
  int p2 = 0;
  if ((rc = check_stats(p, *p->stats_host, validate, &fast, &p2, dD, ldd))) {
    if (ranks) cudaStreamSynchronize(p->aux);  // leave no work behind on the plan
    p->rank_ready = false;
    return rc;
  }
  p->exact = !fast;
  layout_kernel<<<grid_rows(p->n), 256, 0, s>>>(dD, ldd, n, p->ld, fast ? 1 : 0, p2, p->ds,
                                                       p->dnu);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  if (ranks) PALD_CUDA(cudaStreamWaitEvent(s, p->ev_ranks, 0));  // W held the rank scratch
  // W accumulates the pass-1 counts; U needs no clearing (focus_finish
  // writes every entry r, c < n; the row padding is never read)
  PALD_CUDA(cudaMemsetAsync(p->w, 0, p->n * p->ld * 4, s));
  // Triplet: the pair kernel's shared indicator is exact without a scan
  // (its per-element chunks, those inside the row or column tile, cost too
  // little to enter the cost model: tools/time_n.py). Pairwise: the
  // duplicate scan of the columns of D (marks of the tile-pair kernel) is
  // skipped where the pair kernel cannot win even tie-free.
  if (fast && p->algorithm == PALD_GPU_TRIPLET && sym_enabled() && sym_wins(p, 0.0)) p->sym_ready = true;
  p->tri_marks = mark && p->algorithm == PALD_GPU_TRIPLET;
  // (a cached plan made for a strict call keeps its masks when reused for
  // InclusiveSplit: the pair kernel is strict-only)
  const bool tie_scan = fast && p->sym_masks && p->algorithm == PALD_GPU_PAIRWISE && p->policy == PALD_GPU_STRICT &&
                        sym_enabled() && sym_wins(p, 0.0);
  if (tie_scan) {
    if (!mark) {  // no rank codes: scan every column of the layout
      PALD_CUDA(cudaMemsetAsync(p->sym_masks, 0, sym_mask_words(p) * sizeof(uint32_t), s));
      PALD_CUDA(cudaMemsetAsync(p->sym_tile_flags, 0, p->nb * sizeof(uint32_t), s));
      if ((rc = launch_tie_scan(p, p->ds, nullptr, nullptr, s, 0))) return rc;
    }
    if ((rc = tie_summary(p, s))) return rc;
  }
  p->loaded = true;
  p->focus_dirty = false;
  return PALD_GPU_OK;
}

// Validation errors of the reference (types.hpp:45-65) and the range check
// of the FFMA.SAT compare path: scale by 2^p2 so that the largest value lies
// in [0.5, 1); all values must stay >= 2^-102.
int check_stats(const pald_gpu_plan* p, const Stats& st, bool validate, bool* fast_out, int* p2_out,
                const float* d, uint64_t ldd) {
  if (validate && (st.diag_nonzero || st.offdiag_not_positive || st.asymmetric)) {
    // the reference's first violation (types.hpp:50-62): smallest key;
    // positivity before symmetry on the same entry
    const unsigned long long k = std::min(st.key_diag, std::min(st.key_notpos, st.key_asym));
    const unsigned long long x = k / p->n, y = k % p->n;
    if (k == st.key_diag)
      return set_error(PALD_GPU_ERR_VALIDATION, "distance matrix diagonal entry (%llu,%llu) is nonzero", x, x);
    if (k == st.key_notpos) {
      float v = NAN;
      if (d) cudaMemcpy(&v, d + x * ldd + y, sizeof(float), cudaMemcpyDefault);
      char num[64];
      if (std::isnan(v)) snprintf(num, sizeof(num), "%snan", std::signbit(v) ? "-" : "");
      else snprintf(num, sizeof(num), "%f", (double)v);  // std::to_string(double)
      return set_error(PALD_GPU_ERR_VALIDATION,
                       "off-diagonal distance (%llu,%llu) must be positive, got %s (duplicate points are rejected)",
                       x, y, num);
    }
    return set_error(PALD_GPU_ERR_VALIDATION, "distance matrix not symmetric at (%llu,%llu)", x, y);
  }
  bool fast = !(p->flags & PALD_GPU_FLAG_FORCE_EXACT) && !st.offdiag_zero && !st.has_inf &&
              !st.has_nan && st.min_pos_bits != 0xffffffffu;
  int p2 = 0;
  if (fast) {
    float vmax, vmin;
    uint32_t mb = st.max_bits, nbits = st.min_pos_bits;
    std::memcpy(&vmax, &mb, 4);
    std::memcpy(&vmin, &nbits, 4);
    int e = 0;
    std::frexp(vmax, &e);  // vmax = f * 2^e, f in [0.5, 1)
    p2 = -e;
    const double scaled_min = std::ldexp((double)vmin, p2);
    if (!(scaled_min >= std::ldexp(1.0, -102))) fast = false;
  }
  *fast_out = fast;
  *p2_out = p2;
  return PALD_GPU_OK;
}

// Marked-step share of the pair kernel's tie masks (cost model input);
// the pair kernel may run afterwards. Synchronizes s.
int tie_summary(pald_gpu_plan* p, cudaStream_t s) {
  {
    const size_t words = sym_mask_words(p);
    PALD_CUDA(cudaMemsetAsync(p->sym_count, 0, sizeof(unsigned long long), s));
    tie_count_kernel<<<(unsigned)p->sms * 4, 256, 0, s>>>(p->sym_masks, words, p->sym_count);
    PALD_CUDA(cudaGetLastError());
    ++p->launches;
    unsigned long long marked = 0;
    std::vector<uint32_t> tf(p->nb);
    PALD_CUDA(cudaMemcpyAsync(&marked, p->sym_count, sizeof(marked), cudaMemcpyDeviceToHost, s));
    PALD_CUDA(cudaMemcpyAsync(tf.data(), p->sym_tile_flags, tf.size() * 4, cudaMemcpyDeviceToHost, s));
    PALD_CUDA(cudaStreamSynchronize(s));
    // Pairs touching a fully marked tile run the exact step everywhere.
    uint64_t full_pairs = 0, flagged_tiles = 0;
    for (uint64_t P = 0; P < p->nb; ++P) {
      flagged_tiles += tf[P] != 0;
      for (uint64_t Q = P; Q < p->nb; ++Q) full_pairs += (tf[P] | tf[Q]) != 0;
    }
    const double pairs = (double)(p->nb * (p->nb + 1) / 2);
    const double steps = pairs * (double)p->n;
    p->sym_marked = std::min(1.0, ((double)marked + (double)full_pairs * (double)p->n) / steps);
    p->sym_ready = true;
    if (getenv("PALD_GPU_DEBUG_TIES"))
      fprintf(stderr, "[pald_gpu] tie scan: %.4f%% of (pair, k) steps exact, %llu of %llu tiles fully\n",
              100.0 * p->sym_marked, (unsigned long long)flagged_tiles, (unsigned long long)p->nb);
  }
  return PALD_GPU_OK;
}

uint64_t focus_units(const pald_gpu_plan* p) {
  return p->nb * (p->nb + 1) / 2 * ((p->n + kBK - 1) / kBK);
}

int launch_focus_range(pald_gpu_plan* p, long long ub, long long ue, const int2* tile_list, cudaStream_t s,
                       bool peers);

// Pass 1, share `part` of `parts` equal shares of the work units: integer
// focus counts accumulated into the W buffer.
int plan_focus_counts_impl(pald_gpu_plan* p, uint64_t part, uint64_t parts, cudaStream_t s,
                           bool peers = false) {
  if (!p->loaded) return set_error(PALD_GPU_ERR_VALIDATION, "plan has no distances loaded");
  if (parts < 1 || part >= parts) return set_error(PALD_GPU_ERR_VALIDATION, "invalid share %llu of %llu",
                                                   (unsigned long long)part, (unsigned long long)parts);
  if (peers && p->peer_rank < 0) return set_error(PALD_GPU_ERR_VALIDATION, "no peers attached");
  if (peers && p->focus_dirty)  // peers may already be adding into this W
    return set_error(PALD_GPU_ERR_VALIDATION, "fused pass 1 needs a fresh load (W zeroed on every rank)");
  if (p->focus_dirty) {  // counts accumulate into W: start from zero again
    PALD_CUDA(cudaMemsetAsync(p->u, 0, p->n * p->ld * 4, s));
    PALD_CUDA(cudaMemsetAsync(p->w, 0, p->n * p->ld * 4, s));
  }
  p->focus_dirty = true;
  const uint64_t units = focus_units(p);
  const long long ub = (long long)(units * part / parts), ue = (long long)(units * (part + 1) / parts);
  return launch_focus_range(p, ub, ue, p->focus_tiles, s, peers);
}

// Pass-1 work units [ub, ue) of a tile list (unit = tile * nchunks + chunk).
int launch_focus_range(pald_gpu_plan* p, long long ub, long long ue, const int2* tile_list, cudaStream_t s,
                       bool peers) {
  if (ue <= ub) return PALD_GPU_OK;
  const long long tiles = (long long)(p->nb * (p->nb + 1) / 2);
  KernelArgs a{p->ds, p->u, p->w, p->c, (int)p->n, (int)p->ld, (int)p->nb, 0, (int)p->nb, tiles, ub, ue,
               tile_list, kGroupRows, p->peer_w};
  const int grid = (int)std::min<long long>(ue - ub, (long long)p->sms * (p->rank_ready ? ctas_per_sm(kTile, true) : 1));
  int rc;
  const bool tri = p->algorithm == PALD_GPU_TRIPLET;
  const bool split = p->policy == PALD_GPU_INCLUSIVE_SPLIT;
  const CUtensorMap &md = p->tm_d, &mn = p->tm_dnu, &mw = p->tm_w;
  if (p->rank_ready) {  // rank-coded packed compares (exact for both layouts)
    KernelArgs ar = a;
    ar.d = p->rank_a;
    if (tri && p->tri_marks) {
      ar.tie_masks = p->sym_masks;
      ar.tie_tile_flags = p->sym_tile_flags;
      ar.tie_nch = p->sym_nch;
    }
    const CUtensorMap &ra = p->tm_ra, &rb = p->tm_rb;
    if (peers)
      rc = tri     ? launch_tile<0, true, true, true, false, true, false, kTile, false, true, true>(ra, rb, mw, ar, grid, s)
           : split ? launch_tile<0, false, false, true, false, true, false, kTile, false, true, true>(ra, rb, mw, ar, grid, s)
                   : launch_tile<0, false, false, false, false, true, false, kTile, false, true, true>(ra, rb, mw, ar, grid, s);
    else
      rc = tri     ? launch_tile<0, true, true, true, false, true, false, kTile, false, false, true>(ra, rb, mw, ar, grid, s)
           : split ? launch_tile<0, false, false, true, false, true, false, kTile, false, false, true>(ra, rb, mw, ar, grid, s)
                   : launch_tile<0, false, false, false, false, true, false, kTile, false, false, true>(ra, rb, mw, ar, grid, s);
  } else if (peers) {  // counts RED'd straight into every rank's W over NVLink
    if (!p->exact) {
      rc = tri     ? launch_tile<0, true, true, true, false, true, false, kTile, false, true>(md, mn, mw, a, grid, s)
           : split ? launch_tile<0, false, false, true, false, true, false, kTile, false, true>(md, mn, mw, a, grid, s)
                   : launch_tile<0, false, false, false, false, true, false, kTile, false, true>(md, mn, mw, a, grid, s);
    } else {
      rc = tri     ? launch_tile<0, true, true, true, false, false, false, kTile, false, true>(md, mn, mw, a, grid, s)
           : split ? launch_tile<0, false, false, true, false, false, false, kTile, false, true>(md, mn, mw, a, grid, s)
                   : launch_tile<0, false, false, false, false, false, false, kTile, false, true>(md, mn, mw, a, grid, s);
    }
  } else if (!p->exact) {
    rc = tri     ? launch_tile<0, true, true, true, false, true>(md, mn, mw, a, grid, s)
         : split ? launch_tile<0, false, false, true, false, true>(md, mn, mw, a, grid, s)  // <= : < nu(T)
                 : launch_tile<0, false, false, false, false, true>(md, mn, mw, a, grid, s);
  } else {
    rc = tri     ? launch_tile<0, true, true, true, false, false>(md, mn, mw, a, grid, s)
         : split ? launch_tile<0, false, false, true, false, false>(md, mn, mw, a, grid, s)
                 : launch_tile<0, false, false, false, false, false>(md, mn, mw, a, grid, s);
  }
  if (rc) return rc;
  ++p->launches;
  return PALD_GPU_OK;
}

// Counts -> U and W = 1/U over the whole matrix.
int plan_focus_finish_impl(pald_gpu_plan* p, cudaStream_t s) {
  if (!p->loaded) return set_error(PALD_GPU_ERR_VALIDATION, "plan has no distances loaded");
  const uint64_t tiles = p->nb * (p->nb + 1) / 2;
  focus_finish_kernel<false><<<(unsigned)(tiles * 4), 256, 0, s>>>(p->u, p->w, (int)p->n, (int)p->ld, (int)p->nb, 0,
                                                                  FinishPeers{});  // (u_mode unused)
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}

int plan_focus_impl(pald_gpu_plan* p, cudaStream_t s) {
  int rc = plan_focus_counts_impl(p, 0, 1, s);
  if (rc) return rc;
  return plan_focus_finish_impl(p, s);
}

template <int TILE>
int launch_cohesion(pald_gpu_plan* p, uint64_t row0, uint64_t row1, cudaStream_t s) {
  const uint64_t nbt = (p->n + TILE - 1) / TILE;
  const uint64_t tr0 = row0 / TILE, tr1 = (row1 + TILE - 1) / TILE;
  const long long tiles = (long long)((tr1 - tr0) * nbt);
  const long long nch = (long long)((p->n + kBK - 1) / kBK);
  static const int group_rows = [] {
    const char* e = getenv("PALD_GPU_GROUP_ROWS");  // tuning knob (default kGroupRows)
    return e ? std::max(1, atoi(e)) : kGroupRows;
  }();
  KernelArgs a{p->ds, p->u, p->w, p->c, (int)p->n, (int)p->ld, (int)nbt, (int)tr0, (int)tr1, tiles, 0,
               tiles * nch, nullptr, group_rows};
  const int grid = (int)std::min<long long>(tiles, (long long)p->sms * ctas_per_sm(TILE));
  const bool tri = p->algorithm == PALD_GPU_TRIPLET;
  const bool split = p->policy == PALD_GPU_INCLUSIVE_SPLIT;
  const CUtensorMap& md = TILE == 64 ? p->tm_d64 : TILE == 32 ? p->tm_dt32 : p->tm_d;
  const CUtensorMap& mn = TILE == 64 ? p->tm_dnu64 : TILE == 32 ? p->tm_dnut32 : p->tm_dnu;
  const CUtensorMap& mw = TILE == 64 ? p->tm_w64 : TILE == 32 ? p->tm_wt32 : p->tm_w;
  if (accurate(p)) {
    int rc = ensure_c64(p);
    if (rc) return rc;
    a.c64 = p->c64;
    a.acc_chunks = std::max(1, acc_block_terms(p) / kBK);
    if (!p->exact) {
      return tri     ? launch_tile<1, true, true, false, true, true, false, TILE, false, false, false, true>(md, mn, mw, a, grid, s)
             : split ? launch_tile<1, false, false, false, false, true, true, TILE, false, false, false, true>(md, mn, mw, a, grid, s)
                     : launch_tile<1, false, true, false, false, true, false, TILE, false, false, false, true>(md, mn, mw, a, grid, s);
    }
    return tri     ? launch_tile<1, true, true, false, true, false, false, TILE, false, false, false, true>(md, mn, mw, a, grid, s)
           : split ? launch_tile<1, false, false, false, false, false, true, TILE, false, false, false, true>(md, mn, mw, a, grid, s)
                   : launch_tile<1, false, true, false, false, false, false, TILE, false, false, false, true>(md, mn, mw, a, grid, s);
  }
  if (!p->exact) {
    return tri     ? launch_tile<1, true, true, false, true, true, false, TILE>(md, mn, mw, a, grid, s)
           : split ? launch_tile<1, false, false, false, false, true, true, TILE>(md, mn, mw, a, grid, s)
                   : launch_tile<1, false, true, false, false, true, false, TILE>(md, mn, mw, a, grid, s);
  }
  return tri     ? launch_tile<1, true, true, false, true, false, false, TILE>(md, mn, mw, a, grid, s)
         : split ? launch_tile<1, false, false, false, false, false, true, TILE>(md, mn, mw, a, grid, s)
                 : launch_tile<1, false, true, false, false, false, false, TILE>(md, mn, mw, a, grid, s);
}

// Tile-pair cohesion over pairs [t0, t1) of the grouped upper-triangular
// order; writes both C[P][Q] and C[Q][P] of each pair.
// One-sided pass 2 over an explicit list of 64-wide tiles.
template <int TILE>
int launch_cohesion_list(pald_gpu_plan* p, const int2* list, int count, cudaStream_t s) {
  const uint64_t nbt = (p->n + TILE - 1) / TILE;
  const long long nch = (long long)((p->n + kBK - 1) / kBK);
  KernelArgs a{p->ds, p->u, p->w, p->c, (int)p->n, (int)p->ld, (int)nbt, 0, (int)nbt, count, 0,
               (long long)count * nch, list, kGroupRows};
  const int grid = std::min(count, p->sms * ctas_per_sm(TILE));
  const bool tri = p->algorithm == PALD_GPU_TRIPLET;
  const CUtensorMap& md = TILE == 64 ? p->tm_d64 : p->tm_dt32;
  const CUtensorMap& mn = TILE == 64 ? p->tm_dnu64 : p->tm_dnut32;
  const CUtensorMap& mw = TILE == 64 ? p->tm_w64 : p->tm_wt32;
  if (accurate(p)) {
    int rc = ensure_c64(p);
    if (rc) return rc;
    a.c64 = p->c64;
    a.acc_chunks = std::max(1, acc_block_terms(p) / kBK);
    if (tri) return launch_tile<1, true, true, false, true, true, false, TILE, true, false, false, true>(md, mn, mw, a, grid, s);
    return launch_tile<1, false, true, false, false, true, false, TILE, true, false, false, true>(md, mn, mw, a, grid, s);
  }
  if (tri) return launch_tile<1, true, true, false, true, true, false, TILE, true>(md, mn, mw, a, grid, s);
  return launch_tile<1, false, true, false, false, true, false, TILE, true>(md, mn, mw, a, grid, s);
}
int launch_tail(pald_gpu_plan* p, const int2* list, int count, cudaStream_t s) {
  return p->tail_tile == 32 ? launch_cohesion_list<32>(p, list, count, s) : launch_cohesion_list<64>(p, list, count, s);
}

int launch_sym(pald_gpu_plan* p, int t0, int t1, cudaStream_t s, bool peers = false,
               bool round_sync = true) {
  if (t1 <= t0) return PALD_GPU_OK;
  static bool attr_done[64] = {};
  if (!attr_done[p->device & 63]) {
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<false, false, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true, false, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    attr_done[p->device & 63] = true;
  }
  int grid = std::min(t1 - t0, p->sms);
  // Optional round barrier (cooperative launch: all CTAs co-resident, one
  // per SM). It keeps the CTAs of a round at the same k, which cuts the
  // kernel's DRAM reads 7x (1.39 -> 0.20 TB at n = 32768, L2 hit 42 -> 85 %)
  // but costs 4 % of time waiting for each round's slowest CTA; the kernel
  // is operand-bound, not memory-bound, so it is off by default
  // (profiles/round_sync_r01.txt).
  static const int sync_mode = [] {
    const char* e = getenv("PALD_GPU_ROUND_SYNC");  // 1: round barrier on
    return e ? atoi(e) : 0;
  }();
  const bool acc = accurate(p);
  const bool sync = round_sync && sync_mode && !acc && (t1 - t0) / grid >= 2;
  if (acc) {
    const int rc = ensure_c64(p);
    if (rc) return rc;
  }
  if (sync) PALD_CUDA(cudaMemsetAsync(p->round_bar, 0, sizeof(unsigned int), s));
  SymArgs a{p->ds, p->c, p->focus_tiles, p->sym_masks, p->sym_tile_flags,
            (int)p->n, (int)p->ld, (int)p->nb, p->sym_nch, t0, t1, p->peer_c,
            sync ? p->round_bar : nullptr};
  a.c64 = p->c64;
  a.acc_chunks = std::max(1, acc_block_terms(p) / kSymBK);
  a.tri_marks = p->tri_marks ? 1 : 0;
  const bool tri = p->algorithm == PALD_GPU_TRIPLET;
  // accurate mode: whole pairs on the same persistent schedule; the kernel
  // flushes its fp32 sums into the double sums every acc_chunks chunks (the
  // chunk loop stays uniform, so the main loop is the plain kernel's) and
  // only adds into c64: PEERS stores are the rounding pass's job
  (void)peers;
  auto k = acc ? (tri ? pald_sym_cohesion_kernel<true, false, false, false, true>
                      : pald_sym_cohesion_kernel<false, false, false, false, true>)
           : sync ? (peers ? (tri ? pald_sym_cohesion_kernel<true, true, true> : pald_sym_cohesion_kernel<false, true, true>)
                        : (tri ? pald_sym_cohesion_kernel<true, false, true> : pald_sym_cohesion_kernel<false, false, true>))
                : (peers ? (tri ? pald_sym_cohesion_kernel<true, true> : pald_sym_cohesion_kernel<false, true>)
                         : (tri ? pald_sym_cohesion_kernel<true, false> : pald_sym_cohesion_kernel<false, false>));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSymSmem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = sync ? 1 : 0;
  PALD_CUDA(cudaLaunchKernelEx(&cfg, k, p->tm_d32, p->tm_dnu32, p->tm_w32, a));
  PALD_CUDA(cudaGetLastError());
  return PALD_GPU_OK;
}

// Triplet C is compared with a tolerance (the reference's own fp32 triplet C
// depends on its block size), so the pairs of the last partial round of the
// full-range pair launch can be split along k into f parts whose partial
// tiles are summed in a fixed order: ceil(L f / G) / f rounds instead of 1.
// Items: (tile row, tile col, cb | ce << 15, slot); CTA g runs items g,
// g + G, ... In accurate mode the whole pairs of the full rounds run on the
// whole-pair kernel and the list holds only the split parts, each a run of k
// blocks (acc_chunks chunks) on one CTA, all added into the double sums
// (order-independent), the queues padded with empty items.
int build_split(pald_gpu_plan* p, bool acc) {
  auto& sp = p->split[acc ? 1 : 0];
  sp.item_count = 0;
  const std::vector<int2>& order = p->pair_order;
  const int G = p->sms, pairs = (int)order.size(), L = pairs % G;
  if (pairs <= G || L == 0) return PALD_GPU_OK;
  int best_f = 1;
  double best = 1.0;
  for (int f = 2; f <= 8 && f <= p->sym_nch; ++f) {
    const double cost = std::ceil((double)L * f / G) / f;
    if (cost < best - 1e-9) {
      best = cost;
      best_f = f;
    }
  }
  if (best > 0.9) return PALD_GPU_OK;
  const int f = best_f, nch = p->sym_nch;
  auto z = [](int cb, int ce, bool, bool) { return (int)((uint32_t)cb | ((uint32_t)ce << 15)); };
  std::vector<int4> items, prs;
  for (int j = 0; j < L; ++j) {
    const int2 pr = order[pairs - L + j];
    prs.push_back(make_int4(pr.x, pr.y, j * f, f));
  }
  if (!acc) {
    for (int i = 0; i < pairs - L; ++i) items.push_back(make_int4(order[i].x, order[i].y, z(0, nch, true, true), -1));
    for (int j = 0; j < L; ++j)
      for (int q = 0; q < f; ++q)
        items.push_back(make_int4(prs[j].x, prs[j].y, z(nch * q / f, nch * (q + 1) / f, q == 0, false), j * f + q));
  } else {
    // accurate mode: the whole pairs of the full rounds run on the whole-pair
    // kernel (launch_sym); the list holds only the split parts, each cut
    // into k blocks (acc_chunks chunks) that flush into the double sums
    const int ac = std::max(1, acc_block_terms(p) / kSymBK);
    std::vector<std::vector<int4>> queue(G);
    for (int t = 0; t < L * f; ++t) {  // split parts: CTA t % G
      const int j = t / f, q = t % f, pb = nch * q / f, pe = nch * (q + 1) / f;
      for (int cb = pb; cb < pe; cb += ac)
        queue[t % G].push_back(make_int4(prs[j].x, prs[j].y, z(cb, std::min(pe, cb + ac), cb == pb, false), t));
    }
    size_t R = 0;
    for (auto& qu : queue) R = std::max(R, qu.size());
    items.assign(R * G, make_int4(0, 0, 0, -1));  // empty padding items
    for (int g = 0; g < G; ++g)
      for (size_t r = 0; r < queue[g].size(); ++r) items[r * G + g] = queue[g][r];
  }
  PALD_CUDA(cudaMalloc(&sp.items, items.size() * sizeof(int4)));
  PALD_CUDA(cudaMemcpy(sp.items, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice));
  PALD_CUDA(cudaMalloc(&sp.pairs, prs.size() * sizeof(int4)));
  PALD_CUDA(cudaMemcpy(sp.pairs, prs.data(), prs.size() * sizeof(int4), cudaMemcpyHostToDevice));
  if (!acc)  // accurate mode: the parts add straight into the double sums
    PALD_CUDA(cudaMalloc(&sp.partial, (size_t)L * f * 2 * kTile * kTile * sizeof(float)));
  sp.item_count = (int)items.size();
  sp.pair_count = L;
  return PALD_GPU_OK;
}

// Full-range triplet pass 2 through the split items; false if no split.
int launch_sym_split(pald_gpu_plan* p, cudaStream_t s, bool* used) {
  *used = false;
  const bool acc = accurate(p);
  auto& sp = p->split[acc ? 1 : 0];
  if (sp.item_count < 0) {
    const int rc = build_split(p, acc);
    if (rc) return rc;
  }
  if (sp.item_count == 0) return PALD_GPU_OK;
  static bool attr_done[64] = {};
  auto k = acc ? pald_sym_cohesion_kernel<true, false, false, true, true> : pald_sym_cohesion_kernel<true, false, false, true>;
  if (!attr_done[p->device & 63]) {
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true, false, false, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    PALD_CUDA(cudaFuncSetAttribute(pald_sym_cohesion_kernel<true, false, false, true, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem));
    attr_done[p->device & 63] = true;
  }
  int rc;
  if (acc) {  // full rounds on the whole-pair kernel, then the split parts of the last round
    if ((rc = acc_zero_rows(p, 0, p->n, s))) return rc;
    const int pairs = (int)p->pair_order.size();
    if ((rc = launch_sym(p, 0, pairs - sp.pair_count, s, false, false))) return rc;
    ++p->launches;
  }
  SymArgs a{p->ds, p->c, p->focus_tiles, p->sym_masks, p->sym_tile_flags, (int)p->n, (int)p->ld, (int)p->nb,
            p->sym_nch, 0, sp.item_count, p->peer_c, nullptr, sp.items,
            acc ? nullptr : static_cast<float*>(sp.partial), p->c64, std::max(1, acc_block_terms(p) / kSymBK),
            p->tri_marks ? 1 : 0};
  const int grid = std::min(sp.item_count, p->sms);
  k<<<grid, kThreads, kSymSmem, s>>>(p->tm_d32, p->tm_dnu32, p->tm_w32, a);
  PALD_CUDA(cudaGetLastError());
  if (acc) {  // every item added into the double sums: round them all
    if ((rc = acc_round_rows(p, 0, p->n, s))) return rc;
  } else {
    sym_combine_kernel<<<dim3((unsigned)sp.pair_count, 2, kTile / 8), 256, 0, s>>>(
        sp.pairs, static_cast<const float*>(sp.partial), p->c, (int)p->n, (int)p->ld);
    PALD_CUDA(cudaGetLastError());
    ++p->launches;
  }
  ++p->launches;
  *used = true;
  return PALD_GPU_OK;
}

// Rounds-based cost model (in one-sided 128-tile times): a pair does twice
// the outputs at ~1.44x the time of a one-sided tile (tools/microbench3.cu),
// its exact k steps ~2.45x slower than shared ones (measured on all-tied
// data); 64-wide one-sided tiles run 2 per SM at ~0.52 of a 128-tile time.
bool sym_wins(const pald_gpu_plan* p, double marked) {
  if (sym_mode() == 2) return true;
  const double sms = p->sms, nb = (double)p->nb, nb64 = (double)((p->n + 63) / 64);
  // full-range launch: main pair rounds + the 64-wide tail tiles (if any)
  const double t_sym = std::ceil(p->sym_main_pairs / sms) * 1.44 * (1.0 + 1.45 * marked) +
                       tail_rounds(p, p->tail_count) * 1.44;
  const double t_128 = std::ceil(nb * nb / sms);
  const double t_64 = std::ceil(nb64 * nb64 / (2 * sms)) * 0.52;
  return t_sym < std::min(t_128, t_64);
}
// The pair kernel implements the strict policy only (InclusiveSplit takes
// the one-sided kernel).
bool sym_preferred(const pald_gpu_plan* p) { return p->policy == PALD_GPU_STRICT && sym_wins(p, p->sym_marked); }

// Accurate mode around a pass-2 launch: the double sums are zeroed before
// (the kernels add their k-block partials with red.global.add.f64) and
// rounded to the fp32 C after.
int acc_zero_rows(pald_gpu_plan* p, uint64_t r0, uint64_t r1, cudaStream_t s) {
  int rc = ensure_c64(p);
  if (rc) return rc;
  if (r1 > r0) PALD_CUDA(cudaMemsetAsync(p->c64 + r0 * p->ld, 0, (r1 - r0) * p->ld * sizeof(double), s));
  return PALD_GPU_OK;
}
int acc_round_rows(pald_gpu_plan* p, uint64_t r0, uint64_t r1, cudaStream_t s) {
  if (r1 <= r0) return PALD_GPU_OK;
  acc_round_rows_kernel<<<(unsigned)std::min<uint64_t>(r1 - r0, (uint64_t)p->sms * 8), 256, 0, s>>>(
      p->c64, p->c, (int)p->n, (int)p->ld, (int)r0, (int)r1, p->algorithm == PALD_GPU_TRIPLET ? 1 : 0);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}
// Pairs [t0, t1) of the grouped pair order, into every buffer of `out`.
int acc_round_pairs(pald_gpu_plan* p, int t0, int t1, const PeerBufs& out, cudaStream_t s) {
  if (t1 <= t0) return PALD_GPU_OK;
  acc_round_pairs_kernel<<<dim3((unsigned)(t1 - t0), 2), 256, 0, s>>>(p->focus_tiles, t0, p->c64, out, (int)p->n,
                                                                       (int)p->ld, p->algorithm == PALD_GPU_TRIPLET ? 1 : 0);
  PALD_CUDA(cudaGetLastError());
  ++p->launches;
  return PALD_GPU_OK;
}
PeerBufs own_c(pald_gpu_plan* p) {
  PeerBufs b{};
  b.ptr[0] = p->c;
  b.count = 1;
  return b;
}

int plan_cohesion_core(pald_gpu_plan* p, uint64_t row0, uint64_t row1, cudaStream_t s);

int plan_cohesion_impl(pald_gpu_plan* p, uint64_t row0, uint64_t row1, cudaStream_t s) {
  if (!p->loaded) return set_error(PALD_GPU_ERR_VALIDATION, "plan has no distances loaded");
  row1 = std::min(row1, p->n);
  if (row0 >= row1) return PALD_GPU_OK;
  if (row0 % kTile != 0 || (row1 % kTile != 0 && row1 != p->n))
    return set_error(PALD_GPU_ERR_VALIDATION, "cohesion row range must be aligned to %d", kTile);
  const bool acc = accurate(p);
  int rc;
  if (acc && (rc = acc_zero_rows(p, row0, row1, s))) return rc;
  if ((rc = plan_cohesion_core(p, row0, row1, s))) return rc;
  return acc ? acc_round_rows(p, row0, row1, s) : PALD_GPU_OK;
}

// Pass 2 over C rows [row0, row1): the pair kernel for the full range when
// it wins, the one-sided kernel otherwise.
int plan_cohesion_core(pald_gpu_plan* p, uint64_t row0, uint64_t row1, cudaStream_t s) {
  // Less than one wave of 128-wide tiles: use 64-wide tiles (4x the tiles,
  // 2 CTAs per SM) so small problems fill the 148 SMs. Results are
  // identical: every C entry is the same in-order sum either way.
  const uint64_t tiles128 = ((row1 - row0 + kTile - 1) / kTile) * p->nb;
  if (row0 == 0 && row1 == p->n && p->sym_ready && sym_preferred(p)) {
    if (p->algorithm == PALD_GPU_TRIPLET && split_enabled()) {
      bool used = false;
      const int rc = launch_sym_split(p, s, &used);
      if (rc) return rc;
      if (used) {
        p->last_kernel = PALD_GPU_KERNEL_PAIRS;
        return PALD_GPU_OK;
      }
    }
    // 64-wide tail tiles (large n, 2+ tail rounds) run on the aux stream
    // beside the pair launch: their CTAs take the SMs that the pair launch's
    // CTAs free first (disjoint C entries, read-only inputs): n = 32768 pass
    // 2 2483.6 -> 2478.5 ms. A one-round 32-wide tail runs after it (beside
    // it, some tail CTAs were dispatched ahead of pair CTAs: config 3 pass 2
    // 39.66 -> 39.86 ms).
    int rc;
    const bool tail = p->tail_count > 0 && p->tail_tile == 64;
    if (tail) {
      if ((rc = ensure_aux(p))) return rc;
      PALD_CUDA(cudaEventRecord(p->ev_in, s));
    }
    if ((rc = launch_sym(p, 0, p->sym_main_pairs, s))) return rc;
    ++p->launches;
    p->last_kernel = PALD_GPU_KERNEL_PAIRS;
    if (tail) {
      PALD_CUDA(cudaStreamWaitEvent(p->aux, p->ev_in, 0));
      if ((rc = launch_tail(p, p->tail, p->tail_count, p->aux))) return rc;
      ++p->launches;
      PALD_CUDA(cudaEventRecord(p->ev_ranks, p->aux));
      PALD_CUDA(cudaStreamWaitEvent(s, p->ev_ranks, 0));
    } else if (p->tail_count > 0) {
      if ((rc = launch_tail(p, p->tail, p->tail_count, s))) return rc;
      ++p->launches;
    }
    return PALD_GPU_OK;
  }
  static const int force_tile = [] {
    const char* e = getenv("PALD_GPU_COHESION_TILE");  // testing knob: 32, 64 or 128
    return e ? atoi(e) : 0;
  }();
  const bool small = force_tile ? force_tile == 64 : tiles128 < (uint64_t)p->sms;
  const int rc = force_tile == 32 ? launch_cohesion<32>(p, row0, row1, s)
                 : small          ? launch_cohesion<64>(p, row0, row1, s)
                                  : launch_cohesion<kTile>(p, row0, row1, s);
  if (rc == PALD_GPU_OK) {
    ++p->launches;
    p->last_kernel = small ? PALD_GPU_KERNEL_TILE64 : PALD_GPU_KERNEL_TILE128;
  }
  return rc;
}

// Share `part` of `parts` of pass 2 into a zeroed C (see pald_gpu.h).
int plan_cohesion_share_impl(pald_gpu_plan* p, uint64_t part, uint64_t parts, cudaStream_t s) {
  if (!p->loaded) return set_error(PALD_GPU_ERR_VALIDATION, "plan has no distances loaded");
  if (parts < 1 || part >= parts) return set_error(PALD_GPU_ERR_VALIDATION, "invalid share %llu of %llu",
                                                   (unsigned long long)part, (unsigned long long)parts);
  if (parts == 1) return plan_cohesion_impl(p, 0, p->n, s);
  PALD_CUDA(cudaMemsetAsync(p->c, 0, p->n * p->ld * 4, s));
  if (p->sym_ready && sym_preferred(p)) {
    const uint64_t pairs = p->nb * (p->nb + 1) / 2;
    const int t0 = (int)(pairs * part / parts), t1 = (int)(pairs * (part + 1) / parts);
    const bool acc = accurate(p);
    int rc;
    if (acc && (rc = acc_zero_rows(p, 0, p->n, s))) return rc;
    if ((rc = launch_sym(p, t0, t1, s))) return rc;
    ++p->launches;
    p->last_kernel = PALD_GPU_KERNEL_PAIRS;
    return acc ? acc_round_pairs(p, t0, t1, own_c(p), s) : PALD_GPU_OK;
  }
  // Row bands of whole tile rows (every row costs the same).
  const uint64_t t0 = p->nb * part / parts, t1 = p->nb * (part + 1) / parts;
  return plan_cohesion_impl(p, std::min(p->n, t0 * kTile), std::min(p->n, t1 * kTile), s);
}

// Host-memory D, banded: the H2D of D runs in bands of 16 tile rows on a
// copy stream; as each band arrives, its range check (aux stream) and its
// rows' rank codes, tie marks, RA / RB columns and the pass-1 tiles whose
// rows AND columns have all arrived (tiles (P, Q), P <= Q, Q in the band)
// run on the compute stream, so pass 1 overlaps the transfer. Ranks come
// from the raw fp32 bits (sign masked): same order as the layout keys, no
// range check needed. The range check, layout and tie statistics finish
// after the last band; validation errors are reported then (after pass 1).
bool banded_wanted(const pald_gpu_plan* p) {
  static const int m = [] {
    const char* e = getenv("PALD_GPU_BANDED");  // 0: whole H2D, then load + pass 1
    return e ? atoi(e) : 1;
  }();
  return m != 0 && rank_wanted(p) && p->nb > kGroupRows;
}

int build_band_tiles(pald_gpu_plan* p) {
  if (p->band_tiles) return PALD_GPU_OK;
  const int nb = (int)p->nb, nch = (int)((p->n + kBK - 1) / kBK);
  std::vector<int2> list;
  p->band_units.assign(1, 0);
  for (int q0 = 0; q0 < nb; q0 += kGroupRows) {
    const int q1 = std::min(nb, q0 + kGroupRows);
    for (int P = 0; P < q1; ++P)
      for (int Q = std::max(P, q0); Q < q1; ++Q) list.push_back(make_int2(P, Q));
    p->band_units.push_back((long long)list.size() * nch);
  }
  PALD_CUDA(cudaMalloc(&p->band_tiles, list.size() * sizeof(int2)));
  PALD_CUDA(cudaMemcpy(p->band_tiles, list.data(), list.size() * sizeof(int2), cudaMemcpyHostToDevice));
  return PALD_GPU_OK;
}

int load_focus_banded(pald_gpu_plan* p, const float* D, cudaStream_t s, cudaStream_t sc, cudaStream_t sa) {
  const int n = (int)p->n, ld = (int)p->ld;
  const int band_rows = kGroupRows * kTile;
  const int nbands = (n + band_rows - 1) / band_rows;
  int rc;
  if ((rc = ensure_rank_buffers(p, (size_t)nbands + p->n))) return rc;
  if ((rc = build_band_tiles(p))) return rc;
  const bool validate = !(p->flags & PALD_GPU_FLAG_SKIP_VALIDATION);
  Stats init{};
  init.min_pos_bits = 0xffffffffu;
  init.key_diag = init.key_notpos = init.key_asym = ~0ull;
  *p->stats_host = init;
  PALD_CUDA(cudaMemcpyAsync(p->stats, p->stats_host, sizeof(Stats), cudaMemcpyHostToDevice, sa));
  PALD_CUDA(cudaMemsetAsync(p->w, 0, p->n * p->ld * 4, s));  // pass-1 counts
  PALD_CUDA(cudaMemsetAsync(p->rank_fail, 0, nbands * sizeof(int), s));
  const bool mark = tie_marks_wanted(p);
  p->tri_marks = mark && p->algorithm == PALD_GPU_TRIPLET;
  if (mark) {
    PALD_CUDA(cudaMemsetAsync(p->sym_masks, 0, sym_mask_words(p) * sizeof(uint32_t), s));
    PALD_CUDA(cudaMemsetAsync(p->sym_tile_flags, 0, p->nb * sizeof(uint32_t), s));
  }
  p->loaded = false;
  p->rank_ready = true;  // the pass-1 launches below run on RA / RB
  p->sym_ready = false;
  p->sym_marked = 0;
  p->focus_dirty = true;
  const uint32_t* raw = reinterpret_cast<const uint32_t*>(p->c);  // D staged in C (free until pass 2)
  const RankSrc src = rank_src_raw(p->c, p->ld);
  uint16_t* rk = reinterpret_cast<uint16_t*>(p->u);  // U is free until the focus finish
  const TieMarks tm{mark ? p->sym_masks : nullptr, p->sym_tile_flags, (int)p->nb, p->sym_nch};
  // band events (cached with the plan: one per band plus the layout's)
  while ((int)p->band_ev.size() < nbands + 1) {
    cudaEvent_t e;
    PALD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->band_ev.push_back(e);
  }
  cudaEvent_t* ev = p->band_ev.data();
  for (int b = 0; b < nbands; ++b) {
    const int r0 = b * band_rows, r1 = std::min(n, r0 + band_rows);
    hook_rows_needed((uint64_t)r0, (uint64_t)r1);  // f64io: this band converted just in time
    PALD_CUDA(cudaMemcpy2DAsync(p->c + (size_t)r0 * ld, (size_t)ld * 4, D + (size_t)r0 * n, (size_t)n * 4,
                                (size_t)n * 4, r1 - r0, cudaMemcpyHostToDevice, sc));
    PALD_CUDA(cudaEventRecord(ev[b], sc));
    PALD_CUDA(cudaStreamWaitEvent(sa, ev[b], 0));
    stats_kernel<<<std::min(r1 - r0, 148 * 16), 256, 0, sa>>>(p->c, (uint64_t)ld, n, validate ? 1 : 0, p->stats, r0,
                                                               r1);
    PALD_CUDA(cudaGetLastError());
    PALD_CUDA(cudaStreamWaitEvent(s, ev[b], 0));
    int* fail_rows = p->rank_fail + nbands + r0;
    int* fail_count = p->rank_fail + b;
    if ((rc = launch_rank_bins_n(p, src, rk, tm, r0, r1, fail_rows, fail_count, s))) return rc;
    if ((rc = launch_row_rank_n(p, src, rk, fail_rows, fail_count, s))) return rc;
    if (mark && (rc = launch_tie_scan(p, raw, fail_rows, fail_count, s, 0))) return rc;
    if ((rc = launch_rank_layout(p, rk, r0, r1, s))) return rc;
    if ((rc = launch_focus_range(p, p->band_units[b], p->band_units[b + 1], p->band_tiles, s, false))) return rc;
    p->launches += 1;
  }
  PALD_CUDA(cudaMemcpyAsync(p->stats_host, p->stats, sizeof(Stats), cudaMemcpyDeviceToHost, sa));
  PALD_CUDA(cudaStreamSynchronize(sa));
  bool fast = false;
  int p2 = 0;
  if ((rc = check_stats(p, *p->stats_host, validate, &fast, &p2, p->c, p->ld))) {
    cudaStreamSynchronize(s);  // no work left behind on the plan
    p->rank_ready = false;
    return rc;
  }
  p->exact = !fast;
  // layout for pass 2 on the aux stream, concurrent with the pass-1 tail
  layout_kernel<<<grid_rows(p->n), 256, 0, sa>>>(p->c, (uint64_t)ld, n, p->ld, fast ? 1 : 0, p2, p->ds, p->dnu);
  PALD_CUDA(cudaGetLastError());
  p->launches += 2;  // + the stats bands
  cudaEvent_t ev_layout = p->band_ev[nbands];
  PALD_CUDA(cudaEventRecord(ev_layout, sa));
  PALD_CUDA(cudaStreamWaitEvent(s, ev_layout, 0));
  if (fast && p->algorithm == PALD_GPU_TRIPLET && sym_enabled() && sym_wins(p, 0.0)) p->sym_ready = true;
  if (mark && fast && p->algorithm == PALD_GPU_PAIRWISE && sym_wins(p, 0.0) && (rc = tie_summary(p, s))) return rc;
  p->loaded = true;
  return PALD_GPU_OK;
}

// One cached plan per device for the one-shot APIs.
struct Cache {
  std::mutex mu;
  std::unique_ptr<pald_gpu_plan> plan[64];
};
Cache& cache() {
  static Cache c;
  return c;
}

int get_cached_plan(int dev, uint64_t n, const pald_gpu_opts* o, pald_gpu_plan** out) {
  auto& slot = cache().plan[dev & 63];
  if (!slot || slot->n != n) {
    slot.reset();
    pald_gpu_plan* p = nullptr;
    int rc = pald_gpu_plan_create(n, o, &p);
    if (rc) return rc;
    slot.reset(p);
  }
  slot->algorithm = o->algorithm;
  slot->policy = o->policy;
  slot->flags = o->flags;
  slot->loaded = false;
  *out = slot.get();
  return PALD_GPU_OK;
}

// Fused pass-2 share: the pair kernel stores its entries into every rank's C.
int plan_cohesion_share_peers_impl(pald_gpu_plan* p, uint64_t part, uint64_t parts, cudaStream_t s) {
  if (!p->loaded) return set_error(PALD_GPU_ERR_VALIDATION, "plan has no distances loaded");
  if (p->peer_rank < 0) return set_error(PALD_GPU_ERR_VALIDATION, "no peers attached");
  if (parts < 1 || part >= parts) return set_error(PALD_GPU_ERR_VALIDATION, "invalid share %llu of %llu",
                                                   (unsigned long long)part, (unsigned long long)parts);
  if (!(p->sym_ready && sym_preferred(p)))
    return set_error(PALD_GPU_ERR_UNSUPPORTED,
                     "fused pass 2 runs on the pair kernel only (use cohesion_share + a SUM all-reduce)");
  const uint64_t pairs = p->nb * (p->nb + 1) / 2;
  const int t0 = (int)(pairs * part / parts), t1 = (int)(pairs * (part + 1) / parts);
  const bool acc = accurate(p);
  int rc;
  if (acc && (rc = acc_zero_rows(p, 0, p->n, s))) return rc;
  if ((rc = launch_sym(p, t0, t1, s, true))) return rc;
  ++p->launches;
  p->last_kernel = PALD_GPU_KERNEL_PAIRS;
  // accurate: the kernel only adds into the local double sums; the rounding
  // pass stores this share's entries into every rank's C
  return acc ? acc_round_pairs(p, t0, t1, p->peer_c, s) : PALD_GPU_OK;
}

#include "pald_multi.cuh"

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

void pald_gpu_opts_init(pald_gpu_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(pald_gpu_opts);
  o->algorithm = PALD_GPU_PAIRWISE;
  o->policy = PALD_GPU_STRICT;
  o->device = -1;
  o->block = o->block_focus = o->block_cohesion = kTile;
}

const char* pald_gpu_last_error(void) { return g_last_error.c_str(); }

int pald_gpu_abi_version(void) { return PALD_GPU_ABI_VERSION; }

int pald_gpu_visible_devices(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

uint64_t pald_gpu_focus_units(const pald_gpu_plan* p) { return p ? focus_units(p) : 0; }

int pald_gpu_plan_create(uint64_t n, const pald_gpu_opts* o_in, pald_gpu_plan** out) {
  pald_gpu_opts oo;
  int rc = read_opts(o_in, &oo);
  if (rc || (rc = check_opts(&oo))) return rc;
  const pald_gpu_opts* o = &oo;
  if (!out) return set_error(PALD_GPU_ERR_VALIDATION, "null plan output");
  if (n < 2) return set_error(PALD_GPU_ERR_VALIDATION, "distance matrix needs n >= 2, got n=%llu", (unsigned long long)n);
  if (n > (1ull << 24)) return set_error(PALD_GPU_ERR_VALIDATION, "n=%llu exceeds 2^24 (fp32 focus counts)", (unsigned long long)n);
  int dev = o->device;
  if (dev < 0) PALD_CUDA(cudaGetDevice(&dev));
  DeviceGuard g(dev);
  int major = 0;
  PALD_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) return set_error(PALD_GPU_ERR_CUDA, "device %d is not sm_100-class", dev);
  std::unique_ptr<pald_gpu_plan> p(new pald_gpu_plan());
  p->device = dev;
  p->n = n;
  p->ld = round_up(n, 32);
  p->nb = (n + kTile - 1) / kTile;
  p->algorithm = o->algorithm;
  p->policy = o->policy;
  p->flags = o->flags;
  PALD_CUDA(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, dev));
  if ((rc = plan_alloc(p.get()))) return rc;
  *out = p.release();
  return PALD_GPU_OK;
}

int pald_gpu_plan_destroy(pald_gpu_plan* p) {
  delete p;
  return PALD_GPU_OK;
}

int pald_gpu_plan_load(pald_gpu_plan* p, const float* dD, uint64_t ldd, void* stream) {
  if (!p || !dD) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  if (ldd < p->n) return set_error(PALD_GPU_ERR_VALIDATION, "ldd < n");
  DeviceGuard g(p->device);
  return plan_load_impl(p, dD, ldd, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_load_host(pald_gpu_plan* p, const float* D, void* stream) {
  if (!p || !D) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  DeviceGuard g(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Stage the dense host matrix in the C buffer (free until pass 2).
  PALD_CUDA(cudaMemcpy2DAsync(p->c, p->ld * 4, D, p->n * 4, p->n * 4, p->n, cudaMemcpyHostToDevice, s));
  return plan_load_impl(p, p->c, p->ld, s);
}

int pald_gpu_plan_focus(pald_gpu_plan* p, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_focus_impl(p, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_focus_counts(pald_gpu_plan* p, uint64_t part, uint64_t parts, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_focus_counts_impl(p, part, parts, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_focus_finish(pald_gpu_plan* p, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_focus_finish_impl(p, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_cohesion(pald_gpu_plan* p, uint64_t r0, uint64_t r1, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_cohesion_impl(p, r0, r1, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_export_buffers(const pald_gpu_plan* p, pald_gpu_ipc_handle* w, pald_gpu_ipc_handle* c) {
  if (!p || !w || !c) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  static_assert(sizeof(pald_gpu_ipc_handle) == sizeof(cudaIpcMemHandle_t), "IPC handle size");
  DeviceGuard g(p->device);
  PALD_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(w), p->w));
  PALD_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(c), p->c));
  return PALD_GPU_OK;
}

int pald_gpu_plan_attach_peers(pald_gpu_plan* p, int world, int rank, const pald_gpu_ipc_handle* w_handles,
                               const pald_gpu_ipc_handle* c_handles) {
  if (!p || !w_handles || !c_handles) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return set_error(PALD_GPU_ERR_VALIDATION, "peers: world %d / rank %d out of range (max %d)", world, rank,
                     kMaxPeers);
  DeviceGuard g(p->device);
  p->close_peers();
  for (int q = 0; q < world; ++q) {
    if (q == rank) {
      p->peer_w.ptr[q] = p->w;
      p->peer_c.ptr[q] = p->c;
      continue;
    }
    void *pw = nullptr, *pc = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&pw, *reinterpret_cast<const cudaIpcMemHandle_t*>(&w_handles[q]),
                                         cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) {
      e = cudaIpcOpenMemHandle(&pc, *reinterpret_cast<const cudaIpcMemHandle_t*>(&c_handles[q]),
                               cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) cudaIpcCloseMemHandle(pw);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      p->peer_w.count = p->peer_c.count = q;  // close what is open
      p->close_peers();
      return set_error(PALD_GPU_ERR_COMM, "cudaIpcOpenMemHandle of rank %d: %s", q, cudaGetErrorString(e));
    }
    p->peer_w.ptr[q] = static_cast<float*>(pw);
    p->peer_c.ptr[q] = static_cast<float*>(pc);
    p->peer_mapped[q] = true;
    p->peer_w.count = p->peer_c.count = q + 1;
  }
  p->peer_w.count = p->peer_c.count = world;
  p->peer_rank = rank;
  return PALD_GPU_OK;
}

int pald_gpu_plan_export_u(const pald_gpu_plan* p, pald_gpu_ipc_handle* u) {
  if (!p || !u) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  DeviceGuard g(p->device);
  PALD_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(u), p->u));
  return PALD_GPU_OK;
}

int pald_gpu_plan_attach_peers_u(pald_gpu_plan* p, const pald_gpu_ipc_handle* u_handles) {
  if (!p || !u_handles) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  if (p->peer_rank < 0) return set_error(PALD_GPU_ERR_VALIDATION, "attach the W / C peers first");
  DeviceGuard g(p->device);
  p->close_peer_u();
  const int world = p->peer_w.count;
  for (int q = 0; q < world; ++q) {
    if (q == p->peer_rank) {
      p->peer_u.ptr[q] = reinterpret_cast<float*>(p->u);
      continue;
    }
    void* pu = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&pu, *reinterpret_cast<const cudaIpcMemHandle_t*>(&u_handles[q]),
                                               cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p->peer_u.count = q;
      p->close_peer_u();
      return set_error(PALD_GPU_ERR_COMM, "cudaIpcOpenMemHandle (U) of rank %d: %s", q, cudaGetErrorString(e));
    }
    p->peer_u.ptr[q] = static_cast<float*>(pu);
    p->peer_u_mapped[q] = true;
    p->peer_u.count = q + 1;
  }
  p->peer_u.count = world;
  return PALD_GPU_OK;
}

int pald_gpu_plan_focus_finish_peers(pald_gpu_plan* p, uint64_t part, uint64_t parts, int u_mode, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_focus_finish_peers_impl(p, part, parts, u_mode, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_detach_peers(pald_gpu_plan* p) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  p->close_peers();
  return PALD_GPU_OK;
}

int pald_gpu_plan_focus_counts_peers(pald_gpu_plan* p, uint64_t part, uint64_t parts, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_focus_counts_impl(p, part, parts, static_cast<cudaStream_t>(stream), true);
}

int pald_gpu_plan_cohesion_share_peers(pald_gpu_plan* p, uint64_t part, uint64_t parts, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_cohesion_share_peers_impl(p, part, parts, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_cohesion_share(pald_gpu_plan* p, uint64_t part, uint64_t parts, void* stream) {
  if (!p) return set_error(PALD_GPU_ERR_VALIDATION, "null plan");
  DeviceGuard g(p->device);
  return plan_cohesion_share_impl(p, part, parts, static_cast<cudaStream_t>(stream));
}

int pald_gpu_plan_get_info(const pald_gpu_plan* p, pald_gpu_plan_info* out) {
  if (!p || !out) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  if (out->struct_size < offsetof(pald_gpu_plan_info, pair_kernel_preferred))
    return set_error(PALD_GPU_ERR_VALIDATION, "pald_gpu_plan_info.struct_size too small");
  out->cohesion_kernel = p->last_kernel;
  out->exact_path = p->exact ? 1 : 0;
  out->pair_kernel_ready = p->sym_ready ? 1 : 0;
  out->exact_step_share = p->sym_marked;
  out->launches = p->launches;
  out->rank_codes = p->rank_ready ? 1 : 0;
  if (out->struct_size >= offsetof(pald_gpu_plan_info, pair_kernel_preferred) + sizeof(int32_t))
    out->pair_kernel_preferred = (p->loaded && p->sym_ready && sym_preferred(p)) ? 1 : 0;
  return PALD_GPU_OK;
}

int pald_gpu_plan_buffers(const pald_gpu_plan* p, pald_gpu_buffers* out) {
  if (!p || !out) return set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  out->U = p->u;
  out->W = p->w;
  out->C = p->c;
  out->ld = p->ld;
  out->n = p->n;
  out->tile = kTile;
  out->tiles_per_dim = p->nb;
  out->exact_path = p->exact ? 1 : 0;
  out->reserved = 0;
  out->C64 = p->c64;
  return PALD_GPU_OK;
}

uint64_t pald_gpu_plan_launches(const pald_gpu_plan* p) { return p ? p->launches : 0; }

int pald_gpu_cohesion_f32_device(const float* dD, uint64_t ldd, uint64_t n,
                                 const pald_gpu_opts* o_in, int32_t* dU, uint64_t ldu, float* dC,
                                 uint64_t ldc, void* stream) {
  pald_gpu_opts oo;
  int rc = read_opts(o_in, &oo);
  if (rc || (rc = check_opts(&oo))) return rc;
  const pald_gpu_opts* o = &oo;
  if (o->num_devices > 1)
    return set_error(PALD_GPU_ERR_UNSUPPORTED, "the device-pointer API runs on one device (use the host API "
                                               "or a staged plan per device for several)");
  if (!dD || !dC) return set_error(PALD_GPU_ERR_VALIDATION, "null device pointer");
  if (ldd < n || ldc < n || (dU && ldu < n)) return set_error(PALD_GPU_ERR_VALIDATION, "leading dimension < n");
  int dev = o->device;
  if (dev < 0) PALD_CUDA(cudaGetDevice(&dev));
  DeviceGuard g(dev);
  std::lock_guard<std::mutex> lk(cache().mu);
  pald_gpu_plan* p = nullptr;
  if ((rc = get_cached_plan(dev, n, o, &p))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((rc = plan_load_impl(p, dD, ldd, s))) return rc;
  if ((rc = plan_focus_impl(p, s))) return rc;
  if ((rc = plan_cohesion_impl(p, 0, n, s))) return rc;
  if (dU) PALD_CUDA(cudaMemcpy2DAsync(dU, ldu * 4, p->u, p->ld * 4, n * 4, n, cudaMemcpyDeviceToDevice, s));
  PALD_CUDA(cudaMemcpy2DAsync(dC, ldc * 4, p->c, p->ld * 4, n * 4, n, cudaMemcpyDeviceToDevice, s));
  return PALD_GPU_OK;
}


int pald_gpu_cohesion_f32(const float* D, uint64_t n, const pald_gpu_opts* o_in, int32_t* U_out,
                          float* C_out, pald_gpu_phase_times* times) {
  pald_gpu_opts oo;
  int rc = read_opts(o_in, &oo);
  if (rc || (rc = check_opts(&oo))) return rc;
  const pald_gpu_opts* o = &oo;
  if (!D || !C_out) return set_error(PALD_GPU_ERR_VALIDATION, "null host pointer");
  if (n < 2) return set_error(PALD_GPU_ERR_VALIDATION, "distance matrix needs n >= 2, got n=%llu", (unsigned long long)n);
  if (o->num_devices > 1) {
    std::lock_guard<std::mutex> lk(cache().mu);
    DeviceGuard g(-1);
    return run_multi(D, n, o, U_out, C_out, times);
  }
  int dev = o->device;
  if (dev < 0) PALD_CUDA(cudaGetDevice(&dev));
  DeviceGuard g(dev);
  std::lock_guard<std::mutex> lk(cache().mu);
  const auto t_start = std::chrono::steady_clock::now();
  pald_gpu_plan* p = nullptr;
  if ((rc = get_cached_plan(dev, n, o, &p))) return rc;
  // compute stream, copy-out stream, second compute stream and the events of
  // the one-shot call: created once per cached plan
  if ((rc = ensure_oneshot(p))) return rc;
  cudaStream_t s = p->os_s, sc = p->os_sc, s2 = p->os_s2;
  cudaEvent_t* ev = p->os_ev;
  // Pass 2 runs in row bands; each band's C rows are copied to the host on
  // the copy stream while the next band computes, and U is copied during
  // pass 2 (it is final after pass 1). Only the last band's copy is exposed.
  // On the pair kernel a band is a run of whole raster groups of the pair
  // list: once groups [0, g] are done, tile rows [0, kGroupRows * (g + 1))
  // are complete (a pair (P <= Q) writes rows P and Q, and P lies in its
  // group). Bands alternate between two compute streams (they write
  // disjoint entries) so that one band's tail overlaps the next band.
  constexpr int kBands = PALD_HOST_BANDS;
  // (a failed call leaves no work behind on these streams)
  struct Drain {
    cudaStream_t a, b, c;
    ~Drain() {
      cudaStreamSynchronize(a);
      cudaStreamSynchronize(b);
      cudaStreamSynchronize(c);
    }
  } drain{s, sc, s2};
  PALD_CUDA(cudaEventRecord(ev[0], s));
  if (banded_wanted(p)) {  // H2D in bands overlapped with the rank codes and pass 1
    PALD_CUDA(cudaEventRecord(ev[1], s));
    if ((rc = load_focus_banded(p, D, s, sc, s2))) return rc;
    if ((rc = plan_focus_finish_impl(p, s))) return rc;
  } else {
    hook_rows_needed(0, n);
    if ((rc = pald_gpu_plan_load_host(p, D, s))) return rc;
    PALD_CUDA(cudaEventRecord(ev[1], s));
    if ((rc = plan_focus_impl(p, s))) return rc;
  }
  PALD_CUDA(cudaEventRecord(ev[2], s));
  t_msg_next = 0;
  if (U_out) {
    PALD_CUDA(cudaStreamWaitEvent(sc, ev[2], 0));
    PALD_CUDA(cudaMemcpy2DAsync(U_out, n * 4, p->u, p->ld * 4, n * 4, n, cudaMemcpyDeviceToHost, sc));
    queue_landed(sc, 0);
  }
  if (p->sym_ready && sym_preferred(p)) {
    const bool acc = accurate(p);
    if (acc) {  // the double sums zeroed before either band stream starts
      if ((rc = acc_zero_rows(p, 0, n, s))) return rc;
      PALD_CUDA(cudaEventRecord(ev[2], s));
    }
    PALD_CUDA(cudaStreamWaitEvent(s2, ev[2], 0));
    const int nb = (int)p->nb;
    const uint64_t pairs = p->nb * (p->nb + 1) / 2;
    int t0 = 0, t1 = 0, band = 0, g_row0 = 0;
    for (int g0 = 0; g0 < nb; g0 += kGroupRows) {
      const int g1 = std::min(nb, g0 + kGroupRows);
      for (int r = g0; r < g1; ++r) t1 += nb - r;  // pairs of the group
      const uint64_t target = pairs * (uint64_t)(band + 1) / kBands;
      if ((uint64_t)t1 < target && g1 < nb) continue;  // extend the band by one more group
      cudaStream_t cs = (band & 1) ? s2 : s;
      // (bands run concurrently on two streams: no shared round barrier)
      if ((rc = launch_sym(p, t0, t1, cs, false, false))) return rc;
      ++p->launches;
      if (acc && (rc = acc_round_pairs(p, t0, t1, own_c(p), cs))) return rc;
      PALD_CUDA(cudaEventRecord(ev[4 + band], cs));
      PALD_CUDA(cudaStreamWaitEvent(sc, ev[4 + band], 0));
      const uint64_t r0 = (uint64_t)g_row0 * kTile, r1 = std::min(n, (uint64_t)g1 * kTile);
      PALD_CUDA(cudaMemcpy2DAsync(C_out + r0 * n, n * 4, p->c + r0 * p->ld, p->ld * 4, n * 4, r1 - r0,
                                  cudaMemcpyDeviceToHost, sc));
      queue_landed(sc, r1);
      t0 = t1;
      g_row0 = g1;
      ++band;
    }
    p->last_kernel = PALD_GPU_KERNEL_PAIRS;
    for (int b = std::max(0, band - 2); b < band; ++b) PALD_CUDA(cudaStreamWaitEvent(s, ev[4 + b], 0));
  } else {
    const uint64_t rows_per_band = std::max<uint64_t>(kTile, (n / kBands + kTile - 1) / kTile * kTile);
    int nb_used = 0;
    for (uint64_t r0 = 0; r0 < n; r0 += rows_per_band, ++nb_used) {
      const uint64_t r1 = std::min(n, r0 + rows_per_band);
      if ((rc = plan_cohesion_impl(p, r0, r1, s))) return rc;
      PALD_CUDA(cudaEventRecord(ev[4 + nb_used], s));
      PALD_CUDA(cudaStreamWaitEvent(sc, ev[4 + nb_used], 0));
      PALD_CUDA(cudaMemcpy2DAsync(C_out + r0 * n, n * 4, p->c + r0 * p->ld, p->ld * 4, n * 4, r1 - r0,
                                  cudaMemcpyDeviceToHost, sc));
      queue_landed(sc, r1);
    }
  }
  PALD_CUDA(cudaEventRecord(ev[3], s));
  PALD_CUDA(cudaStreamSynchronize(s));
  PALD_CUDA(cudaStreamSynchronize(sc));
  if (times) {
    float f = 0, c = 0;
    PALD_CUDA(cudaEventElapsedTime(&f, ev[1], ev[2]));
    PALD_CUDA(cudaEventElapsedTime(&c, ev[2], ev[3]));
    const double total =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    times->focus_seconds += f * 1e-3;
    times->cohesion_seconds += c * 1e-3;
    times->overhead_seconds += std::max(0.0, total - (f + c) * 1e-3);
    times->total_seconds = total;
  }
  return PALD_GPU_OK;
}

int pald_gpu_fill_diagonal(const int32_t* dU, uint64_t ldu, uint64_t n, double* diag_out,
                           void* stream) {
  if (!dU || !diag_out) return set_error(PALD_GPU_ERR_VALIDATION, "null device pointer");
  fill_diagonal_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      dU, ldu, (int)n, diag_out);
  PALD_CUDA(cudaGetLastError());
  return PALD_GPU_OK;
}

int pald_gpu_points_to_distances(const double* dP, uint64_t n, uint64_t dim, float* dD,
                                 uint64_t ldd, void* stream) {
  if (!dP || !dD) return set_error(PALD_GPU_ERR_VALIDATION, "null device pointer");
  if (n < 2) return set_error(PALD_GPU_ERR_VALIDATION, "point cloud needs at least 2 points");
  if (dim < 1) return set_error(PALD_GPU_ERR_VALIDATION, "points need at least one coordinate");
  if (ldd < n) return set_error(PALD_GPU_ERR_VALIDATION, "ldd < n");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* key = nullptr;
  PALD_CUDA(cudaMallocAsync(&key, sizeof(unsigned long long), s));
  PALD_CUDA(cudaMemsetAsync(key, 0xff, sizeof(unsigned long long), s));
  points_kernel<<<grid_rows(n), 256, 0, s>>>(dP, (int)n, (int)dim, dD, ldd, key);
  PALD_CUDA(cudaGetLastError());
  unsigned long long k = ~0ull;
  PALD_CUDA(cudaMemcpyAsync(&k, key, sizeof(k), cudaMemcpyDeviceToHost, s));
  PALD_CUDA(cudaFreeAsync(key, s));
  PALD_CUDA(cudaStreamSynchronize(s));
  if (k != ~0ull)
    return set_error(PALD_GPU_ERR_VALIDATION, "duplicate points %llu and %llu (zero distance)", k / n, k % n);
  return PALD_GPU_OK;
}

}  // extern "C"

void pald_gpu_set_host_hooks(const pald_gpu_host_hooks* hooks) {
  t_hooks = hooks ? *hooks : pald_gpu_host_hooks{nullptr, nullptr, nullptr, nullptr};
}

int pald_gpu_set_error(int code, const char* message) {
  g_last_error = message;
  return code;
}
