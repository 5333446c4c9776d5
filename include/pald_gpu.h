/*
 * pald_gpu.h -- C ABI of the B200 (sm_100a) PaLD cohesion engine.
 *
 * This is the drop-in boundary for the O(n^3) hot path of the reference
 * library (/root/reference/proj/include/pald). Every entry point names the
 * reference interface it replaces. Plain pointers and sizes only; no torch
 * or C++ types cross this boundary. The header-only C++ shim with the
 * reference's own signatures (pald::gpu::blocked_pairwise<float>, ...)
 * lives in include/pald_gpu.hpp and is the intended caller for C++ code.
 *
 * Semantics (identical to the reference):
 *   Input  D: dense n x n fp32 distance matrix, row-major (element (x,y) at
 *             x*ld + y). Zero diagonal, off-diagonal > 0, exactly symmetric
 *             (types.hpp:45-65). Validated on the device unless
 *             PALD_GPU_FLAG_SKIP_VALIDATION is set.
 *   Output U: focus sizes u_xy, int32 n x n, symmetric, diagonal 0
 *             (types.hpp:79-86). Bit-exact with the reference's strict-<
 *             tie semantics, pairwise (blocked.hpp:101-122) or triplet
 *             (blocked.hpp:195-238, U initialised to 2) as selected.
 *   Output C: unnormalized cohesion, fp32 n x n (the fp32 instantiation of
 *             CohesionMatrix, types.hpp:90-98). Pairwise C is bit-identical
 *             to blocked_pairwise<float> / parallel_pairwise<float>
 *             (ascending-partner summation order). Triplet C matches
 *             blocked_triplet<double> within fp32 tolerance and has its
 *             diagonal left 0 (apply fill_diagonal, reference.hpp:213-220).
 *
 * Return codes mirror the reference CLI's exception -> exit code map
 * (tools/pald.cpp:406-415): 0 ok, 2 ValidationError, 3
 * UnsupportedPolicyError, 4 IoError; 5 CUDA failure, 6 communicator
 * failure. pald_gpu_last_error() gives the message (thread-local).
 */
#ifndef PALD_GPU_H_
#define PALD_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PALD_GPU_ABI_VERSION 4

/* Algorithm variant: blocked_pairwise / parallel_pairwise (blocked.hpp:368,
 * parallel.hpp:159) vs blocked_triplet / parallel_triplet (blocked.hpp:424,
 * parallel.hpp:257). */
enum pald_gpu_algorithm { PALD_GPU_PAIRWISE = 0, PALD_GPU_TRIPLET = 1 };

/* Policy, types.hpp:34. Pairwise supports both (InclusiveSplit: `<=` focus
 * membership, support split 0.5/0.5 on ties, blocked.hpp:117,150-158; C
 * bit-identical to blocked_pairwise<float>(..., InclusiveSplit)); triplet is
 * Strict only and returns PALD_GPU_ERR_UNSUPPORTED otherwise, as the
 * reference throws UnsupportedPolicyError (blocked.hpp:429-430). */
enum pald_gpu_policy { PALD_GPU_STRICT = 0, PALD_GPU_INCLUSIVE_SPLIT = 1 };

enum pald_gpu_status {
  PALD_GPU_OK = 0,
  PALD_GPU_ERR_VALIDATION = 2,
  PALD_GPU_ERR_UNSUPPORTED = 3,
  PALD_GPU_ERR_IO = 4,
  PALD_GPU_ERR_CUDA = 5,
  PALD_GPU_ERR_COMM = 6
};

enum pald_gpu_flags {
  /* The caller guarantees D already passed DistanceMatrix validation
   * (the C++ shim sets this: its DistanceMatrix is validated in double). */
  PALD_GPU_FLAG_SKIP_VALIDATION = 1u,
  /* Use the integer-key compare path even when the fp32 range allows the
   * FFMA.SAT compare path (testing). */
  PALD_GPU_FLAG_FORCE_EXACT = 2u,
  /* Accurate mode: pass 2 keeps each output's fp32 running sum only over
   * blocks of PALD_GPU_ACC_BLOCK (default 1024) third points and adds the
   * block partials into a double sum (exact: see csrc/pald_kernels.cuh
   * acc_flush4), rounded to fp32 at the end. C then stays within ~1e-6 of
   * the fp64-accumulated result at n = 32768 (the default single fp32 chain
   * is the reference's own order, bit-identical to blocked_pairwise<float>,
   * and drifts by ~1.3e-5 there). Deterministic; the double sums are
   * exposed as pald_gpu_buffers.C64. */
  PALD_GPU_FLAG_ACCURATE = 4u
};

#define PALD_GPU_MAX_DEVICES 8

/* Transport of the two exchange steps of a multi-device call (see
 * DESIGN.md section 5 for the traffic model of each):
 *   PEER  pass 1: each device finishes its 1/N of the tiles by reading the
 *         partial counts of every device over peer memory (P2P loads) and
 *         storing U and W = 1/U into every device (P2P stores) -- one fused
 *         reduce + finish + all-gather kernel.
 *         pass 2: the pair kernel stores each finished C tile into every
 *         device (P2P stores, overlapped with the math).
 *   NCCL  pass 1: ncclAllReduce(SUM) of the count buffers, local finish.
 *         pass 2: each device computes its tile-row band; no exchange (the
 *         host reads each band from the device that owns it).
 *   RED   pass 1 only: the focus kernel adds every partial count into every
 *         device's W (red.global.add over NVLink), local finish.
 *   AUTO  PEER where every pair of devices has peer access, else NCCL. */
enum pald_gpu_exchange {
  PALD_GPU_EXCHANGE_AUTO = 0,
  PALD_GPU_EXCHANGE_PEER = 1,
  PALD_GPU_EXCHANGE_NCCL = 2,
  PALD_GPU_EXCHANGE_RED = 3
};

typedef struct pald_gpu_opts {
  uint32_t struct_size;   /* sizeof(pald_gpu_opts) */
  int32_t algorithm;      /* enum pald_gpu_algorithm */
  int32_t policy;         /* enum pald_gpu_policy */
  int32_t device;         /* CUDA device ordinal; -1 = current device */
  /* Block-size hints of the reference drivers (b, b_focus, b_cohesion).
   * Validated >= 1 exactly like blocked.hpp:372 / :431; the GPU tile shape
   * is fixed (128 x 128 x 64), so they do not change results -- neither do
   * they in the reference (C bits of blocked_pairwise<float> are
   * independent of b). */
  uint64_t block;
  uint64_t block_focus;
  uint64_t block_cohesion;
  uint32_t flags;         /* enum pald_gpu_flags */
  uint32_t reserved;
  /* ---- ABI v4: several devices in ONE call (the GPU counterpart of
   * ParallelPlan.workers, parallel.hpp:31-34). num_devices 0 or 1: the
   * single `device` above. num_devices > 1: devices[0..num_devices) (a
   * device may repeat: the plans then share that GPU -- used to test the
   * multi-device path on one GPU). Pass-1 work units and pass-2 tile pairs
   * are split into equal shares, one per listed device; U and C are
   * bit-identical to one device. A caller compiled against ABI v3 passes
   * struct_size = PALD_GPU_OPTS_V3_SIZE and gets one device. */
  int32_t num_devices;
  int32_t devices[PALD_GPU_MAX_DEVICES];
  int32_t exchange_focus;     /* enum pald_gpu_exchange: pass-1 count exchange */
  int32_t exchange_cohesion;  /* enum pald_gpu_exchange: pass-2 C exchange */
} pald_gpu_opts;

/* PhaseTimes, types.hpp:114-119, filled from CUDA events. */
typedef struct pald_gpu_phase_times {
  double focus_seconds;
  double cohesion_seconds;
  double overhead_seconds;
  double total_seconds;
} pald_gpu_phase_times;

/* sizeof(pald_gpu_opts) of ABI v3 (no device list). */
#define PALD_GPU_OPTS_V3_SIZE 48u

/* Fills defaults: pairwise, strict, current device, blocks 128, flags 0,
 * one device, exchange AUTO. */
void pald_gpu_opts_init(pald_gpu_opts* opts);

/* Thread-local message of the last failing call on this thread. */
const char* pald_gpu_last_error(void);

int pald_gpu_abi_version(void);

/* Number of visible CUDA devices (0 without a GPU or driver). */
int pald_gpu_visible_devices(void);

/* One-shot host API. Replaces blocked_pairwise<float> /
 * parallel_pairwise<float> (blocked.hpp:368-418, parallel.hpp:159-222) and
 * blocked_triplet<float> / parallel_triplet<float> (blocked.hpp:424-477,
 * parallel.hpp:257-320) after to_real<float> (blocked.hpp:91-96).
 * D, U_out, C_out are HOST pointers, dense (ld = n). U_out may be NULL.
 * Pinned host memory gives full-speed copies. Synchronous. For
 * 2048 < n <= 32768 D is copied in bands of 2048 rows and pass 1 starts on
 * the bands that have arrived; validation errors are then reported after
 * the last band (the result is the same error code and message). */
int pald_gpu_cohesion_f32(const float* D, uint64_t n, const pald_gpu_opts* opts,
                          int32_t* U_out, float* C_out, pald_gpu_phase_times* times);

/* Double-precision host I/O (ABI v4), for callers holding the reference's
 * own types (DistanceMatrix stores doubles, PaldResult a double C;
 * types.hpp:43-119) -- the C++ shim include/pald_gpu.hpp uses it. Same
 * result as converting D with to_real<float> (blocked.hpp:91-96), calling
 * pald_gpu_cohesion_f32 and widening C like collect_result
 * (blocked.hpp:352-359); the conversions run on all host cores into / out
 * of pinned staging buffers that the library keeps between calls
 * (pald_gpu_release_host_staging frees them), and they are pipelined with
 * the transfers: each row band of D is converted just before its H2D copy
 * (which itself overlaps pass 1), and C is widened band by band as the D2H
 * copies land during pass 2. begin() returns at once (a worker thread runs
 * the GPU call) so the caller can build its result storage meanwhile;
 * outputs() (optional, once, any time before end) hands over U_out
 * (nullable) and C_out so that the widening can start before end();
 * end() waits for the rest and -- if outputs() was not called -- takes
 * U_out / C_out itself (its pointer arguments are ignored otherwise). One
 * job at a time per process (begin blocks until the previous job's end).
 * Errors of the GPU call are returned by end(). */
typedef struct pald_gpu_job pald_gpu_job;
int pald_gpu_cohesion_f64io_begin(const double* D, uint64_t n, const pald_gpu_opts* opts, pald_gpu_job** job);
int pald_gpu_cohesion_f64io_outputs(pald_gpu_job* job, int32_t* U_out, double* C_out);
int pald_gpu_cohesion_f64io_end(pald_gpu_job* job, int32_t* U_out, double* C_out, pald_gpu_phase_times* times);
/* First-touches [p, p + bytes) from all host cores (writes zeros): a caller
 * that has to build a large zero-filled result (std::vector value-
 * initialisation is one thread taking one page fault per 4 KiB) can reserve
 * the storage, prefault it here and then resize. Host memory only. */
int pald_gpu_host_prefault(void* p, uint64_t bytes);
int pald_gpu_cohesion_f64io(const double* D, uint64_t n, const pald_gpu_opts* opts, int32_t* U_out,
                            double* C_out, pald_gpu_phase_times* times);
int pald_gpu_release_host_staging(void);

/* Device API, asynchronous on `stream` (a cudaStream_t; NULL = legacy
 * default stream) except for one small device->host read of the range
 * check. dD, dU, dC are DEVICE pointers with leading dimensions (elements)
 * ldd, ldu, ldc >= n. dU may be NULL. Uses a per-device cached workspace. */
int pald_gpu_cohesion_f32_device(const float* dD, uint64_t ldd, uint64_t n,
                                 const pald_gpu_opts* opts, int32_t* dU, uint64_t ldu,
                                 float* dC, uint64_t ldc, void* stream);

/* ---- Staged plan: the building blocks of the multi-GPU drivers --------
 * A plan owns the device workspace for one n on one device.
 * Pass 1 (focus) is split into work units (a 128 x 128 upper-triangular
 * pair tile x a 64-point chunk of third points). focus_counts(part, parts)
 * accumulates the integer focus counts of share `part` of `parts` equal
 * shares of the units into the W buffer; focus_finish turns the counts
 * into U and W = 1/U (both triangles). A multi-GPU driver gives each rank
 * one share and SUMs the W buffers over ranks between the two calls
 * (integer counts < 2^24 in fp32: exact, order-independent).
 * Pass 2 (cohesion) writes C rows [row_begin, row_end) (tile aligned);
 * each row is one in-order sum, so row bands need no reduction.
 * cohesion_share(part, parts) instead zeroes C and computes share `part`
 * of `parts` of the whole pass-2 work (tile pairs on the pair kernel, row
 * bands otherwise): every C entry belongs to exactly one share and is one
 * in-order sum there, so the elementwise SUM of the C buffers over the
 * parts is the full C, bit-identical to one device. */
typedef struct pald_gpu_plan pald_gpu_plan;

typedef struct pald_gpu_buffers {
  int32_t* U;        /* device, n x ld, focus sizes */
  float* W;          /* device, n x ld, focus counts (after focus_counts) or 1/U (after finish) */
  float* C;          /* device, n x ld, unnormalized cohesion */
  uint64_t ld;       /* leading dimension (elements) of U, W, C */
  uint64_t n;
  uint64_t tile;     /* pair-tile edge (points) */
  uint64_t tiles_per_dim;
  int32_t exact_path;  /* 1 when the integer-key compare path is in use */
  int32_t reserved;
  double* C64;       /* device, n x ld: accurate mode's double C (NULL until used; ABI v4) */
} pald_gpu_buffers;

int pald_gpu_plan_create(uint64_t n, const pald_gpu_opts* opts, pald_gpu_plan** out);
int pald_gpu_plan_destroy(pald_gpu_plan* plan);
/* Validates (unless skipped), range-checks and lays out D (device pointer,
 * leading dimension ldd). Synchronizes `stream` once to read the range
 * check. Zeroes U, W. */
int pald_gpu_plan_load(pald_gpu_plan* plan, const float* dD, uint64_t ldd, void* stream);
/* Same, from a host pointer (dense, ld = n). */
int pald_gpu_plan_load_host(pald_gpu_plan* plan, const float* D, void* stream);
/* focus_counts(0, 1) + focus_finish */
int pald_gpu_plan_focus(pald_gpu_plan* plan, void* stream);
int pald_gpu_plan_focus_counts(pald_gpu_plan* plan, uint64_t part, uint64_t parts, void* stream);
int pald_gpu_plan_focus_finish(pald_gpu_plan* plan, void* stream);
int pald_gpu_plan_cohesion(pald_gpu_plan* plan, uint64_t row_begin, uint64_t row_end,
                           void* stream);
int pald_gpu_plan_cohesion_share(pald_gpu_plan* plan, uint64_t part, uint64_t parts,
                                 void* stream);
int pald_gpu_plan_buffers(const pald_gpu_plan* plan, pald_gpu_buffers* out);
/* Kernel launches issued by this plan so far (evidence counter). */
uint64_t pald_gpu_plan_launches(const pald_gpu_plan* plan);

/* Which pass-2 kernel the last cohesion call ran, and the tie statistics
 * of the loaded D that chose it. */
enum {
  PALD_GPU_KERNEL_NONE = 0,
  PALD_GPU_KERNEL_TILE128 = 1, /* one-sided 128 x 128 output tiles */
  PALD_GPU_KERNEL_TILE64 = 2,  /* one-sided 64 x 64 tiles (small n) */
  PALD_GPU_KERNEL_PAIRS = 3    /* tile pairs: C[P][Q] and C[Q][P] together */
};
typedef struct pald_gpu_plan_info {
  uint32_t struct_size;       /* sizeof(pald_gpu_plan_info) */
  int32_t cohesion_kernel;    /* PALD_GPU_KERNEL_* of the last cohesion call */
  int32_t exact_path;         /* 1: integer-key compare path */
  int32_t pair_kernel_ready;  /* 1: tie scan done, the pair kernel may run */
  double exact_step_share;    /* share of (pair, k) steps on the exact step */
  uint64_t launches;
  int32_t rank_codes;         /* 1: pass 1 runs on per-row rank codes (ABI v3) */
  int32_t pair_kernel_preferred; /* 1: a full-range cohesion of the loaded D would run
                                  * the pair kernel (multi-GPU drivers agree on it
                                  * before a fused pass 2; ABI v4) */
} pald_gpu_plan_info;
int pald_gpu_plan_get_info(const pald_gpu_plan* plan, pald_gpu_plan_info* out);

/* ---- Fused multi-GPU exchange over peer memory (one node, NVLink) ------
 * Replaces the two SUM all-reduces of the staged driver: pass-1 partial
 * counts are added (red.global.add) straight into EVERY rank's W, and the
 * pair kernel stores each C entry into every rank's C, so after the kernels
 * finish every rank holds the full counts / the full C. Setup: each rank
 * exports CUDA IPC handles of its W and C, the handles are all-gathered
 * (any transport), and each rank attaches all of them (its own included,
 * index = rank; world <= 8). Per step the caller orders the ranks with a
 * host barrier after load (every W zeroed), after focus_counts_peers (all
 * counts in) and after cohesion_share_peers (all of C written).
 * cohesion_share_peers needs the pair kernel (PALD_GPU_ERR_UNSUPPORTED
 * otherwise: fall back to cohesion_share + a SUM all-reduce). */
typedef struct pald_gpu_ipc_handle {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} pald_gpu_ipc_handle;
int pald_gpu_plan_export_buffers(const pald_gpu_plan* plan, pald_gpu_ipc_handle* w,
                                 pald_gpu_ipc_handle* c);
int pald_gpu_plan_attach_peers(pald_gpu_plan* plan, int world, int rank,
                               const pald_gpu_ipc_handle* w_handles,
                               const pald_gpu_ipc_handle* c_handles);
int pald_gpu_plan_detach_peers(pald_gpu_plan* plan);
int pald_gpu_plan_focus_counts_peers(pald_gpu_plan* plan, uint64_t part, uint64_t parts,
                                     void* stream);
int pald_gpu_plan_cohesion_share_peers(pald_gpu_plan* plan, uint64_t part, uint64_t parts,
                                       void* stream);

/* Pass-1 exchange by peer pull (ABI v4): instead of the count fan-out of
 * focus_counts_peers, every rank runs plain focus_counts (its share into
 * its OWN W), the ranks meet at a host barrier, and each rank finishes
 * share `part` of `parts` of the upper-triangular tiles: it sums the counts
 * of every rank's W (P2P loads), and stores W = 1/U into every rank's
 * buffer and U as u_mode says (P2P stores). After a
 * second barrier every rank holds the full W. U goes to: u_mode 0 this
 * rank only; 1 every rank; 2 the rank owning the entry's row in the
 * tile-row band split (bands [nb*i/world, nb*(i+1)/world) of tile rows, the
 * split the multi-device host call downloads U by). Replaces the SUM
 * all-reduce of the counts + focus_finish. U peers come from export_u /
 * attach_peers_u (after attach_peers). */
int pald_gpu_plan_export_u(const pald_gpu_plan* plan, pald_gpu_ipc_handle* u);
int pald_gpu_plan_attach_peers_u(pald_gpu_plan* plan, const pald_gpu_ipc_handle* u_handles);
int pald_gpu_plan_focus_finish_peers(pald_gpu_plan* plan, uint64_t part, uint64_t parts, int u_mode,
                                     void* stream);

/* Number of pass-1 work units of the plan. */
uint64_t pald_gpu_focus_units(const pald_gpu_plan* plan);

/* ---- Epilogue and input helpers ---------------------- */
/* fill_diagonal, reference.hpp:213-220: c_xx = sum_{y != x} 1/u_xy,
 * accumulated in double in ascending y and written as double to
 * diag_out[x] (device pointer, n doubles). */
int pald_gpu_fill_diagonal(const int32_t* dU, uint64_t ldu, uint64_t n, double* diag_out,
                           void* stream);
/* Euclidean distances of a point cloud (ingest.hpp:303-322): each pair
 * once, sum of squared differences in double in coordinate order, each
 * step sum = fma(diff, diff, sum) -- the reference as built by its own
 * flags (-O3 -march=native: GCC contracts `sum += diff * diff`; verified
 * bit-exact against oracle/_ref) -- sqrt in double, rounded to fp32
 * (to_real<float>); diagonal 0. Duplicate points (a zero distance) are
 * rejected like the reference: ValidationError "duplicate points x and y
 * (zero distance)" for the first such pair in (x, y > x) order (this reads
 * one word back: the call synchronizes `stream`). Device pointers; points
 * row-major n x dim doubles. */
int pald_gpu_points_to_distances(const double* dP, uint64_t n, uint64_t dim, float* dD,
                                 uint64_t ldd, void* stream);

/* Local depths (reference.hpp:231-241) of the normalized cohesion matrix
 * (normalize, reference.hpp:223-228), straight from the fp32 C on the
 * device: depth_x = sum_z double(c_xz) * (1/(n-1)), z ascending, in double --
 * the reference's arithmetic and order, bit for bit. `diag` (device, n
 * doubles, nullable) replaces c_xx first (the triplet's fill_diagonal). */
int pald_gpu_local_depths(const float* dC, uint64_t ldc, uint64_t n, const double* diag,
                          double* depths_out, void* stream);

/* Strong ties (analyze.hpp:34-53) of the normalized C: edges x < y with
 * min(c'_xy, c'_yx) >= threshold, row-major order. threshold_in (device,
 * nullable) overrides the universal threshold 0.5 * mean(c'_xx), which is
 * written to threshold_out (device). The edge count goes to count_out
 * (device); up to `capacity` edges are written to xs, ys, strength
 * (device arrays, nullable to only count). */
int pald_gpu_strong_ties(const float* dC, uint64_t ldc, uint64_t n, const double* diag,
                         const double* threshold_in, double* threshold_out, uint64_t capacity,
                         uint32_t* xs, uint32_t* ys, double* strength, uint64_t* count_out,
                         void* stream);

/* nearest_neighbors (analyze.hpp:60-75) of the normalized C on the device:
 * the k points z != focus with the largest min(c'_fz, c'_zf), strongest
 * first, equal strengths in ascending z (the reference's stable sort);
 * written to zs / strength (device arrays of k). ValidationError with the
 * reference's messages for focus >= n or k >= n. `diag` as above. */
int pald_gpu_nearest_neighbors(const float* dC, uint64_t ldc, uint64_t n, const double* diag, uint64_t focus,
                               uint64_t k, uint32_t* zs, double* strength, void* stream);

/* The Python mirror's double CohesionMatrix on the device: normalize
 * (reference.hpp:223-228: c *= 1/(n-1) in double) in place, and the
 * sequential (ascending z) double row sums of local_depths
 * (reference.hpp:231-241). Device pointers. */
int pald_gpu_normalize_f64(double* dC, uint64_t ldc, uint64_t n, void* stream);
int pald_gpu_row_sums_f64(const double* dC, uint64_t ldc, uint64_t n, double* out, void* stream);

/* The reference's binary matrix format ("PALD", version 1, width 4 or 8,
 * u64 n, n*n little-endian row-major values; ingest.hpp:214-283).
 * read_binary_header gives n and the width; read_distance_binary streams
 * the payload to the device and applies validate_distances
 * (ingest.hpp:116-149: finite, >= 0, zero diagonal, symmetric within 1e-9
 * relative -> averaged in double, positive) on the GPU, writing the fp32
 * matrix (to_real<float>) to dD (n x ldd). Errors carry the reference's
 * messages: 2 (ValidationError), 4 (IoError, cannot open). */
int pald_gpu_read_binary_header(const char* path, uint64_t* n_out, int32_t* width_out);
int pald_gpu_read_distance_binary(const char* path, float* dD, uint64_t ldd, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PALD_GPU_H_ */
