// pald_internal.h -- shared by the translation units of libpald_gpu.so.
#pragma once

// Records the thread-local message returned by pald_gpu_last_error() and
// returns `code`.
int pald_gpu_set_error(int code, const char* message);

#include <cstdint>

// Host-side hooks of the one-shot host call pald_gpu_cohesion_f32, set by
// pald_hostio.cu (thread-local: the call runs on the thread that set them)
// so that the double <-> float conversions of the f64io entry points are
// pipelined with the banded transfers instead of running before / after
// the whole call:
//   rows_needed(ctx, r0, r1)  called before the H2D copy of rows [r0, r1) of
//                             the fp32 source is queued; returns once those
//                             rows are valid;
//   c_rows_landed(ctx, r1)    rows [0, r1) of C_out are in host memory
//                             (called from a CUDA host callback: no CUDA
//                             calls inside);
//   u_landed(ctx)             all of U_out is in host memory (likewise).
// Paths without hooks (several devices) simply never call them.
struct pald_gpu_host_hooks {
  void (*rows_needed)(void* ctx, uint64_t r0, uint64_t r1);
  void (*c_rows_landed)(void* ctx, uint64_t r1);
  void (*u_landed)(void* ctx);
  void* ctx;
};
void pald_gpu_set_host_hooks(const pald_gpu_host_hooks* hooks);  // nullptr clears
