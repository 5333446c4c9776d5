// pald_hostio.cu -- double-precision host I/O of the C ABI (include/pald_gpu.h,
// pald_gpu_cohesion_f64io*): the entry points the C++ shim
// (include/pald_gpu.hpp) uses for the reference's own types, whose
// DistanceMatrix holds doubles and whose PaldResult holds a double C
// (types.hpp:43-119).
//
// The reference converts D with detail::to_real<float> (blocked.hpp:91-96)
// and widens the fp32 C with detail::collect_result (blocked.hpp:352-359),
// each a single-threaded loop over n^2 elements. Here both conversions run
// on all host cores into / out of pinned staging buffers (cached across
// calls), and the fp32 C-ABI call in between moves the pinned data at full
// PCIe speed with its banded H2D / D2H overlap. The call is split in two so
// that a caller can build its (zero-filled, page-faulting) result vectors
// while the GPU works: begin() returns at once and a worker thread runs
// conversion + GPU; end() joins it and copies out.
#include <cuda_runtime.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pald_gpu.h"
#include "pald_internal.h"

struct pald_gpu_job {
  std::thread worker;     // converts D band by band (hook) and runs the GPU call
  std::thread converter;  // copies U / widens C rows as they land, once the outputs are known
  int status = PALD_GPU_OK;
  std::string error;
  uint64_t n = 0;
  const double* D = nullptr;
  pald_gpu_phase_times times{};
  double convert_in_seconds = 0;   // worker thread only
  uint64_t converted_rows = 0;     // rows [0, converted_rows) of the fp32 staging are valid (worker only)
  // output pipeline (guarded by mu)
  std::mutex mu;
  std::condition_variable cv;
  uint64_t landed_rows = 0;  // rows [0, landed_rows) of the fp32 C staging are in host memory
  bool u_landed = false;
  bool finished = false;     // the GPU call returned (everything landed, or it failed)
  bool abandon = false;      // no outputs will come / the call failed: the converter just exits
  bool outputs_set = false;
  int32_t* U_out = nullptr;
  double* C_out = nullptr;
  double convert_out_seconds = 0;  // converter busy time
  double t_finished = 0;           // when the GPU call returned
};

namespace {

// Pinned staging (D fp32, U, C fp32), grown on demand, one job at a time.
struct Staging {
  std::mutex job_mu;  // held from begin() to end()
  float* d32 = nullptr;
  int32_t* u = nullptr;
  float* c = nullptr;
  size_t elems = 0;
  int ensure(size_t e) {
    if (e <= elems) return PALD_GPU_OK;
    release();
    if (cudaMallocHost(&d32, e * 4) != cudaSuccess || cudaMallocHost(&u, e * 4) != cudaSuccess ||
        cudaMallocHost(&c, e * 4) != cudaSuccess) {
      cudaGetLastError();
      release();
      return pald_gpu_set_error(PALD_GPU_ERR_CUDA, "cannot allocate pinned host staging buffers");
    }
    elems = e;
    return PALD_GPU_OK;
  }
  void release() {
    if (d32) cudaFreeHost(d32);
    if (u) cudaFreeHost(u);
    if (c) cudaFreeHost(c);
    d32 = nullptr;
    u = nullptr;
    c = nullptr;
    elems = 0;
  }
};
Staging& staging() {
  static Staging s;
  return s;
}

int host_threads() {
  cpu_set_t set;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, CPU_COUNT(&set));
  return std::max(1u, std::thread::hardware_concurrency());
}

// fn(begin, end) over [0, count) on all host cores.
template <class F>
void parallel_for(size_t count, F&& fn) {
  const int T = (int)std::min<size_t>((size_t)host_threads(), std::max<size_t>(1, count / (1u << 20)));
  if (T <= 1) {
    fn((size_t)0, count);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const size_t b = count * t / T, e = count * (t + 1) / T;
    th.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& x : th) x.join();
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// detail::to_real<float> (blocked.hpp:91-96): static_cast<float> of each
// value. Rows [converted_rows, r1) are converted when the GPU call is about
// to upload them (rows_needed hook, on the worker thread), so the conversion
// overlaps the banded H2D and pass 1 instead of preceding them.
void convert_rows(pald_gpu_job* j, Staging& st, uint64_t r1) {
  if (r1 <= j->converted_rows) return;
  const double t0 = now_s();
  const uint64_t n = j->n;
  const size_t b0 = (size_t)j->converted_rows * n, e0 = (size_t)r1 * n;
  const double* D = j->D;
  float* d32 = st.d32;
  parallel_for(e0 - b0, [&](size_t b, size_t end) {
    for (size_t i = b0 + b; i < b0 + end; ++i) d32[i] = static_cast<float>(D[i]);
  });
  j->converted_rows = r1;
  j->convert_in_seconds += now_s() - t0;
}

}  // namespace

extern "C" {

int pald_gpu_cohesion_f64io_begin(const double* D, uint64_t n, const pald_gpu_opts* opts, pald_gpu_job** job) {
  if (!D || !opts || !job) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  if (n < 2) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "distance matrix needs n >= 2");
  Staging& st = staging();
  st.job_mu.lock();
  const size_t e = (size_t)n * n;
  int rc = st.ensure(e);
  if (rc) {
    st.job_mu.unlock();
    return rc;
  }
  pald_gpu_opts o;
  pald_gpu_opts_init(&o);  // a shorter (ABI v3) struct leaves the newer fields at their defaults
  std::memcpy(&o, opts, std::min<size_t>(sizeof(o), opts->struct_size ? opts->struct_size : sizeof(o)));
  // "current device" means the caller's, not the worker thread's
  if (o.device < 0 && cudaGetDevice(&o.device) != cudaSuccess) {
    cudaGetLastError();
    o.device = 0;
  }
  auto* j = new pald_gpu_job();
  j->n = n;
  j->D = D;
  j->worker = std::thread([j, n, o, &st] {
    pald_gpu_host_hooks hooks{};
    hooks.ctx = j;
    hooks.rows_needed = [](void* ctx, uint64_t, uint64_t r1) {
      convert_rows(static_cast<pald_gpu_job*>(ctx), staging(), r1);
    };
    hooks.c_rows_landed = [](void* ctx, uint64_t r1) {
      auto* job = static_cast<pald_gpu_job*>(ctx);
      {
        std::lock_guard<std::mutex> lk(job->mu);
        job->landed_rows = std::max(job->landed_rows, r1);
      }
      job->cv.notify_all();
    };
    hooks.u_landed = [](void* ctx) {
      auto* job = static_cast<pald_gpu_job*>(ctx);
      {
        std::lock_guard<std::mutex> lk(job->mu);
        job->u_landed = true;
      }
      job->cv.notify_all();
    };
    if (o.num_devices > 1) convert_rows(j, st, n);  // the multi-device call reads D without hooks
    pald_gpu_set_host_hooks(&hooks);
    j->status = pald_gpu_cohesion_f32(st.d32, n, &o, st.u, st.c, &j->times);
    pald_gpu_set_host_hooks(nullptr);
    j->t_finished = now_s();
    if (j->status) j->error = pald_gpu_last_error();
    {
      std::lock_guard<std::mutex> lk(j->mu);
      j->finished = true;
      if (j->status) {
        j->abandon = true;
      } else {
        j->landed_rows = n;
        j->u_landed = true;
      }
    }
    j->cv.notify_all();
  });
  // detail::collect_result (blocked.hpp:352-359): U as is, C widened to
  // double -- row bands as their D2H copies land, while pass 2 still runs.
  j->converter = std::thread([j, n, &st] {
    uint64_t widened = 0;
    bool u_done = false;
    for (;;) {
      uint64_t landed;
      bool u_ready;
      {
        std::unique_lock<std::mutex> lk(j->mu);
        j->cv.wait(lk, [&] {
          return j->abandon || (j->outputs_set && (j->landed_rows > widened || (j->u_landed && !u_done)));
        });
        if (j->abandon) return;
        landed = j->landed_rows;
        u_ready = j->u_landed;
      }
      const double t0 = now_s();
      if (u_ready && !u_done) {
        if (j->U_out)
          parallel_for((size_t)n * n, [&](size_t b, size_t end) {
            std::memcpy(j->U_out + b, st.u + b, (end - b) * sizeof(int32_t));
          });
        u_done = true;
      }
      if (landed > widened) {
        const size_t b0 = (size_t)widened * n, e0 = (size_t)landed * n;
        double* C_out = j->C_out;
        parallel_for(e0 - b0, [&](size_t b, size_t end) {
          for (size_t i = b0 + b; i < b0 + end; ++i) C_out[i] = static_cast<double>(st.c[i]);
        });
        widened = landed;
      }
      j->convert_out_seconds += now_s() - t0;
      if (widened == n && u_done) return;
    }
  });
  *job = j;
  return PALD_GPU_OK;
}

int pald_gpu_cohesion_f64io_outputs(pald_gpu_job* j, int32_t* U_out, double* C_out) {
  if (!j || !C_out) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  {
    std::lock_guard<std::mutex> lk(j->mu);
    if (j->outputs_set) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "outputs already set");
    j->U_out = U_out;
    j->C_out = C_out;
    j->outputs_set = true;
  }
  j->cv.notify_all();
  return PALD_GPU_OK;
}

int pald_gpu_cohesion_f64io_end(pald_gpu_job* j, int32_t* U_out, double* C_out, pald_gpu_phase_times* times) {
  if (!j) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null job");
  Staging& st = staging();
  j->worker.join();
  int rc = j->status;
  {
    std::lock_guard<std::mutex> lk(j->mu);
    if (rc) {
      pald_gpu_set_error(rc, j->error.c_str());
    } else if (!j->outputs_set) {
      if (!C_out) {
        rc = pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null host pointer");
        j->abandon = true;
      } else {
        j->U_out = U_out;
        j->C_out = C_out;
        j->outputs_set = true;
      }
    }
  }
  j->cv.notify_all();
  j->converter.join();  // the rows that landed after the last pass of the converter
  if (!rc && times) {
    const double tail = std::max(0.0, now_s() - j->t_finished);  // exposed part of the output conversion
    times->focus_seconds += j->times.focus_seconds;
    times->cohesion_seconds += j->times.cohesion_seconds;
    // the input conversion runs inside the GPU call's wall time (hooked), the
    // output conversion overlaps pass 2 except for its tail
    times->overhead_seconds += j->times.overhead_seconds + tail;
    times->total_seconds = j->times.total_seconds + tail;
  }
  delete j;
  st.job_mu.unlock();
  return rc;
}

int pald_gpu_cohesion_f64io(const double* D, uint64_t n, const pald_gpu_opts* opts, int32_t* U_out, double* C_out,
                            pald_gpu_phase_times* times) {
  pald_gpu_job* j = nullptr;
  int rc = pald_gpu_cohesion_f64io_begin(D, n, opts, &j);
  if (rc) return rc;
  if (C_out) pald_gpu_cohesion_f64io_outputs(j, U_out, C_out);  // widen rows as they land
  return pald_gpu_cohesion_f64io_end(j, U_out, C_out, times);
}

int pald_gpu_host_prefault(void* p, uint64_t bytes) {
  if (!p && bytes) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null argument");
  char* c = static_cast<char*>(p);
  parallel_for((size_t)bytes, [c](size_t b, size_t end) { std::memset(c + b, 0, end - b); });
  return PALD_GPU_OK;
}

int pald_gpu_release_host_staging(void) {
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.job_mu);
  st.release();
  return PALD_GPU_OK;
}

}  // extern "C"
