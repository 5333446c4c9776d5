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
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pald_gpu.h"
#include "pald_internal.h"

struct pald_gpu_job {
  std::thread worker;
  int status = PALD_GPU_OK;
  std::string error;
  uint64_t n = 0;
  pald_gpu_phase_times times{};
  double convert_in_seconds = 0;
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
  std::memcpy(&o, opts, std::min<size_t>(sizeof(o), opts->struct_size ? opts->struct_size : sizeof(o)));
  // "current device" means the caller's, not the worker thread's
  if (o.device < 0 && cudaGetDevice(&o.device) != cudaSuccess) {
    cudaGetLastError();
    o.device = 0;
  }
  auto* j = new pald_gpu_job();
  j->n = n;
  j->worker = std::thread([j, D, n, o, e, &st] {
    const double t0 = now_s();
    // detail::to_real<float> (blocked.hpp:91-96): static_cast<float> of each value
    parallel_for(e, [&](size_t b, size_t end) {
      for (size_t i = b; i < end; ++i) st.d32[i] = static_cast<float>(D[i]);
    });
    j->convert_in_seconds = now_s() - t0;
    j->status = pald_gpu_cohesion_f32(st.d32, n, &o, st.u, st.c, &j->times);
    if (j->status) j->error = pald_gpu_last_error();
  });
  *job = j;
  return PALD_GPU_OK;
}

int pald_gpu_cohesion_f64io_end(pald_gpu_job* j, int32_t* U_out, double* C_out, pald_gpu_phase_times* times) {
  if (!j) return pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null job");
  Staging& st = staging();
  j->worker.join();
  int rc = j->status;
  if (rc) {
    pald_gpu_set_error(rc, j->error.c_str());
  } else if (!C_out) {
    rc = pald_gpu_set_error(PALD_GPU_ERR_VALIDATION, "null host pointer");
  } else {
    const double t0 = now_s();
    const size_t e = (size_t)j->n * j->n;
    // detail::collect_result (blocked.hpp:352-359): U as is, C widened to double
    parallel_for(e, [&](size_t b, size_t end) {
      if (U_out) std::memcpy(U_out + b, st.u + b, (end - b) * sizeof(int32_t));
      for (size_t i = b; i < end; ++i) C_out[i] = static_cast<double>(st.c[i]);
    });
    if (times) {
      times->focus_seconds += j->times.focus_seconds;
      times->cohesion_seconds += j->times.cohesion_seconds;
      times->overhead_seconds += j->times.overhead_seconds + j->convert_in_seconds + (now_s() - t0);
      times->total_seconds = j->times.total_seconds + j->convert_in_seconds + (now_s() - t0);
    }
  }
  delete j;
  st.job_mu.unlock();
  return rc;
}

int pald_gpu_cohesion_f64io(const double* D, uint64_t n, const pald_gpu_opts* opts, int32_t* U_out, double* C_out,
                            pald_gpu_phase_times* times) {
  pald_gpu_job* j = nullptr;
  const int rc = pald_gpu_cohesion_f64io_begin(D, n, opts, &j);
  if (rc) return rc;
  return pald_gpu_cohesion_f64io_end(j, U_out, C_out, times);
}

int pald_gpu_release_host_staging(void) {
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.job_mu);
  st.release();
  return PALD_GPU_OK;
}

}  // extern "C"
