// pald_gpu.hpp -- header-only C++ shim with the reference library's entry
// points, running the O(n^3) hot path on a B200 through the C ABI
// (pald_gpu.h).
//
// Drop-in use from code written against the reference
// (/root/reference/proj/include/pald):
//
//     #define PALD_GPU_USE_REFERENCE_TYPES   // reuse pald/types.hpp
//     #include "pald/pald.hpp"
//     #include "pald_gpu.hpp"
//     pald::PaldResult r = pald::gpu::blocked_pairwise<float>(d, b);
//
// Without PALD_GPU_USE_REFERENCE_TYPES the shim declares layout- and
// behaviour-compatible domain types itself (namespace pald), so it also
// works stand-alone.
//
// Contract of every function (same as the reference drivers):
//   * input: a validated DistanceMatrix (double storage), converted to fp32
//     exactly like detail::to_real<float> (blocked.hpp:91-96);
//   * output: PaldResult by value -- U int32 n*n, C double n*n widened from
//     the fp32 result like detail::collect_result (blocked.hpp:352-359),
//     normalized = false;
//   * errors: ValidationError (block sizes < 1, workers < 1),
//     UnsupportedPolicyError (triplet with InclusiveSplit, as the
//     reference), std::runtime_error for CUDA failures. Pairwise supports
//     both policies.
//   * Real: the engine computes in fp32 (the reference's performance
//     instantiation); Real = double is rejected at compile time.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "pald_gpu.h"

#ifdef PALD_GPU_USE_REFERENCE_TYPES
#include "pald/types.hpp"
#else
namespace pald {

// Error hierarchy (reference types.hpp:14-25).
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationError : Error {
  using Error::Error;
};
struct UnsupportedPolicyError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};

// Comparison semantics (types.hpp:27-34).
enum class Policy { Strict, InclusiveSplit };

// Dense symmetric distance matrix; the validation rules are those of
// types.hpp:45-65 (n >= 2, zero diagonal, off-diagonal > 0, symmetric).
class DistanceMatrix {
 public:
  DistanceMatrix(std::size_t n, std::vector<double> values) : n_(n), v_(std::move(values)) {
    if (n_ < 2) throw ValidationError("distance matrix needs n >= 2, got n=" + std::to_string(n_));
    if (v_.size() != n_ * n_) throw ValidationError("distance matrix storage size does not match n*n");
    for (std::size_t x = 0; x < n_; ++x) {
      if (v_[x * n_ + x] != 0.0)
        throw ValidationError("distance matrix diagonal entry (" + std::to_string(x) + "," +
                              std::to_string(x) + ") is nonzero");
      for (std::size_t y = x + 1; y < n_; ++y) {
        const double a = v_[x * n_ + y];
        if (!(a > 0.0))
          throw ValidationError("off-diagonal distance (" + std::to_string(x) + "," +
                                std::to_string(y) + ") must be positive, got " +
                                std::to_string(a) + " (duplicate points are rejected)");
        if (a != v_[y * n_ + x])
          throw ValidationError("distance matrix not symmetric at (" + std::to_string(x) + "," +
                                std::to_string(y) + ")");
      }
    }
  }
  std::size_t size() const { return n_; }
  double operator()(std::size_t x, std::size_t y) const { return v_[x * n_ + y]; }
  const double* row(std::size_t x) const { return v_.data() + x * n_; }
  const std::vector<double>& values() const { return v_; }

 private:
  std::size_t n_;
  std::vector<double> v_;
};

struct FocusSizeMatrix {
  std::size_t n = 0;
  std::vector<std::int32_t> sizes;
  explicit FocusSizeMatrix(std::size_t n_ = 0) : n(n_), sizes(n_ * n_, 0) {}
  std::int32_t& at(std::size_t x, std::size_t y) { return sizes[x * n + y]; }
  std::int32_t at(std::size_t x, std::size_t y) const { return sizes[x * n + y]; }
};

struct CohesionMatrix {
  std::size_t n = 0;
  std::vector<double> values;
  bool normalized = false;
  explicit CohesionMatrix(std::size_t n_ = 0) : n(n_), values(n_ * n_, 0.0) {}
  double& at(std::size_t x, std::size_t z) { return values[x * n + z]; }
  double at(std::size_t x, std::size_t z) const { return values[x * n + z]; }
};

struct PaldResult {
  FocusSizeMatrix focus;
  CohesionMatrix cohesion;
};

struct PhaseTimes {
  double focus_seconds = 0.0;
  double cohesion_seconds = 0.0;
  double overhead_seconds = 0.0;
  double total_seconds = 0.0;
};

}  // namespace pald
#endif

namespace pald {
namespace gpu {

// blocked.hpp:30-32 and parallel.hpp:31-34 counterparts. The functions
// below take the style / plan as template parameters so the reference's own
// pald::UpdateStyle / pald::ParallelPlan can be passed unchanged.
enum class UpdateStyle { Masked, Branchy };

// parallel.hpp:31-34 plus the GPU side of "parallel": the devices one call
// spans (repeats allowed), the exchange transports of the two passes
// (pald_gpu_exchange) and the accurate-summation mode (PALD_GPU_FLAG_ACCURATE).
// A plan WITHOUT a `devices` member (the reference's own ParallelPlan) runs
// on the devices named by the environment variable PALD_GPU_DEVICES ("all"
// or a comma list such as "0,1,2,3"), else on the current device. Results
// do not depend on the device list (U and C bit-identical).
struct ParallelPlan {
  int workers = 1;
  bool deterministic = false;
  std::vector<int> devices;
  int exchange_focus = PALD_GPU_EXCHANGE_AUTO;
  int exchange_cohesion = PALD_GPU_EXCHANGE_AUTO;
  bool accurate = false;
};

namespace detail {

struct RunConfig {
  std::vector<int> devices;  // empty: the current device
  int exchange_focus = PALD_GPU_EXCHANGE_AUTO;
  int exchange_cohesion = PALD_GPU_EXCHANGE_AUTO;
  bool accurate = false;
};

inline RunConfig env_config() {
  RunConfig c;
  if (const char* e = std::getenv("PALD_GPU_DEVICES")) {
    const std::string s(e);
    if (s == "all") {
      for (int i = 0; i < pald_gpu_visible_devices() && i < PALD_GPU_MAX_DEVICES; ++i) c.devices.push_back(i);
    } else {
      std::size_t pos = 0;
      while (pos < s.size()) {
        const std::size_t q = s.find(',', pos);
        const std::string tok = s.substr(pos, q == std::string::npos ? std::string::npos : q - pos);
        if (!tok.empty()) c.devices.push_back(std::stoi(tok));
        if (q == std::string::npos) break;
        pos = q + 1;
      }
    }
  }
  if (const char* a = std::getenv("PALD_GPU_ACCURATE")) c.accurate = std::string(a) == "1";
  return c;
}

// The plan's own device list where it has one (SFINAE), else the environment.
template <class Plan>
auto plan_config(const Plan& p, int) -> decltype(p.devices, p.exchange_focus, p.exchange_cohesion, p.accurate,
                                                 RunConfig()) {
  RunConfig c = env_config();
  if (!p.devices.empty()) c.devices.assign(p.devices.begin(), p.devices.end());
  c.exchange_focus = p.exchange_focus;
  c.exchange_cohesion = p.exchange_cohesion;
  c.accurate = c.accurate || p.accurate;
  return c;
}
template <class Plan>
RunConfig plan_config(const Plan&, long) {
  return env_config();
}

inline void throw_status(int rc) {
  if (rc == PALD_GPU_OK) return;
  const std::string msg = pald_gpu_last_error();
  if (rc == PALD_GPU_ERR_VALIDATION) throw ValidationError(msg);
  if (rc == PALD_GPU_ERR_UNSUPPORTED) throw UnsupportedPolicyError(msg);
  if (rc == PALD_GPU_ERR_IO) throw IoError(msg);
  throw std::runtime_error("pald_gpu: " + msg);
}

// One C-ABI call with the reference's double I/O: D converted like
// to_real<float> (blocked.hpp:91-96) and C widened like collect_result
// (blocked.hpp:352-359), both on all host cores inside the library
// (pald_gpu_cohesion_f64io_*). The result vectors are built (zero-filled,
// as the reference's types do) while the GPU works.
inline PaldResult run(const DistanceMatrix& d, int algorithm, Policy policy, std::size_t b,
                      std::size_t bf, std::size_t bc, PhaseTimes* times, const RunConfig& cfg = env_config()) {
  pald_gpu_opts o;
  pald_gpu_opts_init(&o);
  o.algorithm = algorithm;
  o.policy = policy == Policy::Strict ? PALD_GPU_STRICT : PALD_GPU_INCLUSIVE_SPLIT;
  o.block = b;
  o.block_focus = bf;
  o.block_cohesion = bc;
  o.flags = PALD_GPU_FLAG_SKIP_VALIDATION;  // DistanceMatrix is validated in double
  if (cfg.accurate) o.flags |= PALD_GPU_FLAG_ACCURATE;
  if (cfg.devices.size() > PALD_GPU_MAX_DEVICES)
    throw ValidationError("at most " + std::to_string(PALD_GPU_MAX_DEVICES) + " devices per call");
  if (cfg.devices.size() == 1) o.device = cfg.devices[0];
  if (cfg.devices.size() > 1) {
    o.num_devices = static_cast<int32_t>(cfg.devices.size());
    for (std::size_t i = 0; i < cfg.devices.size(); ++i) o.devices[i] = cfg.devices[i];
  }
  o.exchange_focus = cfg.exchange_focus;
  o.exchange_cohesion = cfg.exchange_cohesion;
  const std::size_t n = d.size();
  pald_gpu_job* job = nullptr;
  throw_status(pald_gpu_cohesion_f64io_begin(d.values().data(), n, &o, &job));
  struct Join {  // end() must run even if building the result throws
    pald_gpu_job* j;
    ~Join() {
      if (j) pald_gpu_cohesion_f64io_end(j, nullptr, nullptr, nullptr);
    }
  } join{job};
  // The result as the reference's types build it (n * n zero-filled
  // entries): the storage is reserved, first-touched by all host cores
  // inside the library, then value-initialised by resize() on the resident
  // pages -- the single-threaded page faults of a fresh 12 GiB result at
  // n = 32768 would otherwise outlast the GPU work.
  PaldResult r{FocusSizeMatrix(0), CohesionMatrix(0)};
  r.focus.n = n;
  r.cohesion.n = n;
  r.focus.sizes.reserve(n * n);
  r.cohesion.values.reserve(n * n);
  pald_gpu_host_prefault(r.focus.sizes.data(), n * n * sizeof(r.focus.sizes[0]));
  pald_gpu_host_prefault(r.cohesion.values.data(), n * n * sizeof(r.cohesion.values[0]));
  r.focus.sizes.resize(n * n);
  r.cohesion.values.resize(n * n);
  // C rows are widened into the result as their copies land during pass 2
  throw_status(pald_gpu_cohesion_f64io_outputs(job, r.focus.sizes.data(), r.cohesion.values.data()));
  pald_gpu_phase_times t{};
  join.j = nullptr;
  throw_status(pald_gpu_cohesion_f64io_end(job, nullptr, nullptr, &t));
  if (times) {
    times->focus_seconds += t.focus_seconds;
    times->cohesion_seconds += t.cohesion_seconds;
    times->overhead_seconds += t.overhead_seconds;
    times->total_seconds = t.total_seconds;
  }
  return r;
}

template <class Real>
constexpr void check_real() {
  static_assert(sizeof(Real) == sizeof(float),
                "pald::gpu computes in fp32: instantiate with Real = float");
}

}  // namespace detail

// blocked.hpp:368-418
template <class Real = float, class Style = UpdateStyle>
PaldResult blocked_pairwise(const DistanceMatrix& d, std::size_t b, Policy policy = Policy::Strict,
                            PhaseTimes* times = nullptr, Style style = Style{}) {
  (void)style;
  detail::check_real<Real>();
  if (b < 1) throw ValidationError("pairwise block size must be >= 1");
  return detail::run(d, PALD_GPU_PAIRWISE, policy, b, 128, 128, times);
}

// blocked.hpp:424-477 (C diagonal left 0; see fill_diagonal)
template <class Real = float, class Style = UpdateStyle>
PaldResult blocked_triplet(const DistanceMatrix& d, std::size_t b_focus, std::size_t b_cohesion,
                           Policy policy = Policy::Strict, PhaseTimes* times = nullptr,
                           Style style = Style{}) {
  (void)style;
  detail::check_real<Real>();
  if (policy != Policy::Strict)
    throw UnsupportedPolicyError("the triplet algorithm supports the strict policy only");
  if (b_focus < 1 || b_cohesion < 1) throw ValidationError("triplet block sizes must be >= 1");
  return detail::run(d, PALD_GPU_TRIPLET, policy, 128, b_focus, b_cohesion, times);
}

// parallel.hpp:159-222. The plan's devices (or PALD_GPU_DEVICES) split the
// work of ONE call across GPUs (pald_gpu_opts.devices); bit-identical to
// blocked_pairwise, as in the reference (test_parallel.cpp:61-76).
template <class Real = float, class Plan = ParallelPlan, class Style = UpdateStyle>
PaldResult parallel_pairwise(const DistanceMatrix& d, std::size_t b, const Plan& plan,
                             Policy policy = Policy::Strict, PhaseTimes* times = nullptr,
                             Style style = Style{}) {
  (void)style;
  detail::check_real<Real>();
  if (plan.workers < 1) throw ValidationError("worker count must be >= 1");
  if (b < 1) throw ValidationError("pairwise block size must be >= 1");
  return detail::run(d, PALD_GPU_PAIRWISE, policy, b, 128, 128, times, detail::plan_config(plan, 0));
}

// parallel.hpp:257-320
template <class Real = float, class Plan = ParallelPlan, class Style = UpdateStyle>
PaldResult parallel_triplet(const DistanceMatrix& d, std::size_t b_focus, std::size_t b_cohesion,
                            const Plan& plan, Policy policy = Policy::Strict,
                            PhaseTimes* times = nullptr, Style style = Style{}) {
  (void)style;
  detail::check_real<Real>();
  if (policy != Policy::Strict)
    throw UnsupportedPolicyError("the triplet algorithm supports the strict policy only");
  if (plan.workers < 1) throw ValidationError("worker count must be >= 1");
  if (b_focus < 1 || b_cohesion < 1) throw ValidationError("triplet block sizes must be >= 1");
  return detail::run(d, PALD_GPU_TRIPLET, policy, 128, b_focus, b_cohesion, times, detail::plan_config(plan, 0));
}

}  // namespace gpu
}  // namespace pald
