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
struct ParallelPlan {
  int workers = 1;
  bool deterministic = false;
};

namespace detail {

inline void throw_status(int rc) {
  if (rc == PALD_GPU_OK) return;
  const std::string msg = pald_gpu_last_error();
  if (rc == PALD_GPU_ERR_VALIDATION) throw ValidationError(msg);
  if (rc == PALD_GPU_ERR_UNSUPPORTED) throw UnsupportedPolicyError(msg);
  if (rc == PALD_GPU_ERR_IO) throw IoError(msg);
  throw std::runtime_error("pald_gpu: " + msg);
}

inline PaldResult run(const DistanceMatrix& d, int algorithm, Policy policy, std::size_t b,
                      std::size_t bf, std::size_t bc, PhaseTimes* times) {
  pald_gpu_opts o;
  pald_gpu_opts_init(&o);
  o.algorithm = algorithm;
  o.policy = policy == Policy::Strict ? PALD_GPU_STRICT : PALD_GPU_INCLUSIVE_SPLIT;
  o.block = b;
  o.block_focus = bf;
  o.block_cohesion = bc;
  o.flags = PALD_GPU_FLAG_SKIP_VALIDATION;  // DistanceMatrix is validated in double
  const std::size_t n = d.size();
  std::vector<float> dd(n * n);  // to_real<float>, blocked.hpp:91-96
  for (std::size_t i = 0; i < dd.size(); ++i) dd[i] = static_cast<float>(d.values()[i]);
  PaldResult r{FocusSizeMatrix(n), CohesionMatrix(n)};
  std::vector<float> c(n * n);
  pald_gpu_phase_times t{};
  throw_status(pald_gpu_cohesion_f32(dd.data(), n, &o, r.focus.sizes.data(), c.data(), &t));
  for (std::size_t i = 0; i < c.size(); ++i) r.cohesion.values[i] = static_cast<double>(c[i]);
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

// parallel.hpp:159-222
template <class Real = float, class Plan = ParallelPlan, class Style = UpdateStyle>
PaldResult parallel_pairwise(const DistanceMatrix& d, std::size_t b, const Plan& plan,
                             Policy policy = Policy::Strict, PhaseTimes* times = nullptr,
                             Style style = Style{}) {
  if (plan.workers < 1) throw ValidationError("worker count must be >= 1");
  return blocked_pairwise<Real>(d, b, policy, times, style);
}

// parallel.hpp:257-320
template <class Real = float, class Plan = ParallelPlan, class Style = UpdateStyle>
PaldResult parallel_triplet(const DistanceMatrix& d, std::size_t b_focus, std::size_t b_cohesion,
                            const Plan& plan, Policy policy = Policy::Strict,
                            PhaseTimes* times = nullptr, Style style = Style{}) {
  if (policy != Policy::Strict)
    throw UnsupportedPolicyError("the triplet algorithm supports the strict policy only");
  if (plan.workers < 1) throw ValidationError("worker count must be >= 1");
  return blocked_triplet<Real>(d, b_focus, b_cohesion, policy, times, style);
}

}  // namespace gpu
}  // namespace pald
