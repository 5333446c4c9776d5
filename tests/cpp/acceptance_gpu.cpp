// acceptance_gpu.cpp -- drop-in proof of the C++ shim: the reference's
// acceptance corpus (200 matrices, n = 2 + i*7919 % 63, seeds 0xACCE0000 + i;
// the corpus of proj/tests/acceptance.cpp:37-43, generated with the
// reference's own detail::random_distances) run through pald::gpu::* compiled
// against the reference's OWN types (PALD_GPU_USE_REFERENCE_TYPES) and through
// the reference's pald::blocked_* / pald::parallel_* in the same process.
//
//   U        exact (every variant, both policies)
//   pairwise C   bit-exact vs blocked_pairwise<float> / parallel_pairwise<float>
//   triplet C    rel_diff <= 1e-5 vs blocked_triplet<double> (helpers.hpp:30-33);
//                after fill_diagonal, <= 1e-5 vs pairwise_entrywise (no ties)
//
// Built by oracle/Makefile (needs the reference headers) into oracle/_ref/;
// run by tests/test_gpu_reference.py on the GPU box. Test code only.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <utility>
#include <vector>

#define PALD_GPU_USE_REFERENCE_TYPES
#include "pald/pald.hpp"
#include "pald_gpu.hpp"

namespace {

int failures = 0;
double worst_tr = 0, worst_fill = 0;

void fail(const char* what, std::size_t i, std::size_t n) {
  if (failures < 20) std::printf("FAIL %s: matrix %zu (n=%zu)\n", what, i, n);
  ++failures;
}

double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double w = 0;
  for (std::size_t k = 0; k < a.size(); ++k)
    w = std::max(w, std::fabs(a[k] - b[k]) / std::max({std::fabs(a[k]), std::fabs(b[k]), 1.0}));
  return w;
}

bool same(const pald::PaldResult& a, const pald::PaldResult& b) {
  return a.focus.sizes == b.focus.sizes && a.cohesion.values == b.cohesion.values;
}

}  // namespace

int main() {
  using pald::Policy;
  std::size_t cases = 0;
  for (std::uint64_t i = 0; i < 200; ++i) {
    const auto d = pald::detail::random_distances(2 + i * 7919 % 63, 0xACCE0000 + i);
    const std::size_t n = d.size();
    // pairwise, both policies: reference fp32 drivers vs the GPU shim
    for (Policy pol : {Policy::Strict, Policy::InclusiveSplit}) {
      const auto ref = pald::blocked_pairwise<float>(d, 8, pol);
      if (!same(ref, pald::parallel_pairwise<float>(d, 8, {4, true}, pol))) fail("reference self-check", i, n);
      for (std::size_t b : {std::size_t(1), std::size_t(3), std::size_t(8), n, n + 7}) {
        ++cases;
        if (!same(ref, pald::gpu::blocked_pairwise<float>(d, b, pol))) fail("gpu blocked_pairwise", i, n);
      }
      for (int p : {2, 4, 8}) {
        ++cases;
        // the reference's own ParallelPlan type, unchanged
        if (!same(ref, pald::gpu::parallel_pairwise<float>(d, 8, pald::ParallelPlan{p, true}, pol)))
          fail("gpu parallel_pairwise", i, n);
      }
    }
    // triplet: U exact; C (diagonal 0) against the fp64 reference
    const auto tref = pald::blocked_triplet<double>(d, 4, 8);
    using P = std::pair<std::size_t, std::size_t>;
    for (auto [bf, bc] : {P{1, 1}, P{4, 8}, P{16, 4}}) {
      ++cases;
      auto g = pald::gpu::blocked_triplet<float>(d, bf, bc);
      if (g.focus.sizes != tref.focus.sizes) fail("gpu blocked_triplet U", i, n);
      worst_tr = std::max(worst_tr, max_rel(g.cohesion.values, tref.cohesion.values));
    }
    {
      ++cases;
      auto g = pald::gpu::parallel_triplet<float>(d, 8, 8, pald::ParallelPlan{4, true});
      if (g.focus.sizes != tref.focus.sizes) fail("gpu parallel_triplet U", i, n);
      worst_tr = std::max(worst_tr, max_rel(g.cohesion.values, tref.cohesion.values));
      // criterion-2 form: triplet + fill_diagonal == the entrywise pairwise pass
      pald::fill_diagonal(g.focus, g.cohesion);
      const auto pe = pald::pairwise_entrywise(d, Policy::Strict);
      if (g.focus.sizes != pe.focus.sizes) fail("triplet vs pairwise U (no ties)", i, n);
      worst_fill = std::max(worst_fill, max_rel(g.cohesion.values, pe.cohesion.values));
    }
    // errors: the reference's exception types
    bool threw = false;
    try {
      pald::gpu::blocked_triplet<float>(d, 1, 1, Policy::InclusiveSplit);
    } catch (const pald::UnsupportedPolicyError&) {
      threw = true;
    }
    if (!threw) fail("UnsupportedPolicyError", i, n);
  }
  if (worst_tr > 1e-5) fail("triplet C rel_diff > 1e-5", 0, 0);
  if (worst_fill > 1e-5) fail("triplet+fill vs pairwise_entrywise > 1e-5", 0, 0);
  std::printf("acceptance corpus: 200 matrices, %zu GPU calls, triplet C max rel_diff %.3g, "
              "triplet+fill vs entrywise %.3g, %d failure(s)\n",
              cases, worst_tr, worst_fill, failures);
  return failures ? 1 : 0;
}
