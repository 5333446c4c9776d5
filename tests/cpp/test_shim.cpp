// C++ shim tests, written like the reference's own tests
// (proj/tests/test_reference.cpp, test_blocked.cpp, test_parallel.cpp) but
// against pald::gpu::*. Plain assertions (doctest is not available).
//
//   test_shim --cpu-only   argument validation only (no GPU needed)
//   test_shim              full run on the GPU, parity against liboracle.so
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#ifdef PALD_GPU_USE_REFERENCE_TYPES
#include "pald/pald.hpp"
#endif
#include "pald_gpu.hpp"

extern "C" void pald_oracle_pairwise_f32(const float* d, uint64_t n, int32_t* u, float* c);
extern "C" void pald_oracle_pairwise_policy_f32(const float* d, uint64_t n, int policy, int32_t* u, float* c);
extern "C" void pald_oracle_triplet_f32in_f64(const float* d, uint64_t n, int32_t* u, double* c);

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
      ++failures;                                                    \
    }                                                                \
  } while (0)

template <class E, class F>
static bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// helpers.hpp:13-19 -- build from the strict upper triangle
static pald::DistanceMatrix dmat(std::size_t n, std::vector<double> upper) {
  std::vector<double> v(n * n, 0.0);
  std::size_t k = 0;
  for (std::size_t x = 0; x < n; ++x)
    for (std::size_t y = x + 1; y < n; ++y) v[x * n + y] = v[y * n + x] = upper[k++];
  return pald::DistanceMatrix(n, std::move(v));
}

static pald::DistanceMatrix random_d(std::size_t n, unsigned seed, bool ties) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.5, 2.0);
  std::uniform_int_distribution<int> ui(1, 16);
  std::vector<double> up;
  for (std::size_t i = 0; i < n * (n - 1) / 2; ++i) up.push_back(ties ? ui(rng) : u(rng));
  return dmat(n, up);
}

static bool close(double a, double b) { return std::fabs(a - b) <= 1e-6; }

static void cpu_only() {
  const auto d3 = dmat(3, {1.0, 2.0, 3.0});
  using pald::Policy;
  CHECK(throws_as<pald::ValidationError>([&] { pald::gpu::blocked_pairwise<float>(d3, 0); }));
  CHECK(throws_as<pald::ValidationError>([&] { pald::gpu::blocked_triplet<float>(d3, 0, 1); }));
  CHECK(throws_as<pald::ValidationError>([&] { pald::gpu::blocked_triplet<float>(d3, 1, 0); }));
  CHECK(throws_as<pald::UnsupportedPolicyError>(
      [&] { pald::gpu::blocked_triplet<float>(d3, 1, 1, Policy::InclusiveSplit); }));
  CHECK(throws_as<pald::ValidationError>(
      [&] { pald::gpu::parallel_pairwise<float>(d3, 1, pald::gpu::ParallelPlan{0, true}); }));
  CHECK(throws_as<pald::ValidationError>(
      [&] { pald::gpu::parallel_pairwise<float>(d3, 0, pald::gpu::ParallelPlan{2, true}); }));
  CHECK(throws_as<pald::UnsupportedPolicyError>([&] {
    pald::gpu::parallel_triplet<float>(d3, 1, 1, pald::gpu::ParallelPlan{2, true},
                                       Policy::InclusiveSplit);
  }));
  CHECK(throws_as<pald::ValidationError>([&] { dmat(3, {1.0, 0.0, 3.0}); }));
#ifdef PALD_GPU_USE_REFERENCE_TYPES
  // the reference's own ParallelPlan / UpdateStyle are accepted unchanged
  CHECK(throws_as<pald::ValidationError>(
      [&] { pald::gpu::parallel_pairwise<float>(d3, 1, pald::ParallelPlan{0, true}); }));
  CHECK(throws_as<pald::ValidationError>([&] {
    pald::gpu::blocked_pairwise<float>(d3, 0, Policy::Strict, nullptr, pald::UpdateStyle::Branchy);
  }));
#endif
}

static void gpu_tests() {
  using pald::Policy;
  // Hand-traced fixtures (test_reference.cpp:70-87, acceptance.cpp:120-146).
  const auto d3 = dmat(3, {1.0, 2.0, 3.0});
  auto r = pald::gpu::blocked_pairwise<float>(d3, 1);
  CHECK(r.focus.at(0, 1) == 2 && r.focus.at(1, 0) == 2);
  CHECK(r.focus.at(0, 2) == 3 && r.focus.at(1, 2) == 3);
  CHECK(!r.cohesion.normalized);
  CHECK(close(r.cohesion.at(0, 0), 5.0 / 6) && close(r.cohesion.at(1, 1), 5.0 / 6));
  CHECK(close(r.cohesion.at(2, 2), 2.0 / 3) && close(r.cohesion.at(0, 1), 1.0 / 3));
  CHECK(r.cohesion.at(0, 2) == 0.0);
  const auto d2 = dmat(2, {5.0});
  auto r2 = pald::gpu::blocked_pairwise<float>(d2, 7);
  CHECK(r2.focus.at(0, 1) == 2 && r2.cohesion.at(0, 0) == 0.5 && r2.cohesion.at(1, 1) == 0.5);
  const auto t3 = dmat(3, {1.0, 1.0, 1.0});
  auto rt = pald::gpu::blocked_pairwise<float>(t3, 2);
  for (std::size_t x = 0; x < 3; ++x)
    for (std::size_t z = 0; z < 3; ++z) {
      CHECK(rt.cohesion.at(x, z) == (x == z ? 1.0 : 0.0));
      if (x != z) CHECK(rt.focus.at(x, z) == 2);
    }
  // Triplet D3 (test_reference.cpp:89-101): diagonal left 0.
  auto tr = pald::gpu::blocked_triplet<float>(d3, 1, 1);
  CHECK(tr.focus.at(0, 1) == 2 && tr.focus.at(0, 2) == 3 && tr.focus.at(1, 2) == 3);
  CHECK(close(tr.cohesion.at(0, 1), 1.0 / 3) && close(tr.cohesion.at(1, 0), 1.0 / 3));
  CHECK(tr.cohesion.at(0, 0) == 0.0);
  auto tr2 = pald::gpu::blocked_triplet<float>(d2, 1, 1);
  CHECK(tr2.focus.at(0, 1) == 2 && tr2.cohesion.at(0, 1) == 0.0);

  // Grid: blocked / parallel vs the fp32 reference-order oracle, bit-exact
  // (test_blocked.cpp:38-50, test_parallel.cpp:61-76).
  for (std::size_t n : {2, 5, 16, 33, 65, 130}) {
    for (bool ties : {false, true}) {
      const auto d = random_d(n, 1000 + n, ties);
      std::vector<float> df(n * n);
      for (std::size_t i = 0; i < n * n; ++i) df[i] = static_cast<float>(d.values()[i]);
      std::vector<int32_t> uo(n * n);
      std::vector<float> co(n * n);
      pald_oracle_pairwise_f32(df.data(), n, uo.data(), co.data());
      for (std::size_t b : {std::size_t(1), std::size_t(3), n + 7}) {
        const auto g = pald::gpu::blocked_pairwise<float>(d, b);
        CHECK(g.focus.sizes == uo);
        bool same = true;
        for (std::size_t i = 0; i < n * n; ++i) same &= g.cohesion.values[i] == (double)co[i];
        CHECK(same);
      }
      {  // InclusiveSplit (blocked.hpp:150-158), bit-exact as well
        std::vector<int32_t> us(n * n);
        std::vector<float> cs(n * n);
        pald_oracle_pairwise_policy_f32(df.data(), n, 1, us.data(), cs.data());
        const auto g = pald::gpu::blocked_pairwise<float>(d, 4, Policy::InclusiveSplit);
        CHECK(g.focus.sizes == us);
        bool same = true;
        for (std::size_t i = 0; i < n * n; ++i) same &= g.cohesion.values[i] == (double)cs[i];
        CHECK(same);
      }
      pald::PhaseTimes pt;
      const auto p = pald::gpu::parallel_pairwise<float>(d, 5, pald::gpu::ParallelPlan{8, true},
                                                         Policy::Strict, &pt);
      CHECK(p.focus.sizes == uo);
      CHECK(pt.total_seconds > 0.0);
      CHECK(pt.focus_seconds + pt.cohesion_seconds + pt.overhead_seconds <= pt.total_seconds * 1.001);
      // triplet: U exact, C within 1e-5 (rel_diff, helpers.hpp:30-33)
      std::vector<int32_t> ut(n * n);
      std::vector<double> ct(n * n);
      pald_oracle_triplet_f32in_f64(df.data(), n, ut.data(), ct.data());
      const auto t = pald::gpu::parallel_triplet<float>(d, 8, 4, pald::gpu::ParallelPlan{4, true});
      CHECK(t.focus.sizes == ut);
      double worst = 0;
      for (std::size_t i = 0; i < n * n; ++i) {
        const double a = t.cohesion.values[i], bb = ct[i];
        worst = std::max(worst, std::fabs(a - bb) / std::max({std::fabs(a), std::fabs(bb), 1.0}));
      }
      CHECK(worst <= 1e-5);
    }
  }
}

// parallel_* over a device list (pald::gpu::ParallelPlan::devices, one C-ABI
// call spanning the listed GPUs) == one device, bit for bit.
static void device_list_tests(const std::vector<int>& devs) {
  using pald::Policy;
  for (std::size_t n : {std::size_t(130), std::size_t(1000), std::size_t(2304)}) {
    for (bool ties : {false, true}) {
      const auto d = random_d(n, 77 + n, ties);
      pald::gpu::ParallelPlan plan;
      plan.workers = 4;
      plan.devices = devs;
      const auto one = pald::gpu::blocked_pairwise<float>(d, 64);
      const auto many = pald::gpu::parallel_pairwise<float>(d, 64, plan);
      CHECK(one.focus.sizes == many.focus.sizes);
      CHECK(one.cohesion.values == many.cohesion.values);
      const auto t1 = pald::gpu::blocked_triplet<float>(d, 64, 64);
      const auto tm = pald::gpu::parallel_triplet<float>(d, 64, 64, plan);
      CHECK(t1.focus.sizes == tm.focus.sizes);
      CHECK(t1.cohesion.values == tm.cohesion.values);
      const auto s1 = pald::gpu::blocked_pairwise<float>(d, 64, Policy::InclusiveSplit);
      const auto sm = pald::gpu::parallel_pairwise<float>(d, 64, plan, Policy::InclusiveSplit);
      CHECK(s1.focus.sizes == sm.focus.sizes);
      CHECK(s1.cohesion.values == sm.cohesion.values);
    }
  }
  if (!failures) std::printf("device list ok (%zu devices)\n", devs.size());
}

int main(int argc, char** argv) {
  const bool cpu = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
  if (argc > 2 && std::strcmp(argv[1], "--devices") == 0) {
    std::vector<int> devs;
    for (const char* p = argv[2]; *p;) {
      devs.push_back(std::atoi(p));
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
    device_list_tests(devs);
    std::printf("devices: %d failure(s)\n", failures);
    return failures ? 1 : 0;
  }
  cpu_only();
  if (!cpu) gpu_tests();
  std::printf("%s: %d failure(s)\n", cpu ? "cpu-only" : "full", failures);
  return failures ? 1 : 0;
}
