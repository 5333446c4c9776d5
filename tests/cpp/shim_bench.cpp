// shim_bench.cpp -- end-to-end timing of the drop-in C++ call a reference
// user makes: pald::gpu::parallel_pairwise<float>(DistanceMatrix, b, plan)
// compiled against the reference's OWN types (PALD_GPU_USE_REFERENCE_TYPES),
// i.e. double D in, PaldResult (int32 U + double C, freshly allocated) out,
// exactly the contract of parallel.hpp:159-222.
//
//   shim_bench <points.f64> <n> <dim> <steps> <warmup> [devices]
//
// The points file holds n*dim doubles (row-major); D is built from them
// with the arithmetic of the reference's points_to_distances
// (ingest.hpp:303-322) on all host cores and validated by the reference's
// DistanceMatrix constructor, outside the timed region. Prints one JSON line. Built by oracle/Makefile into
// oracle/_ref/ (needs the reference headers); run by bench.py.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <algorithm>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#define PALD_GPU_USE_REFERENCE_TYPES
#include "pald/pald.hpp"
#include "pald_gpu.hpp"

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: shim_bench points.f64 n dim steps warmup [devices]\n");
    return 2;
  }
  const std::size_t n = std::strtoull(argv[2], nullptr, 10), dim = std::strtoull(argv[3], nullptr, 10);
  const int steps = std::atoi(argv[4]), warmup = std::atoi(argv[5]);
  pald::PointCloud pc;
  pc.n = n;
  pc.dim = dim;
  pc.coords.resize(n * dim);
  std::ifstream in(argv[1], std::ios::binary);
  in.read(reinterpret_cast<char*>(pc.coords.data()), (std::streamsize)(n * dim * sizeof(double)));
  if (!in) {
    std::fprintf(stderr, "cannot read %zu points from %s\n", n, argv[1]);
    return 2;
  }
  // D (outside the timed region): the arithmetic of the reference's
  // points_to_distances (ingest.hpp:303-322: squared differences summed in
  // coordinate order, sqrt, in double), computed row by row on all host cores
  // -- every entry from its own row, so no strided mirror writes; (a - b)^2 ==
  // (b - a)^2 keeps it exactly symmetric -- and handed to the reference's own
  // DistanceMatrix constructor, which validates it. (The reference function
  // itself takes 75 s single-threaded at n = 32768.)
  const auto t_build0 = std::chrono::steady_clock::now();
  std::vector<double> vals;
  vals.reserve(n * n);
  pald_gpu_host_prefault(vals.data(), n * n * sizeof(double));
  vals.resize(n * n);
  {
    const unsigned T = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    double* v = vals.data();
    const double* c = pc.coords.data();
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([=] {
        for (std::size_t x = n * t / T; x < n * (t + 1) / T; ++x)
          for (std::size_t y = 0; y < n; ++y) {
            double sum = 0.0;
            for (std::size_t k = 0; k < dim; ++k) {
              const double diff = c[x * dim + k] - c[y * dim + k];
              sum += diff * diff;
            }
            v[x * n + y] = x == y ? 0.0 : std::sqrt(sum);
          }
      });
    for (auto& x : th) x.join();
  }
  const pald::DistanceMatrix d(n, std::move(vals));
  const double build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_build0).count();
  pald::gpu::ParallelPlan plan;
  plan.workers = 1;
  if (argc > 6) {
    for (const char* p = argv[6]; *p;) {
      plan.devices.push_back(std::atoi(p));
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
  }
  std::vector<double> times;
  double checksum = 0;
  pald::PhaseTimes last{};
  for (int i = 0; i < warmup + steps; ++i) {
    pald::PhaseTimes pt;
    const auto t0 = std::chrono::steady_clock::now();
    const pald::PaldResult r = pald::gpu::parallel_pairwise<float>(d, 1024, plan, pald::Policy::Strict, &pt);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (i >= warmup) times.push_back(s);
    checksum = 0;
    for (std::size_t z = 0; z < n; ++z) checksum += r.cohesion.values[z];
    last = pt;
  }
  double mean = 0;
  for (double t : times) mean += t;
  mean /= times.empty() ? 1 : (double)times.size();
  std::printf("{\"n\": %zu, \"steps\": %d, \"warmup\": %d, \"seconds_per_step\": %.6f, \"times\": [", n, steps, warmup,
              mean);
  for (std::size_t i = 0; i < times.size(); ++i) std::printf("%s%.6f", i ? ", " : "", times[i]);
  std::printf("], \"phase_times\": {\"focus\": %.6f, \"cohesion\": %.6f, \"overhead\": %.6f, \"total\": %.6f}, "
              "\"devices\": %zu, \"d_build_s\": %.3f, \"row0_sum\": %.17g}\n",
              last.focus_seconds, last.cohesion_seconds, last.overhead_seconds, last.total_seconds,
              plan.devices.size() ? plan.devices.size() : (std::size_t)1, build_s, checksum);
  return 0;
}
