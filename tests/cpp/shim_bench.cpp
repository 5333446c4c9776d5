// shim_bench.cpp -- end-to-end timing of the drop-in C++ call a reference
// user makes: pald::gpu::parallel_pairwise<float>(DistanceMatrix, b, plan)
// compiled against the reference's OWN types (PALD_GPU_USE_REFERENCE_TYPES),
// i.e. double D in, PaldResult (int32 U + double C, freshly allocated) out,
// exactly the contract of parallel.hpp:159-222.
//
//   shim_bench <points.f64> <n> <dim> <steps> <warmup> [devices]
//
// The points file holds n*dim doubles (row-major); D is built with the
// reference's own points_to_distances (ingest.hpp:303-322), outside the
// timed region. Prints one JSON line. Built by oracle/Makefile into
// oracle/_ref/ (needs the reference headers); run by bench.py.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
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
  const auto t_build0 = std::chrono::steady_clock::now();
  const pald::DistanceMatrix d = pald::points_to_distances(pc);
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
