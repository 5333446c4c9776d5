// ref_bridge.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against
// the reference headers where they lie (/root/reference/proj/include; read
// only, never copied) into oracle/_ref/libpald_ref*.so. Used to
//   * generate golden vectors (tests/golden/make_golden.py),
//   * validate the C restatement in oracle/pald_oracle.c,
//   * time the reference CPU implementation (bench.py cpu_baseline and
//     --impl reference).
// Every function forwards to the reference symbol it names; the only logic
// here is marshalling (and, for the bounded timing sample, the body of the
// parallel_pairwise driver loop for a list of block pairs,
// parallel.hpp:178-215, around the reference's own block functions).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pald/pald.hpp"

namespace {

thread_local std::string g_err;

pald::DistanceMatrix make_d(const double* d, uint64_t n) {
  return pald::DistanceMatrix(n, std::vector<double>(d, d + n * n));
}

void out_result(const pald::PaldResult& r, int32_t* u, double* c) {
  const size_t nn = r.focus.sizes.size();
  if (u) std::memcpy(u, r.focus.sizes.data(), sizeof(int32_t) * nn);
  if (c) std::memcpy(c, r.cohesion.values.data(), sizeof(double) * nn);
}

void out_times(const pald::PhaseTimes& t, double* times) {
  if (!times) return;
  times[0] = t.focus_seconds;
  times[1] = t.cohesion_seconds;
  times[2] = t.overhead_seconds;
  times[3] = t.total_seconds;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const pald::UnsupportedPolicyError& e) {
    g_err = e.what();
    return 3;
  } catch (const pald::IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const pald::Error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

pald::Policy pol(int p) { return p == 0 ? pald::Policy::Strict : pald::Policy::InclusiveSplit; }

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// detail::random_distances, blocked.hpp:522-529
int ref_random_distances(uint64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const auto d = pald::detail::random_distances(n, seed);
    std::memcpy(out, d.values().data(), sizeof(double) * n * n);
  });
}

// DistanceMatrix validation, types.hpp:45-65
int ref_validate(const double* d, uint64_t n) {
  return guarded([&] { (void)make_d(d, n); });
}

// focus_size, reference.hpp:31-45
int ref_focus_size(const double* d, uint64_t n, uint64_t x, uint64_t y, int policy, int* out) {
  return guarded([&] { *out = pald::focus_size(make_d(d, n), x, y, pol(policy)); });
}

// pairwise_entrywise, reference.hpp:104-147
int ref_pairwise_entrywise(const double* d, uint64_t n, int policy, int32_t* u, double* c) {
  return guarded([&] { out_result(pald::pairwise_entrywise(make_d(d, n), pol(policy)), u, c); });
}

// triplet_entrywise, reference.hpp:154-208
int ref_triplet_entrywise(const double* d, uint64_t n, int validate_ties, int32_t* u, double* c) {
  return guarded([&] { out_result(pald::triplet_entrywise(make_d(d, n), validate_ties != 0), u, c); });
}

// oracle_cohesion, reference.hpp:73-99 (normalized; no-ties oracle only)
int ref_oracle_cohesion(const double* d, uint64_t n, int policy, double* c) {
  return guarded([&] {
    const auto r = pald::oracle_cohesion(make_d(d, n), pol(policy));
    std::memcpy(c, r.values.data(), sizeof(double) * n * n);
  });
}

// blocked_pairwise<Real>, blocked.hpp:368-418
int ref_blocked_pairwise(const double* d, uint64_t n, uint64_t b, int policy, int use_float,
                         int32_t* u, double* c, double* times) {
  return guarded([&] {
    pald::PhaseTimes t;
    const auto dm = make_d(d, n);
    if (use_float) out_result(pald::blocked_pairwise<float>(dm, b, pol(policy), &t), u, c);
    else out_result(pald::blocked_pairwise<double>(dm, b, pol(policy), &t), u, c);
    out_times(t, times);
  });
}

// blocked_triplet<Real>, blocked.hpp:424-477
int ref_blocked_triplet(const double* d, uint64_t n, uint64_t bf, uint64_t bc, int policy,
                        int use_float, int32_t* u, double* c, double* times) {
  return guarded([&] {
    pald::PhaseTimes t;
    const auto dm = make_d(d, n);
    if (use_float) out_result(pald::blocked_triplet<float>(dm, bf, bc, pol(policy), &t), u, c);
    else out_result(pald::blocked_triplet<double>(dm, bf, bc, pol(policy), &t), u, c);
    out_times(t, times);
  });
}

// parallel_pairwise<Real>, parallel.hpp:159-222
int ref_parallel_pairwise(const double* d, uint64_t n, uint64_t b, int workers, int policy,
                          int use_float, int32_t* u, double* c, double* times) {
  return guarded([&] {
    pald::PhaseTimes t;
    const auto dm = make_d(d, n);
    const pald::ParallelPlan plan{workers, true};
    if (use_float) out_result(pald::parallel_pairwise<float>(dm, b, plan, pol(policy), &t), u, c);
    else out_result(pald::parallel_pairwise<double>(dm, b, plan, pol(policy), &t), u, c);
    out_times(t, times);
  });
}

// parallel_triplet<Real>, parallel.hpp:257-320
int ref_parallel_triplet(const double* d, uint64_t n, uint64_t bf, uint64_t bc, int workers,
                         int policy, int use_float, int32_t* u, double* c, double* times) {
  return guarded([&] {
    pald::PhaseTimes t;
    const auto dm = make_d(d, n);
    const pald::ParallelPlan plan{workers, true};
    if (use_float)
      out_result(pald::parallel_triplet<float>(dm, bf, bc, plan, pol(policy), &t), u, c);
    else
      out_result(pald::parallel_triplet<double>(dm, bf, bc, plan, pol(policy), &t), u, c);
    out_times(t, times);
  });
}

// fill_diagonal / normalize / local_depths, reference.hpp:213-241
int ref_fill_diagonal(const int32_t* u, uint64_t n, double* c) {
  return guarded([&] {
    pald::FocusSizeMatrix f(n);
    std::memcpy(f.sizes.data(), u, sizeof(int32_t) * n * n);
    pald::CohesionMatrix cm(n);
    std::memcpy(cm.values.data(), c, sizeof(double) * n * n);
    pald::fill_diagonal(f, cm);
    std::memcpy(c, cm.values.data(), sizeof(double) * n * n);
  });
}

int ref_normalize_and_depths(double* c, uint64_t n, double* depths) {
  return guarded([&] {
    pald::CohesionMatrix cm(n);
    std::memcpy(cm.values.data(), c, sizeof(double) * n * n);
    pald::normalize(cm);
    const auto ld = pald::local_depths(cm);
    std::memcpy(c, cm.values.data(), sizeof(double) * n * n);
    std::memcpy(depths, ld.depths.data(), sizeof(double) * n);
  });
}

// read_distance_binary, ingest.hpp:280-283 (values copied when n <= cap)
int ref_read_distance_binary(const char* path, uint64_t cap, uint64_t* n_out, double* out) {
  return guarded([&] {
    const auto d = pald::read_distance_binary(path);
    *n_out = d.size();
    if (d.size() <= cap) std::memcpy(out, d.values().data(), sizeof(double) * d.size() * d.size());
  });
}

// default_block_config, blocked.hpp:510-518 (cache_bytes 0 = detect)
int ref_default_block_config(uint64_t element_bytes, uint64_t cache_bytes, uint64_t* out3) {
  return guarded([&] {
    const auto cfg = cache_bytes ? pald::default_block_config(element_bytes, cache_bytes)
                                 : pald::default_block_config(element_bytes);
    out3[0] = cfg.b;
    out3[1] = cfg.b_focus;
    out3[2] = cfg.b_cohesion;
  });
}

// Timing sample of parallel_pairwise<float> by an explicit list of block
// pairs (xb[i], yb[i]), xb <= yb: each is the body of the driver loop of
// parallel.hpp:178-215 (pair_block_focus over the workers' z ranges, the
// rank-order sum of the partial counts, U and the reciprocals, then
// pair_block_cohesion), timed on its own into seconds[i]. The caller
// extrapolates diagonal and off-diagonal block pairs separately.
// policy / style arrive as run-time values exactly as in the real driver
// (a compile-time Strict would let the compiler specialize the block
// functions and time code the reference never runs).
int ref_parallel_pairwise_blockpairs_f32(const float* dd, uint64_t n, uint64_t b, int workers, const uint32_t* xb,
                                         const uint32_t* yb, uint64_t count, double* seconds, int policy_i,
                                         int style_i) {
  return guarded([&] {
    const pald::Policy policy = pol(policy_i);
    const pald::UpdateStyle style = style_i ? pald::UpdateStyle::Branchy : pald::UpdateStyle::Masked;
    using pald::detail::worker_range;
    const int p = workers;
    std::vector<float> c(n * n, 0.0f);
    std::vector<int32_t> u(n * n, 0);
    std::vector<std::vector<int32_t>> partial(p, std::vector<int32_t>(b * b));
    std::vector<float> recip(b * b);
    pald::ThreadPool pool(p);
    for (uint64_t i = 0; i < count; ++i) {
      const uint64_t x0 = (uint64_t)xb[i] * b, y0 = (uint64_t)yb[i] * b;
      const uint64_t x1 = std::min<uint64_t>(x0 + b, n), y1 = std::min<uint64_t>(y0 + b, n);
      const uint64_t ys = y1 - y0, cells = (x1 - x0) * ys;
      const double t0 = pald::detail::PhaseClock::now();
      pool.run([&](int w) {
        auto [z0, z1] = worker_range(n, p, w);
        std::fill(partial[w].begin(), partial[w].begin() + cells, 0);
        pald::detail::pair_block_focus(dd, n, policy, x0, x1, y0, y1, z0, z1, partial[w].data());
      });
      for (int w = 1; w < p; ++w)
        for (uint64_t k = 0; k < cells; ++k) partial[0][k] += partial[w][k];
      for (uint64_t x = x0; x < x1; ++x) {
        const uint64_t ybeg = (y0 > x + 1) ? y0 : x + 1;
        for (uint64_t y = ybeg; y < y1; ++y) {
          const int32_t cnt = partial[0][(x - x0) * ys + (y - y0)];
          u[x * n + y] = u[y * n + x] = cnt;
          recip[(x - x0) * ys + (y - y0)] = 1.0f / static_cast<float>(cnt);
        }
      }
      pool.run([&](int w) {
        auto [z0, z1] = worker_range(n, p, w);
        pald::detail::pair_block_cohesion(dd, n, policy, style, x0, x1, y0,
                                          y1, z0, z1, recip.data(), c.data());
      });
      seconds[i] = pald::detail::PhaseClock::now() - t0;
    }
  });
}

// The O(n^2) part of a parallel_pairwise<float> call (parallel.hpp:167-175,
// :216-219) on a random D of size n: to_real<float>, the zero-filled C / U
// buffers, and collect_result. *seconds = their total.
int ref_pairwise_overhead_f32(uint64_t n, uint64_t seed, double* seconds) {
  return guarded([&] {
    const auto d = pald::detail::random_distances(n, seed);
    const double t0 = pald::detail::PhaseClock::now();
    const std::vector<float> dd = pald::detail::to_real<float>(d);
    std::vector<float> c(n * n, 0.0f);
    std::vector<int32_t> u(n * n, 0);
    pald::PaldResult r = pald::detail::collect_result(n, std::move(u), c);
    *seconds = pald::detail::PhaseClock::now() - t0;
    if (r.focus.sizes.size() != n * n || dd.size() != n * n) throw std::runtime_error("size");
  });
}

// points_to_distances, ingest.hpp:303-322 (row-major n x dim doubles in,
// n x n doubles out; duplicate points -> ValidationError, status 2)
int ref_points_to_distances(const double* pts, uint64_t n, uint64_t dim, double* out) {
  return guarded([&] {
    pald::PointCloud pc;
    pc.n = n;
    pc.dim = dim;
    pc.coords.assign(pts, pts + n * dim);
    const auto d = pald::points_to_distances(pc);
    std::memcpy(out, d.values().data(), sizeof(double) * n * n);
  });
}

namespace {
pald::CohesionMatrix normalized_c(const double* c, uint64_t n) {
  pald::CohesionMatrix cm(n);
  std::memcpy(cm.values.data(), c, sizeof(double) * n * n);
  cm.normalized = true;
  return cm;
}
}  // namespace

// universal_threshold, analyze.hpp:34-40 (c: a normalized C)
int ref_universal_threshold(const double* c, uint64_t n, double* out) {
  return guarded([&] { *out = pald::universal_threshold(normalized_c(c, n)); });
}

// strong_ties, analyze.hpp:42-53. threshold_in NULL = universal threshold.
// Writes up to cap edges; *count_out = the edge count.
int ref_strong_ties(const double* c, uint64_t n, const double* threshold_in, double* threshold_out,
                    uint64_t cap, uint64_t* xs, uint64_t* ys, double* strength, uint64_t* count_out) {
  return guarded([&] {
    const auto cm = normalized_c(c, n);
    const auto g = threshold_in ? pald::strong_ties(cm, *threshold_in) : pald::strong_ties(cm);
    *threshold_out = g.threshold;
    *count_out = g.edges.size();
    for (uint64_t i = 0; i < g.edges.size() && i < cap; ++i) {
      xs[i] = g.edges[i].x;
      ys[i] = g.edges[i].y;
      strength[i] = g.edges[i].strength;
    }
  });
}

// nearest_neighbors, analyze.hpp:60-75
int ref_nearest_neighbors(const double* c, uint64_t n, uint64_t focus, uint64_t k, uint64_t* zs,
                          double* strength) {
  return guarded([&] {
    const auto nb = pald::nearest_neighbors(normalized_c(c, n), focus, k);
    for (uint64_t i = 0; i < nb.size(); ++i) {
      zs[i] = nb[i].z;
      strength[i] = nb[i].strength;
    }
  });
}

}  // extern "C"
