/*
 * pald_oracle.c -- CPU restatement of the reference PaLD algorithms.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker. The product path (paper_2307_16652_b200, the
 * C-ABI in include/pald_gpu.h) never links or calls it.
 *
 * Parity pinning: every function below is checked in tests/test_oracle.py
 * against the reference's own hand-traced fixtures (D2/D3/T3,
 * proj/tests/test_reference.cpp:12-124, acceptance.cpp:120-146) and against
 * golden vectors produced by the reference itself compiled from
 * /root/reference/proj/include (oracle/ref_bridge.cpp ->
 * oracle/_ref/libpald_ref.so; fixtures in tests/golden/, made by
 * tests/golden/make_golden.py).
 *
 * Citations are into /root/reference/proj/include/pald/.
 * Layout: row-major n x n, element (x, y) at x*n + y.
 * Policy: 0 = Strict, 1 = InclusiveSplit (types.hpp:34).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_STRICT 0
#define ORACLE_SPLIT 1

/* focus_size, reference.hpp:31-45: #{z : d_xz < d_xy or d_yz < d_xy}
 * (<= under InclusiveSplit). Evaluated on doubles. */
int pald_oracle_focus_size(const double* d, uint64_t n, uint64_t x, uint64_t y, int policy) {
  const double dxy = d[x * n + y];
  const double* rx = d + x * n;
  const double* ry = d + y * n;
  int u = 0;
  if (policy == ORACLE_STRICT) {
    for (uint64_t z = 0; z < n; ++z) u += (rx[z] < dxy) | (ry[z] < dxy);
  } else {
    for (uint64_t z = 0; z < n; ++z) u += (rx[z] <= dxy) | (ry[z] <= dxy);
  }
  return u;
}

/* pairwise_entrywise, reference.hpp:104-147. U int32 n*n (diagonal 0),
 * C double n*n unnormalized. */
void pald_oracle_pairwise_entrywise(const double* d, uint64_t n, int policy, int32_t* u_out,
                                    double* c) {
  memset(u_out, 0, sizeof(int32_t) * n * n);
  memset(c, 0, sizeof(double) * n * n);
  for (uint64_t x = 0; x < n; ++x) {
    const double* rx = d + x * n;
    for (uint64_t y = x + 1; y < n; ++y) {
      const double* ry = d + y * n;
      const double dxy = rx[y];
      const int u = pald_oracle_focus_size(d, n, x, y, policy);
      u_out[x * n + y] = u_out[y * n + x] = u;
      const double w = 1.0 / u;
      for (uint64_t z = 0; z < n; ++z) {
        if (policy == ORACLE_STRICT) {
          if (rx[z] < dxy || ry[z] < dxy) {
            if (rx[z] < ry[z]) c[x * n + z] += w;
            else c[y * n + z] += w;            /* tie goes to y (types.hpp:29-31) */
          }
        } else {
          if (rx[z] <= dxy || ry[z] <= dxy) {
            if (rx[z] < ry[z]) c[x * n + z] += w;
            else if (ry[z] < rx[z]) c[y * n + z] += w;
            else { c[x * n + z] += 0.5 * w; c[y * n + z] += 0.5 * w; }
          }
        }
      }
    }
  }
}

/* triplet_entrywise, reference.hpp:154-208 (Strict only). Returns 0, or 2
 * when validate_ties is set and an exact tie is found (the reference throws
 * ValidationError there, :167-170). C diagonal left 0. */
int pald_oracle_triplet_entrywise(const double* d, uint64_t n, int validate_ties, int32_t* u,
                                  double* c) {
  memset(u, 0, sizeof(int32_t) * n * n);
  memset(c, 0, sizeof(double) * n * n);
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) u[x * n + y] = 2;
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) {
      const double dxy = d[x * n + y];
      for (uint64_t z = y + 1; z < n; ++z) {
        const double dxz = d[x * n + z], dyz = d[y * n + z];
        if (validate_ties && (dxy == dxz || dxy == dyz || dxz == dyz)) return 2;
        if (dxy < dxz && dxy < dyz) { ++u[x * n + z]; ++u[y * n + z]; }
        else if (dxz < dyz) { ++u[x * n + y]; ++u[y * n + z]; }
        else { ++u[x * n + y]; ++u[x * n + z]; }
      }
    }
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) u[y * n + x] = u[x * n + y];
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) {
      const double dxy = d[x * n + y];
      for (uint64_t z = y + 1; z < n; ++z) {
        const double dxz = d[x * n + z], dyz = d[y * n + z];
        if (dxy < dxz && dxy < dyz) {
          c[x * n + y] += 1.0 / u[x * n + z];
          c[y * n + x] += 1.0 / u[y * n + z];
        } else if (dxz < dyz) {
          c[x * n + z] += 1.0 / u[x * n + y];
          c[z * n + x] += 1.0 / u[y * n + z];
        } else {
          c[y * n + z] += 1.0 / u[x * n + y];
          c[z * n + y] += 1.0 / u[x * n + z];
        }
      }
    }
  return 0;
}

/* fill_diagonal, reference.hpp:213-220: c_xx = sum_{y != x} 1/u_xy (double,
 * ascending y). */
void pald_oracle_fill_diagonal(const int32_t* u, uint64_t n, double* c) {
  for (uint64_t x = 0; x < n; ++x) {
    double s = 0.0;
    for (uint64_t y = 0; y < n; ++y)
      if (y != x) s += 1.0 / u[x * n + y];
    c[x * n + x] = s;
  }
}

/* normalize, reference.hpp:223-228: multiply by 1/(n-1) computed in double. */
void pald_oracle_normalize(double* c, uint64_t n) {
  const double scale = 1.0 / (double)(n - 1);
  for (uint64_t i = 0; i < n * n; ++i) c[i] *= scale;
}

/* local_depths, reference.hpp:231-241: row sums (ascending z) of a
 * normalized C. */
void pald_oracle_local_depths(const double* c, uint64_t n, double* depths) {
  for (uint64_t x = 0; x < n; ++x) {
    double s = 0.0;
    for (uint64_t z = 0; z < n; ++z) s += c[x * n + z];
    depths[x] = s;
  }
}

/* ---- fp32 reference-order restatement of blocked_pairwise<float> -------- */

/* One row x of the pairwise result in fp32, in the reference's summation
 * order. blocked_pairwise<float> (blocked.hpp:368-418) and
 * parallel_pairwise<float> (parallel.hpp:159-222) apply, to every c[x][z],
 * the masked update of pair_block_cohesion (blocked.hpp:143-149) once per
 * partner y, in ascending y, for any block size and worker count: partners
 * y < x arrive through the cy update of pair (y, x), partners y > x through
 * the cx update of pair (x, y). Each update adds 1/u as fp32 or +0.
 * u_xy is pair_block_focus (blocked.hpp:101-122) summed over all z, and
 * 1/u is Real(1)/Real(cnt) (blocked.hpp:401). */
static void pairwise_row_f32(const float* d, uint64_t n, uint64_t x, int32_t* urow, float* crow,
                             float* wrow, int policy) {
  const float* rx = d + x * n;
  for (uint64_t y = 0; y < n; ++y) {
    if (y == x) { urow[y] = 0; wrow[y] = 0.0f; continue; }
    const float* ry = d + y * n;
    const float dxy = rx[y];
    int32_t cnt = 0;
    if (policy == ORACLE_STRICT) {
      for (uint64_t z = 0; z < n; ++z) cnt += (rx[z] < dxy) | (ry[z] < dxy);
    } else {
      for (uint64_t z = 0; z < n; ++z) cnt += (rx[z] <= dxy) | (ry[z] <= dxy);
    }
    urow[y] = cnt;
    wrow[y] = 1.0f / (float)cnt;
  }
  for (uint64_t z = 0; z < n; ++z) crow[z] = 0.0f;
  for (uint64_t y = 0; y < n; ++y) {
    if (y == x) continue;
    const float* ry = d + y * n;
    const float w = wrow[y];
    if (policy == ORACLE_STRICT) {
      /* The masked arithmetic of blocked.hpp:145-148, literally: adding
       * r*s*w with r, s in {0, 1} is exact for finite w, and reproduces the
       * reference's 0*inf = NaN when a pair has u = 0 (an off-diagonal
       * distance that underflows to 0 in fp32). */
      if (y > x) {
        const float dxy = rx[y];  /* pair (x, y): cx update */
        for (uint64_t z = 0; z < n; ++z) {
          const float dxz = rx[z], dyz = ry[z];
          const float r = (dxz < dyz ? dxz : dyz) < dxy ? 1.0f : 0.0f;
          const float s = dxz < dyz ? 1.0f : 0.0f;
          crow[z] += r * s * w;
        }
      } else {
        const float dyx = ry[x];  /* pair (y, x): cy update, x is the second point */
        for (uint64_t z = 0; z < n; ++z) {
          const float dyz = ry[z], dxz = rx[z];
          const float r = (dyz < dxz ? dyz : dxz) < dyx ? 1.0f : 0.0f;
          const float s = dyz < dxz ? 1.0f : 0.0f;
          crow[z] += r * (1.0f - s) * w;
        }
      }
    } else {
      /* InclusiveSplit, masked form blocked.hpp:150-158:
       * r = min(d1z, d2z) <= d12, sx = [d1z < d2z] + 0.5 [d1z == d2z],
       * first point += r*sx*w, second point += r*(1-sx)*w (one addition). */
      const float dxy = rx[y];
      for (uint64_t z = 0; z < n; ++z) {
        const float dxz = rx[z], dyz = ry[z];
        const float r = ((dxz < dyz ? dxz : dyz) <= dxy) ? 1.0f : 0.0f;
        float share;
        if (y > x) {  /* x is the first point */
          share = (dxz < dyz ? 1.0f : 0.0f) + 0.5f * (dxz == dyz ? 1.0f : 0.0f);
        } else {      /* x is the second point of pair (y, x): 1 - s_y */
          const float sy = (dyz < dxz ? 1.0f : 0.0f) + 0.5f * (dyz == dxz ? 1.0f : 0.0f);
          share = 1.0f - sy;
        }
        crow[z] += r * share * w;
      }
    }
  }
}

/* Full pairwise fp32 result (U int32, C fp32) in reference order. O(n^3). */
void pald_oracle_pairwise_f32(const float* d, uint64_t n, int32_t* u, float* c) {
  float* w = (float*)malloc(sizeof(float) * n);
  for (uint64_t x = 0; x < n; ++x) pairwise_row_f32(d, n, x, u + x * n, c + x * n, w, ORACLE_STRICT);
  free(w);
}

/* Same, with a policy (0 Strict, 1 InclusiveSplit). */
void pald_oracle_pairwise_policy_f32(const float* d, uint64_t n, int policy, int32_t* u, float* c) {
  float* w = (float*)malloc(sizeof(float) * n);
  for (uint64_t x = 0; x < n; ++x) pairwise_row_f32(d, n, x, u + x * n, c + x * n, w, policy);
  free(w);
}

/* Selected rows of the fp32 pairwise result. O(n^2) per row: used at sizes
 * where the full oracle is too slow (the n=32768 config). */
void pald_oracle_pairwise_rows_f32(const float* d, uint64_t n, const int64_t* rows,
                                   uint64_t nrows, int32_t* u_rows, float* c_rows) {
  float* w = (float*)malloc(sizeof(float) * n);
  for (uint64_t i = 0; i < nrows; ++i)
    pairwise_row_f32(d, n, (uint64_t)rows[i], u_rows + i * n, c_rows + i * n, w, ORACLE_STRICT);
  free(w);
}

/* Sampled rows of the fp64 pairwise (Strict) oracle below: row x of C
 * (pairwise_entrywise, reference.hpp:108-145) accumulated in double, O(n^2)
 * per row; U as in the fp32 rows. For the fp32-vs-fp64 tolerance at sizes
 * where the O(n^3) oracle is out of reach. */
void pald_oracle_pairwise_rows_f64(const float* d, uint64_t n, const int64_t* rows, uint64_t nrows,
                                   int32_t* u_rows, double* c_rows) {
  double* w = (double*)malloc(sizeof(double) * n);
  for (uint64_t i = 0; i < nrows; ++i) {
    const uint64_t x = (uint64_t)rows[i];
    const float* rx = d + x * n;
    int32_t* urow = u_rows + i * n;
    double* crow = c_rows + i * n;
    for (uint64_t y = 0; y < n; ++y) {
      if (y == x) { urow[y] = 0; w[y] = 0.0; continue; }
      const float* ry = d + y * n;
      const float dxy = rx[y];
      int32_t cnt = 0;
      for (uint64_t z = 0; z < n; ++z) cnt += (rx[z] < dxy) | (ry[z] < dxy);
      urow[y] = cnt;
      w[y] = 1.0 / (double)cnt;
    }
    for (uint64_t z = 0; z < n; ++z) crow[z] = 0.0;
    for (uint64_t y = 0; y < n; ++y) {
      if (y == x) continue;
      const float* ry = d + y * n;
      const float dxy = rx[y];
      for (uint64_t z = 0; z < n; ++z) {
        const float dxz = rx[z], dyz = ry[z];
        if (!((dxz < dyz ? dxz : dyz) < dxy)) continue;
        /* support: x for the pair (x, y) iff dxz < dyz; for (y, x) iff !(dyz < dxz) */
        if (y > x ? (dxz < dyz) : !(dyz < dxz)) crow[z] += w[y];
      }
    }
  }
  free(w);
}

/* fp64 pairwise (Strict) on fp32 inputs: the fp64 oracle for tolerances.
 * Comparisons of the same fp32 values are exact in either precision, so U
 * equals the fp32 U; C is accumulated in double. O(n^3). */
void pald_oracle_pairwise_f32in_f64(const float* d, uint64_t n, int32_t* u, double* c) {
  memset(c, 0, sizeof(double) * n * n);
  for (uint64_t x = 0; x < n; ++x) {
    const float* rx = d + x * n;
    u[x * n + x] = 0;
    for (uint64_t y = x + 1; y < n; ++y) {
      const float* ry = d + y * n;
      const float dxy = rx[y];
      int32_t cnt = 0;
      for (uint64_t z = 0; z < n; ++z) cnt += (rx[z] < dxy) | (ry[z] < dxy);
      u[x * n + y] = u[y * n + x] = cnt;
      const double w = 1.0 / cnt;
      for (uint64_t z = 0; z < n; ++z) {
        if (rx[z] < dxy || ry[z] < dxy) {
          if (rx[z] < ry[z]) c[x * n + z] += w;
          else c[y * n + z] += w;
        }
      }
    }
  }
}

/* Triplet (Strict) on fp32 inputs with fp64 accumulation: the restatement of
 * triplet_entrywise (reference.hpp:154-208) used as the tolerance oracle for
 * the GPU triplet kernels. Returns U (int32) and C (double, diagonal 0). */
void pald_oracle_triplet_f32in_f64(const float* d, uint64_t n, int32_t* u, double* c) {
  memset(u, 0, sizeof(int32_t) * n * n);
  memset(c, 0, sizeof(double) * n * n);
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) u[x * n + y] = 2;
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) {
      const float dxy = d[x * n + y];
      for (uint64_t z = y + 1; z < n; ++z) {
        const float dxz = d[x * n + z], dyz = d[y * n + z];
        if (dxy < dxz && dxy < dyz) { ++u[x * n + z]; ++u[y * n + z]; }
        else if (dxz < dyz) { ++u[x * n + y]; ++u[y * n + z]; }
        else { ++u[x * n + y]; ++u[x * n + z]; }
      }
    }
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) u[y * n + x] = u[x * n + y];
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t y = x + 1; y < n; ++y) {
      const float dxy = d[x * n + y];
      for (uint64_t z = y + 1; z < n; ++z) {
        const float dxz = d[x * n + z], dyz = d[y * n + z];
        if (dxy < dxz && dxy < dyz) {
          c[x * n + y] += 1.0 / u[x * n + z];
          c[y * n + x] += 1.0 / u[y * n + z];
        } else if (dxz < dyz) {
          c[x * n + z] += 1.0 / u[x * n + y];
          c[z * n + x] += 1.0 / u[y * n + z];
        } else {
          c[y * n + z] += 1.0 / u[x * n + y];
          c[z * n + y] += 1.0 / u[x * n + z];
        }
      }
    }
}

/* Row sums of C (double) in ascending z: the row-sum invariant check. */
void pald_oracle_row_sums_f32(const float* c, uint64_t n, double* out) {
  for (uint64_t x = 0; x < n; ++x) {
    double s = 0.0;
    for (uint64_t z = 0; z < n; ++z) s += c[x * n + z];
    out[x] = s;
  }
}

/* ---- sampled-row triplet restatement ----------------------------------- */

/* 1 iff {p, q} is the pair the triplet algorithm credits for the triple
 * {p, q, o} (p, q, o distinct): sort to a < b < c and apply the branch
 * structure of triplet_entrywise, reference.hpp:171-180 / 194-203
 * (r: (a,b); else s: (a,c) if d_ac < d_bc; else t: (b,c)). */
static int triplet_closest_is(const float* d, uint64_t n, uint64_t p, uint64_t q, uint64_t o) {
  uint64_t a = p, b = q, c = o, t;
  if (a > b) { t = a; a = b; b = t; }
  if (b > c) { t = b; b = c; c = t; }
  if (a > b) { t = a; a = b; b = t; }
  const float dab = d[a * n + b], dac = d[a * n + c], dbc = d[b * n + c];
  uint64_t u, v;
  if (dab < dac && dab < dbc) { u = a; v = b; }
  else if (dac < dbc) { u = a; v = c; }
  else { u = b; v = c; }
  return (u == p && v == q) || (u == q && v == p);
}

/* Rows of the triplet result (U int32, C double before fill_diagonal),
 * O(n^2) per row: u_pq = 2 + #{o : (p,q) is incremented} = n - #{o : (p,q)
 * is the credited pair}; c_pq = sum_o 1/u_po over the o for which (p,q) is
 * credited (the two cohesion updates of each case credit the pair's
 * members with 1/u of their pairs with the third point). */
void pald_oracle_triplet_rows_f64(const float* d, uint64_t n, const int64_t* rows, uint64_t nrows,
                                  int32_t* u_rows, double* c_rows) {
  for (uint64_t i = 0; i < nrows; ++i) {
    const uint64_t p = (uint64_t)rows[i];
    int32_t* ur = u_rows + i * n;
    double* cr = c_rows + i * n;
    for (uint64_t q = 0; q < n; ++q) {
      if (q == p) { ur[q] = 0; continue; }
      int32_t cnt = 0;
      for (uint64_t o = 0; o < n; ++o)
        if (o != p && o != q) cnt += triplet_closest_is(d, n, p, q, o);
      ur[q] = (int32_t)n - cnt;
    }
    for (uint64_t q = 0; q < n; ++q) {
      double s = 0.0;
      if (q != p)
        for (uint64_t o = 0; o < n; ++o)
          if (o != p && o != q && triplet_closest_is(d, n, p, q, o)) s += 1.0 / ur[o];
      cr[q] = s;
    }
  }
}

/* points_to_distances, ingest.hpp:303-322, as the reference's own build
 * computes it: -O3 -march=native contracts `sum += diff * diff` into
 * sum = fma(diff, diff, sum) (fused = 1; fused = 0 keeps the separate
 * rounding of the product). Distances in double, written as fp32
 * (to_real<float>, blocked.hpp:91-96). Returns the row-major key x * n + y
 * of the first duplicate pair (zero distance), or -1. */
long long pald_oracle_points_to_distances(const double* p, uint64_t n, uint64_t dim, int fused, float* out) {
  long long dup = -1;
  for (uint64_t x = 0; x < n; ++x) {
    out[x * n + x] = 0.0f;
    for (uint64_t y = x + 1; y < n; ++y) {
      double sum = 0.0;
      for (uint64_t k = 0; k < dim; ++k) {
        const double diff = p[x * dim + k] - p[y * dim + k];
        sum = fused ? fma(diff, diff, sum) : sum + diff * diff;
      }
      const double dist = sqrt(sum);
      if (dist == 0.0 && dup < 0) dup = (long long)(x * n + y);
      out[x * n + y] = out[y * n + x] = (float)dist;
    }
  }
  return dup;
}
