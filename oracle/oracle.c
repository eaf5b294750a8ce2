/*
 * oracle.c — CPU restatement of the reference's space-time K pair path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker; it is never
 * linked into, loaded by, or called from the product library
 * (paper_1912_04753_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load oracle/liboracle.so.
 *
 * Pinned against (tests/test_oracle_cpu.py):
 *   - the reference compiled from its own sources (oracle/_ref, oracle/Makefile),
 *   - the golden proj/data/sample_result.json (committed as tests/golden/sample_*.json),
 *   - the reference's known-answer tests (test_edge_correction.cpp, test_estimator.cpp).
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).  Build flags: -O2 -ffp-contract=off (no -march), so
 * no FMA contraction: the distance is sqrt(RN(RN(dx*dx)+RN(dy*dy))) exactly as
 * the reference Release build computes it.
 *
 * Weighted sums are accumulated EXACTLY as 128-bit fixed point with 53
 * fractional bits (every term 1/w >= 1/2 has ulp >= 2^-53; the reference's
 * omega can exceed 1 by an ulp, so terms just below 1 occur), then rounded once
 * to double.  The reference uses Kahan summation (core/include/stripley/
 * estimator.hpp:61-67), which agrees with the exact sum to ~1 ulp; both are
 * well inside the 1e-9 contract.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (C++ [rand.eng.mers], parameters of [rand.predef]) as used */
/* by rng::Engine (core/include/stripley/rng.hpp:10-40).                      */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t x[MT_N];
  int i;
} orc_mt;

void orc_mt_seed(orc_mt* s, uint64_t seed) {
  s->x[0] = seed;
  for (int k = 1; k < MT_N; ++k)
    s->x[k] = 6364136223846793005ULL * (s->x[k - 1] ^ (s->x[k - 1] >> 62)) + (uint64_t)k;
  s->i = MT_N;
}

static void mt_twist(orc_mt* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  for (int k = 0; k < MT_N; ++k) {
    const uint64_t y = (s->x[k] & UM) | (s->x[(k + 1) % MT_N] & LM);
    s->x[k] = s->x[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
  }
  s->i = 0;
}

uint64_t orc_mt_next(orc_mt* s) {
  if (s->i >= MT_N) mt_twist(s);
  uint64_t z = s->x[s->i++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.hpp:17-25 */
uint64_t orc_below(orc_mt* s, uint64_t n) {
  if (n == 0) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t v;
  do {
    v = orc_mt_next(s);
  } while (v >= limit);
  return v % n;
}
/* rng.hpp:28 */
double orc_real01(orc_mt* s) { return (double)(orc_mt_next(s) >> 11) * 0x1.0p-53; }
/* rng.hpp:31 */
double orc_uniform(orc_mt* s, double lo, double hi) { return lo + (hi - lo) * orc_real01(s); }
/* rng.hpp:34-36 */
int64_t orc_uniform_int(orc_mt* s, int64_t lo, int64_t hi) {
  return lo + (int64_t)orc_below(s, (uint64_t)(hi - lo) + 1);
}

void orc_mt_outputs(uint64_t seed, uint64_t count, uint64_t* out) {
  orc_mt s;
  orc_mt_seed(&s, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = orc_mt_next(&s);
}

/* ------------------------------------------------------------------------ */
/* Geometry (core/src/geometry.cpp)                                          */
/* ring: nv open-ring vertices, interleaved x,y                              */
/* ------------------------------------------------------------------------ */
static double dmax(double a, double b) { return a > b ? a : b; }
static double dmin(double a, double b) { return a < b ? a : b; }

/* geometry.cpp:57-66 */
static int on_segment(double px, double py, double ax, double ay, double bx, double by) {
  const double cross = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
  double scale = 1.0;
  scale = dmax(scale, fabs(ax));
  scale = dmax(scale, fabs(ay));
  scale = dmax(scale, fabs(bx));
  scale = dmax(scale, fabs(by));
  scale = dmax(scale, fabs(px));
  scale = dmax(scale, fabs(py));
  if (fabs(cross) > 1e-12 * scale * scale) return 0;
  return px >= dmin(ax, bx) - 1e-12 * scale && px <= dmax(ax, bx) + 1e-12 * scale &&
         py >= dmin(ay, by) - 1e-12 * scale && py <= dmax(ay, by) + 1e-12 * scale;
}

/* geometry.cpp:81-97: boundary-inclusive even-odd ray cast */
int orc_point_in_polygon(double px, double py, const double* ring, uint32_t nv) {
  if (nv < 3) return 0;
  for (uint32_t i = 0; i < nv; ++i) {
    const uint32_t j = (i + 1) % nv;
    if (on_segment(px, py, ring[2 * i], ring[2 * i + 1], ring[2 * j], ring[2 * j + 1])) return 1;
  }
  int inside = 0;
  for (uint32_t i = 0, j = nv - 1; i < nv; j = i++) {
    const double ax = ring[2 * i], ay = ring[2 * i + 1];
    const double bx = ring[2 * j], by = ring[2 * j + 1];
    if ((ay > py) != (by > py)) {
      const double x_cross = ax + (py - ay) / (by - ay) * (bx - ax);
      if (px < x_cross) inside = !inside;
    }
  }
  return inside;
}

/* geometry.cpp:99-108 */
double orc_polygon_area(const double* ring, uint32_t nv) {
  double acc = 0.0;
  for (uint32_t i = 0, j = nv - 1; i < nv; j = i++)
    acc += ring[2 * j] * ring[2 * i + 1] - ring[2 * i] * ring[2 * j + 1];
  return fabs(acc) / 2.0;
}

/* geometry.cpp:27-34 */
double orc_spatial_distance(double px, double py, double qx, double qy) {
  const double dx = px - qx, dy = py - qy;
  return sqrt(dx * dx + dy * dy);
}

/* ------------------------------------------------------------------------ */
/* Edge correction (core/src/edge_correction.cpp)                            */
/* ------------------------------------------------------------------------ */
static const double kTwoPi = 2.0 * 3.14159265358979323846;
static const double kAngleEps = 1e-9;

/* edge_correction.cpp:18-38 */
static int segment_circle_angles(double ax, double ay, double bx, double by, double cx,
                                 double cy, double r, double* out, int n) {
  const double dx = bx - ax, dy = by - ay;
  const double fx = ax - cx, fy = ay - cy;
  const double qa = dx * dx + dy * dy;
  if (qa == 0.0) return n;
  const double qb = 2.0 * (fx * dx + fy * dy);
  const double qc = fx * fx + fy * fy - r * r;
  const double disc = qb * qb - 4.0 * qa * qc;
  const double scale = qb * qb + fabs(4.0 * qa * qc);
  if (disc <= 1e-9 * scale) return n;
  const double sq = sqrt(disc);
  const double roots[2] = {(-qb - sq) / (2.0 * qa), (-qb + sq) / (2.0 * qa)};
  for (int k = 0; k < 2; ++k) {
    const double t = roots[k];
    if (t < 0.0 || t > 1.0) continue;
    const double px = ax + t * dx, py = ay + t * dy;
    double ang = atan2(py - cy, px - cx);
    if (ang < 0.0) ang += kTwoPi;
    out[n++] = ang;
  }
  return n;
}

/* edge_correction.cpp:42-79.  Returns NaN when the center is outside (the
 * reference throws std::invalid_argument). */
double orc_spatial_weight(double cx, double cy, double d, const double* ring, uint32_t nv) {
  if (d <= 0.0) return 1.0;
  if (!orc_point_in_polygon(cx, cy, ring, nv)) return NAN;
  double stack_buf[64];
  double* angles = nv <= 32 ? stack_buf : (double*)malloc(sizeof(double) * 2 * nv);
  int n = 0;
  for (uint32_t i = 0, j = nv - 1; i < nv; j = i++)
    n = segment_circle_angles(ring[2 * j], ring[2 * j + 1], ring[2 * i], ring[2 * i + 1], cx,
                              cy, d, angles, n);
  double w = 1.0;
  if (n > 0) {
    /* std::sort — insertion sort yields the same ascending sequence */
    for (int a = 1; a < n; ++a) {
      const double v = angles[a];
      int b = a - 1;
      while (b >= 0 && angles[b] > v) {
        angles[b + 1] = angles[b];
        --b;
      }
      angles[b + 1] = v;
    }
    int u = 0; /* dedupe in place */
    for (int a = 0; a < n; ++a)
      if (u == 0 || angles[a] - angles[u - 1] > kAngleEps) angles[u++] = angles[a];
    if (u > 1 && (angles[0] + kTwoPi) - angles[u - 1] <= kAngleEps) --u;
    if (u >= 2) {
      double inside_span = 0.0;
      for (int a = 0; a < u; ++a) {
        const double a0 = angles[a];
        const double a1 = (a + 1 < u) ? angles[a + 1] : angles[0] + kTwoPi;
        const double mid = 0.5 * (a0 + a1);
        const double px = cx + d * cos(mid), py = cy + d * sin(mid);
        if (orc_point_in_polygon(px, py, ring, nv)) inside_span += a1 - a0;
      }
      w = inside_span / kTwoPi;
    }
  }
  if (angles != stack_buf) free(angles);
  return w;
}

/* edge_correction.cpp:81-86 */
double orc_temporal_weight(int64_t center_t, int64_t u, int64_t p0, int64_t p1) {
  return (center_t - u >= p0 && center_t + u <= p1) ? 1.0 : 0.5;
}

/* ------------------------------------------------------------------------ */
/* Estimator (core/src/estimator.cpp)                                        */
/* ------------------------------------------------------------------------ */
/* estimator.cpp:84-92: lower_bound on both axes; 0 = outside the grid */
int orc_bin_pair(const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct,
                 double d, int64_t u, uint32_t* si, uint32_t* ti) {
  uint32_t lo = 0, hi = cs;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    if (s_values[mid] < d) lo = mid + 1; else hi = mid;
  }
  if (lo == cs) return 0;
  *si = lo;
  lo = 0, hi = ct;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    if (t_values[mid] < u) lo = mid + 1; else hi = mid;
  }
  if (lo == ct) return 0;
  *ti = lo;
  return 1;
}

/* 1/w as exact 128-bit fixed point with 53 fractional bits (w = omega*v with
 * omega <= 1 + ulps, v >= 1/2, so 1/w >= 1/2 and its ulp is >= 2^-53). */
static u128 fixed53(double term) {
  int e;
  const double m = frexp(term, &e); /* term = m * 2^e, m in [0.5,1) */
  const uint64_t mant = (uint64_t)ldexp(m, 53); /* exact 53-bit integer */
  const int sh = e;                             /* term * 2^53 = mant * 2^e */
  if (sh >= 0) return (sh >= 128) ? ~(u128)0 : ((u128)mant << sh);
  return (u128)(mant >> (-sh)); /* never taken for term >= 1/2 */
}

/* Correctly rounded double of a 128-bit fixed-point value (53 frac bits). */
double orc_fixed_to_double(uint64_t hi, uint64_t lo) {
  const u128 v = ((u128)hi << 64) | lo;
  return ldexp((double)v, -53); /* gcc's u128 -> double conversion is correctly rounded */
}

typedef struct {
  const double *x, *y;
  const int64_t* t;
  const uint32_t* order; /* indices sorted by x */
  const double* xs;      /* x in sorted order */
  uint64_t n;
  const double* ring;
  uint32_t nv;
  int64_t p0, p1;
  const double* s_values;
  uint32_t cs;
  const int64_t* t_values;
  uint32_t ct;
  uint64_t c0, c1; /* center range (input order) */
  int nthreads, tid;
  /* outputs (private) */
  uint64_t* counts;
  u128* fixed;
  unsigned char* inf; /* bin received 1/0 (omega == 0) */
  uint64_t in_threshold, arc_pairs, half_pairs, bad_center;
} orc_job;

static void pair_worker_center(orc_job* J, uint64_t pos) {
  const uint32_t i = J->order[pos];
  if (i < J->c0 || i >= J->c1) return;
  const double cx = J->x[i], cy = J->y[i];
  const int64_t ctm = J->t[i];
  const double smax = J->s_values[J->cs - 1];
  const int64_t tmax = J->t_values[J->ct - 1];
  const double lim = smax * (1.0 + 0x1p-40);
  for (int dir = -1; dir <= 1; dir += 2) {
    for (int64_t k = (int64_t)pos + dir; k >= 0 && k < (int64_t)J->n; k += dir) {
      const double dxs = cx - J->xs[k];
      if (fabs(dxs) > lim) break; /* d >= |dx| exactly, see header */
      const uint32_t j = J->order[k];
      const double d = orc_spatial_distance(cx, cy, J->x[j], J->y[j]);
      const int64_t u = ctm >= J->t[j] ? ctm - J->t[j] : J->t[j] - ctm;
      if (d > smax || u > tmax) continue;
      uint32_t si, ti;
      if (!orc_bin_pair(J->s_values, J->cs, J->t_values, J->ct, d, u, &si, &ti)) continue;
      const double ws = orc_spatial_weight(cx, cy, d, J->ring, J->nv);
      if (ws != ws) {
        J->bad_center++;
        continue;
      }
      const double wt = orc_temporal_weight(ctm, u, J->p0, J->p1);
      const double w = ws * wt;
      const uint32_t b = si * J->ct + ti;
      J->counts[b]++;
      if (w == 0.0)
        J->inf[b] = 1; /* the reference adds 1/0 = inf; its Kahan sum ends NaN */
      else
        J->fixed[b] += fixed53(1.0 / w);
      J->in_threshold++;
      if (ws != 1.0) J->arc_pairs++;
      if (wt != 1.0) J->half_pairs++;
    }
  }
}

static void* pair_worker(void* arg) {
  orc_job* J = (orc_job*)arg;
  for (uint64_t pos = (uint64_t)J->tid; pos < J->n; pos += (uint64_t)J->nthreads)
    pair_worker_center(J, pos);
  return NULL;
}

static const double* g_sort_x;
static int cmp_by_x(const void* a, const void* b) {
  const uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
  if (g_sort_x[i] < g_sort_x[j]) return -1;
  if (g_sort_x[i] > g_sort_x[j]) return 1;
  return (i > j) - (i < j);
}

/*
 * Per-bin (non-cumulative) in-threshold ordered-pair counts and exact
 * weighted sums over centers with input index in [c0, c1) (pass 0, n for all).
 * Output: counts[cs*ct], sum_hi/sum_lo[cs*ct] (128-bit fixed, 53 frac bits),
 * hist[cs*ct] = correctly rounded double of the exact sum.
 * stats[0..3] = in_threshold, arc (omega != 1), half (v = 1/2), bad centers.
 * Restates estimate_surface's add_pair loop (estimator.cpp:136-144,170-177).
 */
int orc_pair_histogram(const double* x, const double* y, const int64_t* t, uint64_t n,
                       const double* ring, uint32_t nv, int64_t p0, int64_t p1,
                       const double* s_values, uint32_t cs, const int64_t* t_values,
                       uint32_t ct, uint64_t c0, uint64_t c1, int nthreads,
                       uint64_t* counts, uint64_t* sum_hi, uint64_t* sum_lo, double* hist,
                       uint64_t* stats) {
  if (nthreads < 1) nthreads = 1;
  const uint32_t bins = cs * ct;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  double* xs = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  g_sort_x = x;
  qsort(order, n, sizeof(uint32_t), cmp_by_x);
  for (uint64_t k = 0; k < n; ++k) xs[k] = x[order[k]];

  orc_job* jobs = (orc_job*)calloc((size_t)nthreads, sizeof(orc_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int w = 0; w < nthreads; ++w) {
    orc_job* J = &jobs[w];
    J->x = x; J->y = y; J->t = t; J->order = order; J->xs = xs; J->n = n;
    J->ring = ring; J->nv = nv; J->p0 = p0; J->p1 = p1;
    J->s_values = s_values; J->cs = cs; J->t_values = t_values; J->ct = ct;
    J->c0 = c0; J->c1 = c1; J->nthreads = nthreads; J->tid = w;
    J->counts = (uint64_t*)calloc(bins, sizeof(uint64_t));
    J->fixed = (u128*)calloc(bins, sizeof(u128));
    J->inf = (unsigned char*)calloc(bins, 1);
    if (nthreads > 1) pthread_create(&th[w], NULL, pair_worker, J);
  }
  if (nthreads == 1) pair_worker(&jobs[0]);
  for (int w = 0; w < nthreads; ++w)
    if (nthreads > 1) pthread_join(th[w], NULL);

  memset(stats, 0, sizeof(uint64_t) * 4);
  for (uint32_t b = 0; b < bins; ++b) {
    uint64_t c = 0;
    u128 s = 0;
    int inf = 0;
    for (int w = 0; w < nthreads; ++w) {
      c += jobs[w].counts[b];
      s += jobs[w].fixed[b];
      inf |= jobs[w].inf[b];
    }
    if (inf) s += (u128)1 << 120; /* the device library's exported mark (stk.h) */
    counts[b] = c;
    sum_hi[b] = (uint64_t)(s >> 64);
    sum_lo[b] = (uint64_t)s;
    hist[b] = inf ? NAN : orc_fixed_to_double(sum_hi[b], sum_lo[b]);
  }
  for (int w = 0; w < nthreads; ++w) {
    stats[0] += jobs[w].in_threshold;
    stats[1] += jobs[w].arc_pairs;
    stats[2] += jobs[w].half_pairs;
    stats[3] += jobs[w].bad_center;
    free(jobs[w].counts);
    free(jobs[w].fixed);
    free(jobs[w].inf);
  }
  free(jobs); free(th); free(order); free(xs);
  return stats[3] ? 1 : 0;
}

/* estimator.cpp:94-114: 2-D inclusion-exclusion prefix (si outer, ti inner),
 * then x A*D/(n*n). */
void orc_finalize(const double* hist, uint64_t n, double area, int64_t duration, uint32_t cs,
                  uint32_t ct, double* k) {
  const double scale = area * (double)duration / ((double)n * (double)n);
  for (uint32_t si = 0; si < cs; ++si)
    for (uint32_t ti = 0; ti < ct; ++ti) {
      double acc = hist[si * ct + ti];
      if (si > 0) acc += k[(si - 1) * ct + ti];
      if (ti > 0) acc += k[si * ct + ti - 1];
      if (si > 0 && ti > 0) acc -= k[(si - 1) * ct + ti - 1];
      k[si * ct + ti] = acc;
    }
  for (uint32_t b = 0; b < cs * ct; ++b) k[b] *= scale;
}

/* estimator.cpp:51-57,71-82: L = sqrt(K/(2*pi*t)) - s */
void orc_to_l(const double* k, const double* s_values, uint32_t cs, const int64_t* t_values,
              uint32_t ct, double* l) {
  const double pi = 3.14159265358979323846;
  for (uint32_t si = 0; si < cs; ++si)
    for (uint32_t ti = 0; ti < ct; ++ti)
      l[si * ct + ti] = sqrt(k[si * ct + ti] / (2.0 * pi * (double)t_values[ti])) - s_values[si];
}

/* simulation.cpp:86-102 (max/min fold starting at sims[0]) and
 * estimator.cpp:188-202 (diff). */
void orc_envelopes(const double* l_all, uint32_t m, uint32_t bins, double* upper, double* lower) {
  memcpy(upper, l_all, sizeof(double) * bins);
  memcpy(lower, l_all, sizeof(double) * bins);
  for (uint32_t r = 1; r < m; ++r)
    for (uint32_t b = 0; b < bins; ++b) {
      const double v = l_all[(size_t)r * bins + b];
      upper[b] = (upper[b] < v) ? v : upper[b];
      lower[b] = (v < lower[b]) ? v : lower[b];
    }
}

void orc_diff(const double* est, const double* upper, uint32_t bins, double* diff) {
  for (uint32_t b = 0; b < bins; ++b) diff[b] = est[b] > upper[b] ? est[b] - upper[b] : 0.0;
}

/* ------------------------------------------------------------------------ */
/* Simulation (core/src/simulation.cpp)                                      */
/* ------------------------------------------------------------------------ */
/* simulation.cpp:10-24: bbox rejection with PIP, then integer time */
void orc_generate_cstr(uint64_t n, const double* ring, uint32_t nv, int64_t p0, int64_t p1,
                       uint64_t seed, double* x, double* y, int64_t* t) {
  double xmin = ring[0], xmax = ring[0], ymin = ring[1], ymax = ring[1];
  for (uint32_t i = 0; i < nv; ++i) {
    xmin = dmin(xmin, ring[2 * i]);
    xmax = dmax(xmax, ring[2 * i]);
    ymin = dmin(ymin, ring[2 * i + 1]);
    ymax = dmax(ymax, ring[2 * i + 1]);
  }
  orc_mt s;
  orc_mt_seed(&s, seed);
  uint64_t k = 0;
  while (k < n) {
    const double cx = orc_uniform(&s, xmin, xmax);
    const double cy = orc_uniform(&s, ymin, ymax);
    if (!orc_point_in_polygon(cx, cy, ring, nv)) continue;
    x[k] = cx;
    y[k] = cy;
    t[k] = orc_uniform_int(&s, p0, p1);
    ++k;
  }
}

/* simulation.cpp:26-35 */
void orc_generate_bootstrap(const double* x, const double* y, const int64_t* t, uint64_t n,
                            uint64_t seed, double* ox, double* oy, int64_t* ot) {
  orc_mt s;
  orc_mt_seed(&s, seed);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j = orc_below(&s, n);
    ox[i] = x[j];
    oy[i] = y[j];
    ot[i] = t[j];
  }
}

/* simulation.cpp:37-53: Fisher-Yates over the time column */
void orc_generate_permutation(const double* x, const double* y, const int64_t* t, uint64_t n,
                              uint64_t seed, double* ox, double* oy, int64_t* ot) {
  orc_mt s;
  orc_mt_seed(&s, seed);
  memcpy(ox, x, sizeof(double) * n);
  memcpy(oy, y, sizeof(double) * n);
  memcpy(ot, t, sizeof(int64_t) * n);
  for (uint64_t i = n - 1; i > 0; --i) {
    const uint64_t j = orc_below(&s, i + 1);
    const int64_t tmp = ot[i];
    ot[i] = ot[j];
    ot[j] = tmp;
  }
}
