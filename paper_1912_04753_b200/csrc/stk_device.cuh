// stk_device.cuh — device-side geometry, edge weights, MT19937-64 and exact
// fixed-point helpers for the space-time K pair path (sm_100a).
//
// Every FP64 expression here is compiled with -fmad=false, so no mul+add is
// contracted into an FMA: results follow the reference's Release build
// (no -march, no FMA) operation by operation.
#pragma once
#include <cstdint>

#include "stk_types.h"

namespace stk {

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;  // == 2.0 * std::numbers::pi
constexpr double kAngleEps = 1e-9;
constexpr int kMaxAngles = 64;  // circle/boundary crossings handled per weight

// --------------------------------------------------------------- geometry
// Restates geom::on_segment (proj/core/src/geometry.cpp:57-66).
__device__ __forceinline__ bool on_segment(double px, double py, double ax, double ay,
                                           double bx, double by) {
  const double cross = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
  double scale = fmax(fabs(ax), fabs(ay));
  scale = fmax(scale, fmax(fabs(bx), fabs(by)));
  scale = fmax(scale, fmax(fabs(px), fabs(py)));
  scale = fmax(scale, 1.0);
  if (fabs(cross) > 1e-12 * scale * scale) return false;
  return px >= fmin(ax, bx) - 1e-12 * scale && px <= fmax(ax, bx) + 1e-12 * scale &&
         py >= fmin(ay, by) - 1e-12 * scale && py <= fmax(ay, by) + 1e-12 * scale;
}

// Restates geom::point_in_polygon (geometry.cpp:81-97): boundary-inclusive
// even-odd ray cast over the open ring.  on_segment is entered only when the
// cross product passes the bound with the largest possible scale
// (smax = max(1, |ring|, |p|) >= scale): |cross| > 1e-12*smax*smax implies
// |cross| > 1e-12*scale*scale (RN is monotone), i.e. on_segment == false, so
// the skipped calls are exactly the ones that return false.
__device__ __forceinline__ bool point_in_polygon(double px, double py, const double2* ring,
                                                 uint32_t nv, double ring_maxabs = -1.0) {
  if (nv < 3) return false;
  const double smax =
      ring_maxabs < 0.0 ? -1.0 : fmax(fmax(ring_maxabs, 1.0), fmax(fabs(px), fabs(py)));
  const double bound = 1e-12 * smax * smax;
  for (uint32_t i = 0; i < nv; ++i) {
    const double2 a = ring[i];
    const double2 b = ring[(i + 1 == nv) ? 0 : i + 1];
    if (smax > 0.0) {
      const double cross = (b.x - a.x) * (py - a.y) - (b.y - a.y) * (px - a.x);
      if (fabs(cross) > bound) continue;
    }
    if (on_segment(px, py, a.x, a.y, b.x, b.y)) return true;
  }
  bool inside = false;
  for (uint32_t i = 0, j = nv - 1; i < nv; j = i++) {
    const double2 a = ring[i];
    const double2 b = ring[j];
    if ((a.y > py) != (b.y > py)) {
      const double x_cross = a.x + (py - a.y) / (b.y - a.y) * (b.x - a.x);
      if (px < x_cross) inside = !inside;
    }
  }
  return inside;
}

// point_in_polygon restricted to the probe's slab (RegionView::slab_*): the
// same expressions, per edge, as the reference, over the only edges that can
// change its answer.  An edge can pass on_segment only if py lies in its
// y-range widened by 1e-12*scale <= 1e-12*pip_lim, and can toggle the ray
// cast only if (a.y > py) != (b.y > py), i.e. py lies in its y-range; the host
// lists every edge whose y-range widened by 2e-12*pip_lim (plus one slab on
// each side, against rounding of the slab index) meets the slab.  Probes
// outside [pip_ylo, pip_yhi] meet no such edge: false, as the reference.
__device__ __forceinline__ bool pip_slab(double px, double py, const RegionView& R) {
  if (!(py >= R.pip_ylo && py <= R.pip_yhi)) return false;
  int s = (int)floor((py - R.slab_y0) * R.slab_inv_h);
  s = min(max(s, 0), (int)R.nslab - 1);
  const uint32_t b = R.slab_start[s], e = R.slab_start[s + 1];
  const uint32_t nv = R.nv;
  const double2* ring = R.ring;
  const double smax = fmax(fmax(R.maxabs, 1.0), fmax(fabs(px), fabs(py)));
  const double bound = 1e-12 * smax * smax;
  for (uint32_t k = b; k < e; ++k) {  // on_segment(p, ring[i], ring[i+1]) (geometry.cpp:84-86)
    const uint32_t i = R.slab_edge[k];
    const double2 a = ring[i];
    const double2 bb = ring[(i + 1 == nv) ? 0 : i + 1];
    const double cross = (bb.x - a.x) * (py - a.y) - (bb.y - a.y) * (px - a.x);
    if (fabs(cross) > bound) continue;  // see point_in_polygon
    if (on_segment(px, py, a.x, a.y, bb.x, bb.y)) return true;
  }
  bool inside = false;
  for (uint32_t k = b; k < e; ++k) {  // ray cast: the reference's (a, b) = (ring[i+1], ring[i])
    const uint32_t i = R.slab_edge[k];
    const double2 a = ring[(i + 1 == nv) ? 0 : i + 1];
    const double2 bb = ring[i];
    if ((a.y > py) != (bb.y > py)) {
      const double x_cross = a.x + (py - a.y) / (bb.y - a.y) * (bb.x - a.x);
      if (px < x_cross) inside = !inside;
    }
  }
  return inside;
}

// geom::point_in_polygon for the region: slab index when built and the probe
// is within its validity bound, else the full restatement.
__device__ __forceinline__ bool point_in_region(double px, double py, const RegionView& R) {
  if (R.slab_start != nullptr && fabs(px) <= R.pip_lim && fabs(py) <= R.pip_lim)
    return pip_slab(px, py, R);
  return point_in_polygon(px, py, R.ring, R.nv, R.maxabs);
}

// The edge-cell list of a center (RegionView::ec_*), or nullptr (all segments)
// when not built or d exceeds the radius the lists cover.
__device__ __forceinline__ const uint32_t* edge_list(double cx, double cy, double d,
                                                     const RegionView& R, uint32_t* cnt) {
  if (R.ec_start == nullptr || !(d <= R.ec_dmax)) {
    *cnt = R.nv;
    return nullptr;
  }
  int ix = (int)floor((cx - R.ec_x0) * R.ec_inv_w);
  int iy = (int)floor((cy - R.ec_y0) * R.ec_inv_w);
  ix = min(max(ix, 0), R.ec_nx - 1);
  iy = min(max(iy, 0), R.ec_ny - 1);
  const uint32_t cell = (uint32_t)iy * (uint32_t)R.ec_nx + (uint32_t)ix;
  const uint32_t b = R.ec_start[cell];
  uint32_t n = R.ec_start[cell + 1] - b;
  if (d > 0.0) {
    // entries are sorted by a lower bound of their distance to the cell: those
    // beyond d (1 + 4e-6) + 1e-9 S are rejected by the reference (the
    // edge-cell argument with d for s_max) — keep the prefix before them
    const double lim = d * (1.0 + 4e-6) + R.ec_abs;
    const float* dm = R.ec_dmin + b;
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((double)dm[mid] > lim) hi = mid; else lo = mid + 1;
    }
    n = lo;
  }
  *cnt = n;
  return R.ec_edge + b;
}

// atan2 with one division: |y|,|x| -> t in [-tan(pi/8), tan(pi/8)] via
// t = mn/mx (mn <= tan(pi/8) mx) or t = (mn - mx)/(mn + mx) (+ pi/4), then
// atan(t) = t + t*s*R(s), s = t^2, R a degree-10 fit (tools/fit_atan.py;
// approximation error 5e-18 relative), then the octant fix-ups.  About 45
// instructions against ~130 for the library's atan2, within ~2-3 ulp; zeros,
// infinities and NaN go to the library.
__device__ __forceinline__ double fast_atan2(double y, double x) {
  const double ax = fabs(x), ay = fabs(y);
  const bool steep = ay > ax;
  const double mx = steep ? ay : ax, mn = steep ? ax : ay;
  // (0, 0), infinities and NaN never reach this path (crossing vectors are
  // differences of finite points at distance d > 0); the library handles them
  if (!(mx > 0.0 && mx < 1.0e300)) return atan2(y, x);
  constexpr double kTanPi8 = 0.41421356237309504880;
  constexpr double kPi4 = 0.78539816339744830962;
  constexpr double kPi2 = 1.57079632679489661923;
  constexpr double kPi = 3.14159265358979323846;
  const bool small = mn <= kTanPi8 * mx;  // select, then one division for every lane
  const double t = (small ? mn : mn - mx) / (small ? mx : mn + mx);
  const double base = small ? 0.0 : kPi4;
  const double s = t * t;
  double r = -0.0192025292684122813793;
  r = fma(r, s, 0.0392536963206185629612);
  r = fma(r, s, -0.0508625488582314312944);
  r = fma(r, s, 0.0585831181050115303872);
  r = fma(r, s, -0.0666453136980500884962);
  r = fma(r, s, 0.0769218469937177728423);
  r = fma(r, s, -0.090909046476956795219);
  r = fma(r, s, 0.111111110171003266375);
  r = fma(r, s, -0.142857142846913806166);
  r = fma(r, s, 0.199999999999956505772);
  r = fma(r, s, -0.333333333333333302719);
  double a = base + fma(t * s, r, t);  // atan(mn / mx) in [0, pi/4]
  if (steep) a = kPi2 - a;
  if (x < 0.0) a = kPi - a;
  return copysign(a, y);
}

// --------------------------------------------------------- edge weights
// Restates edge::segment_circle_angles (proj/core/src/edge_correction.cpp:18-38).
__device__ __forceinline__ int segment_circle_angles(double2 a, double2 b, double cx,
                                                     double cy, double r, double* out,
                                                     int n) {
  const double dx = b.x - a.x, dy = b.y - a.y;
  const double fx = a.x - cx, fy = a.y - cy;
  const double qa = dx * dx + dy * dy;
  if (qa == 0.0) return n;
  const double qb = 2.0 * (fx * dx + fy * dy);
  const double qc = fx * fx + fy * fy - r * r;
  const double disc = qb * qb - 4.0 * qa * qc;
  const double scale = qb * qb + fabs(4.0 * qa * qc);
  if (disc <= 1e-9 * scale) return n;
  const double sq = sqrt(disc);
  const double t0 = (-qb - sq) / (2.0 * qa);
  const double t1 = (-qb + sq) / (2.0 * qa);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double t = k == 0 ? t0 : t1;
    if (t < 0.0 || t > 1.0) continue;
    const double px = a.x + t * dx, py = a.y + t * dy;
    double ang = atan2(py - cy, px - cx);
    if (ang < 0.0) ang += kTwoPi;
    if (n < kMaxAngles) out[n] = ang;
    ++n;
  }
  return n;
}

// Restates edge::spatial_isotropic_weight (edge_correction.cpp:42-79) for a
// center already known to lie inside the region (the estimator validates
// every point up front, estimator.cpp:123-127, so the reference's throw is
// unreachable on this path), for any number of crossings in bounded storage:
// each pass re-derives every crossing angle (segment_circle_angles, same
// arithmetic) and keeps the kMaxAngles smallest above the previous pass's
// largest, so the passes visit the reference's sorted sequence in order.  The
// de-duplication (v - last kept > 1e-9), the wrap rule and the arc sums then
// run as a stream with one kept angle of delay (an arc is summed once its end
// is known not to be the last kept angle, which the wrap rule may drop), in
// the reference's summation order.  Skipping values equal to the previous
// pass's largest is exact: a duplicate of a value never survives the dedupe.
__device__ __noinline__ double spatial_weight(double cx, double cy, double d, const RegionView* Rp,
                                              int* overflow) {
  (void)overflow;
  if (d <= 0.0) return 1.0;
  const RegionView& R = *Rp;  // device memory (a kernel parameter would be copied to the stack)
  const double2* ring = R.ring;
  const uint32_t nv = R.nv;
  uint32_t cnt;
  const uint32_t* list = edge_list(cx, cy, d, R, &cnt);  // segments that can cross
  const double inner = d * (1.0 - 4e-6) - R.ec_abs;
  double buf[kMaxAngles];
  double lower = -1.0;  // angles are in [0, 2*pi)
  int u = 0;            // kept angles so far
  double first = 0.0, prev = 0.0, cur = 0.0, inside_span = 0.0;
  auto arc = [&](double a0, double a1) {
    const double mid = 0.5 * (a0 + a1);
    double sn, cs;
    sincos(mid, &sn, &cs);
    const double px = cx + d * cs, py = cy + d * sn;
    if (point_in_region(px, py, R)) inside_span += a1 - a0;
  };
  for (;;) {
    int n = 0;
    bool dropped = false;
    for (uint32_t k = 0; k < cnt; ++k) {
      if (list && (double)R.ec_far[(list - R.ec_edge) + k] < inner) continue;  // wholly inside
      const uint32_t i = list ? list[k] : k;
      double two[2];
      const int m = segment_circle_angles(ring[i == 0 ? nv - 1 : i - 1], ring[i], cx, cy, d, two, 0);
      for (int q = 0; q < m; ++q) {
        const double v = two[q];
        if (!(v > lower)) continue;
        if (n == kMaxAngles) {
          if (v >= buf[n - 1]) {
            dropped = true;
            continue;
          }
          --n;  // the largest leaves; it is re-found by a later pass
          dropped = true;
        }
        int b = n - 1;  // insertion (ascending)
        while (b >= 0 && buf[b] > v) {
          buf[b + 1] = buf[b];
          --b;
        }
        buf[b + 1] = v;
        ++n;
      }
    }
    for (int a = 0; a < n; ++a) {
      const double v = buf[a];
      if (u == 0) {
        first = cur = v;
        u = 1;
      } else if (v - cur > kAngleEps) {
        if (u >= 2) arc(prev, cur);  // cur is not the last kept angle
        prev = cur;
        cur = v;
        ++u;
      }
    }
    if (!dropped || n == 0) break;
    lower = buf[n - 1];
  }
  if (u > 1 && (first + kTwoPi) - cur <= kAngleEps) {  // the wrap rule drops the last kept
    --u;
    if (u < 2) return 1.0;
    arc(prev, first + kTwoPi);
    return inside_span / kTwoPi;
  }
  if (u < 2) return 1.0;
  arc(prev, cur);
  arc(cur, first + kTwoPi);
  return inside_span / kTwoPi;
}

__device__ __noinline__ double spatial_weight_ring(double cx, double cy, double d, const double2* ring,
                                              uint32_t nv, double ring_maxabs, int* overflow) {
  if (d <= 0.0) return 1.0;
  double ang[kMaxAngles];
  int n = 0;
  for (uint32_t i = 0, j = nv - 1; i < nv; j = i++)
    n = segment_circle_angles(ring[j], ring[i], cx, cy, d, ang, n);
  if (n > kMaxAngles) {
    *overflow = 1;
    n = kMaxAngles;
  }
  if (n == 0) return 1.0;
  for (int a = 1; a < n; ++a) {  // std::sort (ascending; same sequence)
    const double v = ang[a];
    int b = a - 1;
    while (b >= 0 && ang[b] > v) {
      ang[b + 1] = ang[b];
      --b;
    }
    ang[b + 1] = v;
  }
  int u = 0;
  for (int a = 0; a < n; ++a)
    if (u == 0 || ang[a] - ang[u - 1] > kAngleEps) ang[u++] = ang[a];
  if (u > 1 && (ang[0] + kTwoPi) - ang[u - 1] <= kAngleEps) --u;
  if (u < 2) return 1.0;
  double inside_span = 0.0;
  for (int a = 0; a < u; ++a) {
    const double a0 = ang[a];
    const double a1 = (a + 1 < u) ? ang[a + 1] : ang[0] + kTwoPi;
    const double mid = 0.5 * (a0 + a1);
    double sn, cs;
    sincos(mid, &sn, &cs);
    const double px = cx + d * cs, py = cy + d * sn;
    if (point_in_polygon(px, py, ring, nv, ring_maxabs)) inside_span += a1 - a0;
  }
  return inside_span / kTwoPi;
}

// spatial_isotropic_weight for rings of at most 32 vertices, organised for
// SIMT: (1) a uniform pass over the segments marks those whose quadratic has
// an accepted discriminant; (2) each lane walks only its accepted segments
// (recomputing the same quadratic) and records the crossing vectors; (3) one
// loop of atan2 over the crossings; then sort / de-duplicate / arc midpoints
// exactly as spatial_weight().  Lanes crossing different edges no longer
// serialise their atan2 and divisions.  Crossing data live in a caller
// scratch (shared memory, element k at buf[k * stride], 2*cap elements).
// Same arithmetic and order as the reference; returns -1 when more than `cap`
// crossings occur (caller falls back to spatial_weight()).
// point_in_polygon for an axis-aligned rectangle ring [x0,x1] x [y0,y1]
// (RegionView::rect), exactly equal to the general routine on that ring:
// * ray cast: horizontal edges never satisfy (a.y > py) != (b.y > py); a
//   vertical edge at X gives x_cross = X + q*(b.x-a.x) = X + q*0 = X exactly
//   and toggles iff y0 <= py < y1; two toggles cancel, so the parity is
//   (y0 <= py < y1) && (x0 <= px < x1);
// * boundary: on_segment is evaluated (exactly as the reference) only for the
//   edges whose cross product passes the tolerance with the largest scale;
//   all other edges return false there (see point_in_polygon).
__device__ __forceinline__ bool point_in_rect(double px, double py, const RegionView& R) {
  if (py >= R.ymin && py < R.ymax && px >= R.xmin && px < R.xmax) {
    // strictly-inside parity is true; on_segment could only add true
    return true;
  }
  // outside the box expanded by box_m no edge's on_segment can hold: its
  // cross product exceeds 1e-12*scale^2 or the point leaves the segment's
  // bounding box by more than 1e-12*scale (box_m bounds both, host-side)
  if (px < R.xmin - R.box_m || px > R.xmax + R.box_m || py < R.ymin - R.box_m ||
      py > R.ymax + R.box_m)
    return false;
  const double smax = fmax(fmax(R.maxabs, 1.0), fmax(fabs(px), fabs(py)));
  const double bound = 1e-12 * smax * smax;
  for (uint32_t i = 0; i < 4; ++i) {
    const double2 a = R.ring[i];
    const double2 b = R.ring[(i + 1) & 3];
    const double cross = (b.x - a.x) * (py - a.y) - (b.y - a.y) * (px - a.x);
    if (fabs(cross) > bound) continue;
    if (on_segment(px, py, a.x, a.y, b.x, b.y)) return true;
  }
  return false;
}

// Certified point_in_rect of the probe c + d*(cos mid, sin mid) from an FP32
// approximation: |__sincosf error| <= 2^-21.4 on [-pi, pi] plus the float
// rounding of the reduced angle (<= 2^-24 * pi) bounds the approximate probe's
// distance to the exact one by d * 2e-6 (+ rounding).  When the approximate
// probe is farther than that from the decision boundaries (strict interior,
// expanded exterior) the exact probe is on the same side; otherwise return -1
// and the caller evaluates the exact probe.
__device__ __forceinline__ int rect_probe_certified(double cx, double cy, double d, double mid,
                                                    const RegionView& R) {
  double m = mid;
  if (m > 3.14159265358979323846) m -= kTwoPi;
  if (m > 3.14159265358979323846) m -= kTwoPi;
  float sf, cf;
  __sincosf((float)m, &sf, &cf);
  const double px = cx + d * (double)cf, py = cy + d * (double)sf;
  const double e = d * 2e-6 + 1e-12 * (R.maxabs + d + 1.0);
  if (px >= R.xmin + e && px < R.xmax - e && py >= R.ymin + e && py < R.ymax - e) return 1;
  const double o = e + R.box_m;
  if (px < R.xmin - o || px > R.xmax + o || py < R.ymin - o || py > R.ymax + o) return 0;
  return -1;
}

// spatial_isotropic_weight for rings of at most 32 vertices, organised for
// SIMT: (1) a uniform pass over the segments marks those whose quadratic has
// an accepted discriminant; (2) each lane walks only its accepted segments
// (recomputing the same quadratic) and records the crossing vectors; (3) one
// loop of atan2 over the crossings; then sort / de-duplicate / arc midpoints
// exactly as spatial_weight().  Lanes crossing different edges no longer
// serialise their atan2 and divisions.  Crossing data live in a caller
// scratch (shared memory, element k at buf[k * stride], 2*cap elements).
// For rectangles, pass (1) skips edges whose line lies farther than
// r*(1 + 1e-6) from the center: their true discriminant is negative by a
// margin far above the rounding error (<~1e-15 * scale), so the reference
// rejects them too; and PIP uses point_in_rect.
// Same arithmetic and order as the reference; returns -1 when more than `cap`
// crossings occur (caller falls back to spatial_weight()).
// Rings of at most 32 segments visited in full (the rectangle kernel's
// deferred drain).  Kept with runtime R.rect tests: specialising them away
// changes the pair kernel's register allocation for the worse (the hot loop
// then reloads its neighbour from local memory).
__device__ __noinline__ double spatial_weight_buf_rect(double cx, double cy, double d,
                                                       const RegionView& R, double* buf,
                                                       int stride, int cap) {
  if (d <= 0.0) return 1.0;
  const uint32_t nv = R.nv;
  const double2* ring = R.ring;
  const double r2 = d * d;
  const double reach = d * (1.0 + 1e-6);
  uint32_t acc = 0;
  for (uint32_t i = 0; i < nv; ++i) {  // segment (ring[i-1], ring[i])
    const double2 A = ring[i == 0 ? nv - 1 : i - 1], Bv = ring[i];
    if (R.rect) {
      const double h = A.x == Bv.x ? fabs(A.x - cx) : fabs(A.y - cy);
      if (h > reach) continue;
    }
    const double dx = Bv.x - A.x, dy = Bv.y - A.y;
    const double fx = A.x - cx, fy = A.y - cy;
    const double qa = dx * dx + dy * dy;
    const double qb = 2.0 * (fx * dx + fy * dy);
    const double qc = fx * fx + fy * fy - r2;
    const double disc = qb * qb - 4.0 * qa * qc;
    const double scale = qb * qb + fabs(4.0 * qa * qc);
    if (qa != 0.0 && disc > 1e-9 * scale) acc |= 1u << i;
  }
  if (acc == 0) return 1.0;
  int n = 0;
  while (acc) {
    const uint32_t i = __ffs(acc) - 1;
    acc &= acc - 1;
    const double2 A = ring[i == 0 ? nv - 1 : i - 1], Bv = ring[i];
    const double dx = Bv.x - A.x, dy = Bv.y - A.y;
    const double fx = A.x - cx, fy = A.y - cy;
    const double qa = dx * dx + dy * dy;
    const double qb = 2.0 * (fx * dx + fy * dy);
    const double qc = fx * fx + fy * fy - r2;
    const double disc = qb * qb - 4.0 * qa * qc;
    const double sq = sqrt(disc);
    const double t0 = (-qb - sq) / (2.0 * qa);
    const double t1 = (-qb + sq) / (2.0 * qa);
    if (t0 >= 0.0 && t0 <= 1.0) {
      if (n >= cap) return -1.0;
      buf[(2 * n) * stride] = (A.y + t0 * dy) - cy;
      buf[(2 * n + 1) * stride] = (A.x + t0 * dx) - cx;
      ++n;
    }
    if (t1 >= 0.0 && t1 <= 1.0) {
      if (n >= cap) return -1.0;
      buf[(2 * n) * stride] = (A.y + t1 * dy) - cy;
      buf[(2 * n + 1) * stride] = (A.x + t1 * dx) - cx;
      ++n;
    }
  }
  if (n == 0) return 1.0;
  for (int k = 0; k < n; ++k) {  // angle k overwrites slot k (vector k sits at 2k, 2k+1)
    double ang = fast_atan2(buf[(2 * k) * stride], buf[(2 * k + 1) * stride]);
    if (ang < 0.0) ang += kTwoPi;
    buf[k * stride] = ang;
  }
  for (int a = 1; a < n; ++a) {  // std::sort (ascending; same sequence)
    const double v = buf[a * stride];
    int b = a - 1;
    while (b >= 0 && buf[b * stride] > v) {
      buf[(b + 1) * stride] = buf[b * stride];
      --b;
    }
    buf[(b + 1) * stride] = v;
  }
  int u = 0;
  for (int a = 0; a < n; ++a) {
    const double v = buf[a * stride];
    if (u == 0 || v - buf[(u - 1) * stride] > kAngleEps) buf[(u++) * stride] = v;
  }
  const double first = buf[0];
  if (u > 1 && (first + kTwoPi) - buf[(u - 1) * stride] <= kAngleEps) --u;
  if (u < 2) return 1.0;
  double inside_span = 0.0;
  for (int a = 0; a < u; ++a) {
    const double a0 = buf[a * stride];
    const double a1 = (a + 1 < u) ? buf[(a + 1) * stride] : first + kTwoPi;
    const double mid = 0.5 * (a0 + a1);
    int dec = R.rect ? rect_probe_certified(cx, cy, d, mid, R) : -1;
    if (dec < 0) {
      double sn, cs;
      sincos(mid, &sn, &cs);
      const double px = cx + d * cs, py = cy + d * sn;
      dec = (R.rect ? point_in_rect(px, py, R) : point_in_polygon(px, py, ring, nv, R.maxabs)) ? 1 : 0;
    }
    if (dec) inside_span += a1 - a0;
  }
  return inside_span / kTwoPi;
}

// RECT: the region is RegionView::rect (4 segments, rectangle PIP); else a
// general ring through the edge cells and the slab PIP.
template <bool RECT>
__device__ __forceinline__ double spatial_weight_buf(double cx, double cy, double d,
                                                       const RegionView& R, double* buf,
                                                       int stride, int cap) {
  if (d <= 0.0) return 1.0;
  const uint32_t nv = R.nv;
  const double2* ring = R.ring;
  const double r2 = d * d;
  const double reach = d * (1.0 + 1e-6);
  uint32_t cnt = 4;
  const uint32_t* list = RECT ? nullptr : edge_list(cx, cy, d, R, &cnt);
  const double inner = d * (1.0 - 4e-6) - R.ec_abs;  // farthest point nearer: wholly inside
  int n = 0;
  for (uint32_t base = 0; base < cnt; base += 32) {  // 32 segments per accept mask
  const uint32_t m = RECT ? 4u : min(32u, cnt - base);
  uint32_t acc = 0;
  for (uint32_t k = 0; k < m; ++k) {  // segment (ring[i-1], ring[i])
    // a segment lying inside the circle by the reach margin has both roots
    // outside [0, 1] by far more than their error: the reference takes none
    if (!RECT && list && (double)R.ec_far[(list - R.ec_edge) + base + k] < inner) continue;
    const uint32_t i = (!RECT && list) ? list[base + k] : base + k;
    const double2 A = ring[i == 0 ? nv - 1 : i - 1], Bv = ring[i];
    if (RECT) {
      const double h = A.x == Bv.x ? fabs(A.x - cx) : fabs(A.y - cy);
      if (h > reach) continue;
    }
    const double dx = Bv.x - A.x, dy = Bv.y - A.y;
    const double fx = A.x - cx, fy = A.y - cy;
    const double qa = dx * dx + dy * dy;
    const double qb = 2.0 * (fx * dx + fy * dy);
    const double qc = fx * fx + fy * fy - r2;
    const double disc = qb * qb - 4.0 * qa * qc;
    const double scale = qb * qb + fabs(4.0 * qa * qc);
    if (qa != 0.0 && disc > 1e-9 * scale) acc |= 1u << k;
  }
  while (acc) {
    const uint32_t k = __ffs(acc) - 1;
    acc &= acc - 1;
    const uint32_t i = (!RECT && list) ? list[base + k] : base + k;
    const double2 A = ring[i == 0 ? nv - 1 : i - 1], Bv = ring[i];
    const double dx = Bv.x - A.x, dy = Bv.y - A.y;
    const double fx = A.x - cx, fy = A.y - cy;
    const double qa = dx * dx + dy * dy;
    const double qb = 2.0 * (fx * dx + fy * dy);
    const double qc = fx * fx + fy * fy - r2;
    const double disc = qb * qb - 4.0 * qa * qc;
    const double sq = sqrt(disc);
    const double t0 = (-qb - sq) / (2.0 * qa);
    const double t1 = (-qb + sq) / (2.0 * qa);
    if (t0 >= 0.0 && t0 <= 1.0) {
      if (n >= cap) return -1.0;
      buf[(2 * n) * stride] = (A.y + t0 * dy) - cy;
      buf[(2 * n + 1) * stride] = (A.x + t0 * dx) - cx;
      ++n;
    }
    if (t1 >= 0.0 && t1 <= 1.0) {
      if (n >= cap) return -1.0;
      buf[(2 * n) * stride] = (A.y + t1 * dy) - cy;
      buf[(2 * n + 1) * stride] = (A.x + t1 * dx) - cx;
      ++n;
    }
  }
  }
  if (n == 0) return 1.0;
  for (int k = 0; k < n; ++k) {  // angle k overwrites slot k (vector k sits at 2k, 2k+1)
    double ang = fast_atan2(buf[(2 * k) * stride], buf[(2 * k + 1) * stride]);
    if (ang < 0.0) ang += kTwoPi;
    buf[k * stride] = ang;
  }
  for (int a = 1; a < n; ++a) {  // std::sort (ascending; same sequence)
    const double v = buf[a * stride];
    int b = a - 1;
    while (b >= 0 && buf[b * stride] > v) {
      buf[(b + 1) * stride] = buf[b * stride];
      --b;
    }
    buf[(b + 1) * stride] = v;
  }
  int u = 0;
  for (int a = 0; a < n; ++a) {
    const double v = buf[a * stride];
    if (u == 0 || v - buf[(u - 1) * stride] > kAngleEps) buf[(u++) * stride] = v;
  }
  const double first = buf[0];
  if (u > 1 && (first + kTwoPi) - buf[(u - 1) * stride] <= kAngleEps) --u;
  if (u < 2) return 1.0;
  double inside_span = 0.0;
  for (int a = 0; a < u; ++a) {
    const double a0 = buf[a * stride];
    const double a1 = (a + 1 < u) ? buf[(a + 1) * stride] : first + kTwoPi;
    const double mid = 0.5 * (a0 + a1);
    int dec = RECT ? rect_probe_certified(cx, cy, d, mid, R) : -1;
    if (dec < 0) {
      double sn, cs;
      sincos(mid, &sn, &cs);
      const double px = cx + d * cs, py = cy + d * sn;
      dec = (RECT ? point_in_rect(px, py, R) : point_in_region(px, py, R)) ? 1 : 0;
    }
    if (dec) inside_span += a1 - a0;
  }
  return inside_span / kTwoPi;
}

// spatial_isotropic_weight in closed form for the dominant rectangle case:
// the center strictly inside, exactly one side crossed, the other three out of
// reach d*(1+1e-6), and that side's quadratic accepted.  The reference then
// finds two crossings strictly inside the side (the perpendicular sides are
// out of reach, so the chord ends lie >= 1e-6 d inside the segment), two
// distinct angles, an outside arc of 2*theta whose midpoint probe lies beyond
// the side by ~(d - h) > 4 box_m (PIP false) and an inside arc whose probe is
// >= 1e-6 d inside (PIP true):
//   omega_ref = (2*pi - 2*theta_ref) / (2*pi),  cos(theta) = h / d.
// theta_ref carries the reference's own rounding (the quadratic's
// cancellation: <= 2^-53 * scale / (len * sqrt(disc) * d) rad), which the
// gate qa*disc*d^2 >= 1e-10*scale^2 bounds by ~1e-11.
// 1/x for a normal positive x to ~1 ulp: the hardware approximation plus two
// Newton steps, without the IEEE division's special-case path (the arc
// drains' operands are bounded away from zero and infinity by their gates).
__device__ __forceinline__ double rcp_pos(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// The single-edge closed form, per center and q = d^2 (the pair kernel's arc
// drains), without forming d = RN(sqrt(q)).  Sufficient conditions in q for the
// reference's own decisions with d = RN(sqrt(q)) (d^2 = q (1 +- 2.3e-16)),
// slack included for the roundings of the reference's quadratic (DESIGN.md
// §4.4), with h the nearest side's distance, h2 the second nearest and fa the
// along-side offset of the reference's segment start (fa^2 >= h2^2 > q):
//   the other three sides out of reach h_s >= d (1 + 1e-6) <=  q < h2^2 / (1 + 2.1e-6)
//   d >= sw_dmin                                          <=  q >= sw_q_min
//   d - h > 4 box_m + 1e-12 d                             <=  q (1 - 2.5e-12) > (h + 4 box_m)^2
//   disc > 1e-9 scale (accept) and qa disc d^2 >= 1e-10 scale^2, with
//   disc = 4 D^2 (d^2 - h^2) +- 3e-15 (fa^2 + d^2) 4 D^2 and
//   scale = 4 D^2 (fa^2 + |h^2 + fa^2 - d^2|) (1 +- 1e-15) = 4 D^2 (K - d^2), K = 2 fa^2 + h^2:
//     E > 1.00001e-9 S + 4e-15 (fa^2 + q)  and
//     (E - 4e-15 (fa^2 + q)) q >= 4.0001e-10 (S + 3e-16 q)^2,  E = q - h^2, S = K - q.
// All are intervals in q: the last is q >= the larger root of a quadratic.  So
// each center carries {h, [q_lo, q_hi)} (rect_arc_record, computed once per
// point in the grid build, bounds widened by 1e-12 relative against their own
// rounding), stored as the high words of q_lo rounded up and of q_hi rounded
// down: hi32(q) in [lo, hi) implies q in [q_lo, q_hi).  Then
// omega = 1 - atan2(sqrt(E), h) / pi, within ~1e-13 of the d-based form (theta
// moves by h * 2.3e-16 / (2 w), w = sqrt(E) bounded below by the interval).
// An empty interval (lo = ~0) sends every arc pair of the center to the exact
// path.
__device__ __forceinline__ double2 rect_arc_record(double cx, double cy, const RegionView& R) {
  const double hl = cx - R.xmin, hr = R.xmax - cx, hb = cy - R.ymin, ht = R.ymax - cy;
  const bool xr = hr < hl, yt = ht < hb;
  const double a = xr ? hr : hl, A = xr ? hl : hr;
  const double b = yt ? ht : hb, Bm = yt ? hb : ht;
  const bool hz = b < a;  // the nearest side is horizontal (y = ymin / ymax)
  const double h = hz ? b : a;
  const double h2 = fmin(hz ? a : b, fmin(A, Bm));
  const int sd = hz ? (yt ? 3 : 2) : (xr ? 1 : 0);
  const double fa = R.sd_start[sd] - (hz ? cx : cy);
  const double h_2 = h * h, fa2 = fa * fa, K = 2.0 * fa2 + h_2;
  const double c1 = 1.00001e-9, c2 = 4e-15, c4 = 4.0001e-10, k = 1.0 - 3e-16;
  const double hm = h + R.sw_margin;
  double lo = fmax(R.sw_q_min, hm * hm / (1.0 - 2.5e-12));
  lo = fmax(lo, (h_2 * (1.0 + c1) + fa2 * (2.0 * c1 + c2)) / (1.0 + c1 - c2));
  const double qa = (1.0 - c2) - c4 * k * k, qb = h_2 + c2 * fa2 - 2.0 * c4 * K * k,
               qc = c4 * K * K;
  lo = fmax(lo, (qb + sqrt(qb * qb + 4.0 * qa * qc)) / (2.0 * qa));
  lo *= 1.0 + 1e-12;
  const double hi = h2 * h2 / (1.0 + 2.1e-6) * (1.0 - 1e-12);
  uint32_t lo_h = ~0u, hi_h = 0u;
  if (h > 0.0 && lo < hi && lo < 1e300) {
    const uint64_t lb = (uint64_t)__double_as_longlong(lo);
    lo_h = (uint32_t)(lb >> 32) + ((uint32_t)lb != 0u ? 1u : 0u);
    hi_h = (uint32_t)__double2hiint(hi);
  }
  return make_double2(h, __longlong_as_double((long long)(((uint64_t)hi_h << 32) | lo_h)));
}

// Constants of the arc drains' closed form in the constant bank: FP64
// instructions take a constant-bank operand directly, whereas a literal
// double costs two uniform moves per use.
// [0, 11): the atan polynomial of fast_atan2 (highest degree first);
// [11, 15): tan(pi/8), pi/4, pi/2, -1/pi
static __constant__ double kArcC[15] = {
    -0.0192025292684122813793, 0.0392536963206185629612, -0.0508625488582314312944,
    0.0585831181050115303872,  -0.0666453136980500884962, 0.0769218469937177728423,
    -0.090909046476956795219,  0.111111110171003266375,   -0.142857142846913806166,
    0.199999999999956505772,   -0.333333333333333302719,
    0.41421356237309504880,    0.78539816339744830962,    1.57079632679489661923,
    -0.31830988618379067154};

// atan2(y, x) for y > 0, x > 0 finite (fast_atan2 without the sign cases).
__device__ __forceinline__ double atan2_pos(double y, double x) {
  const bool steep = y > x;
  const double mx = steep ? y : x, mn = steep ? x : y;
  const bool small = mn <= kArcC[11] * mx;
  const double t = (small ? mn : mn - mx) * rcp_pos(small ? mx : mn + mx);
  const double s = t * t;
  double r = kArcC[0];
#pragma unroll
  for (int i = 1; i < 11; ++i) r = fma(r, s, kArcC[i]);
  const double a = (small ? 0.0 : kArcC[12]) + fma(t * s, r, t);
  return steep ? kArcC[13] - a : a;
}

// omega of a pair at q from its center's rect_arc_record, or -1 (exact path).
__device__ __forceinline__ double rect_single_edge_omega(double q, double2 rec) {
  const uint64_t iv = (uint64_t)__double_as_longlong(rec.y);
  const uint32_t qh = (uint32_t)__double2hiint(q);
  if (!(qh >= (uint32_t)iv && qh < (uint32_t)(iv >> 32))) return -1.0;
  const double h = rec.x;
  const double theta = atan2_pos(sqrt(fma(-h, h, q)), h);
  return fma(theta, kArcC[14], 1.0);  // 1 - theta / pi
}

// spatial_isotropic_weight in closed form for a rectangle and a circle that
// reaches several sides (corners; circles larger than the region).  For each
// side within reach the reference's own quadratic decides accept / reject; an
// accepted side s at distance h contributes the line crossings phi_s +- theta_s
// (cos theta = h / d; phi = 0, pi/2, pi, 3pi/2 for the right, top, left, bottom
// side), each of which lies on the segment iff the corner on its side of the
// foot is outside the circle.  Gates (else -1, the general routine): the
// single-side gates of rect_single_edge_omega for every accepted side, no side
// rejected while its line is nearer than d (a tangency the reference drops),
// and every corner between two sides within reach away from the circle by
// |g| = ||K - c|^2 - d^2| > 1e-4 d^2 — then crossings are 2.5e-5 d or more from
// the segment ends and from each other, far above the reference's root error,
// and its de-duplication keeps them all.  No crossing at all gives 1.0 (the
// reference's rule when the circle contains the whole rectangle).
//
// The crossings come out in increasing angle without sorting: side s's
// clockwise end phi - theta precedes its counter-clockwise end, and the next
// side's clockwise end follows unless the corner between them is inside the
// circle (then both are dropped; theta_s + theta_s1 < pi/2 exactly when that
// corner is outside).  So ends alternate clockwise / counter-clockwise, arcs
// from a clockwise end to the next end are outside and the others inside, and
// each end borders one inside arc:
//   inside span = pi/2 * (sum_cw s - sum_ccw s) + 2 pi [first end is cw]
//                 - sum over ends of theta_s.
// The theta sum is the argument of the product of (h_s + i w_s), w_s =
// sqrt((d - h_s)(d + h_s)), one factor per end: one atan2 per pair instead of
// one per side, with whole turns counted as the running product's imaginary
// part turns non-negative again.
// The reference classifies each arc by a PIP probe at its midpoint, which its
// crossing angles place within ~1e-11 d of the true midpoint; the corner gate
// keeps every true midpoint farther than that (plus on_segment's 1e-12 scale)
// from the boundary, so the probe returns the pattern above:
//  * a side's own outside arc: beyond the side by d - h_s > 4 box_m (as in the
//    single-side form);
//  * an arc around a corner K inside the circle (its two ends dropped): outside,
//    at least d - |K - c| > d (1 - sqrt(1 - 1e-4)) > 5e-5 d from the region;
//  * an inside arc between sides s and s+1 around an outside corner: its ends
//    P1, P2 lie g / (h + w) >= 5e-5 d from K along the sides, so its span is
//    >= 7e-5 and its midpoint clears side s by 2 w_s sin(span / 4) >= 3.5e-8 d
//    under the gate w >= 1e-3 d on every side with an end (likewise side
//    s+1), and the two opposite sides by more than their distance h to the
//    center (the midpoint lies in the quadrant between sides s and s+1).
// With T = 1e-11 d + 4 box_m + 1e-12 (max|coord| + d + 1) the reference's
// probe error plus every on_segment tolerance, the gates 3.5e-8 d > T and
// min h > T leave each probe on the expected side.  (The round-1 form probed
// every midpoint under a 1e-5 d^2 corner gate, where clearances fall to
// ~1e-12 d.)
// Results below 1e-3 go to the general routine (see the end).
__device__ __forceinline__ double rect_multi_edge_weight(double cx, double cy, double d,
                                                         const RegionView& R) {
  if (d <= 0.0) return 1.0;
  if (!(cx > R.xmin && cx < R.xmax && cy > R.ymin && cy < R.ymax) || d < R.sw_dmin) return -1.0;
  if (!(d > 1e-30 && d < 1e30)) return -1.0;  // keeps the product of <= 8 factors of size d finite
  const double reach = d * (1.0 + 1e-6);
  const double r2 = d * d;
  // sides in angular order: right (x = xmax), top, left (x = xmin), bottom; the
  // RegionView side tables are ordered left, right, bottom, top
  const double h[4] = {R.xmax - cx, R.ymax - cy, cx - R.xmin, cy - R.ymin};
  const int tab[4] = {1, 3, 0, 2};
  const double along[4] = {cy, cx, cy, cx};
  double w[4] = {0.0, 0.0, 0.0, 0.0};
  unsigned acc = 0, inr = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (!(h[s] <= reach)) continue;
    inr |= 1u << s;
    const double fa = R.sd_start[tab[s]] - along[s];
    const double D = R.sd_len[tab[s]];
    const double qa = D * D;
    const double qb = 2.0 * (fa * D);
    const double qc = h[s] * h[s] + fa * fa - r2;
    const double disc = qb * qb - 4.0 * qa * qc;
    const double scale = qb * qb + fabs(4.0 * qa * qc);
    if (!(qa != 0.0 && disc > 1e-9 * scale)) {
      if (h[s] < d) return -1.0;  // a crossing line the reference drops as tangent
      continue;
    }
    if (qa * disc * r2 < 1e-10 * scale * scale) return -1.0;
    const double dm = d - h[s];
    if (dm <= R.sw_margin + 1e-12 * d) return -1.0;
    w[s] = sqrt(dm * (d + h[s]));
    acc |= 1u << s;
  }
  if (acc == 0) return 1.0;
  const double T = 1e-11 * d + 4.0 * R.box_m + 1e-12 * (R.maxabs + d + 1.0);
  if (!(3.5e-8 * d > T && fmin(fmin(h[0], h[1]), fmin(h[2], h[3])) > T)) return -1.0;
  // corner k sits between side k and side k+1 (counter-clockwise)
  unsigned cin = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int k1 = (k + 1) & 3;
    if (!((inr >> k) & 1u) || !((inr >> k1) & 1u)) continue;  // beyond reach: outside
    const double g = h[k] * h[k] + h[k1] * h[k1] - r2;
    if (fabs(g) <= 1e-4 * r2) return -1.0;
    if (g < 0.0) cin |= 1u << k;
  }
  // crossing ends: slot 2s = side s's clockwise end (dropped when corner s-1
  // is inside), slot 2s+1 its counter-clockwise end (dropped when corner s is)
  unsigned E = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (!((acc >> s) & 1u)) continue;
    E |= (((cin >> ((s + 3) & 3)) & 1u) ^ 1u) << (2 * s);
    E |= (((cin >> s) & 1u) ^ 1u) << (2 * s + 1);
  }
  if (E == 0) return 1.0;
  if (__popc(E) & 1) return -1.0;  // cannot happen (ends alternate); defensive
#pragma unroll
  for (int s = 0; s < 4; ++s)  // the inside-arc clearance gate (above)
    if (((E >> (2 * s)) & 3u) && w[s] < 1e-3 * d) return -1.0;
  // theta sum = argument of prod_s (h_s + i w_s)^{c_s}, c_s = ends of side s;
  // each factor adds c_s * theta_s < pi, so whole turns show as the imaginary
  // part turning non-negative again
  double pr = 1.0, pim = 0.0;
  int turns = 0, ksum = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const unsigned cw = (E >> (2 * s)) & 1u, ccw = (E >> (2 * s + 1)) & 1u;
    ksum += s * ((int)cw - (int)ccw);
    if (!(cw | ccw)) continue;
    double zr = h[s], zi = w[s];
    if (cw & ccw) {  // (h + i w)^2
      zr = (h[s] - w[s]) * (h[s] + w[s]);
      zi = 2.0 * h[s] * w[s];
    }
    const double nr = pr * zr - pim * zi;
    const double ni = pr * zi + pim * zr;
    turns += (pim < 0.0) & (ni >= 0.0);
    pr = nr;
    pim = ni;
  }
  const bool first_cw = !((__ffs(E) - 1) & 1);  // the lowest end is a clockwise one
  const double kHalfPi = 1.57079632679489661923;
  double a = fast_atan2(pim, pr);
  if (a < 0.0) a += kTwoPi;
  const double tsum = a + kTwoPi * turns;
  const double span = kHalfPi * ksum + (first_cw ? kTwoPi : 0.0) - tsum;
  // the reference's crossing points carry its own rounding (up to ~1e-12 rad at
  // large coordinate offsets); a small omega would turn that into a large
  // relative difference, so small results come from the general routine,
  // which reproduces those crossing points
  const double wt = span * 0.15915494309189533577;  // / (2 pi)
  return wt >= 1e-3 ? wt : -1.0;
}

// Squared radius below which spatial_weight() provably returns exactly 1.0
// for this center (the circle stays strictly inside every edge's reach by a
// relative margin far above the rounding error of the reference's quadratic;
// DESIGN.md §4.4).  Returns -1 when no such radius exists.
// With edge cells (general polygons) only the cell's segments are visited:
// every other segment is farther than ec_reach from the point, so the true
// nearest distance is >= min(listed nearest, ec_reach) and the radius below
// stays a lower bound.
__device__ __forceinline__ double safe_q(double cx, double cy, const RegionView& R) {
  if (R.rect) {  // the nearest boundary point of a rectangle lies on a side's perpendicular
    const double rs = fmin(fmin(cx - R.xmin, R.xmax - cx), fmin(cy - R.ymin, R.ymax - cy));
    const double scale = fmax(R.maxabs, fmax(fabs(cx), fabs(cy)));
    const double r_ok = rs - 1e-6 * (rs + scale);
    return r_ok > 0.0 ? r_ok * r_ok * (1.0 - 1e-9) : -1.0;
  }
  const double2* ring = R.ring;
  const uint32_t nv = R.nv;
  double r2 = 1.0e308;
  uint32_t cnt = nv;
  const uint32_t* list = nullptr;
  if (!R.rect && R.ec_start != nullptr) {
    list = edge_list(cx, cy, 0.0, R, &cnt);
    r2 = R.ec_reach * R.ec_reach;
  }
  const double ring_maxabs = R.maxabs;
  const float* dml = list ? R.ec_dmin + (list - R.ec_edge) : nullptr;
  for (uint32_t k = 0; k < cnt; ++k) {
    // sorted lower bounds: nothing further down the list can come nearer
    if (dml && (double)dml[k] * (double)dml[k] >= r2) break;
    const uint32_t i = list ? list[k] : k;
    const double2 a = ring[i == 0 ? nv - 1 : i - 1], b = ring[i];
    const double ex = b.x - a.x, ey = b.y - a.y;
    const double len2 = ex * ex + ey * ey;
    double t = 0.0;
    if (len2 > 0.0) {
      t = ((cx - a.x) * ex + (cy - a.y) * ey) / len2;
      t = fmin(fmax(t, 0.0), 1.0);
    }
    const double px = a.x + t * ex - cx, py = a.y + t * ey - cy;
    r2 = fmin(r2, px * px + py * py);
  }
  const double rs = sqrt(r2);
  const double scale = fmax(ring_maxabs, fmax(fabs(cx), fabs(cy)));
  const double r_ok = rs - 1e-6 * (rs + scale);
  return r_ok > 0.0 ? r_ok * r_ok * (1.0 - 1e-9) : -1.0;
}

// -------------------------------------------------- exact accumulation
// Term 1/w minus 1 as a signed 128-bit fixed-point integer with 53 fractional
// bits (two's complement in lo/hi).  w = omega * v with v in {1, 1/2} and
// omega <= 1 up to the reference's own rounding (its arc sum can exceed 2*pi by
// an ulp: omega = 1 + 2^-52 happens), so 1/w >= 1/2 and its ulp is >= 2^-53:
// the conversion is exact, and terms just below 1 give small negative values.
__device__ __forceinline__ void fixed_term_minus_one(double term, uint64_t* lo, uint64_t* hi) {
  const uint64_t one = 1ULL << kFixedFracBits;
  if (term < 2048.0) {  // term * 2^53 is an integer below 2^64: one exact conversion
    const uint64_t v = __double2ull_rn(term * 0x1p53);
    *lo = v - one;
    *hi = (v < one) ? ~0ULL : 0ULL;
    return;
  }
  const uint64_t bits = __double_as_longlong(term);
  const int e = int((bits >> 52) & 0x7FF) - 1023;            // term = 1.m * 2^e, e >= -1
  const uint64_t mant = (bits & 0xFFFFFFFFFFFFFULL) | (1ULL << 52);
  const int sh = e + 1;                                       // term * 2^53 = mant << sh
  uint64_t l, h;
  if (sh < 0 || sh >= 75) {  // cannot happen for w in (0, 1 + tiny]; saturate visibly
    l = ~0ULL;
    h = ~0ULL >> 1;
  } else if (sh == 0) {
    l = mant;
    h = 0;
  } else if (sh < 64) {
    l = mant << sh;
    h = mant >> (64 - sh);
  } else {
    l = 0;
    h = mant << (sh - 64);
  }
  // subtract 1.0 == 2^53 (borrows into hi: negative results wrap to two's complement)
  h -= (l < one) ? 1ULL : 0ULL;
  l -= one;
  *lo = l;
  *hi = h;
}

// Correctly rounded double of the 128-bit unsigned value (hi:lo) * 2^-53.
__device__ __forceinline__ double fixed128_to_double(uint64_t hi, uint64_t lo) {
  if (hi == 0) return ldexp((double)lo, -kFixedFracBits);  // u64 -> f64 rounds to nearest
  const int lz = __clzll((long long)hi);
  const int sh = 64 - lz;  // bits of hi above position 64
  uint64_t top = lz == 0 ? hi : ((hi << lz) | (lo >> sh));
  const uint64_t rest = lo << lz;  // low bits that do not fit in top
  if (rest != 0) top |= 1ULL;      // sticky bit (below the 53-bit rounding point)
  return ldexp((double)top, sh - kFixedFracBits);
}

// ------------------------------------------------------ MT19937-64
// std::mt19937_64 tempering ([rand.eng.mers]); rng::Engine wraps it
// (proj/core/include/stripley/rng.hpp:10-40).
__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}
__device__ __forceinline__ uint64_t mt_mag(uint64_t y) {
  return (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}
constexpr uint64_t kMtUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kMtLower = 0x7FFFFFFFULL;

// rng::Engine::real01 (rng.hpp:28) and uniform (rng.hpp:31)
__device__ __forceinline__ double mt_uniform(uint64_t v, double lo, double hi) {
  const double r01 = (double)(v >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * r01;
}

}  // namespace stk
