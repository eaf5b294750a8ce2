// stripley_api.cpp — the reference's C++ entry points (include/stripley_gpu.hpp)
// implemented over the C ABI (include/stk.h).  Host code only: validation
// and small host-side surface utilities follow the reference line by line;
// every estimation / simulation runs on the device.
#include "../../include/stripley_gpu.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>
#include <string>

#include "../../include/stk.h"

namespace stripley {
namespace {

constexpr double kPi = std::numbers::pi;

[[noreturn]] void raise(int rc, const std::string& msg) {
  if (rc == STK_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("stk error " + std::to_string(rc) + ": " + msg);
}

// One context per device per process (a context is single-threaded; the
// mutex serialises host threads sharing it, like the reference's
// single-writer WeightCache contract).
struct Ctx {
  stk_ctx* h = nullptr;
  std::mutex mu;
  std::vector<double> ring;
  std::int64_t p0 = 0, p1 = 0;
  std::vector<double> s;
  std::vector<std::int64_t> t;
  bool have_region = false, have_grid = false;
  ~Ctx() {
    if (h) stk_destroy(h);
  }
  void check(int rc) {
    if (rc != STK_OK) raise(rc, stk_last_error(h));
  }
  void region(const geom::StudyRegion& r) {
    std::vector<double> flat;
    for (const auto& v : r.boundary()) {
      flat.push_back(v.x);
      flat.push_back(v.y);
    }
    if (have_region && flat == ring && p0 == r.period_start() && p1 == r.period_end()) return;
    check(stk_set_region(h, flat.data(), (uint32_t)r.boundary().size(), r.period_start(),
                         r.period_end()));
    ring = std::move(flat);
    p0 = r.period_start();
    p1 = r.period_end();
    have_region = true;
  }
  void grid(const est::DistanceGrid& g) {
    if (have_grid && g.s_values == s && g.t_values == t) return;
    check(stk_set_grid(h, g.s_values.data(), (uint32_t)g.s_values.size(), g.t_values.data(),
                       (uint32_t)g.t_values.size()));
    s = g.s_values;
    t = g.t_values;
    have_grid = true;
  }
};

Ctx& context(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Ctx>> ctxs;
  std::lock_guard<std::mutex> lk(mu);
  auto& c = ctxs[device];
  if (!c) {
    c = std::make_unique<Ctx>();
    if (stk_create(&c->h, device) != STK_OK) {
      c.reset();
      throw std::runtime_error("stk_create failed: no usable CUDA device (no CPU fallback)");
    }
  }
  return *c;
}

struct SoA {
  std::vector<double> x, y;
  std::vector<std::int64_t> t;
  explicit SoA(std::span<const geom::STPoint> pts) : x(pts.size()), y(pts.size()), t(pts.size()) {
    for (std::size_t i = 0; i < pts.size(); ++i) {
      x[i] = pts[i].x;
      y[i] = pts[i].y;
      t[i] = pts[i].start_time;
    }
  }
};

std::vector<geom::STPoint> to_points(const std::vector<double>& x, const std::vector<double>& y,
                                     const std::vector<std::int64_t>& t) {
  std::vector<geom::STPoint> out(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) out[i] = geom::make_point(x[i], y[i], t[i]);
  return out;
}

est::KSurface surface(const est::DistanceGrid& g, const double* flat, est::SurfaceKind kind) {
  est::KSurface s;
  s.grid = g;
  s.kind = kind;
  s.values.assign(g.cells_s(), std::vector<double>(g.cells_t(), 0.0));
  for (std::size_t si = 0; si < g.cells_s(); ++si)
    for (std::size_t ti = 0; ti < g.cells_t(); ++ti) s.values[si][ti] = flat[si * g.cells_t() + ti];
  return s;
}

int method_code(sim::Method m) {
  switch (m) {
    case sim::Method::Cstr: return STK_METHOD_CSR;
    case sim::Method::Bootstrap: return STK_METHOD_BOOTSTRAP;
    case sim::Method::Permutation: return STK_METHOD_PERMUTATION;
  }
  throw std::invalid_argument("unknown simulation method");
}

void check_cache(const est::EstimatorOptions& o, const cache::WeightCache* wc) {
  const bool tol = o.coord_tolerance != 0.0 || o.dist_tolerance != 0.0 ||
                   (wc && (wc->coord_tolerance() != 0.0 || wc->dist_tolerance() != 0.0));
  if (o.use_cache && tol)
    throw std::runtime_error("nonzero weight-cache tolerances are not supported on the device path");
}

}  // namespace

// ------------------------------------------------------------------- geom
namespace geom {

bool point_in_polygon(const PlanarPoint& pt, const std::vector<PlanarPoint>& ring) {
  const std::size_t n = ring.size();
  if (n < 3) return false;
  auto on_segment = [](const PlanarPoint& p, const PlanarPoint& a, const PlanarPoint& b) {
    const double cross = (b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x);
    const double scale = std::max({std::abs(a.x), std::abs(a.y), std::abs(b.x), std::abs(b.y),
                                   std::abs(p.x), std::abs(p.y), 1.0});
    if (std::abs(cross) > 1e-12 * scale * scale) return false;
    return p.x >= std::min(a.x, b.x) - 1e-12 * scale && p.x <= std::max(a.x, b.x) + 1e-12 * scale &&
           p.y >= std::min(a.y, b.y) - 1e-12 * scale && p.y <= std::max(a.y, b.y) + 1e-12 * scale;
  };
  for (std::size_t i = 0; i < n; ++i)
    if (on_segment(pt, ring[i], ring[(i + 1) % n])) return true;
  bool inside = false;
  for (std::size_t i = 0, j = n - 1; i < n; j = i++) {
    const PlanarPoint& a = ring[i];
    const PlanarPoint& b = ring[j];
    if ((a.y > pt.y) != (b.y > pt.y)) {
      const double x_cross = a.x + (pt.y - a.y) / (b.y - a.y) * (b.x - a.x);
      if (pt.x < x_cross) inside = !inside;
    }
  }
  return inside;
}

StudyRegion::StudyRegion(std::vector<PlanarPoint> ring, std::int64_t period_start,
                         std::int64_t period_end)
    : ring_(std::move(ring)), period_start_(period_start), period_end_(period_end) {
  std::vector<double> flat;
  for (const auto& v : ring_) {
    flat.push_back(v.x);
    flat.push_back(v.y);
  }
  double area = 0.0;
  std::int64_t dur = 0;
  char msg[256];
  const int rc = stk_check_region(flat.data(), (uint32_t)ring_.size(), period_start, period_end,
                                  &area, &dur, msg, sizeof msg);
  if (rc != STK_OK) raise(rc, msg);
  if (ring_.size() >= 2 && ring_.front().x == ring_.back().x && ring_.front().y == ring_.back().y)
    ring_.pop_back();
  area_ = area;
  duration_ = dur;
}

// geometry.cpp:27-44 (host side; the device computes the same expressions)
double spatial_distance(const STPoint& p, const STPoint& q) {
  const double dx = p.x - q.x;
  const double dy = p.y - q.y;
  return std::sqrt(dx * dx + dy * dy);
}

std::int64_t temporal_distance(const STPoint& p, const STPoint& q) {
  return p.start_time >= q.start_time ? p.start_time - q.start_time
                                      : q.start_time - p.start_time;
}

bool within_cylinder(const STCylinder& cyl, const STPoint& p) {
  return spatial_distance(cyl.center, p) <= cyl.spatial_radius &&
         temporal_distance(cyl.center, p) <= cyl.temporal_radius;
}

STEnvelope StudyRegion::bounding_envelope() const {
  STEnvelope env;
  env.x_min = env.x_max = ring_[0].x;
  env.y_min = env.y_max = ring_[0].y;
  for (const auto& v : ring_) {
    env.x_min = std::min(env.x_min, v.x);
    env.x_max = std::max(env.x_max, v.x);
    env.y_min = std::min(env.y_min, v.y);
    env.y_max = std::max(env.y_max, v.y);
  }
  env.t_min = period_start_;
  env.t_max = period_end_;
  return env;
}

}  // namespace geom

// -------------------------------------------------------------------- est
namespace est {

void DistanceGrid::validate() const {
  char msg[256];
  const int rc = stk_check_grid(s_values.data(), (uint32_t)s_values.size(), t_values.data(),
                                (uint32_t)t_values.size(), msg, sizeof msg);
  if (rc != STK_OK) raise(rc, msg);
}

DistanceGrid DistanceGrid::regular(double s_step, double s_max, std::int64_t t_step,
                                   std::int64_t t_max) {
  DistanceGrid grid;  // estimator.cpp:24-32 (accumulating s += step)
  for (double s = s_step; s <= s_max * (1.0 + 1e-12); s += s_step) grid.s_values.push_back(s);
  for (std::int64_t t = t_step; t <= t_max; t += t_step) grid.t_values.push_back(t);
  grid.validate();
  return grid;
}

double intensity(std::size_t n, const geom::StudyRegion& region) {
  if (n == 0) throw std::invalid_argument("intensity needs n >= 1");
  return static_cast<double>(n) / (region.area() * static_cast<double>(region.duration()));
}

double theoretical_k(double s, double t) { return 2.0 * kPi * s * s * t; }

double k_to_l(double k, double s, double t) {
  if (t == 0.0) throw std::invalid_argument("L transform undefined at t=0");
  if (k < 0.0) throw std::invalid_argument("K value must be >= 0");
  return std::sqrt(k / (2.0 * kPi * t)) - s;
}

KSurface theoretical_surface(const DistanceGrid& grid) {
  KSurface surf;
  surf.grid = grid;
  surf.kind = SurfaceKind::K;
  surf.values.assign(grid.cells_s(), std::vector<double>(grid.cells_t(), 0.0));
  for (std::size_t si = 0; si < grid.cells_s(); ++si)
    for (std::size_t ti = 0; ti < grid.cells_t(); ++ti)
      surf.values[si][ti] = theoretical_k(grid.s_values[si], static_cast<double>(grid.t_values[ti]));
  return surf;
}

KSurface to_l(const KSurface& k_surface) {
  KSurface surf = k_surface;
  surf.kind = SurfaceKind::L;
  for (std::size_t si = 0; si < surf.grid.cells_s(); ++si)
    for (std::size_t ti = 0; ti < surf.grid.cells_t(); ++ti)
      surf.values[si][ti] = k_to_l(k_surface.values[si][ti], surf.grid.s_values[si],
                                   static_cast<double>(surf.grid.t_values[ti]));
  return surf;
}

std::optional<std::pair<std::size_t, std::size_t>> bin_pair(const DistanceGrid& grid, double d,
                                                            std::int64_t u) {
  auto s_it = std::lower_bound(grid.s_values.begin(), grid.s_values.end(), d);
  if (s_it == grid.s_values.end()) return std::nullopt;
  auto t_it = std::lower_bound(grid.t_values.begin(), grid.t_values.end(), u);
  if (t_it == grid.t_values.end()) return std::nullopt;
  return std::make_pair(static_cast<std::size_t>(s_it - grid.s_values.begin()),
                        static_cast<std::size_t>(t_it - grid.t_values.begin()));
}

KSurface estimate_surface(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                          const DistanceGrid& grid, const EstimatorOptions& options,
                          cache::WeightCache* weight_cache, EstimatorTelemetry* telemetry) {
  grid.validate();
  if (points.size() < 2) throw std::invalid_argument("K estimation needs n >= 2");
  check_cache(options, weight_cache);
  Ctx& c = context(0);
  std::lock_guard<std::mutex> lk(c.mu);
  c.region(region);
  c.grid(grid);
  const SoA p(points);
  std::vector<double> k(grid.cells_s() * grid.cells_t());
  stk_telemetry tel{};
  c.check(stk_estimate_surface(c.h, p.x.data(), p.y.data(), p.t.data(), points.size(), k.data(),
                               &tel));
  if (telemetry) {  // accumulated with += like the reference (estimator.cpp:180-184)
    telemetry->pair_comparisons += tel.candidate_pairs;
    telemetry->in_threshold_pairs += tel.in_threshold_pairs;
    telemetry->index_build_seconds += tel.grid_ms * 1e-3;
  }
  return surface(grid, k.data(), SurfaceKind::K);
}

KSurface diff_surface(const KSurface& estimated_l, const KSurface& upper_l) {
  if (estimated_l.grid != upper_l.grid) throw std::invalid_argument("grid mismatch between surfaces");
  KSurface surf = estimated_l;
  surf.kind = SurfaceKind::Diff;
  for (std::size_t si = 0; si < surf.grid.cells_s(); ++si)
    for (std::size_t ti = 0; ti < surf.grid.cells_t(); ++ti) {
      const double est = estimated_l.values[si][ti];
      const double up = upper_l.values[si][ti];
      surf.values[si][ti] = est > up ? est - up : 0.0;
    }
  return surf;
}

}  // namespace est

// -------------------------------------------------------------------- sim
namespace sim {

std::vector<geom::STPoint> generate(Method method, std::size_t n,
                                    std::span<const geom::STPoint> observed,
                                    const geom::StudyRegion& region, std::uint64_t seed) {
  Ctx& c = context(0);
  std::lock_guard<std::mutex> lk(c.mu);
  c.region(region);
  const std::size_t m = method == Method::Cstr ? n : observed.size();
  const SoA o(observed);
  std::vector<double> x(m), y(m);
  std::vector<std::int64_t> t(m);
  c.check(stk_generate(c.h, method_code(method), m, o.x.data(), o.y.data(), o.t.data(), seed,
                       x.data(), y.data(), t.data()));
  return to_points(x, y, t);
}

std::vector<geom::STPoint> generate_cstr(std::size_t n, const geom::StudyRegion& region,
                                         std::uint64_t seed) {
  return generate(Method::Cstr, n, {}, region, seed);
}

namespace {
// bootstrap / permutation never read the region; any valid one configures the context
const geom::StudyRegion& unit_region() {
  static const geom::StudyRegion r({{0, 0}, {1, 0}, {1, 1}, {0, 1}}, 0, 1);
  return r;
}
}  // namespace

std::vector<geom::STPoint> generate_bootstrap(std::span<const geom::STPoint> points,
                                              std::uint64_t seed) {
  if (points.empty()) throw std::invalid_argument("bootstrap needs n >= 1");
  return generate(Method::Bootstrap, points.size(), points, unit_region(), seed);
}

std::vector<geom::STPoint> generate_permutation(std::span<const geom::STPoint> points,
                                                std::uint64_t seed) {
  if (points.empty()) throw std::invalid_argument("permutation needs n >= 1");
  return generate(Method::Permutation, points.size(), points, unit_region(), seed);
}

std::vector<est::KSurface> run_simulations(std::span<const geom::STPoint> points,
                                           const geom::StudyRegion& region,
                                           const est::DistanceGrid& grid, Method method,
                                           std::size_t m, std::uint64_t base_seed,
                                           const est::EstimatorOptions& options,
                                           cache::WeightCache* weight_cache) {
  if (m < 1) throw std::invalid_argument("need at least one simulation");
  if (weight_cache) weight_cache->freeze();
  grid.validate();
  if (points.size() < 2) throw std::invalid_argument("K estimation needs n >= 2");
  check_cache(options, weight_cache);
  Ctx& c = context(0);
  std::lock_guard<std::mutex> lk(c.mu);
  c.region(region);
  c.grid(grid);
  const SoA p(points);
  const std::size_t bins = grid.cells_s() * grid.cells_t();
  std::vector<double> l_all(m * bins), up(bins), lo(bins);
  stk_telemetry tel{};
  const bool obs = method != Method::Cstr;
  c.check(stk_simulate(c.h, obs ? p.x.data() : nullptr, obs ? p.y.data() : nullptr,
                       obs ? p.t.data() : nullptr, points.size(), method_code(method), base_seed,
                       0, (uint32_t)m, l_all.data(), up.data(), lo.data(), &tel));
  std::vector<est::KSurface> out;
  out.reserve(m);
  for (std::size_t r = 0; r < m; ++r)
    out.push_back(surface(grid, l_all.data() + r * bins, est::SurfaceKind::L));
  return out;
}

std::pair<est::KSurface, est::KSurface> envelopes(std::span<const est::KSurface> sims) {
  if (sims.empty()) throw std::invalid_argument("envelopes need >= 1 surface");
  for (const auto& s : sims)
    if (s.grid != sims.front().grid)
      throw std::invalid_argument("grid mismatch between simulated surfaces");
  est::KSurface upper = sims.front(), lower = sims.front();
  for (std::size_t k = 1; k < sims.size(); ++k)
    for (std::size_t si = 0; si < upper.grid.cells_s(); ++si)
      for (std::size_t ti = 0; ti < upper.grid.cells_t(); ++ti) {
        upper.values[si][ti] = std::max(upper.values[si][ti], sims[k].values[si][ti]);
        lower.values[si][ti] = std::min(lower.values[si][ti], sims[k].values[si][ti]);
      }
  return {upper, lower};
}

}  // namespace sim

// --------------------------------------------------------------------- rt
namespace rt {

JobPlan build_plan(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                   const JobSpec& spec) {
  (void)points;
  (void)region;
  if (spec.partitions < 1) throw std::invalid_argument("partitions must be >= 1");
  JobPlan plan;
  plan.choice = spec.partitioner;
  plan.partitions = 1;  // the device grid replaces the KDB leaves
  return plan;
}

std::vector<TaskData> make_tasks(const JobPlan& plan, std::span<const geom::STPoint> dataset,
                                 const JobSpec& spec, std::uint64_t* redundancy_out) {
  std::vector<TaskData> tasks(plan.partitions);
  for (std::uint32_t t = 0; t < plan.partitions; ++t) tasks[t].task_id = t;
  std::uint64_t redundancy = 0;
  for (std::size_t i = 0; i < dataset.size(); ++i) {
    const auto idx = static_cast<std::uint32_t>(i);
    tasks[plan.locate(dataset[i], idx)].points.push_back({dataset[i], idx});
    geom::STCylinder cyl;
    cyl.center = dataset[i];
    cyl.spatial_radius = spec.grid.s_max();
    cyl.temporal_radius = spec.grid.t_max();
    cyl.temporal_unit = spec.time_unit;
    for (std::uint32_t t : plan.assign(cyl)) {
      tasks[t].cylinders.push_back({cyl, idx});
      ++redundancy;
    }
  }
  if (redundancy_out) *redundancy_out += redundancy;
  return tasks;
}

namespace {
int device_from_env() {
  const char* d = std::getenv("STK_DEVICE");
  return d ? std::atoi(d) : 0;
}
}  // namespace

PartialResult execute_task(const TaskData& task, const geom::StudyRegion& region,
                           const est::DistanceGrid& grid, const est::EstimatorOptions& options,
                           cache::WeightCache* weight_cache) {
  check_cache(options, weight_cache);
  grid.validate();
  Ctx& c = context(device_from_env());
  std::lock_guard<std::mutex> lk(c.mu);
  c.region(region);
  c.grid(grid);
  const std::size_t np = task.points.size(), nc = task.cylinders.size();
  std::vector<double> px(np), py(np), cx(nc), cy(nc), cr(nc);
  std::vector<std::int64_t> pt(np), ct(nc), ctr(nc);
  std::vector<std::uint32_t> pi(np), ci(nc);
  for (std::size_t j = 0; j < np; ++j) {
    px[j] = task.points[j].pt.x;
    py[j] = task.points[j].pt.y;
    pt[j] = task.points[j].pt.start_time;
    pi[j] = task.points[j].record_index;
  }
  for (std::size_t k = 0; k < nc; ++k) {
    const auto& a = task.cylinders[k];
    cx[k] = a.cyl.center.x;
    cy[k] = a.cyl.center.y;
    ct[k] = a.cyl.center.start_time;
    cr[k] = a.cyl.spatial_radius;
    ctr[k] = a.cyl.temporal_radius;
    ci[k] = a.center_index;
  }
  PartialResult partial;
  partial.task_id = task.task_id;
  partial.histogram.assign(grid.cells_s() * grid.cells_t(), 0.0);
  c.check(stk_task_histogram(c.h, px.data(), py.data(), pt.data(), pi.data(), np, cx.data(),
                             cy.data(), ct.data(), ci.data(), cr.data(), ctr.data(), nc,
                             partial.histogram.data(), &partial.in_threshold_pairs,
                             &partial.pair_comparisons));
  return partial;
}

est::KSurface aggregate(std::span<const PartialResult> partials, std::size_t n,
                        const geom::StudyRegion& region, const est::DistanceGrid& grid) {
  const std::size_t bins = grid.cells_s() * grid.cells_t();
  std::vector<const PartialResult*> ordered;
  for (const auto& p : partials) ordered.push_back(&p);
  std::sort(ordered.begin(), ordered.end(),
            [](const PartialResult* a, const PartialResult* b) { return a->task_id < b->task_id; });
  // PairHistogram::add_flat (estimator.cpp:39-43): Kahan, in task order
  std::vector<double> sum(bins, 0.0), comp(bins, 0.0);
  for (const auto* p : ordered) {
    if (p->histogram.size() != bins)
      throw std::invalid_argument("partial histogram dimension mismatch");
    for (std::size_t b = 0; b < bins; ++b) {
      const double y = p->histogram[b] - comp[b];
      const double t = sum[b] + y;
      comp[b] = (t - sum[b]) - y;
      sum[b] = t;
    }
  }
  // finalize_surface (estimator.cpp:94-114)
  est::KSurface k = surface(grid, sum.data(), est::SurfaceKind::K);
  const std::size_t cs = grid.cells_s(), ct = grid.cells_t();
  for (std::size_t si = 0; si < cs; ++si)
    for (std::size_t ti = 0; ti < ct; ++ti) {
      double acc = sum[si * ct + ti];
      if (si > 0) acc += k.values[si - 1][ti];
      if (ti > 0) acc += k.values[si][ti - 1];
      if (si > 0 && ti > 0) acc -= k.values[si - 1][ti - 1];
      k.values[si][ti] = acc;
    }
  const double scale =
      region.area() * static_cast<double>(region.duration()) /
      (static_cast<double>(n) * static_cast<double>(n));
  for (auto& row : k.values)
    for (double& v : row) v *= scale;
  return k;
}

LocalExecutor::LocalExecutor(std::uint32_t workers, const geom::StudyRegion& region,
                             const est::DistanceGrid& grid, const est::EstimatorOptions& options)
    : workers_(std::max<std::uint32_t>(1, workers)), region_(region), grid_(grid),
      options_(options), device_(device_from_env()) {
  check_cache(options_, nullptr);
}

std::vector<PartialResult> LocalExecutor::run(const std::vector<TaskData>& tasks,
                                              bool simulation_phase) {
  (void)simulation_phase;  // caches are replaced by per-center recomputation
  std::vector<PartialResult> partials(tasks.size());
  for (std::size_t t = 0; t < tasks.size(); ++t) {
    partials[t] = execute_task(tasks[t], region_, grid_, options_);
    partials[t].worker_id = static_cast<std::uint32_t>(t % workers_);
  }
  return partials;
}

void LocalExecutor::collect_telemetry(RunTelemetry& out) const { (void)out; }

DeviceExecutor::DeviceExecutor(int device, std::uint32_t rank, std::uint32_t world,
                               SumHook sum_u64, MaxMinHook max_min)
    : device_(device), rank_(rank), world_(world), sum_(std::move(sum_u64)),
      maxmin_(std::move(max_min)) {
  if (world_ < 1 || rank_ >= world_) throw std::invalid_argument("rank must be < world");
  if (world_ > 1 && !(sum_ && maxmin_))
    throw std::invalid_argument(
        "DeviceExecutor with world > 1 needs an NCCL unique id or both exchange hooks");
}

DeviceExecutor::DeviceExecutor(int device, std::uint32_t rank, std::uint32_t world,
                               const std::array<unsigned char, 128>& nccl_unique_id)
    : device_(device), rank_(rank), world_(world) {
  if (world_ < 1 || rank_ >= world_) throw std::invalid_argument("rank must be < world");
  Ctx& c = context(device_);
  std::lock_guard<std::mutex> lk(c.mu);
  c.check(stk_comm_init(c.h, nccl_unique_id.data(), static_cast<int>(world_),
                        static_cast<int>(rank_)));
  comm_ = true;
}

std::array<unsigned char, 128> DeviceExecutor::nccl_unique_id() {
  std::array<unsigned char, 128> id{};
  const int rc = stk_comm_unique_id(id.data());
  if (rc != STK_OK) throw std::runtime_error("stk_comm_unique_id failed (NCCL unavailable)");
  return id;
}

std::vector<PartialResult> DeviceExecutor::run(const std::vector<TaskData>& tasks,
                                               bool simulation_phase) {
  (void)simulation_phase;
  // the tasks of a region / grid configured by the last run_job on this device
  Ctx& c = context(device_);
  if (!c.have_region || !c.have_grid)
    throw std::runtime_error("DeviceExecutor::run needs a configured region and grid");
  const geom::StudyRegion region(
      [&] {
        std::vector<geom::PlanarPoint> r;
        for (std::size_t i = 0; i + 1 < c.ring.size(); i += 2) r.push_back({c.ring[i], c.ring[i + 1]});
        return r;
      }(),
      c.p0, c.p1);
  est::DistanceGrid g;
  g.s_values = c.s;
  g.t_values = c.t;
  std::vector<PartialResult> partials(tasks.size());
  for (std::size_t t = 0; t < tasks.size(); ++t) {
    partials[t] = execute_task(tasks[t], region, g, est::EstimatorOptions{});
    partials[t].worker_id = rank_;
  }
  return partials;
}

namespace {

double seconds_since(const std::chrono::steady_clock::time_point& t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void add_tel(RunTelemetry& r, const stk_telemetry& t) {
  r.pair_comparisons += t.candidate_pairs;
  r.in_threshold_pairs += t.in_threshold_pairs;
  r.exact_path_pairs += t.exact_path_pairs;
  r.device_ms += t.total_ms;
  r.pair_kernel_ms += t.pair_ms;
}

// The reference's flow for executors that do not name a GPU: plan, tasks,
// executor.run, aggregate per pattern (runtime.cpp:190-249); realisations
// are generated on the device (sim::generate).
RunResult run_job_tasks(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                        const JobSpec& spec, Executor& executor) {
  RunResult result;
  auto t0 = std::chrono::steady_clock::now();
  const JobPlan plan = build_plan(points, region, spec);
  result.telemetry.plan_seconds = seconds_since(t0);
  result.telemetry.partition_count = plan.partitions;
  executor.broadcast_plan(plan);
  auto accumulate = [&](const std::vector<PartialResult>& partials) {
    for (const auto& p : partials) {
      result.telemetry.pair_comparisons += p.pair_comparisons;
      result.telemetry.in_threshold_pairs += p.in_threshold_pairs;
    }
  };
  t0 = std::chrono::steady_clock::now();
  const auto tasks = make_tasks(plan, points, spec, &result.telemetry.cylinder_assignments);
  result.telemetry.partition_point_counts.assign(plan.partitions, 0);
  for (const auto& task : tasks)
    result.telemetry.partition_point_counts[task.task_id] = task.points.size();
  const auto partials = executor.run(tasks, false);
  accumulate(partials);
  result.k_hat = aggregate(partials, points.size(), region, spec.grid);
  result.l_hat = est::to_l(result.k_hat);
  result.theoretical = est::theoretical_surface(spec.grid);
  result.telemetry.estimation_seconds = seconds_since(t0);
  if (spec.sims > 0) {
    t0 = std::chrono::steady_clock::now();
    std::vector<est::KSurface> sims;
    for (std::uint32_t r = 0; r < spec.sims; ++r) {
      const auto sp = sim::generate(spec.method, points.size(), points, region, spec.seed + r);
      const auto st = make_tasks(plan, sp, spec, &result.telemetry.cylinder_assignments);
      const auto sp_partials = executor.run(st, true);
      accumulate(sp_partials);
      sims.push_back(est::to_l(aggregate(sp_partials, sp.size(), region, spec.grid)));
    }
    auto [upper, lower] = sim::envelopes(sims);
    result.diff_upper = est::diff_surface(result.l_hat, upper);
    result.upper_l = std::move(upper);
    result.lower_l = std::move(lower);
    result.telemetry.simulation_seconds = seconds_since(t0);
  }
  executor.collect_telemetry(result.telemetry);
  return result;
}

}  // namespace

RunResult run_job(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                  const JobSpec& spec, Executor& executor) {
  spec.grid.validate();
  if (points.size() < 2) throw std::invalid_argument("K estimation needs n >= 2");
  check_cache(spec.options, nullptr);
  if (executor.device() < 0) return run_job_tasks(points, region, spec, executor);
  const std::uint32_t W = executor.world(), rk = executor.rank();
  if (W > 1 && !executor.has_communicator() && !executor.has_hooks())
    throw std::invalid_argument(
        "executor with world > 1 needs an NCCL communicator or both exchange hooks");
  if (rk >= W) throw std::invalid_argument("rank must be < world");
  auto t0 = std::chrono::steady_clock::now();
  Ctx& c = context(executor.device());
  std::lock_guard<std::mutex> lk(c.mu);
  c.region(region);
  c.grid(spec.grid);
  const SoA p(points);
  const auto& g = spec.grid;
  const std::size_t bins = g.cells_s() * g.cells_t(), n = points.size();
  const int meth = method_code(spec.method);
  RunResult res;
  res.telemetry.plan_seconds = seconds_since(t0);
  res.telemetry.partition_count = 1;
  res.telemetry.partition_point_counts.assign(1, n);
  res.telemetry.cylinder_assignments = static_cast<std::uint64_t>(n) * (1 + spec.sims);
  res.telemetry.bytes_sent = 24ull * n;  // host -> device upload of the points
  stk_telemetry tel{};
  std::vector<double> up(bins), lo(bins), k(bins), l(bins), diff(bins);
  t0 = std::chrono::steady_clock::now();
  if (W <= 1) {
    // the observed pattern (estimation), then the realisations (simulation):
    // two device pipelines so the reference's two timings stay meaningful
    c.check(stk_run_job(c.h, p.x.data(), p.y.data(), p.t.data(), n, 0, spec.seed, meth,
                        k.data(), l.data(), nullptr, nullptr, nullptr, &tel));
    res.telemetry.estimation_seconds = seconds_since(t0);
    res.k_hat = surface(g, k.data(), est::SurfaceKind::K);
    res.l_hat = surface(g, l.data(), est::SurfaceKind::L);
    res.telemetry.bytes_received += 16ull * bins;
    if (spec.sims > 0) {
      t0 = std::chrono::steady_clock::now();
      const bool obs = meth != STK_METHOD_CSR;
      c.check(stk_simulate(c.h, obs ? p.x.data() : nullptr, obs ? p.y.data() : nullptr,
                           obs ? p.t.data() : nullptr, n, meth, spec.seed, 0, spec.sims,
                           nullptr, up.data(), lo.data(), &tel));
      res.upper_l = surface(g, up.data(), est::SurfaceKind::L);
      res.lower_l = surface(g, lo.data(), est::SurfaceKind::L);
      res.diff_upper = est::diff_surface(res.l_hat, *res.upper_l);
      res.telemetry.simulation_seconds = seconds_since(t0);
      res.telemetry.bytes_received += 16ull * bins;
    }
  } else if (executor.has_communicator()) {
    // one collective: this rank's shard + realisation block, exact NCCL
    // exchange and finalize inside the library
    c.check(stk_run_job_dist(c.h, p.x.data(), p.y.data(), p.t.data(), n, spec.sims, spec.seed,
                             meth, k.data(), l.data(), up.data(), lo.data(), diff.data(), &tel));
    res.telemetry.estimation_seconds = seconds_since(t0);
    res.k_hat = surface(g, k.data(), est::SurfaceKind::K);
    res.l_hat = surface(g, l.data(), est::SurfaceKind::L);
    if (spec.sims > 0) {
      res.upper_l = surface(g, up.data(), est::SurfaceKind::L);
      res.lower_l = surface(g, lo.data(), est::SurfaceKind::L);
      res.diff_upper = surface(g, diff.data(), est::SurfaceKind::Diff);
    }
    res.telemetry.bytes_sent += 8ull * bins * (6 + 2);  // NCCL all-reduce payloads
    res.telemetry.bytes_received += 8ull * bins * (6 + 2 + 5);
  } else {
    // one rank's share, then the two exact exchange steps through the hooks
    const std::uint32_t base = spec.sims / W, extra = spec.sims % W;
    const std::uint32_t r0 = rk * base + std::min(rk, extra);
    const std::uint32_t r1 = r0 + base + (rk < extra ? 1 : 0);
    std::vector<std::uint64_t> cnt(bins), hi(bins), lw(bins);
    std::fill(up.begin(), up.end(), -INFINITY);
    std::fill(lo.begin(), lo.end(), INFINITY);
    c.check(stk_run_job_shard(c.h, p.x.data(), p.y.data(), p.t.data(), n, rk, W, r0, r1,
                              spec.seed, meth, cnt.data(), hi.data(), lw.data(), up.data(),
                              lo.data(), &tel));
    // 128-bit sums as three 32/64-bit limbs so a uint64 SUM carries every bit
    std::vector<std::uint64_t> limbs(3 * bins);
    for (std::size_t b = 0; b < bins; ++b) {
      limbs[b] = hi[b];
      limbs[bins + b] = lw[b] >> 32;
      limbs[2 * bins + b] = lw[b] & 0xFFFFFFFFull;
    }
    executor.allreduce_sum_u64(limbs);
    for (std::size_t b = 0; b < bins; ++b) {
      const unsigned __int128 v = ((unsigned __int128)limbs[b] << 64) +
                                  ((unsigned __int128)limbs[bins + b] << 32) + limbs[2 * bins + b];
      hi[b] = (std::uint64_t)(v >> 64);
      lw[b] = (std::uint64_t)v;
    }
    c.check(stk_finalize(c.h, n, hi.data(), lw.data(), k.data(), l.data()));
    res.k_hat = surface(g, k.data(), est::SurfaceKind::K);
    res.l_hat = surface(g, l.data(), est::SurfaceKind::L);
    if (spec.sims > 0) {
      executor.allreduce_max_min(up, lo);
      res.upper_l = surface(g, up.data(), est::SurfaceKind::L);
      res.lower_l = surface(g, lo.data(), est::SurfaceKind::L);
      res.diff_upper = est::diff_surface(res.l_hat, *res.upper_l);
    }
    res.telemetry.estimation_seconds = seconds_since(t0);
  }
  res.theoretical = est::theoretical_surface(g);
  add_tel(res.telemetry, tel);
  executor.collect_telemetry(res.telemetry);
  return res;
}

double speedup_factor(double t_original, double t_optimized) {
  if (!(t_original > 0.0) || !(t_optimized > 0.0))
    throw std::invalid_argument("times must be > 0");
  return t_original / t_optimized;
}

double acceleration_factor(double t_standalone, double t_distributed) {
  return speedup_factor(t_standalone, t_distributed);
}

}  // namespace rt
}  // namespace stripley
