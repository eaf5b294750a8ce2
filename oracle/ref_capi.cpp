// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI over the *unmodified* reference sources (/root/reference/proj/core),
// compiled by oracle/Makefile with -Dstripley=stripley_ref into
// oracle/_ref/libstripley_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it, and only as the
// checker or the CPU baseline.  Every entry point forwards to the reference's
// own public API:
//   ref_estimate_surface -> est::estimate_surface   (core/src/estimator.cpp:116-186)
//   ref_run_job          -> rt::run_job + LocalExecutor (core/src/runtime.cpp:190-249)
//   ref_run_simulations  -> sim::run_simulations    (core/src/simulation.cpp:67-84)
//   ref_generate_cstr    -> sim::generate_cstr      (core/src/simulation.cpp:10-24)
//   ref_spatial_weight   -> edge::spatial_isotropic_weight (core/src/edge_correction.cpp:42-79)
//   ref_temporal_weight  -> edge::temporal_isotropic_weight (:81-86)
//   ref_pair_counts      -> per-bin counts from geom::spatial_distance /
//                           temporal_distance / est::bin_pair (the reference
//                           exposes only the total)
//   ref_pair_counts_indexed -> the same per-bin counts over index::STRTree::range_query
//                           (core/src/st_index.cpp:108-130), centers split over threads
//   ref_job_open / ref_job_pattern / ref_job_close -> rt::run_job's body split per
//                           pattern (core/src/runtime.cpp:190-249): plan once, then the
//                           observed pattern or realisation r (seed + r) through
//                           make_tasks -> executor.run -> aggregate -> to_l
//   ref_brute_force_k    -> testutil::brute_force_k (tests/helpers.hpp:95-139)
//   ref_*_ring / ref_*_points -> the reference test generators (tests/helpers.hpp:18-90)
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "helpers.hpp"
#include "stripley/estimator.hpp"
#include "stripley/rng.hpp"
#include "stripley/runtime.hpp"
#include "stripley/simulation.hpp"
#include "stripley/st_index.hpp"

using namespace stripley_ref;

namespace {

thread_local std::string g_err;

geom::StudyRegion make_region(const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1) {
  std::vector<geom::PlanarPoint> ring(nv);
  for (uint32_t i = 0; i < nv; ++i) ring[i] = {ring_xy[2 * i], ring_xy[2 * i + 1]};
  return geom::StudyRegion(std::move(ring), p0, p1);
}

est::DistanceGrid make_grid(const double* s, uint32_t cs, const int64_t* t, uint32_t ct) {
  est::DistanceGrid g;
  g.s_values.assign(s, s + cs);
  g.t_values.assign(t, t + ct);
  return g;
}

std::vector<geom::STPoint> make_points(const double* x, const double* y, const int64_t* t,
                                       uint64_t n) {
  std::vector<geom::STPoint> pts(n);
  for (uint64_t i = 0; i < n; ++i) pts[i] = geom::make_point(x[i], y[i], t[i]);
  return pts;
}

void flatten(const est::KSurface& s, double* out) {
  const size_t ct = s.grid.cells_t();
  for (size_t si = 0; si < s.grid.cells_s(); ++si)
    for (size_t ti = 0; ti < ct; ++ti) out[si * ct + ti] = s.values[si][ti];
}

void unpack_points(const std::vector<geom::STPoint>& pts, double* x, double* y, int64_t* t) {
  for (size_t i = 0; i < pts.size(); ++i) {
    x[i] = pts[i].x;
    y[i] = pts[i].y;
    t[i] = pts[i].start_time;
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_estimate_surface(const double* x, const double* y, const int64_t* t, uint64_t n,
                         const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                         const double* s_values, uint32_t cs, const int64_t* t_values,
                         uint32_t ct, int use_index, int use_cache, double* out_k,
                         uint64_t* out_in_threshold, uint64_t* out_comparisons) {
  return guarded([&] {
    const auto region = make_region(ring_xy, nv, p0, p1);
    const auto grid = make_grid(s_values, cs, t_values, ct);
    const auto pts = make_points(x, y, t, n);
    est::EstimatorOptions opt;
    opt.use_index = use_index != 0;
    opt.use_cache = use_cache != 0;
    est::EstimatorTelemetry tel;
    const auto k = est::estimate_surface(pts, region, grid, opt, nullptr, &tel);
    flatten(k, out_k);
    if (out_in_threshold) *out_in_threshold = tel.in_threshold_pairs;
    if (out_comparisons) *out_comparisons = tel.pair_comparisons;
  });
}

// method: 0 = CSR, 1 = bootstrap, 2 = permutation.  workers <= 0 -> hardware threads.
// Outputs (cs*ct each, row-major [s][t]); upper/lower/diff only written when sims > 0.
int ref_run_job(const double* x, const double* y, const int64_t* t, uint64_t n,
                const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct,
                uint32_t sims, uint64_t seed, int method, uint32_t partitions, int workers,
                int use_index, int use_cache, double* out_k, double* out_l,
                double* out_upper, double* out_lower, double* out_diff,
                uint64_t* out_in_threshold, uint64_t* out_comparisons, double* out_seconds) {
  return guarded([&] {
    const auto region = make_region(ring_xy, nv, p0, p1);
    const auto pts = make_points(x, y, t, n);
    rt::JobSpec spec;
    spec.grid = make_grid(s_values, cs, t_values, ct);
    spec.method = method == 0 ? sim::Method::Cstr
                  : method == 1 ? sim::Method::Bootstrap
                                : sim::Method::Permutation;
    spec.sims = sims;
    spec.seed = seed;
    spec.options.use_index = use_index != 0;
    spec.options.use_cache = use_cache != 0;
    spec.partitions = partitions;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    spec.workers = workers > 0 ? static_cast<uint32_t>(workers) : hw;
    spec.time_unit = geom::TimeUnit::Seconds;
    rt::LocalExecutor exec(spec.workers, region, spec.grid, spec.options);
    const auto r = rt::run_job(pts, region, spec, exec);
    flatten(r.k_hat, out_k);
    flatten(r.l_hat, out_l);
    if (sims > 0) {
      flatten(*r.upper_l, out_upper);
      flatten(*r.lower_l, out_lower);
      flatten(*r.diff_upper, out_diff);
    }
    if (out_in_threshold) *out_in_threshold = r.telemetry.in_threshold_pairs;
    if (out_comparisons) *out_comparisons = r.telemetry.pair_comparisons;
    if (out_seconds) {
      out_seconds[0] = r.telemetry.plan_seconds;
      out_seconds[1] = r.telemetry.estimation_seconds;
      out_seconds[2] = r.telemetry.simulation_seconds;
    }
  });
}

// m L-surfaces (m*cs*ct) via sim::run_simulations, method as above.
int ref_run_simulations(const double* x, const double* y, const int64_t* t, uint64_t n,
                        const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                        const double* s_values, uint32_t cs, const int64_t* t_values,
                        uint32_t ct, int method, uint32_t m, uint64_t base_seed,
                        int use_index, double* out_l_all) {
  return guarded([&] {
    const auto region = make_region(ring_xy, nv, p0, p1);
    const auto grid = make_grid(s_values, cs, t_values, ct);
    const auto pts = make_points(x, y, t, n);
    est::EstimatorOptions opt;
    opt.use_index = use_index != 0;
    const auto meth = method == 0 ? sim::Method::Cstr
                      : method == 1 ? sim::Method::Bootstrap
                                    : sim::Method::Permutation;
    const auto sims = sim::run_simulations(pts, region, grid, meth, m, base_seed, opt);
    for (uint32_t r = 0; r < m; ++r) flatten(sims[r], out_l_all + size_t(r) * cs * ct);
  });
}

int ref_generate_cstr(uint64_t n, const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                      uint64_t seed, double* x, double* y, int64_t* t) {
  return guarded([&] {
    const auto region = make_region(ring_xy, nv, p0, p1);
    unpack_points(sim::generate_cstr(n, region, seed), x, y, t);
  });
}

int ref_generate_bootstrap(const double* x, const double* y, const int64_t* t, uint64_t n,
                           uint64_t seed, double* ox, double* oy, int64_t* ot) {
  return guarded([&] {
    unpack_points(sim::generate_bootstrap(make_points(x, y, t, n), seed), ox, oy, ot);
  });
}

int ref_generate_permutation(const double* x, const double* y, const int64_t* t, uint64_t n,
                             uint64_t seed, double* ox, double* oy, int64_t* ot) {
  return guarded([&] {
    unpack_points(sim::generate_permutation(make_points(x, y, t, n), seed), ox, oy, ot);
  });
}

// Returns NaN and sets the error on a throw (center outside the region).
double ref_spatial_weight(double cx, double cy, double d, const double* ring_xy, uint32_t nv) {
  double w = 0.0;
  const int rc = guarded([&] {
    const auto region = make_region(ring_xy, nv, 0, 1);
    w = edge::spatial_isotropic_weight({cx, cy}, d, region);
  });
  return rc == 0 ? w : __builtin_nan("");
}

double ref_temporal_weight(int64_t center_t, int64_t u, int64_t p0, int64_t p1) {
  const double ring[8] = {0, 0, 1, 0, 1, 1, 0, 1};
  const auto region = make_region(ring, 4, p0, p1);
  return edge::temporal_isotropic_weight(center_t, u, region);
}

int ref_point_in_polygon(double px, double py, const double* ring_xy, uint32_t nv) {
  std::vector<geom::PlanarPoint> ring(nv);
  for (uint32_t i = 0; i < nv; ++i) ring[i] = {ring_xy[2 * i], ring_xy[2 * i + 1]};
  return geom::point_in_polygon({px, py}, ring) ? 1 : 0;
}

// Region validation through the reference StudyRegion constructor
// (core/src/geometry.cpp:110-136).  Returns 0 and writes area/duration, or 1
// with the reference's message in ref_last_error().
int ref_region_info(const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                    double* area, int64_t* duration) {
  return guarded([&] {
    const auto region = make_region(ring_xy, nv, p0, p1);
    *area = region.area();
    *duration = region.duration();
  });
}

// Per-bin in-threshold ordered-pair counts (cs*ct, non-cumulative), built on
// the reference's own distance and binning functions.
int ref_pair_counts(const double* x, const double* y, const int64_t* t, uint64_t n,
                    const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct,
                    uint64_t* out_counts) {
  return guarded([&] {
    const auto grid = make_grid(s_values, cs, t_values, ct);
    const auto pts = make_points(x, y, t, n);
    std::memset(out_counts, 0, sizeof(uint64_t) * cs * ct);
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t j = 0; j < n; ++j) {
        if (i == j) continue;
        const double d = geom::spatial_distance(pts[i], pts[j]);
        const int64_t u = geom::temporal_distance(pts[i], pts[j]);
        const auto bin = est::bin_pair(grid, d, u);
        if (bin) ++out_counts[bin->first * ct + bin->second];
      }
  });
}

// Per-bin counts as above, over the reference's own STR R-tree: every center's
// cylinder query (estimator.cpp:150-167) with centers split round-robin over
// threads (the tree is immutable and safe for concurrent queries,
// st_index.hpp:26-27).  Test infrastructure for patterns too large for the
// O(n^2) loop.
int ref_pair_counts_indexed(const double* x, const double* y, const int64_t* t, uint64_t n,
                            const double* s_values, uint32_t cs, const int64_t* t_values,
                            uint32_t ct, int threads, uint64_t* out_counts,
                            uint64_t* out_in_threshold) {
  return guarded([&] {
    const auto grid = make_grid(s_values, cs, t_values, ct);
    grid.validate();
    const auto pts = make_points(x, y, t, n);
    std::vector<index::IndexedPoint> indexed(n);
    for (uint64_t i = 0; i < n; ++i) indexed[i] = {pts[i], static_cast<uint32_t>(i)};
    const auto tree = index::STRTree::build(std::move(indexed), 16);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = threads > 0 ? static_cast<unsigned>(threads) : hw;
    std::vector<std::vector<uint64_t>> part(nt, std::vector<uint64_t>(size_t(cs) * ct, 0));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nt; ++w)
      pool.emplace_back([&, w] {
        geom::STCylinder cyl;
        cyl.spatial_radius = grid.s_max();
        cyl.temporal_radius = grid.t_max();
        auto& cnt = part[w];
        for (uint64_t i = w; i < n; i += nt) {
          cyl.center = pts[i];
          for (const auto& item : tree.range_query(cyl)) {
            if (item.record_index == i) continue;
            const double d = geom::spatial_distance(pts[i], item.pt);
            const int64_t u = geom::temporal_distance(pts[i], item.pt);
            const auto bin = est::bin_pair(grid, d, u);
            if (bin) ++cnt[bin->first * ct + bin->second];
          }
        }
      });
    for (auto& th : pool) th.join();
    uint64_t total = 0;
    for (size_t b = 0; b < size_t(cs) * ct; ++b) {
      uint64_t c = 0;
      for (unsigned w = 0; w < nt; ++w) c += part[w][b];
      out_counts[b] = c;
      total += c;
    }
    if (out_in_threshold) *out_in_threshold = total;
  });
}

// rt::run_job (core/src/runtime.cpp:190-249) split per pattern so a caller can
// time or check one pattern at a time: ref_job_open validates and plans once
// (build_plan on the observed points, as run_job does); ref_job_pattern(which)
// runs the observed pattern (which < 0: make_tasks -> executor.run(false) ->
// aggregate -> to_l) or realisation r = which (sim::generate(method, n, points,
// region, seed + r) -> make_tasks -> executor.run(true) -> aggregate -> to_l),
// the exact loop body of run_job.
struct RefJob {
  geom::StudyRegion region;
  std::vector<geom::STPoint> points;
  rt::JobSpec spec;
  rt::JobPlan plan;
  std::unique_ptr<rt::LocalExecutor> exec;
  RefJob(geom::StudyRegion r) : region(std::move(r)) {}
};

void* ref_job_open(const double* x, const double* y, const int64_t* t, uint64_t n,
                   const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                   const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct,
                   uint64_t seed, int method, uint32_t partitions, int workers, int use_index,
                   int use_cache) {
  RefJob* job = nullptr;
  const int rc = guarded([&] {
    auto j = std::make_unique<RefJob>(make_region(ring_xy, nv, p0, p1));
    j->points = make_points(x, y, t, n);
    auto& spec = j->spec;
    spec.grid = make_grid(s_values, cs, t_values, ct);
    spec.method = method == 0 ? sim::Method::Cstr
                  : method == 1 ? sim::Method::Bootstrap
                                : sim::Method::Permutation;
    spec.seed = seed;
    spec.options.use_index = use_index != 0;
    spec.options.use_cache = use_cache != 0;
    spec.partitions = partitions;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    spec.workers = workers > 0 ? static_cast<uint32_t>(workers) : hw;
    spec.time_unit = geom::TimeUnit::Seconds;
    spec.grid.validate();
    if (j->points.size() < 2) throw std::invalid_argument("K estimation needs n >= 2");
    for (const auto& p : j->points)
      if (!j->region.contains(p))
        throw std::invalid_argument("point outside study region or period");
    j->plan = rt::build_plan(j->points, j->region, spec);
    j->exec = std::make_unique<rt::LocalExecutor>(spec.workers, j->region, spec.grid,
                                                  spec.options);
    j->exec->broadcast_plan(j->plan);
    job = j.release();
  });
  return rc == 0 ? job : nullptr;
}

int ref_job_pattern(void* handle, int64_t which, double* out_k, double* out_l,
                    uint64_t* out_in_threshold, uint64_t* out_comparisons) {
  return guarded([&] {
    auto* j = static_cast<RefJob*>(handle);
    const auto& spec = j->spec;
    std::vector<geom::STPoint> sim_points;
    const bool sim_phase = which >= 0;
    if (sim_phase)
      sim_points = sim::generate(spec.method, j->points.size(), j->points, j->region,
                                 spec.seed + static_cast<uint64_t>(which));
    const auto& pts = sim_phase ? sim_points : j->points;
    const auto tasks = rt::make_tasks(j->plan, pts, spec, nullptr);
    const auto partials = j->exec->run(tasks, sim_phase);
    uint64_t in_thr = 0, comps = 0;
    for (const auto& p : partials) {
      in_thr += p.in_threshold_pairs;
      comps += p.pair_comparisons;
    }
    const auto k = rt::aggregate(partials, pts.size(), j->region, spec.grid);
    if (out_k) flatten(k, out_k);
    if (out_l) flatten(est::to_l(k), out_l);
    if (out_in_threshold) *out_in_threshold = in_thr;
    if (out_comparisons) *out_comparisons = comps;
  });
}

void ref_job_close(void* handle) { delete static_cast<RefJob*>(handle); }

int ref_brute_force_k(const double* x, const double* y, const int64_t* t, uint64_t n,
                      const double* ring_xy, uint32_t nv, int64_t p0, int64_t p1,
                      const double* s_values, uint32_t cs, const int64_t* t_values,
                      uint32_t ct, double* out_k) {
  return guarded([&] {
    const auto region = make_region(ring_xy, nv, p0, p1);
    const auto grid = make_grid(s_values, cs, t_values, ct);
    flatten(testutil::brute_force_k(make_points(x, y, t, n), region, grid), out_k);
  });
}

int ref_regular_grid(double s_step, double s_max, int64_t t_step, int64_t t_max,
                     double* s_out, uint32_t* cs, int64_t* t_out, uint32_t* ct,
                     uint32_t capacity) {
  return guarded([&] {
    const auto g = est::DistanceGrid::regular(s_step, s_max, t_step, t_max);
    if (g.s_values.size() > capacity || g.t_values.size() > capacity)
      throw std::runtime_error("grid capacity exceeded");
    *cs = static_cast<uint32_t>(g.s_values.size());
    *ct = static_cast<uint32_t>(g.t_values.size());
    std::copy(g.s_values.begin(), g.s_values.end(), s_out);
    std::copy(g.t_values.begin(), g.t_values.end(), t_out);
  });
}

// Reference test generators, each on a fresh rng::Engine(seed).
int ref_random_convex_ring(uint64_t seed, double rx, double ry, uint32_t vertices,
                           double* out_xy) {
  return guarded([&] {
    rng::Engine eng(seed);
    const auto ring = testutil::random_convex_ring(eng, rx, ry, vertices);
    for (size_t i = 0; i < ring.size(); ++i) {
      out_xy[2 * i] = ring[i].x;
      out_xy[2 * i + 1] = ring[i].y;
    }
  });
}

int ref_random_star_ring(uint64_t seed, double radius, uint32_t vertices, double* out_xy) {
  return guarded([&] {
    rng::Engine eng(seed);
    const auto ring = testutil::random_star_ring(eng, radius, vertices);
    for (size_t i = 0; i < ring.size(); ++i) {
      out_xy[2 * i] = ring[i].x;
      out_xy[2 * i + 1] = ring[i].y;
    }
  });
}

int ref_uniform_points(uint64_t seed, const double* ring_xy, uint32_t nv, int64_t p0,
                       int64_t p1, uint64_t n, double* x, double* y, int64_t* t) {
  return guarded([&] {
    rng::Engine eng(seed);
    const auto region = make_region(ring_xy, nv, p0, p1);
    unpack_points(testutil::uniform_points(eng, region, n), x, y, t);
  });
}

int ref_clustered_points(uint64_t seed, const double* ring_xy, uint32_t nv, int64_t p0,
                         int64_t p1, uint64_t n, uint32_t clusters, double sigma_s,
                         double sigma_t, double* x, double* y, int64_t* t) {
  return guarded([&] {
    rng::Engine eng(seed);
    const auto region = make_region(ring_xy, nv, p0, p1);
    unpack_points(testutil::clustered_points(eng, region, n, clusters, sigma_s, sigma_t), x,
                  y, t);
  });
}

// Raw std::mt19937_64 outputs through the reference's rng::Engine.
void ref_mt_outputs(uint64_t seed, uint64_t count, uint64_t* out) {
  rng::Engine eng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = eng.next_u64();
}

}  // extern "C"
