// stripley_gpu.hpp — the reference's C++ API for the space-time K pair path,
// backed by the B200 library (libstk.so, C ABI in stk.h).
//
// Drop-in at the source level for the hot path: the namespaces, type names,
// member names and function signatures follow the reference headers
// (paths relative to /root/reference/proj/core/include/stripley/):
//   geom::STPoint / make_point / PlanarPoint / STEnvelope / StudyRegion  geometry.hpp:9-120
//   est::DistanceGrid / KSurface / EstimatorOptions / EstimatorTelemetry  estimator.hpp:15-51
//   est::intensity / theoretical_k / k_to_l / theoretical_surface / to_l
//   est::bin_pair / estimate_surface / diff_surface                       estimator.hpp:83-114
//   cache::WeightCache (tolerance-0 semantics)                            weight_cache.hpp:39-129
//   sim::Method / generate_cstr / generate_bootstrap / generate_permutation
//   sim::run_simulations / envelopes                                      simulation.hpp:14-47
//   rt::JobSpec / RunTelemetry / RunResult / Executor / run_job           runtime.hpp:21-153
// Errors: std::invalid_argument with the reference's messages; device
// failures as std::runtime_error.  There is no CPU fallback.
//
// What differs, by design: rt::Executor is the device plug-in point (the
// reference's KDB plan / TaskData decomposition is replaced by the on-device
// grid), so run_job takes a DeviceExecutor; multi-process runs supply two
// exact reduction hooks (see DeviceExecutor).
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

namespace stripley {

namespace geom {

enum class TimeUnit : std::uint8_t { Seconds = 0, Minutes = 1, Hours = 2, Days = 3, Months = 4 };

struct STPoint {
  double x = 0.0;
  double y = 0.0;
  std::uint32_t overlap_count = 1;
  std::int64_t start_time = 0;
  std::int64_t end_time = 0;
  std::int32_t zone_id = 0;
  bool operator==(const STPoint&) const = default;
};

inline STPoint make_point(double x, double y, std::int64_t t) { return STPoint{x, y, 1, t, t, 0}; }

struct PlanarPoint {
  double x = 0.0;
  double y = 0.0;
};

struct STEnvelope {
  double x_min = 0.0, x_max = 0.0;
  double y_min = 0.0, y_max = 0.0;
  std::int64_t t_min = 0, t_max = 0;
  std::int32_t zone_id = 0;
  std::int64_t envelope_id = 0;
};

/// Boundary-inclusive even-odd test (geometry.cpp:81-97), host side.
bool point_in_polygon(const PlanarPoint& pt, const std::vector<PlanarPoint>& ring);

/// Simple polygon + study period; validated like the reference constructor.
class StudyRegion {
 public:
  StudyRegion(std::vector<PlanarPoint> ring, std::int64_t period_start, std::int64_t period_end);
  const std::vector<PlanarPoint>& boundary() const { return ring_; }
  std::int64_t period_start() const { return period_start_; }
  std::int64_t period_end() const { return period_end_; }
  double area() const { return area_; }
  std::int64_t duration() const { return duration_; }
  bool contains(const PlanarPoint& pt) const { return point_in_polygon(pt, ring_); }
  bool contains(const STPoint& p) const {
    return point_in_polygon({p.x, p.y}, ring_) && p.start_time >= period_start_ &&
           p.start_time <= period_end_;
  }
  STEnvelope bounding_envelope() const;

 private:
  std::vector<PlanarPoint> ring_;
  std::int64_t period_start_;
  std::int64_t period_end_;
  double area_;
  std::int64_t duration_;
};

}  // namespace geom

namespace cache {
/// At tolerance 0 the reference cache never changes results; the device
/// recomputes weights per center.  Nonzero tolerances are rejected.
class WeightCache {
 public:
  WeightCache(double coord_tolerance = 0.0, double dist_tolerance = 0.0)
      : coord_tol_(coord_tolerance), dist_tol_(dist_tolerance) {}
  void freeze() { frozen_ = true; }
  bool frozen() const { return frozen_; }
  double coord_tolerance() const { return coord_tol_; }
  double dist_tolerance() const { return dist_tol_; }

 private:
  double coord_tol_, dist_tol_;
  bool frozen_ = false;
};
}  // namespace cache

namespace est {

struct DistanceGrid {
  std::vector<double> s_values;
  std::vector<std::int64_t> t_values;

  void validate() const;
  double s_max() const { return s_values.back(); }
  std::int64_t t_max() const { return t_values.back(); }
  std::size_t cells_s() const { return s_values.size(); }
  std::size_t cells_t() const { return t_values.size(); }
  static DistanceGrid regular(double s_step, double s_max, std::int64_t t_step, std::int64_t t_max);
  bool operator==(const DistanceGrid&) const = default;
};

enum class SurfaceKind { K, L, Diff };

struct KSurface {
  DistanceGrid grid;
  std::vector<std::vector<double>> values;  // [s index][t index]
  SurfaceKind kind = SurfaceKind::K;
};

struct EstimatorOptions {
  bool use_index = false;
  bool use_cache = false;
  double coord_tolerance = 0.0;
  double dist_tolerance = 0.0;
  std::uint32_t node_capacity = 16;
};

struct EstimatorTelemetry {
  std::uint64_t pair_comparisons = 0;
  std::uint64_t in_threshold_pairs = 0;
  double index_build_seconds = 0.0;
};

double intensity(std::size_t n, const geom::StudyRegion& region);
double theoretical_k(double s, double t);
double k_to_l(double k, double s, double t);
KSurface theoretical_surface(const DistanceGrid& grid);
KSurface to_l(const KSurface& k_surface);
std::optional<std::pair<std::size_t, std::size_t>> bin_pair(const DistanceGrid& grid, double d,
                                                            std::int64_t u);

/// Full space-time K on the device (grid build, pair kernel, finalize).
KSurface estimate_surface(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                          const DistanceGrid& grid, const EstimatorOptions& options,
                          cache::WeightCache* weight_cache = nullptr,
                          EstimatorTelemetry* telemetry = nullptr);

KSurface diff_surface(const KSurface& estimated_l, const KSurface& upper_l);

}  // namespace est

namespace sim {

enum class Method { Cstr, Bootstrap, Permutation };

std::vector<geom::STPoint> generate_cstr(std::size_t n, const geom::StudyRegion& region,
                                         std::uint64_t seed);
std::vector<geom::STPoint> generate_bootstrap(std::span<const geom::STPoint> points,
                                              std::uint64_t seed);
std::vector<geom::STPoint> generate_permutation(std::span<const geom::STPoint> points,
                                                std::uint64_t seed);
std::vector<geom::STPoint> generate(Method method, std::size_t n,
                                    std::span<const geom::STPoint> observed,
                                    const geom::StudyRegion& region, std::uint64_t seed);

std::vector<est::KSurface> run_simulations(std::span<const geom::STPoint> points,
                                           const geom::StudyRegion& region,
                                           const est::DistanceGrid& grid, Method method,
                                           std::size_t m, std::uint64_t base_seed,
                                           const est::EstimatorOptions& options,
                                           cache::WeightCache* weight_cache = nullptr);

std::pair<est::KSurface, est::KSurface> envelopes(std::span<const est::KSurface> sims);

}  // namespace sim

namespace rt {

enum class PartitionerChoice { Kdb, Hash };
enum class Mode { Local, Distributed };

struct JobSpec {
  est::DistanceGrid grid;
  sim::Method method = sim::Method::Cstr;
  std::uint32_t sims = 99;
  std::uint64_t seed = 1;
  est::EstimatorOptions options;
  PartitionerChoice partitioner = PartitionerChoice::Kdb;  // accepted, no effect on device
  std::uint32_t partitions = 1;                              // accepted, no effect on device
  std::uint32_t workers = 1;                                 // accepted, no effect on device
  Mode mode = Mode::Local;
  double sample_fraction = 0.01;
  geom::TimeUnit time_unit = geom::TimeUnit::Days;
};

struct RunTelemetry {
  std::uint64_t pair_comparisons = 0;
  std::uint64_t in_threshold_pairs = 0;
  std::uint64_t exact_path_pairs = 0;
  double plan_seconds = 0.0;
  double estimation_seconds = 0.0;
  double simulation_seconds = 0.0;
  double device_ms = 0.0;
  double pair_kernel_ms = 0.0;
};

struct RunResult {
  est::KSurface k_hat;
  est::KSurface l_hat;
  est::KSurface theoretical;
  std::optional<est::KSurface> upper_l;
  std::optional<est::KSurface> lower_l;
  std::optional<est::KSurface> diff_upper;
  RunTelemetry telemetry;
};

/// The plug-in point of run_job (runtime.hpp:108-117 role).  One executor
/// drives one GPU.  For one process per GPU (rank of world), the two exact
/// exchange steps are supplied by the caller (e.g. NCCL all-reduces):
///   allreduce_sum_u64: in-place SUM of a uint64 array across ranks
///                      (observed pattern's exact per-bin partials, as limbs),
///   allreduce_max_min: in-place MAX of `upper` and MIN of `lower`.
class Executor {
 public:
  virtual ~Executor() = default;
  virtual int device() const = 0;
  virtual std::uint32_t rank() const { return 0; }
  virtual std::uint32_t world() const { return 1; }
  virtual void allreduce_sum_u64(std::vector<std::uint64_t>& v) const { (void)v; }
  virtual void allreduce_max_min(std::vector<double>& upper, std::vector<double>& lower) const {
    (void)upper;
    (void)lower;
  }
};

class DeviceExecutor : public Executor {
 public:
  explicit DeviceExecutor(int device = 0, std::uint32_t rank = 0, std::uint32_t world = 1,
                          std::function<void(std::vector<std::uint64_t>&)> sum_u64 = {},
                          std::function<void(std::vector<double>&, std::vector<double>&)>
                              max_min = {})
      : device_(device), rank_(rank), world_(world), sum_(std::move(sum_u64)),
        maxmin_(std::move(max_min)) {}
  int device() const override { return device_; }
  std::uint32_t rank() const override { return rank_; }
  std::uint32_t world() const override { return world_; }
  void allreduce_sum_u64(std::vector<std::uint64_t>& v) const override {
    if (sum_) sum_(v);
  }
  void allreduce_max_min(std::vector<double>& u, std::vector<double>& l) const override {
    if (maxmin_) maxmin_(u, l);
  }

 private:
  int device_;
  std::uint32_t rank_, world_;
  std::function<void(std::vector<std::uint64_t>&)> sum_;
  std::function<void(std::vector<double>&, std::vector<double>&)> maxmin_;
};

RunResult run_job(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                  const JobSpec& spec, Executor& executor);

}  // namespace rt
}  // namespace stripley
