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
// rt::Executor keeps the reference's virtuals (broadcast_plan / run /
// collect_telemetry) and rt::LocalExecutor its constructor, so a program
// written against runtime.hpp compiles unchanged; an executor that names a GPU
// makes run_job take the fused device pipeline (the KDB plan / TaskData
// decomposition is replaced by the on-device grid), and task lists given to
// run() execute on the device.  Multi-GPU: DeviceExecutor with an NCCL
// communicator inside the library (or two exact reduction hooks).
#pragma once

#include <array>
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

/// geometry.hpp:62-69
struct STCylinder {
  STPoint center;
  double spatial_radius = 0.0;
  std::int64_t temporal_radius = 0;
  TimeUnit temporal_unit = TimeUnit::Days;
  bool operator==(const STCylinder&) const = default;
};

double spatial_distance(const STPoint& p, const STPoint& q);
std::int64_t temporal_distance(const STPoint& p, const STPoint& q);
bool within_cylinder(const STCylinder& cyl, const STPoint& p);

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

namespace index {
/// st_index.hpp:12-19: a point plus the record index that identifies it.
struct IndexedPoint {
  geom::STPoint pt;
  std::uint32_t record_index = 0;
  bool operator==(const IndexedPoint&) const = default;
};
}  // namespace index

namespace cache {
/// weight_cache.hpp:13-25
struct TableStats {
  std::uint64_t hits = 0;
  std::uint64_t misses = 0;
  std::uint64_t insertions = 0;
  TableStats& operator+=(const TableStats& o) {
    hits += o.hits;
    misses += o.misses;
    insertions += o.insertions;
    return *this;
  }
};

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

/// runtime.hpp:35-38
struct IndexedCylinder {
  geom::STCylinder cyl;
  std::uint32_t center_index = 0;
};

/// One unit of work (runtime.hpp:40-46): a partition's points plus every
/// query cylinder assigned to it.
struct TaskData {
  std::uint32_t task_id = 0;
  std::vector<index::IndexedPoint> points;
  std::vector<IndexedCylinder> cylinders;
};

/// runtime.hpp:48-57
struct PartialResult {
  std::uint32_t task_id = 0;
  std::uint32_t worker_id = 0;
  std::vector<double> histogram;  // cells_s * cells_t, pre-cumulative
  std::uint64_t pair_comparisons = 0;
  std::uint64_t in_threshold_pairs = 0;
  cache::TableStats spatial_cache;
  cache::TableStats temporal_cache;
};

/// runtime.hpp:59-72, plus device counters.  On the device: one "partition"
/// per pattern (the uniform grid replaces the KDB plan), so partition_count
/// is 1 and cylinder_assignments counts one cylinder per point and pattern;
/// the weight caches are replaced by per-center recomputation (stats stay 0);
/// bytes_sent / bytes_received count host<->device and NCCL exchange bytes.
struct RunTelemetry {
  std::uint64_t pair_comparisons = 0;
  std::uint64_t in_threshold_pairs = 0;
  std::uint64_t cylinder_assignments = 0;
  std::uint64_t partition_count = 0;
  std::vector<std::uint64_t> partition_point_counts;
  cache::TableStats spatial_cache;
  cache::TableStats temporal_cache;
  std::uint64_t bytes_sent = 0;
  std::uint64_t bytes_received = 0;
  double plan_seconds = 0.0;
  double estimation_seconds = 0.0;
  double simulation_seconds = 0.0;
  // device extras
  std::uint64_t exact_path_pairs = 0;
  double device_ms = 0.0;
  double pair_kernel_ms = 0.0;
};

/// runtime.hpp:74-84.  The device's uniform space-time grid replaces the
/// KDB partitioner (out of scope: it never changes results), so a plan has
/// one partition holding every point and every cylinder.
struct JobPlan {
  PartitionerChoice choice = PartitionerChoice::Kdb;
  std::uint32_t partitions = 1;
  std::uint32_t locate(const geom::STPoint& p, std::uint32_t record_index) const {
    (void)p;
    (void)record_index;
    return 0;
  }
  std::vector<std::uint32_t> assign(const geom::STCylinder& cyl) const {
    (void)cyl;
    return {0};
  }
};

JobPlan build_plan(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                   const JobSpec& spec);

std::vector<TaskData> make_tasks(const JobPlan& plan, std::span<const geom::STPoint> dataset,
                                 const JobSpec& spec, std::uint64_t* redundancy_out = nullptr);

/// rt::execute_task on the device (stk_task_histogram).
PartialResult execute_task(const TaskData& task, const geom::StudyRegion& region,
                           const est::DistanceGrid& grid, const est::EstimatorOptions& options,
                           cache::WeightCache* weight_cache = nullptr);

/// Elementwise-sum partial histograms in task order, cumulative-sum, scale
/// (runtime.cpp:119-136).
est::KSurface aggregate(std::span<const PartialResult> partials, std::size_t n,
                        const geom::StudyRegion& region, const est::DistanceGrid& grid);

/// Task execution backend (runtime.hpp:106-117).  The reference's interface is
/// kept verbatim; device() is this framework's extension: an executor that
/// names a GPU (LocalExecutor, DeviceExecutor) lets run_job take the fused
/// device pipeline, any other executor is driven through run() with tasks as
/// the reference does.
class Executor {
 public:
  virtual ~Executor() = default;
  virtual void broadcast_plan(const JobPlan& plan) { (void)plan; }
  virtual std::vector<PartialResult> run(const std::vector<TaskData>& tasks,
                                         bool simulation_phase) = 0;
  virtual void collect_telemetry(RunTelemetry& out) const = 0;
  // ---- device extension
  virtual int device() const { return -1; }
  virtual std::uint32_t rank() const { return 0; }
  virtual std::uint32_t world() const { return 1; }
  /// world > 1: the context of device() holds an NCCL communicator (stk_comm_init)
  virtual bool has_communicator() const { return false; }
  /// world > 1 without a communicator: caller-supplied exact exchange hooks
  virtual bool has_hooks() const { return false; }
  virtual void allreduce_sum_u64(std::vector<std::uint64_t>& v) const { (void)v; }
  virtual void allreduce_max_min(std::vector<double>& upper, std::vector<double>& lower) const {
    (void)upper;
    (void)lower;
  }
};

/// The reference's in-process executor (runtime.hpp:119-136), on the GPU:
/// `workers` is recorded (task t reports worker t mod workers) but the device
/// replaces the thread pool; tasks run through execute_task on the device
/// (STK_DEVICE, default 0).
class LocalExecutor : public Executor {
 public:
  LocalExecutor(std::uint32_t workers, const geom::StudyRegion& region,
                const est::DistanceGrid& grid, const est::EstimatorOptions& options);

  std::vector<PartialResult> run(const std::vector<TaskData>& tasks,
                                 bool simulation_phase) override;
  void collect_telemetry(RunTelemetry& out) const override;
  int device() const override { return device_; }

 private:
  std::uint32_t workers_;
  const geom::StudyRegion& region_;
  est::DistanceGrid grid_;
  est::EstimatorOptions options_;
  int device_;
};

/// One GPU per process.  world > 1 needs the exact exchange: either an NCCL
/// communicator inside the library (the constructor taking the unique id of
/// stk_comm_unique_id, distributed from rank 0 by any means) -- the
/// DistributedExecutor replacement (distributed.cpp:116-245) -- or two
/// caller-supplied hooks (in-place uint64 SUM of the exact limbs; in-place MAX
/// of upper and MIN of lower).  Constructing world > 1 with neither throws.
class DeviceExecutor : public Executor {
 public:
  using SumHook = std::function<void(std::vector<std::uint64_t>&)>;
  using MaxMinHook = std::function<void(std::vector<double>&, std::vector<double>&)>;
  explicit DeviceExecutor(int device = 0, std::uint32_t rank = 0, std::uint32_t world = 1,
                          SumHook sum_u64 = {}, MaxMinHook max_min = {});
  DeviceExecutor(int device, std::uint32_t rank, std::uint32_t world,
                 const std::array<unsigned char, 128>& nccl_unique_id);
  /// rank 0's side: a fresh NCCL unique id (stk_comm_unique_id)
  static std::array<unsigned char, 128> nccl_unique_id();

  std::vector<PartialResult> run(const std::vector<TaskData>& tasks,
                                 bool simulation_phase) override;
  void collect_telemetry(RunTelemetry& out) const override { (void)out; }
  int device() const override { return device_; }
  std::uint32_t rank() const override { return rank_; }
  std::uint32_t world() const override { return world_; }
  bool has_communicator() const override { return comm_; }
  bool has_hooks() const override { return sum_ && maxmin_; }
  void allreduce_sum_u64(std::vector<std::uint64_t>& v) const override {
    if (sum_) sum_(v);
  }
  void allreduce_max_min(std::vector<double>& u, std::vector<double>& l) const override {
    if (maxmin_) maxmin_(u, l);
  }

 private:
  int device_;
  std::uint32_t rank_, world_;
  SumHook sum_;
  MaxMinHook maxmin_;
  bool comm_ = false;
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

/// Full pipeline: plan, estimate, simulate, envelope (runtime.cpp:190-249).
/// Simulation replicate r uses seed spec.seed + r.
RunResult run_job(std::span<const geom::STPoint> points, const geom::StudyRegion& region,
                  const JobSpec& spec, Executor& executor);

/// Performance ratios; both operands must be > 0 (runtime.hpp:155-157).
double speedup_factor(double t_original, double t_optimized);
double acceleration_factor(double t_standalone, double t_distributed);

}  // namespace rt
}  // namespace stripley
