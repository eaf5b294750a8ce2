// A program written against the reference's runtime interface
// (/root/reference/proj/core/include/stripley/runtime.hpp:106-157), compiled
// unchanged against this framework's drop-in headers (include/stripley/).
// It uses the reference's LocalExecutor constructor, a user-defined Executor
// plug-in that implements the three virtuals with rt::execute_task (the way a
// reference backend does), run_job with both, RunTelemetry, speedup_factor.
//   reference_program <points.bin> <ring.bin> p0 p1 <grid.bin> sims seed
// (binary layouts as tests/cpp/test_api.cpp); prints one JSON object.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "stripley/runtime.hpp"
#include "stripley/simulation.hpp"

using namespace stripley;

namespace {

/// A reference-style executor plug-in: tasks run one after the other through
/// rt::execute_task; it counts plans and tasks like a backend's telemetry.
class SerialExecutor : public rt::Executor {
 public:
  SerialExecutor(const geom::StudyRegion& region, const est::DistanceGrid& grid,
                 const est::EstimatorOptions& options)
      : region_(region), grid_(grid), options_(options) {}

  void broadcast_plan(const rt::JobPlan& plan) override { plans_ += plan.partitions; }

  std::vector<rt::PartialResult> run(const std::vector<rt::TaskData>& tasks,
                                     bool simulation_phase) override {
    std::vector<rt::PartialResult> out;
    for (const auto& t : tasks) {
      out.push_back(rt::execute_task(t, region_, grid_, options_));
      out.back().worker_id = simulation_phase ? 1 : 0;
      ++tasks_;
    }
    return out;
  }

  void collect_telemetry(rt::RunTelemetry& out) const override {
    out.bytes_sent += tasks_;  // a backend's counters land in the run telemetry
    out.bytes_received += plans_;
  }

 private:
  const geom::StudyRegion& region_;
  est::DistanceGrid grid_;
  est::EstimatorOptions options_;
  std::uint64_t plans_ = 0, tasks_ = 0;
};

template <class T>
std::vector<T> read_vec(std::ifstream& f, std::uint64_t n) {
  std::vector<T> v(n);
  f.read(reinterpret_cast<char*>(v.data()), sizeof(T) * n);
  return v;
}

void dump(const char* name, const est::KSurface& s, bool comma = true) {
  std::printf("\"%s\": [", name);
  bool first = true;
  for (const auto& row : s.values)
    for (double v : row) {
      std::printf(first ? "%.17g" : ", %.17g", v);
      first = false;
    }
  std::printf("]%s", comma ? ", " : "");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 8) return 2;
  std::ifstream pf(argv[1], std::ios::binary), rf(argv[2], std::ios::binary),
      gf(argv[5], std::ios::binary);
  std::uint64_t n = 0, nv = 0, cs = 0, ct = 0;
  pf.read(reinterpret_cast<char*>(&n), 8);
  const auto x = read_vec<double>(pf, n), y = read_vec<double>(pf, n);
  const auto t = read_vec<std::int64_t>(pf, n);
  rf.read(reinterpret_cast<char*>(&nv), 8);
  const auto ring_xy = read_vec<double>(rf, nv);
  gf.read(reinterpret_cast<char*>(&cs), 8);
  const auto s_values = read_vec<double>(gf, cs);
  gf.read(reinterpret_cast<char*>(&ct), 8);
  const auto t_values = read_vec<std::int64_t>(gf, ct);

  std::vector<geom::PlanarPoint> ring;
  for (std::uint64_t i = 0; i + 1 < nv; i += 2) ring.push_back({ring_xy[i], ring_xy[i + 1]});
  const geom::StudyRegion region(ring, std::stoll(argv[3]), std::stoll(argv[4]));
  std::vector<geom::STPoint> points;
  for (std::uint64_t i = 0; i < n; ++i) points.push_back(geom::make_point(x[i], y[i], t[i]));

  rt::JobSpec spec;
  spec.grid.s_values = s_values;
  spec.grid.t_values = t_values;
  spec.sims = static_cast<std::uint32_t>(std::stoul(argv[6]));
  spec.seed = std::stoull(argv[7]);
  spec.partitions = 8;
  spec.workers = 4;
  spec.options.use_index = true;
  spec.options.use_cache = true;
  spec.time_unit = geom::TimeUnit::Days;

  try {
    rt::LocalExecutor exec(spec.workers, region, spec.grid, spec.options);
    const rt::RunResult r = rt::run_job(points, region, spec, exec);
    SerialExecutor plug(region, spec.grid, spec.options);
    const rt::RunResult q = rt::run_job(points, region, spec, plug);
    // the executor's own task path on the observed pattern
    const auto plan = rt::build_plan(points, region, spec);
    const auto tasks = rt::make_tasks(plan, points, spec);
    const auto partials = exec.run(tasks, false);
    const auto k_tasks = rt::aggregate(partials, points.size(), region, spec.grid);
    const double ratio = rt::speedup_factor(2.0, 0.5);
    std::printf("{");
    dump("k", r.k_hat);
    dump("l", r.l_hat);
    dump("upper", *r.upper_l);
    dump("lower", *r.lower_l);
    dump("diff", *r.diff_upper);
    dump("k_plugin", q.k_hat);
    dump("upper_plugin", *q.upper_l);
    dump("k_tasks", k_tasks);
    std::printf("\"in_threshold\": %llu, \"in_threshold_plugin\": %llu, ",
                (unsigned long long)r.telemetry.in_threshold_pairs,
                (unsigned long long)q.telemetry.in_threshold_pairs);
    std::printf("\"partition_count\": %llu, \"cylinder_assignments\": %llu, ",
                (unsigned long long)r.telemetry.partition_count,
                (unsigned long long)r.telemetry.cylinder_assignments);
    std::printf("\"plugin_bytes_sent\": %llu, \"plugin_bytes_received\": %llu, ",
                (unsigned long long)q.telemetry.bytes_sent,
                (unsigned long long)q.telemetry.bytes_received);
    std::printf("\"estimation_seconds\": %.9g, \"simulation_seconds\": %.9g, \"ratio\": %.17g}\n",
                r.telemetry.estimation_seconds, r.telemetry.simulation_seconds, ratio);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
