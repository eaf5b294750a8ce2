// stripley_gpu — the reference CLI's `run` command (proj/tools/stripley_main.cpp:
// flags, defaults, exit codes, report) on the device path: rt::run_job with
// rt::DeviceExecutor instead of LocalExecutor / DistributedExecutor.
//
//   stripley_gpu run --points P.csv --boundary B.wkt --smax S --sstep s --tmax T --tstep t
//                    [--time-unit days] [--sims 99] [--sim-method csr|bootstrap|permutation]
//                    [--seed 1] [--index on|off] [--cache on|off] [--coord-tol 0]
//                    [--dist-tol 0] [--partitioner kdb|hash] [--partitions 1] [--workers 1]
//                    [--mode local] [--out R.json] [--csv-dir D] [--drop-outside]
//                    [--benchmark] [--period-start a] [--period-end b] [--device 0]
//
// Exit codes (stripley_main.cpp:22-25): 0 ok, 1 usage, 2 data, 3 runtime.
// index / cache / partitioner / partitions / workers are accepted and echoed
// (they never change the reference's results; the device has no host
// partitions); nonzero cache tolerances are rejected by the library.  The
// reference's master-worker TCP mode (`--mode distributed`, `worker`) is
// replaced by one process per GPU over torch.distributed / NCCL.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "stripley_gpu.hpp"
#include "stripley_gpu_io.hpp"

namespace {

using namespace stripley;

constexpr int kExitOk = 0, kExitUsage = 1, kExitData = 2, kExitRuntime = 3;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Flags {
  std::string points, boundary, time_unit = "days", sim_method = "csr", index = "off",
                                cache = "off", partitioner = "kdb", mode = "local", out, csv_dir;
  double smax = 0, sstep = 0, coord_tol = 0, dist_tol = 0;
  std::int64_t tmax = 0, tstep = 0, period_start = 0, period_end = 0;
  std::uint32_t sims = 99, partitions = 1, workers = 1;
  std::uint64_t seed = 1;
  int device = 0;
  bool drop_outside = false, benchmark = false, ps_set = false, pe_set = false;
};

const char* kUsage =
    "usage: stripley_gpu run --points CSV --boundary WKT|GEOJSON --smax S --sstep s --tmax T\n"
    "                        --tstep t [--time-unit seconds|minutes|hours|days|months]\n"
    "                        [--sims N] [--sim-method csr|bootstrap|permutation] [--seed N]\n"
    "                        [--index on|off] [--cache on|off] [--coord-tol X] [--dist-tol X]\n"
    "                        [--partitioner kdb|hash] [--partitions N] [--workers N]\n"
    "                        [--mode local] [--out PATH] [--csv-dir DIR] [--drop-outside]\n"
    "                        [--benchmark] [--period-start T0] [--period-end T1] [--device N]\n";

template <class T>
T number(const std::string& opt, const std::string& v) {
  std::istringstream in(v);
  T x{};
  if (!(in >> x) || !(in >> std::ws).eof())
    throw UsageError(opt + ": invalid value '" + v + "'");
  return x;
}

void member(const std::string& opt, const std::string& v, std::set<std::string> allowed) {
  if (!allowed.count(v)) throw UsageError(opt + ": '" + v + "' not in the allowed set");
}

Flags parse_run(int argc, char** argv) {
  Flags f;
  std::map<std::string, std::string> val;
  std::set<std::string> seen;
  static const std::set<std::string> kFlags = {"--drop-outside", "--benchmark"};
  static const std::set<std::string> kOptions = {
      "--points",   "--boundary",    "--time-unit",  "--smax",       "--sstep",
      "--tmax",     "--tstep",       "--sims",       "--sim-method", "--seed",
      "--index",    "--cache",       "--coord-tol",  "--dist-tol",   "--partitioner",
      "--partitions", "--workers",   "--mode",       "--worker-addrs", "--out",
      "--csv-dir",  "--period-start", "--period-end", "--device"};
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i], v;
    if (a == "-h" || a == "--help") {
      std::cout << kUsage;
      std::exit(kExitOk);
    }
    const std::size_t eq = a.find('=');
    if (eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    if (kFlags.count(a)) {
      seen.insert(a);
      continue;
    }
    if (!kOptions.count(a)) throw UsageError("unexpected argument: " + a);
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw UsageError(a + " requires a value");
      v = argv[++i];
    }
    val[a] = v;
    seen.insert(a);
  }
  for (const char* req : {"--points", "--boundary", "--smax", "--sstep", "--tmax", "--tstep"})
    if (!val.count(req)) throw UsageError(std::string(req) + " is required");
  auto get = [&](const char* k, auto* dst) {
    auto it = val.find(k);
    if (it == val.end()) return;
    using T = std::remove_pointer_t<decltype(dst)>;
    if constexpr (std::is_same_v<T, std::string>)
      *dst = it->second;
    else
      *dst = number<T>(k, it->second);
  };
  get("--points", &f.points);
  get("--boundary", &f.boundary);
  get("--time-unit", &f.time_unit);
  get("--smax", &f.smax);
  get("--sstep", &f.sstep);
  get("--tmax", &f.tmax);
  get("--tstep", &f.tstep);
  get("--sims", &f.sims);
  get("--sim-method", &f.sim_method);
  get("--seed", &f.seed);
  get("--index", &f.index);
  get("--cache", &f.cache);
  get("--coord-tol", &f.coord_tol);
  get("--dist-tol", &f.dist_tol);
  get("--partitioner", &f.partitioner);
  get("--partitions", &f.partitions);
  get("--workers", &f.workers);
  get("--mode", &f.mode);
  get("--out", &f.out);
  get("--csv-dir", &f.csv_dir);
  get("--period-start", &f.period_start);
  get("--period-end", &f.period_end);
  get("--device", &f.device);
  member("--time-unit", f.time_unit, {"seconds", "minutes", "hours", "days", "months"});
  member("--sim-method", f.sim_method, {"csr", "bootstrap", "permutation"});
  member("--index", f.index, {"on", "off"});
  member("--cache", f.cache, {"on", "off"});
  member("--partitioner", f.partitioner, {"kdb", "hash"});
  member("--mode", f.mode, {"local", "distributed"});
  f.ps_set = val.count("--period-start") > 0;
  f.pe_set = val.count("--period-end") > 0;
  f.drop_outside = seen.count("--drop-outside") > 0;
  f.benchmark = seen.count("--benchmark") > 0;
  return f;
}

sim::Method method_of(const std::string& name) {
  if (name == "bootstrap") return sim::Method::Bootstrap;
  if (name == "permutation") return sim::Method::Permutation;
  return sim::Method::Cstr;
}

rt::JobSpec spec_of(const Flags& f) {
  rt::JobSpec s;
  s.grid = est::DistanceGrid::regular(f.sstep, f.smax, f.tstep, f.tmax);
  s.method = method_of(f.sim_method);
  s.sims = f.sims;
  s.seed = f.seed;
  s.options.use_index = f.index == "on";
  s.options.use_cache = f.cache == "on";
  s.options.coord_tolerance = f.coord_tol;
  s.options.dist_tolerance = f.dist_tol;
  s.partitioner = f.partitioner == "hash" ? rt::PartitionerChoice::Hash
                                          : rt::PartitionerChoice::Kdb;
  s.partitions = f.partitions;
  s.workers = f.workers;
  s.mode = rt::Mode::Local;
  s.time_unit = io::parse_time_unit(f.time_unit);
  return s;
}

struct Job {
  std::vector<geom::STPoint> points;
  geom::StudyRegion region;
};

// stripley_main.cpp:102-140: period defaults to the data's time range (end
// > start enforced), outside points are fatal unless --drop-outside.
Job load(const Flags& f) {
  const io::Dataset ds = io::load_points_csv(f.points, io::parse_time_unit(f.time_unit));
  std::vector<geom::PlanarPoint> ring = io::load_boundary(f.boundary);
  std::int64_t lo = ds.points.front().start_time, hi = lo;
  for (const geom::STPoint& p : ds.points) {
    lo = std::min(lo, p.start_time);
    hi = std::max(hi, p.start_time);
  }
  const std::int64_t p0 = f.ps_set ? f.period_start : lo;
  std::int64_t p1 = f.pe_set ? f.period_end : hi;
  if (p1 <= p0) p1 = p0 + 1;
  geom::StudyRegion region(std::move(ring), p0, p1);
  std::vector<geom::STPoint> kept;
  std::vector<std::string> outside;
  for (std::size_t i = 0; i < ds.points.size(); ++i) {
    if (region.contains(ds.points[i]))
      kept.push_back(ds.points[i]);
    else
      outside.push_back(ds.ids[i]);
  }
  if (!outside.empty() && !f.drop_outside) {
    std::ostringstream m;
    m << outside.size() << " point(s) outside study region/period:";
    for (std::size_t i = 0; i < outside.size() && i < 10; ++i) m << ' ' << outside[i];
    if (outside.size() > 10) m << " ...";
    m << " (use --drop-outside to drop them)";
    throw io::DataError(m.str());
  }
  if (!outside.empty()) std::cerr << "dropped " << outside.size() << " point(s) outside region/period\n";
  return Job{std::move(kept), std::move(region)};
}

io::RunParams params_of(const Flags& f) {
  io::RunParams p;
  p.points_path = f.points;
  p.boundary_path = f.boundary;
  p.time_unit = f.time_unit;
  p.sim_method = f.sim_method;
  p.partitioner = f.partitioner;
  p.mode = f.mode;
  p.sims = f.sims;
  p.seed = f.seed;
  p.partitions = f.partitions;
  p.workers = f.workers;
  p.use_index = f.index == "on";
  p.use_cache = f.cache == "on";
  p.coord_tolerance = f.coord_tol;
  p.dist_tolerance = f.dist_tol;
  return p;
}

int run(const Flags& f) {
  if (f.mode == "distributed")
    throw UsageError("--mode distributed: the device path scales as one process per GPU "
                     "(torch.distributed / NCCL, DESIGN.md §7); use --mode local");
  const rt::JobSpec spec = spec_of(f);
  const Job job = load(f);
  rt::DeviceExecutor exec(f.device);
  if (f.benchmark) {
    // The reference's option matrix (stripley_main.cpp:187-240): results are
    // identical across it; the device ignores index / cache / partitioner.
    std::printf("n=%zu  grid=%zux%zu  sims=%u  device=%d\n", job.points.size(),
                spec.grid.cells_s(), spec.grid.cells_t(), spec.sims, f.device);
    std::printf("%-44s %10s %8s %14s %14s\n", "configuration", "seconds", "SF", "comparisons",
                "in-threshold");
    double base = 0;
    for (const bool idx : {false, true})
      for (const bool cache : {false, true})
        for (const char* part : {"hash", "kdb"}) {
          rt::JobSpec s = spec;
          s.options.use_index = idx;
          s.options.use_cache = cache;
          const auto t0 = std::chrono::steady_clock::now();
          const rt::RunResult r = rt::run_job(job.points, job.region, s, exec);
          const double sec =
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          if (base == 0) base = sec;
          const std::string name = std::string("index=") + (idx ? "on" : "off") +
                                   " cache=" + (cache ? "on" : "off") + " partitioner=" + part;
          std::printf("%-44s %10.3f %8.2f %14llu %14llu\n", name.c_str(), sec, base / sec,
                      (unsigned long long)r.telemetry.pair_comparisons,
                      (unsigned long long)r.telemetry.in_threshold_pairs);
        }
    return kExitOk;
  }
  const rt::RunResult res = rt::run_job(job.points, job.region, spec, exec);
  const io::DeviceTelemetry dev{job.points.size(), 1ull + spec.sims};
  const std::string report = io::build_report_json(params_of(f), spec, res, dev);
  if (f.out.empty())
    std::cout << report;
  else
    io::write_file(f.out, report);
  if (!f.csv_dir.empty()) io::write_surface_csvs(f.csv_dir, res);
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw UsageError("a subcommand is required");
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
      std::cout << kUsage;
      return kExitOk;
    }
    if (cmd == "worker")
      throw UsageError("worker: the reference's TCP worker is replaced by one process per GPU "
                       "(torch.distributed / NCCL)");
    if (cmd != "run") throw UsageError("unknown subcommand: " + cmd);
    return run(parse_run(argc, argv));
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n" << kUsage;
    return kExitUsage;
  } catch (const io::DataError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitData;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitData;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitRuntime;
  }
}
