// C++ checks of the reference-facing API (include/stripley_gpu.hpp) on the GPU.
// Mirrors proj/tests/test_estimator.cpp / test_edge_correction.cpp style checks,
// and runs rt::run_job on an input file for the Python harness to compare with
// the golden fixtures.  Usage:
//   test_api selftest
//   test_api runjob <points.bin> <ring.bin> p0 p1 <grid.bin> sims seed world
// Binary files: little-endian; points.bin = u64 n, f64 x[n], f64 y[n], i64 t[n];
// ring.bin = u64 nv, f64 xy[2nv]; grid.bin = u64 cs, f64 s[cs], u64 ct, i64 t[ct].
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "stripley_gpu.hpp"

using namespace stripley;

static int failures = 0;
#define EXPECT(cond)                                                      \
  do {                                                                    \
    if (!(cond)) {                                                        \
      ++failures;                                                         \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                     \
  } while (0)

template <class F>
static std::string throws(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    return e.what();
  } catch (const std::exception& e) {
    return std::string("other: ") + e.what();
  }
  return "";
}

static int selftest() {
  // validation messages (geometry.cpp:110-136, estimator.cpp:14-22)
  EXPECT(throws([] { geom::StudyRegion({{0, 0}, {1, 0}}, 0, 1); }) == "polygon needs >= 3 vertices");
  EXPECT(throws([] { geom::StudyRegion({{0, 0}, {10, 10}, {10, 0}, {0, 10}}, 0, 1); }) ==
         "polygon is self-intersecting");
  EXPECT(throws([] { geom::StudyRegion({{0, 0}, {10, 0}, {10, 10}}, 5, 5); }) ==
         "study period duration must be > 0");
  EXPECT(throws([] { est::DistanceGrid{{1.0, 1.0}, {1}}.validate(); }) ==
         "distance grid must be strictly increasing");
  const auto g = est::DistanceGrid::regular(500.0, 2000.0, 2, 10);
  EXPECT((g.s_values == std::vector<double>{500, 1000, 1500, 2000}));
  // bin_pair (test_estimator.cpp:52-60)
  const est::DistanceGrid bg{{1.0, 2.0, 3.0}, {10, 20}};
  EXPECT((est::bin_pair(bg, 1.5, 11) == std::pair<std::size_t, std::size_t>{1, 1}));
  EXPECT(!est::bin_pair(bg, 3.1, 5).has_value());
  // two interior points: K = 5e9 (test_estimator.cpp:62-76)
  const geom::StudyRegion sq({{0, 0}, {10000, 0}, {10000, 10000}, {0, 10000}}, 0, 100);
  const std::vector<geom::STPoint> pts{geom::make_point(4000, 5000, 50), geom::make_point(5000, 5000, 55)};
  const auto k = est::estimate_surface(pts, sq, est::DistanceGrid{{2000.0}, {10}}, {});
  EXPECT(std::abs(k.values[0][0] - 5.0e9) <= 1e-6);
  // preconditions (test_estimator.cpp:77-90)
  EXPECT(throws([&] { est::estimate_surface(std::vector<geom::STPoint>{geom::make_point(1, 1, 1)}, sq,
                                            est::DistanceGrid{{10.0}, {10}}, {}); }) ==
         "K estimation needs n >= 2");
  EXPECT(throws([&] { est::estimate_surface(std::vector<geom::STPoint>{geom::make_point(1, 1, 1),
                                                                       geom::make_point(2, 2, 999)},
                                            sq, est::DistanceGrid{{10.0}, {10}}, {}); }) ==
         "point outside study region or period");
  // CSR determinism + bootstrap/permutation properties (test_simulation.cpp)
  const auto a = sim::generate_cstr(500, sq, 7), b = sim::generate_cstr(500, sq, 7);
  EXPECT(a == b);
  for (const auto& p : a) EXPECT(sq.contains(p));
  const auto perm = sim::generate_permutation(a, 3);
  std::vector<std::int64_t> t0, t1;
  for (std::size_t i = 0; i < a.size(); ++i) {
    EXPECT(perm[i].x == a[i].x && perm[i].y == a[i].y);
    t0.push_back(a[i].start_time);
    t1.push_back(perm[i].start_time);
  }
  std::sort(t0.begin(), t0.end());
  std::sort(t1.begin(), t1.end());
  EXPECT(t0 == t1);
  // envelopes (test_simulation.cpp:99-110)
  const auto sims = sim::run_simulations(a, sq, est::DistanceGrid{{500.0, 1000.0}, {10, 20}},
                                         sim::Method::Cstr, 5, 11, {});
  const auto [up, lo] = sim::envelopes(sims);
  for (const auto& s : sims)
    for (std::size_t i = 0; i < 2; ++i)
      for (std::size_t j = 0; j < 2; ++j) EXPECT(lo.values[i][j] <= s.values[i][j] && s.values[i][j] <= up.values[i][j]);
  // executors (runtime.hpp:106-136): LocalExecutor, the NCCL-communicator
  // DeviceExecutor at world 1 (stk_run_job_dist: exact device exchange) and a
  // world > 1 executor without communicator or hooks (rejected)
  {
    rt::JobSpec spec;
    spec.grid = est::DistanceGrid{{250.0, 500.0, 1000.0}, {10, 20, 40}};
    spec.sims = 4;
    spec.seed = 21;
    rt::LocalExecutor local(4, sq, spec.grid, spec.options);
    const auto r1 = rt::run_job(a, sq, spec, local);
    rt::DeviceExecutor coll(0, 0, 1, rt::DeviceExecutor::nccl_unique_id());
    const auto r2 = rt::run_job(a, sq, spec, coll);
    EXPECT(r1.k_hat.values == r2.k_hat.values && r1.l_hat.values == r2.l_hat.values);
    EXPECT(r1.upper_l->values == r2.upper_l->values && r1.lower_l->values == r2.lower_l->values);
    EXPECT(r1.diff_upper->values == r2.diff_upper->values);
    EXPECT(r1.telemetry.in_threshold_pairs == r2.telemetry.in_threshold_pairs);
    EXPECT(throws([] { rt::DeviceExecutor bad(0, 0, 2); }).find("needs an NCCL unique id") !=
           std::string::npos);
    EXPECT(throws([] { rt::DeviceExecutor bad(0, 2, 2); }) == "rank must be < world");
    EXPECT(rt::speedup_factor(10.0, 2.5) == 4.0);
    EXPECT(throws([] { rt::speedup_factor(0.0, 1.0); }) == "times must be > 0");
  }
  std::printf("selftest failures=%d\n", failures);
  return failures ? 1 : 0;
}

template <class T>
static std::vector<T> read_vec(std::ifstream& f) {
  std::uint64_t n = 0;
  f.read(reinterpret_cast<char*>(&n), 8);
  std::vector<T> v(n);
  f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(n * sizeof(T)));
  return v;
}

static void print_surface(const char* name, const est::KSurface& s, bool last = false) {
  std::printf("\"%s\": [", name);
  bool first = true;
  for (const auto& row : s.values)
    for (double v : row) {
      std::printf("%s%.17g", first ? "" : ",", v);
      first = false;
    }
  std::printf("]%s\n", last ? "" : ",");
}

static int runjob(int argc, char** argv) {
  if (argc < 10) return 2;
  std::ifstream fp(argv[2], std::ios::binary), fr(argv[3], std::ios::binary), fg(argv[6], std::ios::binary);
  std::uint64_t n = 0;
  fp.read(reinterpret_cast<char*>(&n), 8);
  std::vector<double> x(n), y(n);
  std::vector<std::int64_t> t(n);
  fp.read(reinterpret_cast<char*>(x.data()), 8 * n);
  fp.read(reinterpret_cast<char*>(y.data()), 8 * n);
  fp.read(reinterpret_cast<char*>(t.data()), 8 * n);
  const auto ring_xy = read_vec<double>(fr);
  std::vector<geom::PlanarPoint> ring;
  for (std::size_t i = 0; i + 1 < ring_xy.size(); i += 2) ring.push_back({ring_xy[i], ring_xy[i + 1]});
  const geom::StudyRegion region(ring, std::stoll(argv[4]), std::stoll(argv[5]));
  rt::JobSpec spec;
  spec.grid.s_values = read_vec<double>(fg);
  spec.grid.t_values = read_vec<std::int64_t>(fg);
  spec.sims = (std::uint32_t)std::stoul(argv[7]);
  spec.seed = std::stoull(argv[8]);
  const std::uint32_t world = (std::uint32_t)std::stoul(argv[9]);
  std::vector<geom::STPoint> pts(n);
  for (std::size_t i = 0; i < n; ++i) pts[i] = geom::make_point(x[i], y[i], t[i]);
  rt::RunResult res;
  if (world <= 1) {
    rt::DeviceExecutor ex(0);
    res = rt::run_job(pts, region, spec, ex);
  } else {
    // ranks run one after another in this process; the reduction hooks
    // accumulate into the shared state, so the last rank holds the combined
    // (exact SUM / MAX / MIN) values of all ranks
    std::vector<std::uint64_t> acc;
    std::vector<double> aup, alo;
    for (std::uint32_t r = 0; r < world; ++r) {
      rt::DeviceExecutor ex(
          0, r, world,
          [&](std::vector<std::uint64_t>& v) {
            if (acc.empty()) acc.assign(v.size(), 0);
            for (std::size_t i = 0; i < v.size(); ++i) acc[i] += v[i];
            v = acc;
          },
          [&](std::vector<double>& u, std::vector<double>& l) {
            if (aup.empty()) { aup = u; alo = l; }
            for (std::size_t i = 0; i < u.size(); ++i) {
              aup[i] = std::max(aup[i], u[i]);
              alo[i] = std::min(alo[i], l[i]);
            }
            u = aup;
            l = alo;
          });
      res = rt::run_job(pts, region, spec, ex);
    }
  }
  std::printf("{\n\"in_threshold\": %llu,\n", (unsigned long long)res.telemetry.in_threshold_pairs);
  print_surface("k", res.k_hat);
  print_surface("l", res.l_hat);
  if (res.upper_l) {
    print_surface("upper", *res.upper_l);
    print_surface("lower", *res.lower_l);
    print_surface("diff", *res.diff_upper, true);
  } else {
    std::printf("\"none\": 0\n");
  }
  std::printf("}\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::strcmp(argv[1], "selftest") == 0) return selftest();
  if (argc >= 2 && std::strcmp(argv[1], "runjob") == 0) return runjob(argc, argv);
  std::fprintf(stderr, "usage: test_api selftest | runjob ...\n");
  return 2;
}
