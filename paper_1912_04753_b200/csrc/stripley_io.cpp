// stripley_io.cpp — CSV / WKT / GeoJSON ingest and the JSON / CSV result
// writers of the device CLI (interface: include/stripley_gpu_io.hpp; behaviour
// of proj/core/src/io.cpp: same accepted formats, messages and schema).
// The JSON is produced by nlohmann::ordered_json (the header the reference's
// io.cpp uses, found in this image under cudnn_frontend's thirdparty tree) so
// number formatting and key order match the reference's reports.
#include "stripley_gpu_io.hpp"

#include <charconv>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <sstream>

#include <nlohmann/json.hpp>

namespace stripley::io {

namespace {

using Json = nlohmann::ordered_json;

const char* const kSpace = " \t\r\n";

std::string strip(const std::string& s) {
  const std::size_t b = s.find_first_not_of(kSpace);
  if (b == std::string::npos) return std::string();
  return s.substr(b, s.find_last_not_of(kSpace) - b + 1);
}

std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw DataError("cannot open " + path);
  std::stringstream buf;
  buf << f.rdbuf();
  return buf.str();
}

std::vector<std::string> split_commas(const std::string& line) {
  std::vector<std::string> out(1);
  for (const char ch : line) {
    if (ch == ',')
      out.emplace_back();
    else
      out.back() += ch;
  }
  return out;
}

// Days since 1970-01-01 of a proleptic Gregorian date (era arithmetic: a
// 400-year era has 146,097 days; March-based years put Feb 29 last).
std::int64_t civil_to_days(std::int64_t year, int month, int day) {
  const std::int64_t y = month <= 2 ? year - 1 : year;
  const std::int64_t era = (y >= 0 ? y : y - 399) / 400;
  const std::int64_t yoe = y - era * 400;                               // [0, 399]
  const int mp = month > 2 ? month - 3 : month + 9;                      // March = 0
  const std::int64_t doy = (153 * mp + 2) / 5 + day - 1;                 // [0, 365]
  const std::int64_t doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;       // [0, 146096]
  return era * 146097 + doe - 719468;
}

std::int64_t div_floor(std::int64_t a, std::int64_t b) {
  const std::int64_t q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

template <class T>
bool parse_int(const char* b, const char* e, T* out) {
  const auto r = std::from_chars(b, e, *out);
  return r.ec == std::errc{} && r.ptr == e;
}

std::vector<geom::PlanarPoint> ring_from_wkt(const std::string& text) {
  const std::size_t lo = text.find("((");
  const std::size_t hi = text.find("))");
  if (lo == std::string::npos || hi == std::string::npos || hi < lo)
    throw DataError("malformed WKT POLYGON");
  const std::string body = text.substr(lo + 2, hi - lo - 2);
  if (body.find('(') != std::string::npos) throw DataError("polygon holes are not supported");
  std::vector<geom::PlanarPoint> ring;
  std::size_t pos = 0;
  while (pos <= body.size()) {
    const std::size_t next = std::min(body.find(',', pos), body.size());
    const std::string item = body.substr(pos, next - pos);
    std::istringstream in(strip(item));
    geom::PlanarPoint v;
    if (!(in >> v.x >> v.y)) throw DataError("malformed WKT coordinate: " + item);
    ring.push_back(v);
    pos = next + 1;
  }
  return ring;
}

std::vector<geom::PlanarPoint> ring_from_geojson(const std::string& text) {
  Json doc;
  try {
    doc = Json::parse(text);
  } catch (const std::exception& e) {
    throw DataError(std::string("invalid GeoJSON: ") + e.what());
  }
  const Json& g = doc.contains("geometry") ? doc["geometry"] : doc;  // Feature or geometry
  if (!g.contains("type") || g["type"] != "Polygon" || !g.contains("coordinates"))
    throw DataError("GeoJSON boundary must be a Polygon");
  const Json& rings = g["coordinates"];
  if (!rings.is_array() || rings.empty()) throw DataError("GeoJSON polygon has no rings");
  if (rings.size() > 1) throw DataError("polygon holes are not supported");
  std::vector<geom::PlanarPoint> ring;
  for (const Json& v : rings[0]) {
    if (!v.is_array() || v.size() < 2) throw DataError("malformed GeoJSON vertex");
    ring.push_back({v[0].get<double>(), v[1].get<double>()});
  }
  return ring;
}

Json matrix(const est::KSurface& s) {
  Json m = Json::array();
  for (const std::vector<double>& row : s.values) m.push_back(row);
  return m;
}

void matrix_csv(const std::filesystem::path& path, const est::KSurface& s) {
  std::ostringstream out;
  out << std::setprecision(17);
  for (const std::vector<double>& row : s.values) {
    for (std::size_t j = 0; j < row.size(); ++j) out << (j ? "," : "") << row[j];
    out << '\n';
  }
  write_file(path.string(), out.str());
}

}  // namespace

geom::TimeUnit parse_time_unit(const std::string& name) {
  static const std::pair<const char*, geom::TimeUnit> kUnits[] = {
      {"seconds", geom::TimeUnit::Seconds}, {"minutes", geom::TimeUnit::Minutes},
      {"hours", geom::TimeUnit::Hours},     {"days", geom::TimeUnit::Days},
      {"months", geom::TimeUnit::Months}};
  for (const auto& [n, u] : kUnits)
    if (name == n) return u;
  throw DataError("unknown time unit: " + name);
}

std::string time_unit_name(geom::TimeUnit unit) {
  switch (unit) {
    case geom::TimeUnit::Seconds: return "seconds";
    case geom::TimeUnit::Minutes: return "minutes";
    case geom::TimeUnit::Hours: return "hours";
    case geom::TimeUnit::Months: return "months";
    case geom::TimeUnit::Days: break;
  }
  return "days";
}

std::int64_t parse_timestamp(const std::string& field, geom::TimeUnit unit) {
  const std::string s = strip(field);
  const char* p = s.data();
  if (s.size() == 10 && s[4] == '-' && s[7] == '-') {  // YYYY-MM-DD
    int y = 0, m = 0, d = 0;
    if (!parse_int(p, p + 4, &y) || !parse_int(p + 5, p + 7, &m) ||
        !parse_int(p + 8, p + 10, &d) || m < 1 || m > 12 || d < 1 || d > 31)
      throw DataError("invalid ISO date: " + s);
    const std::int64_t days = civil_to_days(y, m, d);
    switch (unit) {
      case geom::TimeUnit::Seconds: return days * 86400;
      case geom::TimeUnit::Minutes: return days * 1440;
      case geom::TimeUnit::Hours: return days * 24;
      case geom::TimeUnit::Months: return div_floor(days, 30);
      case geom::TimeUnit::Days: break;
    }
    return days;
  }
  std::int64_t v = 0;
  if (!parse_int(p, p + s.size(), &v)) throw DataError("invalid timestamp: " + s);
  return v;
}

Dataset load_points_csv(const std::string& path, geom::TimeUnit unit) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open " + path);
  std::string line;
  if (!std::getline(in, line)) throw DataError(path + ": empty file");
  std::vector<std::string> head = split_commas(strip(line));
  for (std::string& h : head) h = strip(h);
  if (head.size() < 4 || head[0] != "id" || head[1] != "x" || head[2] != "y" || head[3] != "t")
    throw DataError(path + ":1: expected header id,x,y,t");
  Dataset ds;
  for (std::size_t no = 2; std::getline(in, line); ++no) {
    const std::string row = strip(line);
    if (row.empty()) continue;
    const std::vector<std::string> f = split_commas(row);
    const std::string at = path + ":" + std::to_string(no);
    if (f.size() < 4) throw DataError(at + ": expected 4 columns");
    geom::STPoint pt;
    try {  // std::stod, as the reference: a numeric prefix is accepted
      pt.x = std::stod(strip(f[1]));
      pt.y = std::stod(strip(f[2]));
    } catch (const std::exception&) {
      throw DataError(at + ": invalid coordinate");
    }
    if (!std::isfinite(pt.x) || !std::isfinite(pt.y)) throw DataError(at + ": coordinate not finite");
    try {
      pt.start_time = pt.end_time = parse_timestamp(f[3], unit);
    } catch (const DataError& e) {
      throw DataError(at + ": " + e.what());
    }
    ds.ids.push_back(strip(f[0]));
    ds.points.push_back(pt);
  }
  if (ds.points.empty()) throw DataError(path + ": no data rows");
  return ds;
}

std::vector<geom::PlanarPoint> load_boundary(const std::string& path) {
  const std::string text = strip(slurp(path));
  if (text.empty()) throw DataError(path + ": empty boundary file");
  std::vector<geom::PlanarPoint> ring;
  if (text.compare(0, 7, "POLYGON") == 0)
    ring = ring_from_wkt(text);
  else if (text[0] == '{')
    ring = ring_from_geojson(text);
  else
    throw DataError(path + ": boundary must be WKT POLYGON or GeoJSON Polygon");
  if (ring.size() >= 2 && ring.front().x == ring.back().x && ring.front().y == ring.back().y)
    ring.pop_back();  // stored open
  if (ring.size() < 3) throw DataError(path + ": polygon needs >= 3 vertices");
  return ring;
}

std::string build_report_json(const RunParams& prm, const rt::JobSpec& spec,
                              const rt::RunResult& res, const DeviceTelemetry& dev) {
  Json j;
  j["params"] = {{"points", prm.points_path},
                 {"boundary", prm.boundary_path},
                 {"time_unit", prm.time_unit},
                 {"smax", spec.grid.s_max()},
                 {"tmax", spec.grid.t_max()},
                 {"sims", prm.sims},
                 {"sim_method", prm.sim_method},
                 {"seed", prm.seed},
                 {"index", prm.use_index ? "on" : "off"},
                 {"cache", prm.use_cache ? "on" : "off"},
                 {"coord_tol", prm.coord_tolerance},
                 {"dist_tol", prm.dist_tolerance},
                 {"partitioner", prm.partitioner},
                 {"partitions", prm.partitions},
                 {"workers", prm.workers},
                 {"mode", prm.mode}};
  j["grid"] = {{"s", res.k_hat.grid.s_values}, {"t", res.k_hat.grid.t_values}};
  j["k_hat"] = matrix(res.k_hat);
  j["l_hat"] = matrix(res.l_hat);
  j["theoretical_k"] = matrix(res.theoretical);
  if (res.upper_l && res.lower_l) {
    j["envelope"] = {{"upper_l", matrix(*res.upper_l)}, {"lower_l", matrix(*res.lower_l)}};
    if (res.diff_upper) j["diff_upper"] = matrix(*res.diff_upper);
  }
  const rt::RunTelemetry& t = res.telemetry;
  // The device keeps no weight cache and no host partitions: cache counters
  // are zero, the whole pattern is one "partition" assigned once per pattern.
  const Json zero_cache = {{"hits", 0}, {"misses", 0}, {"insertions", 0}};
  j["telemetry"] = {
      {"timings",
       {{"plan_seconds", t.plan_seconds},
        {"estimation_seconds", t.estimation_seconds},
        {"simulation_seconds", t.simulation_seconds}}},
      {"comparisons",
       {{"pair_comparisons", t.pair_comparisons}, {"in_threshold_pairs", t.in_threshold_pairs}}},
      {"cache", {{"spatial", zero_cache}, {"temporal", zero_cache}}},
      {"redundancy",
       {{"cylinder_assignments", dev.points * dev.patterns},
        {"partitions", 1},
        {"partition_point_counts", Json::array({dev.points})}}},
      {"bytes", {{"sent", 0}, {"received", 0}}},
      {"device",
       {{"device_ms", t.device_ms},
        {"pair_kernel_ms", t.pair_kernel_ms},
        {"exact_path_pairs", t.exact_path_pairs}}},
  };
  return j.dump(2) + "\n";
}

void write_file(const std::string& path, const std::string& contents) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw DataError("cannot write " + path);
  out << contents;
}

void write_surface_csvs(const std::string& dir, const rt::RunResult& res) {
  const std::filesystem::path d(dir);
  std::filesystem::create_directories(d);
  matrix_csv(d / "k_hat.csv", res.k_hat);
  matrix_csv(d / "l_hat.csv", res.l_hat);
  matrix_csv(d / "theoretical_k.csv", res.theoretical);
  if (res.upper_l) matrix_csv(d / "upper_l.csv", *res.upper_l);
  if (res.lower_l) matrix_csv(d / "lower_l.csv", *res.lower_l);
  if (res.diff_upper) matrix_csv(d / "diff_upper.csv", *res.diff_upper);
}

}  // namespace stripley::io
