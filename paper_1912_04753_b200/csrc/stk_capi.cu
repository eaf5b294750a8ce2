// stk_capi.cu — host runtime behind the C ABI in include/stk.h.
//
// One context = one device + one stream.  The runtime validates inputs with
// the reference's rules and messages, derives the exact bin thresholds and
// the cell grid, sizes pattern batches to a memory budget, and drives the
// kernels of stk_kernels.cu:
//
//   per batch of R patterns:  generate (K4) -> grid (K1) -> pairs (K2) -> finalize/envelopes (K5)
//
// All device work of one call is enqueued on the context stream; the host
// synchronises once at the end (plus one tiny read-back for validation).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and constants only: libnccl.so.2 is dlopen'ed on first use

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/stk.h"
#include "stk_kernels.h"
#include "stk_types.h"

using namespace stk;

namespace {

struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// NCCL entry points, resolved from libnccl.so.2 at the first communicator call
// (the library loads, and single-GPU calls run, without NCCL installed; in a
// process that already loaded torch's NCCL the soname resolves to that copy).
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.load_error = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
    a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
    a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce ||
        !a.group_start || !a.group_end || !a.error_string) {
      a.load_error = "libnccl.so.2 lacks the expected symbols";
      a.get_unique_id = nullptr;
    }
    return a;
  }();
  if (!api.get_unique_id) throw NcclFail(api.load_error);
  return api;
}

#define NK(expr)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (expr);                                                             \
    if (r_ != ncclSuccess) throw NcclFail(std::string(#expr) + ": " + nccl().error_string(r_)); \
  } while (0)

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw CudaFail(std::string(#expr) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

// Bumped by every device (re)allocation: a captured CUDA graph holds raw
// buffer addresses and is replayed only while this is unchanged.
uint64_t g_alloc_gen = 0;

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  void ensure(size_t n) {
    if (n <= cap) return;
    ++g_alloc_gen;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    cap = std::max<size_t>(n, 1);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Largest q with RN(sqrt(q)) <= s: d <= s  <=>  q <= Q(s), exactly, because
// the correctly rounded sqrt is monotone (lets the kernels bin on q).
double sqrt_threshold(double s) {
  double q = s * s;
  while (q > 0 && std::sqrt(q) > s) q = std::nextafter(q, 0.0);
  for (;;) {
    const double qn = std::nextafter(q, std::numeric_limits<double>::infinity());
    if (std::sqrt(qn) <= s) q = qn; else break;
  }
  return q;
}

// geom::segments_properly_intersect (geometry.cpp:70-79)
bool segments_properly_intersect(const double* a, const double* b, const double* c,
                                 const double* d) {
  auto orient = [](const double* p, const double* q, const double* r) {
    const double v = (q[0] - p[0]) * (r[1] - p[1]) - (q[1] - p[1]) * (r[0] - p[0]);
    return (v > 0.0) - (v < 0.0);
  };
  const int o1 = orient(a, b, c), o2 = orient(a, b, d);
  const int o3 = orient(c, d, a), o4 = orient(c, d, b);
  return o1 != o2 && o3 != o4 && o1 != 0 && o2 != 0 && o3 != 0 && o4 != 0;
}

}  // namespace

namespace {
struct GraphCache;  // captured pipeline of the last repeated job (run_pipeline)
}

struct stk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int num_sms = 148;
  uint64_t mem_budget = 16ull << 30;
  int time_radius = 0;     // time layers of the stencil, 0 = the spatial radius (STK_TIME_RADIUS env)
  double min_cell_pop = 8.0;  // finer cells only when this populous (STK_MIN_CELL_POP env)
  double min_cell_pop_t = 12.5;  // ... and finer time layers only from here (STK_MIN_CELL_POP_T)
  int stencil_radius = 2;  // preferred cell refinement (STK_STENCIL_RADIUS env overrides)
  int rng = STK_RNG_MT19937_64;  // realisation generator (stk_set_rng)

  // region (geom::StudyRegion)
  bool have_region = false;
  std::vector<double> ring;  // open, interleaved
  uint32_t nv = 0;
  int64_t p0 = 0, p1 = 0;
  double area = 0;
  int64_t duration = 0;
  double xmin = 0, xmax = 0, ymin = 0, ymax = 0, maxabs = 0;
  bool fast_rect = false;  // axis-aligned rectangle: every bbox draw is inside
  DevBuf<double2> d_ring;
  // general-polygon indexes: slabs (region only) and edge
  // cells (region + grid), built lazily by region_view()
  bool slab_ok = false, ec_ok = false;
  uint32_t nslab = 0;
  double slab_y0 = 0, slab_inv_h = 0, pip_lim = 0, pip_ylo = 0, pip_yhi = 0;
  DevBuf<uint32_t> d_slab_start, d_slab_edge;
  int ec_nx = 0, ec_ny = 0;
  double ec_x0 = 0, ec_y0 = 0, ec_inv_w = 0, ec_dmax = 0, ec_reach = 0;
  DevBuf<uint32_t> d_ec_start, d_ec_edge;
  DevBuf<float> d_ec_dmin, d_ec_dmax;
  DevBuf<RegionView> d_rv;  // device copy of region_view() for out-of-line device code

  // grid (est::DistanceGrid)
  bool have_grid = false;
  std::vector<double> s_values;
  std::vector<int64_t> t_values;
  std::vector<double> Q;
  std::vector<QBucket> qtab;
  std::vector<TBucket<int64_t>> ttab;
  int q_shift = 0, q_base = 0;
  int t_shift = 0;
  bool single_step = false;
  bool q_single = false;  // the q table alone is single-step
  int t_uni = 0;          // BinView::t_uni and its constants
  int32_t t_add = 0, t_lo = 0;
  uint32_t t_magic = 0;
  int t_sh = 0;
  DevBuf<double> d_Q, d_s;
  DevBuf<int64_t> d_T;
  DevBuf<QBucket> d_qtab;
  DevBuf<TBucket<int64_t>> d_ttab;

  // batch buffers (grow-only)
  DevBuf<double> x, y;
  DevBuf<int64_t> t;
  DevBuf<double2> pxy;
  DevBuf<double2> parc;  // rectangles: per sorted point arc record (Batch::parc)
  DevBuf<unsigned char> pmeta;
  DevBuf<uint32_t> key, rank, sidx, cell_count, cell_start, item_start, task_start, task_counter;
  DevBuf<uint2> items;
  DevBuf<uint32_t> sel_start, center_pos;
  DevBuf<uint4> arcq;
  DevBuf<double> angs;
  DevBuf<unsigned long long> hist, stats, bad;
  DevBuf<double> K, L, env, obs;
  DevBuf<int> flags, ovf;
  DevBuf<double> scratch;
  DevBuf<uint32_t> perm;  // parallel permutation scratch (draws, lists, scans)
  DevBuf<unsigned long long> perm_mx;
  DevBuf<uint2> scan_part;  // multi-CTA scan: chunk sums
  DevBuf<double> sx, sy;  // host-upload staging of the observed pattern
  DevBuf<int64_t> st;

  uint64_t launches = 0;  // kernels launched by the current call
  DevBuf<unsigned long long> obsraw;  // observed pattern's exact sums [4][bins] (h_cnt, h_half, h_lo, h_hi)
  DevBuf<unsigned long long> limbs;   // their exact-exchange limbs [6][bins]

  // multi-GPU (stk_comm_init): one communicator per context, one rank per GPU
  ncclComm_t comm = nullptr;
  int comm_rank = 0, nranks = 1;

  // Pinned host staging of a call's outputs: device results land here and are
  // copied to the caller's buffers only after the end-of-call checks (a failed
  // validation writes nothing, like the reference's throw before any work).
  unsigned char* hstage = nullptr;
  size_t hstage_cap = 0, hstage_used = 0;
  struct Out {
    void* dst;        // resolved host destination (field < 0) ...
    int field;        // ... or a JobOut field (bound per call: graphs replay the layout)
    uint64_t elem;    // element offset into that field
    size_t off, bytes;
  };
  std::vector<Out> outs;
  bool check_points = false;  // validate_kernel ran: read c->bad at the end of the call

  // pair-kernel occupancy per (wide, mode, smem): set once, not per batch
  struct Occ {
    int wide, mode;
    size_t smem;
    int per_sm;
  };
  std::vector<Occ> occ;
  bool rv_dev_valid = false;  // d_rv holds region_view() of the current region + grid
  std::unique_ptr<GraphCache> graph;

  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  cudaEvent_t ev() {
    if (evnext == evpool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      evpool.push_back(e);
    }
    return evpool[evnext++];
  }
};

namespace {

// Exported per-bin sums (128-bit fixed point, 53 fractional bits) of a bin
// that received an infinite term (omega == 0) carry + 2^120: real sums stay
// far below (< 2^110), so summing partials of up to 255 ranks/shards keeps
// the mark, and fixed_or_nan() turns it into the reference's NaN.
constexpr unsigned __int128 kInfSentinel = (unsigned __int128)1 << 120;
double fixed_or_nan(unsigned __int128 v) {
  if (v >= ((unsigned __int128)1 << 119)) return std::nan("");
  return std::ldexp((double)v, -kFixedFracBits);  // correctly rounded u128 -> f64
}

void upload_u32(stk_ctx* c, DevBuf<uint32_t>& buf, const std::vector<uint32_t>& v) {
  buf.ensure(std::max<size_t>(v.size(), 1));
  if (!v.empty())
    CK(cudaMemcpyAsync(buf.p, v.data(), sizeof(uint32_t) * v.size(), cudaMemcpyHostToDevice,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// Horizontal slabs for point_in_polygon (stk_device.cuh pip_slab): edge k
// (ring[k] -> ring[k+1]) goes to every slab its y-range, widened by
// tol = 2e-12 * pip_lim (>= the reference's on_segment tolerance 1e-12*scale
// for any probe with |x|, |y| <= pip_lim) and by one slab each side, meets.
void build_slabs(stk_ctx* c) {
  const uint32_t m = c->nv;
  const double* r = c->ring.data();
  const double ext = std::max(c->xmax - c->xmin, c->ymax - c->ymin);
  c->pip_lim = 2.0 * (c->maxabs + ext) + 1.0;
  const double tol = 2e-12 * c->pip_lim;
  const uint32_t ns = std::min<uint32_t>(4096, std::max<uint32_t>(1, m / 2));
  c->nslab = ns;
  c->slab_y0 = c->ymin;
  c->slab_inv_h = (double)ns / (c->ymax - c->ymin);
  c->pip_ylo = c->ymin - tol;
  c->pip_yhi = c->ymax + tol;
  auto slab_of = [&](double y) {
    const double f = std::floor((y - c->slab_y0) * c->slab_inv_h);
    return (int64_t)std::max(-2.0, std::min((double)ns + 1.0, f));
  };
  std::vector<uint32_t> count(ns + 1, 0), start(ns + 1, 0), edge;
  auto range = [&](uint32_t k, int64_t* s0, int64_t* s1) {
    const uint32_t k1 = (k + 1 == m) ? 0 : k + 1;
    const double lo = std::min(r[2 * k + 1], r[2 * k1 + 1]) - tol;
    const double hi = std::max(r[2 * k + 1], r[2 * k1 + 1]) + tol;
    *s0 = std::max<int64_t>(0, slab_of(lo) - 1);
    *s1 = std::min<int64_t>(ns - 1, slab_of(hi) + 1);
  };
  for (uint32_t k = 0; k < m; ++k) {
    int64_t s0, s1;
    range(k, &s0, &s1);
    for (int64_t q = s0; q <= s1; ++q) ++count[q];
  }
  for (uint32_t q = 0; q < ns; ++q) start[q + 1] = start[q] + count[q];
  edge.resize(start[ns]);
  std::vector<uint32_t> fill(start.begin(), start.end() - 1);
  for (uint32_t k = 0; k < m; ++k) {
    int64_t s0, s1;
    range(k, &s0, &s1);
    for (int64_t q = s0; q <= s1; ++q) edge[fill[q]++] = k;
  }
  upload_u32(c, c->d_slab_start, start);
  upload_u32(c, c->d_slab_edge, edge);
  c->slab_ok = true;
}

// Edge cells for the arc weight and the safe radius (general polygons): a
// square grid of width w >= s_max/2 over the ring's bbox; cell (ix, iy) lists
// segment i (ring[i-1] -> ring[i]) unless the segment is farther than
// reach + half-diagonal from the cell center, i.e. farther than
// reach = s_max (1 + 4e-6) + 1e-9 S from every point of the cell.  For
// d <= s_max the reference rejects every unlisted segment.
double seg_dist(double px, double py, double ax, double ay, double bx, double by) {
  const double ex = bx - ax, ey = by - ay, l2 = ex * ex + ey * ey;
  double t = 0.0;
  if (l2 > 0.0) t = std::min(1.0, std::max(0.0, ((px - ax) * ex + (py - ay) * ey) / l2));
  const double qx = ax + t * ex - px, qy = ay + t * ey - py;
  return std::sqrt(qx * qx + qy * qy);
}

void build_edge_cells(stk_ctx* c) {
  const uint32_t m = c->nv;
  const double* r = c->ring.data();
  const double smax = c->s_values.back();
  const double S = c->pip_lim;
  const double reach = smax * (1.0 + 4e-6) + 1e-9 * S;
  const double W = c->xmax - c->xmin, H = c->ymax - c->ymin;
  const double ew = std::max(smax / 16.0, std::max(W, H) / 1024.0);
  const int nx = std::max(1, (int)std::ceil(W / ew)), ny = std::max(1, (int)std::ceil(H / ew));
  const double half_diag = ew * 0.70710678118654757 * (1.0 + 1e-9) + 1e-9 * S;
  c->ec_nx = nx;
  c->ec_ny = ny;
  c->ec_x0 = c->xmin;
  c->ec_y0 = c->ymin;
  c->ec_inv_w = 1.0 / ew;
  c->ec_dmax = smax;
  c->ec_reach = reach * (1.0 - 1e-9);
  const uint64_t cells = (uint64_t)nx * ny;
  // per cell: (lower, upper bound of the segment's distance from the cell's
  // points, segment)
  struct Entry {
    float lb, ub;
    uint32_t seg;
    bool operator<(const Entry& o) const { return lb < o.lb || (lb == o.lb && seg < o.seg); }
  };
  std::vector<std::vector<Entry>> lists(cells);
  for (uint32_t i = 0; i < m; ++i) {
    const uint32_t j = i == 0 ? m - 1 : i - 1;
    const double ax = r[2 * j], ay = r[2 * j + 1], bx = r[2 * i], by = r[2 * i + 1];
    const double lim = reach + half_diag;
    auto cell_lo = [&](double v, double v0) { return (int)std::floor((v - v0) / ew) - 1; };
    const int ix0 = std::max(0, cell_lo(std::min(ax, bx) - lim, c->xmin));
    const int ix1 = std::min(nx - 1, cell_lo(std::max(ax, bx) + lim, c->xmin) + 2);
    const int iy0 = std::max(0, cell_lo(std::min(ay, by) - lim, c->ymin));
    const int iy1 = std::min(ny - 1, cell_lo(std::max(ay, by) + lim, c->ymin) + 2);
    for (int iy = iy0; iy <= iy1; ++iy)
      for (int ix = ix0; ix <= ix1; ++ix) {
        const double cx = c->xmin + (ix + 0.5) * ew, cy = c->ymin + (iy + 0.5) * ew;
        const double dist = seg_dist(cx, cy, ax, ay, bx, by);
        if (dist <= lim) {
          // no point of the cell is nearer than dist - half_diag (rounded
          // down), none farther than the far endpoint + half_diag (rounded up)
          float lb = (float)std::max(0.0, (dist - half_diag) * (1.0 - 1e-9));
          if ((double)lb > std::max(0.0, dist - half_diag)) lb = std::nextafter(lb, 0.0f);
          const double far = std::max(std::hypot(ax - cx, ay - cy), std::hypot(bx - cx, by - cy));
          float ub = (float)((far + half_diag) * (1.0 + 1e-9));
          if ((double)ub < far + half_diag) ub = std::nextafter(ub, std::numeric_limits<float>::infinity());
          lists[(uint64_t)iy * nx + ix].push_back({lb, ub, i});
        }
      }
  }
  std::vector<uint32_t> start(cells + 1, 0), edge;
  std::vector<float> dmin, dmax;
  for (uint64_t q = 0; q < cells; ++q) start[q + 1] = start[q] + (uint32_t)lists[q].size();
  edge.reserve(start[cells]);
  dmin.reserve(start[cells]);
  dmax.reserve(start[cells]);
  for (auto& l : lists) {  // nearest first: a circle of radius d stops at the first lb > reach(d)
    std::sort(l.begin(), l.end());
    for (const Entry& e : l) {
      dmin.push_back(e.lb);
      dmax.push_back(e.ub);
      edge.push_back(e.seg);
    }
  }
  upload_u32(c, c->d_ec_start, start);
  upload_u32(c, c->d_ec_edge, edge);
  c->d_ec_dmin.ensure(std::max<size_t>(dmin.size(), 1));
  c->d_ec_dmax.ensure(std::max<size_t>(dmax.size(), 1));
  if (!dmin.empty()) {
    CK(cudaMemcpyAsync(c->d_ec_dmin.p, dmin.data(), sizeof(float) * dmin.size(),
                       cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_ec_dmax.p, dmax.data(), sizeof(float) * dmax.size(),
                       cudaMemcpyHostToDevice, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  c->ec_ok = true;
}

RegionView region_view(stk_ctx* c);

// A device-memory copy of a RegionView (pageable H2D: the source is consumed
// before cudaMemcpyAsync returns).
const RegionView* device_region(stk_ctx* c, const RegionView& rv) {
  if (!c->rv_dev_valid) {  // refreshed after stk_set_region / stk_set_grid only
    c->d_rv.ensure(1);
    CK(cudaMemcpyAsync(c->d_rv.p, &rv, sizeof(RegionView), cudaMemcpyHostToDevice, c->stream));
    c->rv_dev_valid = true;
  }
  return c->d_rv.p;
}

RegionView region_view(stk_ctx* c) {
  // STK_NO_SLABS / STK_NO_EDGE_CELLS (debugging): full-ring loops instead
  static const bool no_slabs = std::getenv("STK_NO_SLABS") != nullptr;
  static const bool no_ec = std::getenv("STK_NO_EDGE_CELLS") != nullptr;
  if (c->have_region && !c->fast_rect && !c->slab_ok && !no_slabs) build_slabs(c);
  if (c->have_region && c->have_grid && !c->fast_rect && !c->ec_ok && !no_ec) build_edge_cells(c);
  RegionView r;
  r.ring = c->d_ring.p;
  r.nv = c->nv;
  r.p0 = c->p0;
  r.p1 = c->p1;
  r.xmin = c->xmin;
  r.xmax = c->xmax;
  r.ymin = c->ymin;
  r.ymax = c->ymax;
  r.maxabs = c->maxabs;
  r.rect = c->fast_rect ? 1 : 0;
  // Largest coordinate magnitude a probe can have: the ring's plus the largest
  // distance (a probe is at distance d <= s_max from a center in the region).
  const double smax = c->s_values.empty() ? 0.0 : c->s_values.back();
  const double S = std::max(1.0, c->maxabs + smax);
  const double min_edge = std::max(std::min(c->xmax - c->xmin, c->ymax - c->ymin), 1e-300);
  r.box_m = 4e-12 * S * std::max(1.0, S / min_edge);
  for (int i = 0; i < 4; ++i) {
    r.rv[i] = (r.rect && c->ring.size() == 8) ? make_double2(c->ring[2 * i], c->ring[2 * i + 1])
                                              : make_double2(0.0, 0.0);
    r.sd_start[i] = r.sd_len[i] = 0.0;
  }
  if (r.rect && c->ring.size() == 8) {
    for (int i = 0; i < 4; ++i) {  // segment (ring[i-1], ring[i]) as the reference's loop
      const double ax = c->ring[2 * ((i + 3) & 3)], ay = c->ring[2 * ((i + 3) & 3) + 1];
      const double bx = c->ring[2 * i], by = c->ring[2 * i + 1];
      if (ax == bx) {  // vertical: x = xmin (side 0) or x = xmax (side 1)
        const int sd = ax == c->xmin ? 0 : 1;
        r.sd_start[sd] = ay;
        r.sd_len[sd] = by - ay;
      } else {         // horizontal: y = ymin (side 2) or y = ymax (side 3)
        const int sd = ay == c->ymin ? 2 : 3;
        r.sd_start[sd] = ax;
        r.sd_len[sd] = bx - ax;
      }
    }
  }
  // the closed form needs the reach margin d*1e-6 far above
  // coordinate rounding (d >= 1e-8 S) and the outside probe clear of every
  // on_segment tolerance (d - h > 4 box_m)
  r.sw_dmin = 1e-8 * S;
  r.sw_margin = 4.0 * r.box_m;
  r.sw_q_min = r.sw_dmin * r.sw_dmin * (1.0 + 1e-12);
  r.slab_start = c->slab_ok ? c->d_slab_start.p : nullptr;
  r.slab_edge = c->slab_ok ? c->d_slab_edge.p : nullptr;
  r.nslab = c->nslab;
  r.slab_y0 = c->slab_y0;
  r.slab_inv_h = c->slab_inv_h;
  r.pip_lim = c->pip_lim;
  r.pip_ylo = c->pip_ylo;
  r.pip_yhi = c->pip_yhi;
  r.ec_start = c->ec_ok ? c->d_ec_start.p : nullptr;
  r.ec_edge = c->ec_ok ? c->d_ec_edge.p : nullptr;
  r.ec_dmin = c->ec_ok ? c->d_ec_dmin.p : nullptr;
  r.ec_far = c->ec_ok ? c->d_ec_dmax.p : nullptr;
  r.ec_abs = 1e-9 * c->pip_lim;
  r.ec_nx = c->ec_nx;
  r.ec_ny = c->ec_ny;
  r.ec_x0 = c->ec_x0;
  r.ec_y0 = c->ec_y0;
  r.ec_inv_w = c->ec_inv_w;
  r.ec_dmax = c->ec_dmax;
  r.ec_reach = c->ec_reach;
  static const bool no_safe = std::getenv("STK_NO_SAFE_RADIUS") != nullptr;
  r.no_safe = no_safe ? 1 : 0;
  return r;
}

BinView bin_view(stk_ctx* c) {
  BinView b;
  b.Q = c->d_Q.p;
  b.T = c->d_T.p;
  b.q_tab = c->d_qtab.p;
  b.t_tab = c->d_ttab.p;
  b.cs = (uint32_t)c->s_values.size();
  b.ct = (uint32_t)c->t_values.size();
  b.Qmax = c->Q.back();
  b.Tmax = c->t_values.back();
  b.q_shift = c->q_shift;
  b.q_base = c->q_base;
  b.t_shift = c->t_shift;
  b.single_step = c->single_step ? 1 : 0;
  b.t_uni = c->t_uni;
  b.t_add = c->t_add;
  b.t_lo = c->t_lo;
  b.t_magic = c->t_magic;
  b.t_sh = c->t_sh;
  return b;
}

// Uniform grid with cells >= (s_max / R, t_max / R): every in-threshold
// neighbour of a point lies within R cells in each dimension.  R = 2 (finer
// cells: the half-stencil holds ~0.56x the candidates of R = 1) when the
// pattern is dense enough to fill the cells, else R = 1.
GridGeom make_grid_geom(stk_ctx* c, uint64_t n) {
  GridGeom g;
  const double smax = c->s_values.back();
  const int64_t tmax = c->t_values.back();
  const double ex = c->xmax - c->xmin, ey = c->ymax - c->ymin;
  const uint64_t cap = std::max<uint64_t>(4096, std::min<uint64_t>(2 * n, 1ull << 26));
  auto ncell = [](double extent, double width) {
    const double k = std::floor(extent / width) + 1.0;
    return (int64_t)std::min(k, 1e9);
  };
  for (int R = c->stencil_radius; R >= 1; --R) {
    // w * R = s_max * (1 + 1e-6): a true |dx| <= s_max (the computed d <= s_max
    // implies it up to 1e-16) spans at most R cells even after FP rounding of
    // the cell index; integer time cells of width ceil(t_max / R) are exact.
    double w = smax * (1.0 + 1e-6) / R;
    // time cells may be finer or coarser than space cells (RT layers; the
    // half-stencil's (R + 1) + RT (2R + 1) rows must fit a warp); the density
    // test below uses the population of cells with R time layers
    int RT = std::max(1, std::min(c->time_radius > 0 ? c->time_radius : R,
                                  (32 - (R + 1)) / (2 * R + 1)));
    int64_t tw, nx, ny, nt;
    auto size_cells = [&]() {
      tw = std::max<int64_t>((tmax + RT - 1) / RT, 1);
      for (;;) {
        nx = ncell(ex, w);
        ny = ncell(ey, w);
        nt = (c->p1 - c->p0) / tw + 1;
        if ((double)nx * (double)ny * (double)nt <= (double)cap) break;
        if (nx * ny >= nt) w *= 1.5; else tw = tw + tw / 2 + 1;
      }
    };
    size_cells();
    const double per_cell = (double)n / ((double)nx * ny * nt) * (double)RT / R;
    if (R > 1 && per_cell < c->min_cell_pop) continue;  // too sparse for finer cells
    // Finer space cells but too few points per cell for R time layers as well:
    // one time layer per t_max (twice the centers per item for 1.23x the
    // candidates).  Measured crossover on B200 at ~12.5 points per cell
    // (C2, 10 per cell: -5%; C4 at 800k points, 12.8: equal; C4, 16: +3.7%).
    if (R > 1 && c->time_radius <= 0 && RT > 1 && per_cell < c->min_cell_pop_t) {
      RT = 1;
      size_cells();
    }
    g.x0 = c->xmin;
    g.y0 = c->ymin;
    g.inv_w = 1.0 / w;
    g.t0 = c->p0;
    g.tw = tw;
    g.inv_tw = 1.0 / (double)tw;
    g.nx = (int32_t)nx;
    g.ny = (int32_t)ny;
    g.nt = (int32_t)nt;
    g.cells = (uint32_t)(nx * ny * nt);
    g.rs = R;
    g.rt = RT;
    break;
  }
  return g;
}

struct Plan {
  uint64_t n;
  GridGeom G;
  uint32_t bins;
  uint32_t max_items;
  int R;  // patterns per batch
};

Plan make_plan(stk_ctx* c, uint64_t n, uint64_t patterns) {
  Plan P;
  P.n = n;
  P.G = make_grid_geom(c, n);
  P.bins = (uint32_t)(c->s_values.size() * c->t_values.size());
  P.max_items = (uint32_t)((n + kItemCenters - 1) / kItemCenters + P.G.cells);
  const uint64_t per = n * (8 * 3 + 16 + 16 + 24 + 4 * 5) + (uint64_t)(P.G.cells + 1) * 4 * 3 +
                       (uint64_t)P.max_items * 8 + (uint64_t)P.bins * 8 * 6 + 64;
  uint64_t R = std::max<uint64_t>(1, c->mem_budget / per);
  R = std::min<uint64_t>(R, std::max<uint64_t>(patterns, 1));
  R = std::min<uint64_t>(R, 4096);
  // the pair kernel indexes a batch with 32-bit offsets (pattern * n + j etc.)
  const uint64_t widest = std::max<uint64_t>({n, (uint64_t)P.G.cells + 1, P.max_items});
  R = std::max<uint64_t>(1, std::min<uint64_t>(R, 0xffffffffull / widest));
  if (patterns > R) {  // equal batches: ceil(patterns / number of batches)
    const uint64_t nb = (patterns + R - 1) / R;
    R = (patterns + nb - 1) / nb;
  }
  P.R = (int)R;
  return P;
}

Batch alloc_batch(stk_ctx* c, const Plan& P) {
  const uint64_t R = P.R, n = P.n;
  c->x.ensure(R * n);
  c->y.ensure(R * n);
  c->t.ensure(R * n);
  const int wide = (c->p1 - c->p0) >= 0x7fffffffLL ? 1 : 0;
  c->pxy.ensure(R * n);
  if (c->fast_rect) c->parc.ensure(R * n);
  c->pmeta.ensure(R * n * (wide ? sizeof(PtMeta<int64_t>) : sizeof(PtMeta<int32_t>)));
  c->key.ensure(R * n);
  c->rank.ensure(R * n);
  c->sidx.ensure(R * n);
  c->cell_count.ensure(R * P.G.cells);
  c->cell_start.ensure(R * (P.G.cells + 1));
  c->item_start.ensure(R * (P.G.cells + 1));
  c->items.ensure(R * P.max_items);
  c->task_start.ensure(R + 1);
  c->task_counter.ensure(3);
  c->hist.ensure(R * P.bins * 4);
  c->stats.ensure(8);
  c->K.ensure(R * P.bins);
  c->L.ensure(R * P.bins);
  c->flags.ensure(R);
  Batch B;
  B.R = (int)R;
  B.n = n;
  B.x = c->x.p;
  B.y = c->y.p;
  B.t = c->t.p;
  B.pxy = c->pxy.p;
  B.parc = c->fast_rect ? c->parc.p : nullptr;
  B.pmeta = c->pmeta.p;
  B.wide = wide;
  B.key = c->key.p;
  B.rank = c->rank.p;
  B.perm = c->sidx.p;
  B.cell_count = c->cell_count.p;
  B.cell_start = c->cell_start.p;
  B.item_start = c->item_start.p;
  B.items = c->items.p;
  B.max_items = P.max_items;
  B.task_start = c->task_start.p;
  B.task_counter = c->task_counter.p;
  B.h_cnt = c->hist.p;
  B.h_half = c->hist.p + R * P.bins;
  B.h_lo = c->hist.p + 2 * R * P.bins;
  B.h_hi = c->hist.p + 3 * R * P.bins;
  B.K = c->K.p;
  B.L = c->L.p;
  B.stats = c->stats.p;
  B.flags = c->flags.p;
  B.n_sel = 0;
  B.shard = 0;
  B.nshards = 1;
  B.c0 = 0;
  B.c1 = ~0ULL;
  B.sel_start = nullptr;
  B.center_pos = nullptr;
  return B;
}

// Timing events of the pipeline.  cudaEventRecordExternal makes a record
// inside stream capture a real event-record node of the graph (a plain record
// there only expresses a dependency), so graph replays keep device timings.
cudaError_t rec_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  const cudaError_t q = cudaStreamIsCapturing(s, &st);
  if (q != cudaSuccess) return q;
  return st == cudaStreamCaptureStatusActive
             ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
             : cudaEventRecord(e, s);
}

struct Timers {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gen, grid, pair, fin;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
};

void require_ready(stk_ctx* c) {
  if (!c->have_region) throw StateErr("study region not set (stk_set_region)");
  if (!c->have_grid) throw StateErr("distance grid not set (stk_set_grid)");
}

// Check region.contains(p) for the n points at (dx,dy,dt) on the device.  No
// host round trip: the first failing index lands in c->bad, which the pair
// kernel reads to skip its work, and finish_call() raises the reference's
// invalid_argument before any output reaches the caller.
void validate_points(stk_ctx* c, const double* dx, const double* dy, const int64_t* dt,
                     uint64_t n) {
  c->bad.ensure(1);
  CK(cudaMemsetAsync(c->bad.p, 0xff, sizeof(unsigned long long), c->stream));
  const int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)c->num_sms * 16);
  validate_kernel<<<std::max(blocks, 1), 256, 0, c->stream>>>(dx, dy, dt, n, region_view(c),
                                                               c->bad.p);
  CK(cudaGetLastError());
  ++c->launches;
  c->check_points = true;
}

// Pinned staging of a call's host outputs (see stk_ctx::hstage).
void stage_reset(stk_ctx* c, size_t bytes) {
  c->outs.clear();
  c->hstage_used = 0;
  bytes += 256;
  if (bytes > c->hstage_cap) {
    if (c->hstage) cudaFreeHost(c->hstage);
    c->hstage = nullptr;
    c->hstage_cap = 0;
    CK(cudaHostAlloc((void**)&c->hstage, bytes, cudaHostAllocDefault));
    c->hstage_cap = bytes;
  }
}

// Enqueue a device -> staging copy whose bytes go to host `dst` at finish_call.
void* stage_d2h(stk_ctx* c, void* dst, const void* dsrc, size_t bytes, int field = -1,
                uint64_t elem = 0) {
  const size_t off = (c->hstage_used + 15) & ~size_t(15);
  if (off + bytes > c->hstage_cap) throw CudaFail("internal error: output staging overflow");
  CK(cudaMemcpyAsync(c->hstage + off, dsrc, bytes, cudaMemcpyDeviceToHost, c->stream));
  c->hstage_used = off + bytes;
  if (dst || field >= 0) c->outs.push_back({dst, field, elem, off, bytes});
  return c->hstage + off;
}

enum class Source { Observed, Csr, Bootstrap, Permutation };

// Fill patterns [p_first, p_first+count) of the batch.  Observed: copy from
// device pointers (count must be 1).  Otherwise realisation seeds seed0 + j.
void generate(stk_ctx* c, const Batch& B, Source src, int p_first, int count, uint64_t seed0,
              const double* ox, const double* oy, const int64_t* ot,
              unsigned long long* validate_into = nullptr) {
  if (count <= 0) return;
  const uint64_t n = B.n;
  if (src == Source::Observed) {  // one kernel for the three arrays (one graph node),
                                  // validating them on the way when asked
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)c->num_sms * 8);
    copy_points_kernel<<<std::max(blocks, 1u), 256, 0, c->stream>>>(
        B.x + (uint64_t)p_first * n, B.y + (uint64_t)p_first * n, B.t + (uint64_t)p_first * n,
        ox, oy, ot, n, region_view(c), validate_into);
    CK(cudaGetLastError());
    ++c->launches;
    return;
  }
  CK(cudaMemsetAsync(B.flags + p_first, 0, sizeof(int) * count, c->stream));
  if (c->rng == STK_RNG_PHILOX) {  // opt-in counter-based generator (statistical parity)
    const dim3 gp((unsigned)((n + 255) / 256), (unsigned)count);
    if (src == Source::Csr) {
      const uint64_t ntl = (uint64_t)(c->p1 - c->p0) + 1;
      csr_philox_kernel<<<gp, 256, 0, c->stream>>>(B, p_first, seed0, region_view(c), ntl);
    } else if (src == Source::Bootstrap) {
      bootstrap_philox_kernel<<<gp, 256, 0, c->stream>>>(B, p_first, seed0, ox, oy, ot);
    } else {
      throw Unsupported("permutation draws Fisher-Yates on the reference's sequential stream; "
                        "the Philox generator covers CSR and bootstrap");
    }
    CK(cudaGetLastError());
    ++c->launches;
    return;
  }
  if (src == Source::Csr) {
    const uint64_t ntl = (uint64_t)(c->p1 - c->p0) + 1;  // uniform_int(p0, p1)
    const uint64_t limit = ~0ULL - (~0ULL % ntl);
    const RegionView rv = region_view(c);
    if (c->fast_rect) {
      csr_gen_kernel<<<count, kGenThreads, 0, c->stream>>>(B, p_first, seed0, rv.xmin, rv.xmax, rv.ymin,
                                                   rv.ymax);
      CK(cudaGetLastError());
      ++c->launches;
      const dim3 gf((unsigned)((n + 255) / 256), (unsigned)count);
      csr_finish_kernel<<<gf, 256, 0, c->stream>>>(B, p_first, rv, ntl, ~0ULL / ntl, limit);
    } else {
      csr_poly_kernel<<<count, 320, 0, c->stream>>>(B, p_first, seed0, rv, ntl, limit);
    }
    CK(cudaGetLastError());
    ++c->launches;
    // patterns a parallel kernel flagged (probability ~0): sequential, exact
    csr_seq_kernel<<<(count + 31) / 32, 32, 0, c->stream>>>(B, p_first, count, seed0, rv, ntl,
                                                            limit, 0);
    CK(cudaGetLastError());
  ++c->launches;
  } else if (src == Source::Bootstrap) {
    const uint64_t limit = ~0ULL - (~0ULL % n);
    bootstrap_kernel<<<count, 320, 0, c->stream>>>(B, p_first, seed0, ox, oy, ot, limit);
    CK(cudaGetLastError());
  ++c->launches;
    resample_seq_kernel<<<(count + 31) / 32, 32, 0, c->stream>>>(B, p_first, count, seed0, ox,
                                                                 oy, ot, 1);
    CK(cudaGetLastError());
  ++c->launches;
  } else {
    // permutation: parallel Fisher-Yates (stk_kernels.cu perm_*), bit-exact; a
    // realisation whose stream hits a below() rejection reruns sequentially
    static const bool seq = std::getenv("STK_SEQ_PERMUTATION") != nullptr;
    if (seq) {
      resample_seq_kernel<<<(count + 31) / 32, 32, 0, c->stream>>>(B, p_first, count, seed0, ox,
                                                                   oy, ot, 2);
      CK(cudaGetLastError());
      ++c->launches;
      return;
    }
    const uint64_t cn = (uint64_t)count * n, cn1 = (uint64_t)count * (n + 1);
    c->perm.ensure(4 * cn + 2 * cn1);
    uint32_t* J = c->perm.p;
    uint32_t* cnt = J + cn;
    uint32_t* rank = cnt + cn;
    uint32_t* list = rank + cn;
    uint32_t* start = list + cn;
    uint32_t* istart = start + cn1;
    c->perm_mx.ensure(1);
    perm_draw_kernel<<<count, 320, 0, c->stream>>>(B, p_first, seed0, J);
    CK(cudaMemsetAsync(cnt, 0, 4 * cn, c->stream));
    const dim3 g((unsigned)((n + 255) / 256), (unsigned)count);
    perm_count_kernel<<<g, 256, 0, c->stream>>>(n, J, cnt, rank);
    c->scan_part.ensure(scan_scratch((uint32_t)n, (unsigned)count));
    c->launches += scan_launch(cnt, start, istart, (uint32_t)n, (unsigned)count, c->perm_mx.p,
                               c->scan_part.p, c->stream) - 1;
    perm_scatter_kernel<<<g, 256, 0, c->stream>>>(n, J, start, rank, list);
    perm_sort_kernel<<<g, 256, 0, c->stream>>>(n, start, list);
    perm_final_kernel<<<g, 256, 0, c->stream>>>(B, p_first, ox, oy, ot, J, start, list);
    resample_seq_kernel<<<(count + 31) / 32, 32, 0, c->stream>>>(B, p_first, count, seed0, ox,
                                                                 oy, ot, 3);
    CK(cudaGetLastError());
    c->launches += 7;
  }
}

// Resident pair-kernel CTAs per SM for (wide, mode, smem), cached per context.
// The function's dynamic shared-memory limit is raised to the largest size
// requested so far, so every cached configuration stays launchable.
int pair_occupancy(stk_ctx* c, int wide, int mode, size_t smem) {
  size_t mx = smem;
  for (const auto& o : c->occ) {
    if (o.wide == wide && o.mode == mode && o.smem == smem) return o.per_sm;
    if (o.wide == wide && o.mode == mode) mx = std::max(mx, o.smem);
  }
  int per_sm = 0;
  CK(pair_kernel_prepare(wide, mode, smem, mx, &per_sm));
  if (per_sm < 1) throw Unsupported("distance grid too large for the pair kernel's shared histogram");
  c->occ.push_back({wide, mode, smem, per_sm});
  return per_sm;
}

// Grid build + pair kernel + finalize for patterns [0, R) of the batch.
// Grid build + pair kernel (+ finalize) for the batch.  Center selection
// (shard of nshards by input index, and input-index range [c0, c1)) applies to
// patterns [0, n_sel).
void run_batch(stk_ctx* c, const Plan& P, Batch& B, Timers& tm, int n_sel, uint32_t shard,
               uint32_t nshards, uint64_t c0, uint64_t c1, bool finalize,
               unsigned long long* obs_raw = nullptr, double* obs_kl = nullptr) {
  const GridGeom& G = P.G;
  const int R = B.R;
  cudaEvent_t e0 = c->ev(), e1 = c->ev(), e2 = c->ev();
  CK(rec_event(e0, c->stream));
  CK(cudaMemsetAsync(B.cell_count, 0, sizeof(uint32_t) * (uint64_t)R * G.cells, c->stream));
  CK(cudaMemsetAsync(B.h_cnt, 0, sizeof(unsigned long long) * (uint64_t)R * P.bins * 4, c->stream));
  // K1 point kernels: 4 points per thread (kK1Per), 1,024 per CTA
  dim3 gp((unsigned)((B.n + 1023) / 1024), (unsigned)R);
  key_kernel<<<gp, 256, 0, c->stream>>>(B, G, 0);
  CK(cudaGetLastError());
  ++c->launches;
  c->scan_part.ensure(scan_scratch(G.cells, (unsigned)R));
  c->launches += scan_launch(B.cell_count, B.cell_start, B.item_start, G.cells, (unsigned)R,
                             B.stats + 5, c->scan_part.p, c->stream);
  CK(cudaGetLastError());
  place_kernel<<<gp, 256, 0, c->stream>>>(B, G, 0);
  CK(cudaGetLastError());
  ++c->launches;
  uint64_t qbits;
  std::memcpy(&qbits, &c->Q.back(), 8);
  gather_kernel<<<gp, 256, 0, c->stream>>>(B, region_view(c), 0, (uint32_t)(qbits >> 32));
  CK(cudaGetLastError());
  ++c->launches;
  B.n_sel = std::min(n_sel, R);
  B.shard = shard;
  B.nshards = std::max<uint32_t>(nshards, 1);
  B.c0 = c0;
  B.c1 = c1;
  if (B.n_sel > 0) {
    c->sel_start.ensure((uint64_t)B.n_sel * (G.cells + 1));
    c->center_pos.ensure((uint64_t)B.n_sel * B.n);
    B.sel_start = c->sel_start.p;
    B.center_pos = c->center_pos.p;
    CK(cudaMemsetAsync(B.cell_count, 0, sizeof(uint32_t) * (uint64_t)B.n_sel * G.cells, c->stream));
    dim3 gs((unsigned)((B.n + 255) / 256), (unsigned)B.n_sel);
    select_count_kernel<<<gs, 256, 0, c->stream>>>(B, G);
    CK(cudaGetLastError());
    ++c->launches;
    c->launches += scan_launch(B.cell_count, B.sel_start, B.item_start, G.cells,
                               (unsigned)B.n_sel, B.stats + 5, c->scan_part.p, c->stream);
    CK(cudaGetLastError());
    select_scatter_kernel<<<gs, 256, 0, c->stream>>>(B, G);
    CK(cudaGetLastError());
    ++c->launches;
  }
  dim3 gc((G.cells + 255) / 256, (unsigned)R);
  items_kernel<<<gc, 256, 0, c->stream>>>(B, G, 0);
  CK(cudaGetLastError());
  ++c->launches;
  const size_t smem = pair_kernel_smem(P.bins, B.wide);
  // bit 2: q table single-step and evenly spaced time thresholds (32-bit lags)
  const bool tuni = c->t_uni && !B.wide && c->q_single;
  const int mode = (c->fast_rect ? 1 : 0) | ((c->single_step || tuni) ? 2 : 0) | (tuni ? 4 : 0);
  const int per_sm = pair_occupancy(c, B.wide, mode, smem);
  tasks_kernel<<<1, 1, 0, c->stream>>>(B, G, (uint32_t)(c->num_sms * per_sm));
  CK(cudaGetLastError());
  ++c->launches;
  CK(rec_event(e1, c->stream));

  PairArgs A;
  A.B = B;
  A.G = G;
  A.bins = bin_view(c);
  A.reg = region_view(c);
  A.reg_g = device_region(c, A.reg);
  A.abort_flag = c->check_points ? c->bad.p : nullptr;
  const uint64_t ctas = (uint64_t)c->num_sms * per_sm;
  c->arcq.ensure(ctas * kPairWarps * (kArcRing + kCplxRing));
  A.B.arcq = c->arcq.p;
  // crossing scratch of the general weight: <= 8 crossings per lane (more use
  // the bounded-storage fallback), global and L1-resident
  c->angs.ensure(ctas * kPairWarps * kAngleSlots * 32);
  A.angs_g = c->angs.p;
  pair_kernel_launch(B.wide, mode, (unsigned)ctas, smem, c->stream, A);
  CK(cudaGetLastError());
  ++c->launches;
  CK(rec_event(e2, c->stream));
  tm.grid.push_back({e0, e1});
  tm.pair.push_back({e1, e2});
  if (finalize) {
    cudaEvent_t e3 = c->ev();
    finalize_kernel<<<R, 256, 0, c->stream>>>(B, A.bins.cs, A.bins.ct, c->d_s.p, c->d_T.p,
                                              c->area, c->duration, 0, obs_raw, obs_kl);
    CK(cudaGetLastError());
  ++c->launches;
    CK(rec_event(e3, c->stream));
    tm.fin.push_back({e2, e3});
  }
}

double elapsed(const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
  double s = 0;
  for (auto& pr : v) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) s += ms;
    else (void)cudaGetLastError();  // never leave a sticky error for the next CK
  }
  return s;
}

// The pipeline shared by estimate / simulate / run_job: an optional observed
// pattern (device pointers) followed by realisations [r_begin, r_end).
struct JobOut {
  double* k_obs = nullptr;   // host
  double* l_obs = nullptr;   // host
  double* l_all = nullptr;   // host (r_end - r_begin) * bins
  double* upper = nullptr;   // host
  double* lower = nullptr;   // host
  double* diff = nullptr;    // host
  uint64_t* obs_counts = nullptr;  // host: exact pre-cumulative results of the observed
  uint64_t* obs_hi = nullptr;      //       pattern (or of its shard)
  uint64_t* obs_lo = nullptr;
  // collective (stk_run_job_dist): this rank computed shard `rank` of the
  // observed pattern's pairs and its block of the realisations; the exact
  // all-reduces over the context's communicator combine them on the device
  bool dist = false;
  uint32_t sims_total = 0;   // realisations of the whole job (dist)
  bool validate = false;     // run validate_kernel on the observed points first
};

enum JobField { F_K = 0, F_L, F_LALL, F_UP, F_LO, F_DIFF };
double* field_ptr(const JobOut& o, int f) {
  switch (f) {
    case F_K: return o.k_obs;
    case F_L: return o.l_obs;
    case F_LALL: return o.l_all;
    case F_UP: return o.upper;
    case F_LO: return o.lower;
    default: return o.diff;
  }
}



// End of a call: ONE synchronisation, then the checks in the reference's order
// (invalid points first: estimator.cpp:123-127 throws before any work), then
// the staged outputs go to the caller's buffers and the telemetry is added.
void finish_call(stk_ctx* c, Timers& tm, stk_telemetry* tel, uint64_t patterns,
                 const JobOut* jo = nullptr) {
  const unsigned long long* st =
      (const unsigned long long*)stage_d2h(c, nullptr, c->stats.p, 8 * sizeof(unsigned long long));
  const unsigned long long* bad =
      c->check_points ? (const unsigned long long*)stage_d2h(c, nullptr, c->bad.p, 8) : nullptr;
  CK(cudaStreamSynchronize(c->stream));
  c->check_points = false;
  if (bad && *bad != ~0ULL) throw InvalidArg("point outside study region or period");
  // stats[3]: bit 1 = arc ring overflow (pair kernel), bit 0 = more crossings
  // than the rectangle weight's buffer holds; neither can happen by
  // construction (<= 31 + kArcChunk*64 ring entries; <= 8 crossings on 4 sides)
  if (st[3] & 2) throw CudaFail("internal error: arc ring overflow in the pair kernel");
  if (st[3] & 1) throw CudaFail("internal error: crossing buffer overflow in the rectangle edge weight");
  if (st[3] & 8)
    throw Unsupported("a grid cell's stencil holds more points than the pair kernel's 32-bit "
                      "per-task counters can take (about 3e7 in one cell)");
  if (st[3] & 4)
    throw Unsupported("Philox CSR: 4096 rejections for one point (the region covers too small a "
                      "share of its bounding box)");
  for (const auto& o : c->outs) {
    void* dst = o.field >= 0 ? (void*)(field_ptr(*jo, o.field) + o.elem) : o.dst;
    if (dst) std::memcpy(dst, c->hstage + o.off, o.bytes);
  }
  c->outs.clear();
  if (!tel) return;
  tel->in_threshold_pairs += st[0];
  tel->candidate_pairs += st[1];
  tel->exact_path_pairs += st[2];
  tel->arc_pairs += st[4];
  tel->patterns += patterns;
  tel->batches += tm.pair.size();
  tel->kernel_launches += c->launches;
  tel->gen_ms += elapsed(tm.gen);
  tel->grid_ms += elapsed(tm.grid);
  tel->pair_ms += elapsed(tm.pair);
  tel->finalize_ms += elapsed(tm.fin);
  if (tm.t0 && tm.t1) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, tm.t0, tm.t1) == cudaSuccess) tel->total_ms += ms;
    else (void)cudaGetLastError();
  }
}

Source source_of(int method) {
  switch (method) {
    case STK_METHOD_CSR: return Source::Csr;
    case STK_METHOD_BOOTSTRAP: return Source::Bootstrap;
    case STK_METHOD_PERMUTATION: return Source::Permutation;
  }
  throw InvalidArg("unknown simulation method");
}

// Exact exchange of the observed partials and the partial envelopes over the
// context's NCCL communicator, then finalize / diff on the device (the
// reference's DistributedExecutor gather + aggregate, distributed.cpp:197-245,
// runtime.cpp:119-136, done as two exact all-reduces: bit-identical at any
// GPU count).
void exchange(stk_ctx* c, const Plan& P, uint64_t n, bool have_env, uint32_t sims_total) {
  const uint32_t bins = P.bins;
  const unsigned g = (bins + 255) / 256;
  unsigned long long* raw = c->obsraw.p;
  c->limbs.ensure(6 * (uint64_t)bins);
  pack_exact_kernel<<<g, 256, 0, c->stream>>>(raw, raw + bins, raw + 2 * bins, raw + 3 * bins,
                                              bins, c->limbs.p);
  CK(cudaGetLastError());
  ++c->launches;
  if (sims_total > 0 && !have_env) {  // no realisations on this rank: neutral elements
    fill_kernel<<<g, 256, 0, c->stream>>>(c->env.p, bins, -INFINITY);
    fill_kernel<<<g, 256, 0, c->stream>>>(c->env.p + bins, bins, INFINITY);
    CK(cudaGetLastError());
    c->launches += 2;
  }
  const NcclApi& api = nccl();
  NK(api.group_start());
  NK(api.all_reduce(c->limbs.p, c->limbs.p, 6 * (size_t)bins, ncclUint64, ncclSum, c->comm,
                    c->stream));
  if (sims_total > 0) {
    NK(api.all_reduce(c->env.p, c->env.p, bins, ncclFloat64, ncclMax, c->comm, c->stream));
    NK(api.all_reduce(c->env.p + bins, c->env.p + bins, bins, ncclFloat64, ncclMin, c->comm,
                      c->stream));
  }
  NK(api.group_end());
  unpack_exact_kernel<<<g, 256, 0, c->stream>>>(c->limbs.p, bins, raw, raw + bins,
                                                raw + 2 * bins, raw + 3 * bins);
  CK(cudaGetLastError());
  ++c->launches;
  Batch F{};
  F.R = 1;
  F.n = n;
  F.h_cnt = raw;
  F.h_half = raw + bins;
  F.h_lo = raw + 2 * bins;
  F.h_hi = raw + 3 * bins;
  F.K = c->obs.p;
  F.L = c->obs.p + bins;
  finalize_kernel<<<1, 256, 0, c->stream>>>(F, (uint32_t)c->s_values.size(),
                                            (uint32_t)c->t_values.size(), c->d_s.p, c->d_T.p,
                                            c->area, c->duration, 0, nullptr, nullptr);
  CK(cudaGetLastError());
  ++c->launches;
}

// What one enqueue of the pipeline leaves for the host epilogue (kept with a
// captured graph so a replay needs no re-enqueue).
struct PipeInfo {
  Timers tm;
  uint64_t patterns = 0;
  uint64_t launches = 0;
  const void* raw_host = nullptr;  // staged observed sums (obs_counts requested)
  uint32_t bins = 0;
  bool validated = false;
  std::vector<stk_ctx::Out> outs;
};

// Enqueue the whole pipeline on the context stream (no host synchronisation).
PipeInfo enqueue_pipeline(stk_ctx* c, const double* dx, const double* dy, const int64_t* dt,
                          uint64_t n, bool with_observed, int method, uint64_t base_seed,
                          uint32_t r_begin, uint32_t r_end, const JobOut& out,
                          uint32_t obs_shard, uint32_t obs_nshards, const Plan& P) {
  PipeInfo info;
  c->evnext = 0;
  Timers& tm = info.tm;
  tm.t0 = c->ev();
  tm.t1 = c->ev();
  CK(rec_event(tm.t0, c->stream));
  const uint64_t sims = r_end > r_begin ? r_end - r_begin : 0;
  const uint64_t patterns = (with_observed ? 1 : 0) + sims;
  info.patterns = patterns;
  const Source src = source_of(method);
  const uint32_t bins = P.bins;
  info.bins = bins;
  // the observed pattern is validated by its copy-in kernel (no separate pass)
  const bool fuse_validate = out.validate && with_observed;
  if (fuse_validate) {
    c->bad.ensure(1);
    CK(cudaMemsetAsync(c->bad.p, 0xff, sizeof(unsigned long long), c->stream));
    c->check_points = true;
  } else if (out.validate) {
    validate_points(c, dx, dy, dt, n);
  }
  info.validated = c->check_points;
  CK(cudaMemsetAsync(c->stats.p, 0, sizeof(unsigned long long) * 8, c->stream));
  bool env_init = true;
  uint64_t done = 0;
  uint32_t next_r = r_begin;
  while (done < patterns) {
    const uint64_t R = std::min<uint64_t>((uint64_t)P.R, patterns - done);
    Plan PB = P;
    PB.R = (int)R;
    Batch B = alloc_batch(c, PB);
    int p = 0;
    cudaEvent_t g0 = c->ev(), g1 = c->ev();
    CK(rec_event(g0, c->stream));
    const bool obs_here = with_observed && done == 0;
    if (obs_here) {
      generate(c, B, Source::Observed, 0, 1, 0, dx, dy, dt, fuse_validate ? c->bad.p : nullptr);
      p = 1;
    }
    const int nsim = (int)(R - (obs_here ? 1 : 0));
    generate(c, B, src, p, nsim, base_seed + next_r, dx, dy, dt);
    CK(rec_event(g1, c->stream));
    tm.gen.push_back({g0, g1});
    // finalize also keeps the observed pattern's exact sums and its K, L
    run_batch(c, PB, B, tm, (obs_here && obs_nshards > 1) ? 1 : 0, obs_shard, obs_nshards, 0,
              ~0ULL, true, obs_here ? c->obsraw.p : nullptr, obs_here ? c->obs.p : nullptr);
    cudaEvent_t f0 = c->ev(), f1 = c->ev();
    CK(rec_event(f0, c->stream));
    if (nsim > 0) {
      envelope_kernel<<<(bins + 255) / 256, 256, 0, c->stream>>>(
          B, bins, p, nsim, env_init ? 1 : 0, c->env.p, c->env.p + bins);
      CK(cudaGetLastError());
      ++c->launches;
      env_init = false;
      if (out.l_all)
        stage_d2h(c, nullptr, B.L + (uint64_t)p * bins, sizeof(double) * bins * nsim, F_LALL,
                  (uint64_t)(next_r - r_begin) * bins);
    }
    CK(rec_event(f1, c->stream));
    tm.fin.push_back({f0, f1});
    next_r += (uint32_t)nsim;
    done += R;
  }
  const uint32_t sims_job = out.dist ? out.sims_total : (uint32_t)sims;
  if (with_observed && out.obs_counts)  // this rank's own observed sums, before any exchange
    info.raw_host = stage_d2h(c, nullptr, c->obsraw.p, 32 * (uint64_t)bins);
  if (out.dist) exchange(c, P, n, sims > 0, sims_job);
  if (with_observed && sims_job > 0 && out.diff) {
    diff_kernel<<<(bins + 255) / 256, 256, 0, c->stream>>>(c->obs.p + bins, c->env.p, bins,
                                                           c->scratch.p);
    CK(cudaGetLastError());
    ++c->launches;
    stage_d2h(c, nullptr, c->scratch.p, sizeof(double) * bins, F_DIFF);
  }
  if (with_observed && out.k_obs) stage_d2h(c, nullptr, c->obs.p, sizeof(double) * bins, F_K);
  if (with_observed && out.l_obs)
    stage_d2h(c, nullptr, c->obs.p + bins, sizeof(double) * bins, F_L);
  if (sims_job > 0 && out.upper) stage_d2h(c, nullptr, c->env.p, sizeof(double) * bins, F_UP);
  if (sims_job > 0 && out.lower)
    stage_d2h(c, nullptr, c->env.p + bins, sizeof(double) * bins, F_LO);
  CK(rec_event(tm.t1, c->stream));
  info.launches = c->launches;
  info.outs = c->outs;
  return info;
}

// Everything a captured pipeline depends on besides the context's region /
// grid / budget (whose setters drop the graph): a replay needs all equal.
struct PipeKey {
  const void *dx = nullptr, *dy = nullptr, *dt = nullptr;
  uint64_t n = 0, seed = 0, gen = 0;
  int method = 0;
  uint32_t r_begin = 0, r_end = 0, shard = 0, nshards = 0;
  unsigned flags = 0;
  const void* hstage = nullptr;
  bool operator==(const PipeKey& o) const {
    return dx == o.dx && dy == o.dy && dt == o.dt && n == o.n && seed == o.seed &&
           gen == o.gen && method == o.method && r_begin == o.r_begin && r_end == o.r_end &&
           shard == o.shard && nshards == o.nshards && flags == o.flags && hstage == o.hstage;
  }
};

struct GraphCache {
  cudaGraphExec_t exec = nullptr;
  PipeKey key, last;  // key of the captured graph; key of the last plain call
  PipeInfo info;
  ~GraphCache() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

void drop_graph(stk_ctx* c) { c->graph.reset(); }

// The pipeline shared by estimate / simulate / run_job: an optional observed
// pattern (device pointers) followed by realisations [r_begin, r_end).
// Small single-batch jobs repeated with identical arguments (a service loop,
// the bench, one rank's share of C2 at 8 GPUs) are captured as one CUDA graph
// on the second identical call and replayed after that: one launch and one
// synchronisation per call instead of ~30 API calls.
void run_pipeline(stk_ctx* c, const double* dx, const double* dy, const int64_t* dt, uint64_t n,
                  bool with_observed, int method, uint64_t base_seed, uint32_t r_begin,
                  uint32_t r_end, const JobOut& out, stk_telemetry* tel,
                  uint32_t obs_shard = 0, uint32_t obs_nshards = 1) {
  require_ready(c);
  const uint64_t sims = r_end > r_begin ? r_end - r_begin : 0;
  const uint64_t patterns = (with_observed ? 1 : 0) + sims;
  const Plan P = make_plan(c, n, patterns);
  const uint32_t bins = P.bins;
  stage_reset(c, 8 * (uint64_t)bins * (5 + 4 + (out.l_all ? sims : 0)) + 128);
  c->env.ensure(2 * (uint64_t)bins);
  c->obs.ensure(2 * (uint64_t)bins);
  c->obsraw.ensure(4 * (uint64_t)bins);
  c->scratch.ensure(bins);
  static const bool no_graph = std::getenv("STK_NO_GRAPH") != nullptr;
  const bool graphable = !no_graph && !out.dist && patterns <= (uint64_t)P.R &&
                         n * patterns <= (32ull << 20);
  PipeKey key;
  if (graphable) {
    key.dx = dx; key.dy = dy; key.dt = dt; key.n = n; key.seed = base_seed;
    key.method = method; key.r_begin = r_begin; key.r_end = r_end;
    key.shard = obs_shard; key.nshards = obs_nshards; key.hstage = c->hstage;
    key.flags = (with_observed ? 1u : 0u) | (out.validate ? 2u : 0u) | (out.k_obs ? 4u : 0u) |
                (out.l_obs ? 8u : 0u) | (out.l_all ? 16u : 0u) | (out.upper ? 32u : 0u) |
                (out.lower ? 64u : 0u) | (out.diff ? 128u : 0u) | (out.obs_counts ? 256u : 0u);
    key.gen = g_alloc_gen;
  }
  PipeInfo info;
  bool replayed = false;
  if (graphable && !c->graph) c->graph = std::make_unique<GraphCache>();
  GraphCache* gc = c->graph.get();
  if (graphable && gc->exec && gc->key == key) {
    CK(cudaGraphLaunch(gc->exec, c->stream));
    info = gc->info;
    replayed = true;
  } else if (graphable && gc->last == key) {
    // second identical call: capture (nothing allocates: same sizes as the last call)
    if (gc->exec) cudaGraphExecDestroy(gc->exec);
    gc->exec = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    cudaGraph_t graph = nullptr;
    try {
      info = enqueue_pipeline(c, dx, dy, dt, n, with_observed, method, base_seed, r_begin, r_end,
                              out, obs_shard, obs_nshards, P);
    } catch (...) {
      cudaStreamEndCapture(c->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess || g_alloc_gen != key.gen) {  // not replayable: run it plainly
      (void)cudaGetLastError();
      if (exec) cudaGraphExecDestroy(exec);
      c->launches = 0;
      c->outs.clear();
      c->hstage_used = 0;
      info = enqueue_pipeline(c, dx, dy, dt, n, with_observed, method, base_seed, r_begin, r_end,
                              out, obs_shard, obs_nshards, P);
    } else {
      gc->exec = exec;
      gc->key = key;
      gc->info = info;
      CK(cudaGraphLaunch(exec, c->stream));
      replayed = true;
    }
  } else {
    info = enqueue_pipeline(c, dx, dy, dt, n, with_observed, method, base_seed, r_begin, r_end,
                            out, obs_shard, obs_nshards, P);
    if (graphable) {
      gc->last = key;
      gc->last.gen = g_alloc_gen;  // as left by this call's allocations
    }
  }
  if (replayed) {
    c->launches = info.launches;
    c->outs = info.outs;
    c->check_points = info.validated;
    c->hstage_used = 0;
    for (const auto& o : info.outs) c->hstage_used = std::max(c->hstage_used, o.off + o.bytes);
    if (info.raw_host)
      c->hstage_used = std::max(c->hstage_used, (size_t)((const unsigned char*)info.raw_host -
                                                         c->hstage) + 32 * (size_t)bins);
  }
  finish_call(c, info.tm, tel, info.patterns, &out);
  if (info.raw_host) {
    const unsigned long long* r = (const unsigned long long*)info.raw_host;
    for (uint32_t i = 0; i < bins; ++i) {
      const unsigned long long raw = r[i], half = r[bins + i], lo = r[2 * bins + i],
                               hi = r[3 * bins + i];
      const unsigned long long cnt = raw & ~1ULL;
      out.obs_counts[i] = cnt;
      const unsigned __int128 v = ((unsigned __int128)hi << 64 | lo) +
                                  ((unsigned __int128)(cnt + half) << kFixedFracBits) +
                                  ((raw & 1ULL) ? kInfSentinel : (unsigned __int128)0);
      if (out.obs_hi) out.obs_hi[i] = (uint64_t)(v >> 64);
      if (out.obs_lo) out.obs_lo[i] = (uint64_t)v;
    }
  }
}

template <class F>
int guarded(stk_ctx* c, F&& f) {
  if (!c) return STK_ESTATE;
  try {
    CK(cudaSetDevice(c->device));
    c->launches = 0;
    c->check_points = false;
    c->outs.clear();
    f();
    c->err.clear();
    return STK_OK;
  } catch (const InvalidArg& e) {
    c->err = e.what();
    return STK_EINVAL;
  } catch (const Unsupported& e) {
    c->err = e.what();
    return STK_EUNSUPPORTED;
  } catch (const StateErr& e) {
    c->err = e.what();
    return STK_ESTATE;
  } catch (const NcclFail& e) {
    c->err = e.what();
    return STK_ENCCL;
  } catch (const std::exception& e) {
    c->err = e.what();
    return STK_ECUDA;
  }
}

// Upload the host observed pattern into the context's staging buffers.
void upload_points(stk_ctx* c, const double* x, const double* y, const int64_t* t, uint64_t n) {
  c->sx.ensure(n);
  c->sy.ensure(n);
  c->st.ensure(n);
  CK(cudaMemcpyAsync(c->sx.p, x, n * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->sy.p, y, n * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->st.p, t, n * 8, cudaMemcpyHostToDevice, c->stream));
}

void check_n(uint64_t n) {
  if (n < 2) throw InvalidArg("K estimation needs n >= 2");
  if (n > 0xFFFFFFF0ull) throw Unsupported("more than 2^32 points per pattern");
}

}  // namespace

// =====================================================================
extern "C" {

const char* stk_version(void) { return "stk 0.1 (sm_100a)"; }

int stk_create(stk_ctx** out, int device) {
  if (!out) return STK_EINVAL;
  *out = nullptr;
  stk_ctx* c = new stk_ctx();
  c->device = device;
  try {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (const char* r = std::getenv("STK_STENCIL_RADIUS")) c->stencil_radius = std::max(1, std::min(4, std::atoi(r)));
    if (const char* r = std::getenv("STK_MIN_CELL_POP")) c->min_cell_pop = std::atof(r);
    if (const char* r = std::getenv("STK_MIN_CELL_POP_T")) c->min_cell_pop_t = std::atof(r);
    if (const char* r = std::getenv("STK_TIME_RADIUS")) c->time_radius = std::max(0, std::min(8, std::atoi(r)));
    {  // batch budget: 40% of the free device memory, between 4 and 64 GiB (a B200's
       // 180 GB gives 64 GiB: C5 runs 3 batches of 67 patterns instead of 12 of 17, so
       // the one-CTA-per-realisation generators and the pair kernel's tail see 4x the work)
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
        c->mem_budget = std::min<uint64_t>(64ull << 30, std::max<uint64_t>(4ull << 30, fr / 5 * 2));
      else
        (void)cudaGetLastError();
    }
    c->stats.ensure(8);
  } catch (const std::exception& e) {
    delete c;
    return STK_ECUDA;
  }
  *out = c;
  return STK_OK;
}

void stk_destroy(stk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto e : c->evpool) cudaEventDestroy(e);
  c->d_ring.release(); c->d_Q.release(); c->d_s.release(); c->d_T.release();
  c->d_qtab.release(); c->d_ttab.release();
  c->x.release(); c->y.release(); c->t.release();
  c->pxy.release(); c->parc.release(); c->pmeta.release(); c->key.release(); c->rank.release(); c->sidx.release();
  c->cell_count.release(); c->cell_start.release(); c->item_start.release();
  c->task_start.release(); c->task_counter.release(); c->items.release();
  c->hist.release(); c->stats.release(); c->bad.release(); c->K.release(); c->L.release();
  c->env.release(); c->obs.release(); c->flags.release(); c->ovf.release();
  c->sel_start.release(); c->center_pos.release(); c->arcq.release(); c->angs.release();
  c->scratch.release(); c->sx.release(); c->sy.release(); c->st.release();
  c->graph.reset();
  c->obsraw.release(); c->limbs.release(); c->d_rv.release();
  c->perm.release(); c->perm_mx.release(); c->scan_part.release();
  if (c->comm) nccl().comm_destroy(c->comm);
  if (c->hstage) cudaFreeHost(c->hstage);
  cudaStreamDestroy(c->stream);
  delete c;
}

const char* stk_last_error(const stk_ctx* c) { return c ? c->err.c_str() : "null context"; }

void* stk_stream(stk_ctx* c) { return c ? (void*)c->stream : nullptr; }

int stk_set_memory_budget(stk_ctx* c, uint64_t bytes) {
  return guarded(c, [&] {
    if (bytes < (1ull << 20)) throw InvalidArg("memory budget must be >= 1 MiB");
    c->mem_budget = bytes;
    drop_graph(c);
  });
}

namespace {

struct RegionInfo {
  std::vector<double> ring;
  uint32_t nv;
  double area;
  int64_t duration;
};

// geom::StudyRegion constructor checks (geometry.cpp:113-136), in order.
RegionInfo check_region(const double* ring_xy, uint32_t nv, int64_t period_start,
                        int64_t period_end) {
  if (!ring_xy && nv) throw InvalidArg("null ring");
  std::vector<double> r(ring_xy, ring_xy + 2 * (size_t)nv);
  if (r.size() >= 4 && r[0] == r[r.size() - 2] && r[1] == r[r.size() - 1]) r.resize(r.size() - 2);
  const uint32_t m = (uint32_t)(r.size() / 2);
  if (m < 3) throw InvalidArg("polygon needs >= 3 vertices");
  for (double v : r)
    if (!std::isfinite(v)) throw InvalidArg("polygon vertex not finite");
  for (uint32_t i = 0; i < m; ++i)
    for (uint32_t j = i + 1; j < m; ++j) {
      if (j == i + 1 || (i == 0 && j == m - 1)) continue;
      if (segments_properly_intersect(&r[2 * i], &r[2 * ((i + 1) % m)], &r[2 * j],
                                      &r[2 * ((j + 1) % m)]))
        throw InvalidArg("polygon is self-intersecting");
    }
  double acc = 0.0;  // polygon_area (geometry.cpp:99-108)
  for (uint32_t i = 0, j = m - 1; i < m; j = i++)
    acc += r[2 * j] * r[2 * i + 1] - r[2 * i] * r[2 * j + 1];
  const double area = std::abs(acc) / 2.0;
  if (!(area > 0.0)) throw InvalidArg("degenerate polygon (zero area)");
  const int64_t duration = period_end - period_start;
  if (duration <= 0) throw InvalidArg("study period duration must be > 0");
  return RegionInfo{std::move(r), m, area, duration};
}

// DistanceGrid::validate (estimator.cpp:14-22).
void check_grid(const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct) {
  if (cs == 0 || ct == 0) throw InvalidArg("distance grid must be non-empty");
  if (!(s_values[0] > 0.0) || t_values[0] <= 0)
    throw InvalidArg("distance grid must exclude s=0 and t=0");
  for (uint32_t i = 1; i < cs; ++i)
    if (!(s_values[i - 1] < s_values[i])) throw InvalidArg("distance grid must be strictly increasing");
  for (uint32_t i = 1; i < ct; ++i)
    if (!(t_values[i - 1] < t_values[i])) throw InvalidArg("distance grid must be strictly increasing");
}

int write_msg(const std::exception& e, char* msg, size_t msglen, int code) {
  if (msg && msglen) {
    std::strncpy(msg, e.what(), msglen - 1);
    msg[msglen - 1] = 0;
  }
  return code;
}

}  // namespace

int stk_check_region(const double* ring_xy, uint32_t nv, int64_t period_start,
                     int64_t period_end, double* area, int64_t* duration, char* msg,
                     size_t msglen) {
  try {
    const RegionInfo ri = check_region(ring_xy, nv, period_start, period_end);
    if (area) *area = ri.area;
    if (duration) *duration = ri.duration;
    return STK_OK;
  } catch (const InvalidArg& e) {
    return write_msg(e, msg, msglen, STK_EINVAL);
  } catch (const std::exception& e) {
    return write_msg(e, msg, msglen, STK_ECUDA);
  }
}

int stk_check_grid(const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct,
                   char* msg, size_t msglen) {
  try {
    check_grid(s_values, cs, t_values, ct);
    return STK_OK;
  } catch (const InvalidArg& e) {
    return write_msg(e, msg, msglen, STK_EINVAL);
  }
}

int stk_set_region(stk_ctx* c, const double* ring_xy, uint32_t nv, int64_t period_start,
                   int64_t period_end) {
  return guarded(c, [&] {
    c->have_region = false;
    c->slab_ok = c->ec_ok = false;
    c->rv_dev_valid = false;
    drop_graph(c);
    const RegionInfo ri = check_region(ring_xy, nv, period_start, period_end);
    const std::vector<double>& r = ri.ring;
    const uint32_t m = ri.nv;
    c->ring = r;
    c->nv = m;
    c->p0 = period_start;
    c->p1 = period_end;
    c->area = ri.area;
    c->duration = ri.duration;
    c->xmin = c->xmax = r[0];
    c->ymin = c->ymax = r[1];
    c->maxabs = 0;
    for (uint32_t i = 0; i < m; ++i) {
      c->xmin = std::min(c->xmin, r[2 * i]);
      c->xmax = std::max(c->xmax, r[2 * i]);
      c->ymin = std::min(c->ymin, r[2 * i + 1]);
      c->ymax = std::max(c->ymax, r[2 * i + 1]);
      c->maxabs = std::max(c->maxabs, std::max(std::abs(r[2 * i]), std::abs(r[2 * i + 1])));
    }
    bool rect = (m == 4);
    for (uint32_t i = 0; rect && i < m; ++i) {
      const uint32_t j = (i + 1) % m;
      rect = (r[2 * i] == r[2 * j]) || (r[2 * i + 1] == r[2 * j + 1]);
    }
    c->fast_rect = rect && ri.area == (c->xmax - c->xmin) * (c->ymax - c->ymin);
    c->d_ring.ensure(m);
    CK(cudaMemcpyAsync(c->d_ring.p, r.data(), sizeof(double) * r.size(), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_region = true;
  });
}

namespace {

// Distance buckets on q = d^2 indexed by the high word of q's IEEE bits (sign,
// 11 exponent bits, top 20 mantissa bits; q >= 0 orders as an integer): with m
// mantissa bits per octave (shift = 20 - m) the buckets are log-spaced, so one
// table covers the grid's whole dynamic range, and bucket i holds exactly the
// q in [D((base + i) << shift : 0), D((base + i + 1) << shift : 0)) — no
// conversion and no rounding on the device.  Its entry is the first bin with
// Q[bin] >= the bucket's lower bound (a lower bound of the true bin) and
// Q[bin].  Single-step when the next threshold lies at or above the bucket's
// upper bound.  Bucket 0 takes everything below.  The largest m whose table is
// single-step everywhere wins; else m = 5 with the compare loop on the device.
bool build_q_buckets(stk_ctx* c) {
  const std::vector<double>& Q = c->Q;
  const int cs = (int)Q.size();
  const double qmax = Q.back();
  uint64_t qbits;
  std::memcpy(&qbits, &qmax, 8);
  const uint32_t top_hi = (uint32_t)(qbits >> 32);
  auto from_hi = [](uint64_t hi) {  // the double with high word hi and low word 0
    if (hi >= 0x7ff00000ull) return std::numeric_limits<double>::infinity();
    const uint64_t bits = hi << 32;
    double d;
    std::memcpy(&d, &bits, 8);
    return d;
  };
  auto build = [&](int m, std::vector<QBucket>* tab, int* shift, int* base) {
    *shift = 20 - m;
    const int64_t top = (int64_t)(top_hi >> *shift);
    *base = (int)std::max<int64_t>(0, top - (kQBuckets - 1));
    tab->assign(kQBuckets, QBucket{qmax, (uint32_t)(cs - 1), 0});
    bool single = true;
    for (int i = 0; i < kQBuckets; ++i) {
      const uint64_t idx = (uint64_t)*base + i;
      const double lo = i > 0 ? from_hi(idx << *shift) : 0.0;
      const double hi = from_hi((idx + 1) << *shift);
      int k = 0;
      while (k < cs - 1 && Q[k] < lo) ++k;
      (*tab)[i] = QBucket{Q[k], (uint32_t)k, 0};
      // a second step is needed iff some in-threshold q of the bucket exceeds Q[k + 1]
      if (lo <= qmax && k + 1 < cs && Q[k + 1] < hi && Q[k + 1] < qmax) single = false;
    }
    return single;
  };
  for (int m = 8; m >= 2; --m) {
    std::vector<QBucket> tab;
    int shift, base;
    if (build(m, &tab, &shift, &base)) {
      c->qtab = std::move(tab);
      c->q_shift = shift;
      c->q_base = base;
      return true;
    }
  }
  build(5, &c->qtab, &c->q_shift, &c->q_base);
  return false;
}

}  // namespace

int stk_set_grid(stk_ctx* c, const double* s_values, uint32_t cs, const int64_t* t_values,
                 uint32_t ct) {
  return guarded(c, [&] {
    c->have_grid = false;
    c->ec_ok = false;
    c->rv_dev_valid = false;
    drop_graph(c);
    check_grid(s_values, cs, t_values, ct);
    if ((uint64_t)cs * ct > (1u << 20)) throw Unsupported("more than 2^20 grid cells");
    if (cs > (uint32_t)kMaxAxis || ct > (uint32_t)kMaxAxis)
      throw Unsupported("more than " + std::to_string(kMaxAxis) + " distance thresholds per axis");
    c->s_values.assign(s_values, s_values + cs);
    c->t_values.assign(t_values, t_values + ct);
    c->Q.resize(cs);
    for (uint32_t k = 0; k < cs; ++k) c->Q[k] = sqrt_threshold(s_values[k]);
    if (cs > 65535 || ct > 65535) throw Unsupported("more than 65535 bins per axis");
    const bool q_single = build_q_buckets(c);
    // time buckets (linear, width 2^t_shift): bucket b holds exactly the lags
    // u in [b 2^k, (b + 1) 2^k), so the first bin at or above b 2^k is a lower
    // bound of the true bin; single-step when the next threshold covers the
    // bucket's last lag
    const int64_t tmax = t_values[ct - 1];
    int tsh = 0;
    while ((tmax >> tsh) >= (int64_t)kBucketTable) ++tsh;
    c->t_shift = tsh;
    c->ttab.assign(kBucketTable, TBucket<int64_t>{0, 0});
    bool t_single = true;
    for (int b = 0, k = 0; b < kBucketTable; ++b) {
      const int64_t lo = (int64_t)b << tsh, last = (((int64_t)b + 1) << tsh) - 1;
      while (k < (int)ct - 1 && t_values[k] < lo) ++k;
      c->ttab[b] = TBucket<int64_t>{t_values[k], (uint32_t)k};
      if (lo <= tmax && k + 1 < (int)ct && t_values[k + 1] < std::min(last, tmax)) t_single = false;
    }
    c->single_step = q_single && t_single;
    c->q_single = q_single;
    // evenly spaced time thresholds: exact multiply-high division (BinView::t_uni)
    c->t_uni = 0;
    if (ct >= 2 && t_values[0] >= 0) {
      const int64_t D = t_values[1] - t_values[0], T0 = t_values[0];
      bool even = D >= 2 && (int64_t)ct * D < (1ll << 31) && T0 < (1ll << 31);
      for (uint32_t k = 0; even && k < ct; ++k) even = t_values[k] == T0 + (int64_t)k * D;
      if (even) {
        int N = 0, l = 0;
        while ((1ll << N) < (int64_t)ct * D) ++N;
        while ((1ll << l) < D) ++l;
        const int E = N + l;  // m = ceil(2^E / D) < 2^(N+1) <= 2^32
        const unsigned __int128 pw = (unsigned __int128)1 << E;
        const uint64_t m = (uint64_t)((pw + (unsigned __int128)(D - 1)) / (unsigned __int128)D);
        const uint64_t magic = E >= 32 ? m : m << (32 - E);
        const int sh = E >= 32 ? E - 32 : 0;
        bool exact = magic < (1ull << 32);
        auto div = [&](uint64_t x) { return ((x * magic) >> 32) >> sh; };
        for (int64_t j = 0; exact && j <= (int64_t)ct; ++j)
          for (int64_t x : {j * D - 1, j * D})
            if (x >= D - 1 && x <= (int64_t)ct * D - 1) exact = div((uint64_t)x) == (uint64_t)(x / D);
        if (exact) {
          c->t_uni = 1;
          c->t_add = (int32_t)(D - 1 - T0);
          c->t_lo = (int32_t)(D - 1);
          c->t_magic = (uint32_t)magic;
          c->t_sh = sh;
        }
      }
    }
    c->d_Q.ensure(cs);
    c->d_s.ensure(cs);
    c->d_T.ensure(ct);
    c->d_qtab.ensure(kQBuckets);
    c->d_ttab.ensure(kBucketTable);
    CK(cudaMemcpyAsync(c->d_Q.p, c->Q.data(), 8 * cs, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_s.p, s_values, 8 * cs, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_T.p, t_values, 8 * ct, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_qtab.p, c->qtab.data(), sizeof(QBucket) * kQBuckets,
                       cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_ttab.p, c->ttab.data(), sizeof(TBucket<int64_t>) * kBucketTable,
                       cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_grid = true;
  });
}

int stk_set_options(stk_ctx* c, int use_index, int use_cache, double coord_tolerance,
                    double dist_tolerance) {
  return guarded(c, [&] {
    (void)use_index;
    if (use_cache && (coord_tolerance != 0.0 || dist_tolerance != 0.0))
      throw Unsupported("nonzero weight-cache tolerances are order-dependent in the reference "
                        "and are not supported on the device path");
  });
}

int stk_estimate_surface(stk_ctx* c, const double* x, const double* y, const int64_t* t,
                         uint64_t n, double* k_out, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    upload_points(c, x, y, t, n);
    JobOut o;
    o.k_obs = k_out;
    o.validate = true;
    run_pipeline(c, c->sx.p, c->sy.p, c->st.p, n, true, STK_METHOD_CSR, 0, 0, 0, o, tel);
  });
}

int stk_pair_histogram(stk_ctx* c, const double* x, const double* y, const int64_t* t,
                       uint64_t n, uint32_t shard, uint32_t nshards, uint64_t* counts,
                       uint64_t* sum_hi, uint64_t* sum_lo, double* hist, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    if (nshards == 0 || shard >= nshards) throw InvalidArg("shard index out of range");
    upload_points(c, x, y, t, n);
    validate_points(c, c->sx.p, c->sy.p, c->st.p, n);
    c->evnext = 0;
    Timers tm;
    tm.t0 = c->ev();
    tm.t1 = c->ev();
    CK(cudaEventRecord(tm.t0, c->stream));
    Plan P = make_plan(c, n, 1);
    P.R = 1;
    stage_reset(c, 32 * (uint64_t)P.bins + 128);
    Batch B = alloc_batch(c, P);
    CK(cudaMemsetAsync(c->stats.p, 0, sizeof(unsigned long long) * 8, c->stream));
    generate(c, B, Source::Observed, 0, 1, 0, c->sx.p, c->sy.p, c->st.p);
    run_batch(c, P, B, tm, nshards > 1 ? 1 : 0, shard, nshards, 0, ~0ULL, false);
    const uint32_t bins = P.bins;
    const unsigned long long* h = (const unsigned long long*)stage_d2h(
        c, nullptr, B.h_cnt, sizeof(unsigned long long) * 4 * bins);
    CK(cudaEventRecord(tm.t1, c->stream));
    finish_call(c, tm, tel, 1);
    for (uint32_t b = 0; b < bins; ++b) {
      const unsigned long long raw = h[b], half = h[bins + b], lo = h[2 * bins + b],
                               hi = h[3 * bins + b];
      const unsigned long long cnt = raw & ~1ULL;  // bit 0: the bin received 1/0 (omega == 0)
      if (counts) counts[b] = cnt;
      const unsigned __int128 v = ((unsigned __int128)hi << 64 | lo) +
                                  ((unsigned __int128)(cnt + half) << kFixedFracBits) +
                                  ((raw & 1ULL) ? kInfSentinel : (unsigned __int128)0);
      if (sum_hi) sum_hi[b] = (uint64_t)(v >> 64);
      if (sum_lo) sum_lo[b] = (uint64_t)v;
      if (hist) hist[b] = fixed_or_nan(v);
    }
  });
}

int stk_finalize(stk_ctx* c, uint64_t n, const uint64_t* sum_hi, const uint64_t* sum_lo,
                 double* k_out, double* l_out) {
  return guarded(c, [&] {
    require_ready(c);
    if (n == 0) throw InvalidArg("intensity needs n >= 1");
    const uint32_t cs = (uint32_t)c->s_values.size(), ct = (uint32_t)c->t_values.size();
    std::vector<double> K((size_t)cs * ct);
    for (uint32_t si = 0; si < cs; ++si)
      for (uint32_t ti = 0; ti < ct; ++ti) {
        const uint32_t b = si * ct + ti;
        const unsigned __int128 v = ((unsigned __int128)sum_hi[b] << 64) | sum_lo[b];
        double acc = fixed_or_nan(v);
        if (si > 0) acc += K[b - ct];
        if (ti > 0) acc += K[b - 1];
        if (si > 0 && ti > 0) acc -= K[b - ct - 1];
        K[b] = acc;
      }
    const double scale = c->area * (double)c->duration / ((double)n * (double)n);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (uint32_t b = 0; b < cs * ct; ++b) {
      K[b] *= scale;
      if (k_out) k_out[b] = K[b];
      if (l_out)
        l_out[b] = std::sqrt(K[b] / (two_pi * (double)c->t_values[b % ct])) - c->s_values[b / ct];
    }
  });
}

int stk_simulate(stk_ctx* c, const double* x, const double* y, const int64_t* t, uint64_t n,
                 int method, uint64_t base_seed, uint32_t r_begin, uint32_t r_end,
                 double* l_all, double* upper_l, double* lower_l, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    const Source src = source_of(method);
    const double *dx = nullptr, *dy = nullptr;
    const int64_t* dt = nullptr;
    if (src != Source::Csr) {
      if (!x || !y || !t) throw InvalidArg("bootstrap/permutation need the observed points");
      upload_points(c, x, y, t, n);
      dx = c->sx.p;
      dy = c->sy.p;
      dt = c->st.p;
    }
    if (r_end < r_begin) throw InvalidArg("r_end < r_begin");
    JobOut o;
    o.validate = src != Source::Csr;  // the observed points feed bootstrap / permutation
    o.l_all = l_all;
    o.upper = upper_l;
    o.lower = lower_l;
    run_pipeline(c, dx, dy, dt, n, false, method, base_seed, r_begin, r_end, o, tel);
  });
}

static int run_job_impl(stk_ctx* c, const double* dx, const double* dy, const int64_t* dt,
                        uint64_t n, uint32_t sims, uint64_t seed, int method, double* k_out,
                        double* l_out, double* upper_l, double* lower_l, double* diff_upper,
                        stk_telemetry* tel) {
  JobOut o;
  o.validate = true;
  o.k_obs = k_out;
  o.l_obs = l_out;
  o.upper = upper_l;
  o.lower = lower_l;
  o.diff = diff_upper;
  run_pipeline(c, dx, dy, dt, n, true, method, seed, 0, sims, o, tel);
  return 0;
}

int stk_run_job(stk_ctx* c, const double* x, const double* y, const int64_t* t, uint64_t n,
                uint32_t sims, uint64_t seed, int method, double* k_out, double* l_out,
                double* upper_l, double* lower_l, double* diff_upper, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    (void)source_of(method);
    upload_points(c, x, y, t, n);
    run_job_impl(c, c->sx.p, c->sy.p, c->st.p, n, sims, seed, method, k_out, l_out, upper_l, lower_l,
                 diff_upper, tel);
  });
}

int stk_run_job_device(stk_ctx* c, const double* d_x, const double* d_y, const int64_t* d_t,
                       uint64_t n, uint32_t sims, uint64_t seed, int method, double* k_out,
                       double* l_out, double* upper_l, double* lower_l, double* diff_upper,
                       stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    (void)source_of(method);
    run_job_impl(c, d_x, d_y, d_t, n, sims, seed, method, k_out, l_out, upper_l, lower_l,
                 diff_upper, tel);
  });
}

static void run_shard_impl(stk_ctx* c, const double* dx, const double* dy, const int64_t* dt,
                           uint64_t n, uint32_t obs_shard, uint32_t obs_nshards, uint32_t r_begin,
                           uint32_t r_end, uint64_t seed, int method, uint64_t* obs_counts,
                           uint64_t* obs_sum_hi, uint64_t* obs_sum_lo, double* upper_l,
                           double* lower_l, stk_telemetry* tel) {
  if (obs_nshards == 0 || obs_shard >= obs_nshards) throw InvalidArg("shard index out of range");
  if (r_end < r_begin) throw InvalidArg("r_end < r_begin");
  if (!obs_counts) throw InvalidArg("obs_counts is required");
  JobOut o;
  o.validate = true;
  o.upper = upper_l;
  o.lower = lower_l;
  o.obs_counts = obs_counts;
  o.obs_hi = obs_sum_hi;
  o.obs_lo = obs_sum_lo;
  run_pipeline(c, dx, dy, dt, n, true, method, seed, r_begin, r_end, o, tel, obs_shard,
               obs_nshards);
}

int stk_run_job_shard(stk_ctx* c, const double* x, const double* y, const int64_t* t, uint64_t n,
                      uint32_t obs_shard, uint32_t obs_nshards, uint32_t r_begin, uint32_t r_end,
                      uint64_t seed, int method, uint64_t* obs_counts, uint64_t* obs_sum_hi,
                      uint64_t* obs_sum_lo, double* upper_l, double* lower_l, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    (void)source_of(method);
    upload_points(c, x, y, t, n);
    run_shard_impl(c, c->sx.p, c->sy.p, c->st.p, n, obs_shard, obs_nshards, r_begin, r_end, seed,
                   method, obs_counts, obs_sum_hi, obs_sum_lo, upper_l, lower_l, tel);
  });
}

int stk_run_job_shard_device(stk_ctx* c, const double* d_x, const double* d_y,
                             const int64_t* d_t, uint64_t n, uint32_t obs_shard,
                             uint32_t obs_nshards, uint32_t r_begin, uint32_t r_end,
                             uint64_t seed, int method, uint64_t* obs_counts,
                             uint64_t* obs_sum_hi, uint64_t* obs_sum_lo, double* upper_l,
                             double* lower_l, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    (void)source_of(method);
    run_shard_impl(c, d_x, d_y, d_t, n, obs_shard, obs_nshards, r_begin, r_end, seed, method,
                   obs_counts, obs_sum_hi, obs_sum_lo, upper_l, lower_l, tel);
  });
}

int stk_comm_unique_id(unsigned char* id_out) {
  if (!id_out) return STK_EINVAL;
  try {
    ncclUniqueId id;
    NK(nccl().get_unique_id(&id));
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return STK_OK;
  } catch (const std::exception&) {
    return STK_ENCCL;
  }
}

int stk_comm_init(stk_ctx* c, const unsigned char* id, int nranks, int rank) {
  return guarded(c, [&] {
    if (!id) throw InvalidArg("null NCCL unique id");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArg("rank out of range");
    if (c->comm) {
      NK(nccl().comm_destroy(c->comm));
      c->comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm = nullptr;
    NK(nccl().comm_init_rank(&comm, nranks, uid, rank));
    c->comm = comm;
    c->comm_rank = rank;
    c->nranks = nranks;
  });
}

int stk_comm_destroy(stk_ctx* c) {
  return guarded(c, [&] {
    if (c->comm) {
      CK(cudaStreamSynchronize(c->stream));
      NK(nccl().comm_destroy(c->comm));
    }
    c->comm = nullptr;
    c->comm_rank = 0;
    c->nranks = 1;
  });
}

int stk_comm_rank(stk_ctx* c, int* rank, int* nranks) {
  if (!c) return STK_ESTATE;
  if (rank) *rank = c->comm ? c->comm_rank : 0;
  if (nranks) *nranks = c->comm ? c->nranks : 1;
  return c->comm ? STK_OK : STK_ESTATE;
}

static void run_dist_impl(stk_ctx* c, const double* dx, const double* dy, const int64_t* dt,
                          uint64_t n, uint32_t sims, uint64_t seed, int method, double* k_out,
                          double* l_out, double* upper_l, double* lower_l, double* diff_upper,
                          stk_telemetry* tel) {
  if (!c->comm) throw StateErr("no communicator (stk_comm_init)");
  const uint32_t G = (uint32_t)c->nranks, g = (uint32_t)c->comm_rank;
  const uint32_t base = sims / G, extra = sims % G;  // contiguous blocks of the seed ladder
  const uint32_t r0 = g * base + std::min(g, extra);
  const uint32_t r1 = r0 + base + (g < extra ? 1u : 0u);
  JobOut o;
  o.k_obs = k_out;
  o.l_obs = l_out;
  o.upper = upper_l;
  o.lower = lower_l;
  o.diff = diff_upper;
  o.dist = true;
  o.sims_total = sims;
  o.validate = true;
  run_pipeline(c, dx, dy, dt, n, true, method, seed, r0, r1, o, tel, g, G);
}

int stk_run_job_dist(stk_ctx* c, const double* x, const double* y, const int64_t* t, uint64_t n,
                     uint32_t sims, uint64_t seed, int method, double* k_out, double* l_out,
                     double* upper_l, double* lower_l, double* diff_upper, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    (void)source_of(method);
    upload_points(c, x, y, t, n);
    run_dist_impl(c, c->sx.p, c->sy.p, c->st.p, n, sims, seed, method, k_out, l_out, upper_l,
                  lower_l, diff_upper, tel);
  });
}

int stk_run_job_dist_device(stk_ctx* c, const double* d_x, const double* d_y,
                            const int64_t* d_t, uint64_t n, uint32_t sims, uint64_t seed,
                            int method, double* k_out, double* l_out, double* upper_l,
                            double* lower_l, double* diff_upper, stk_telemetry* tel) {
  return guarded(c, [&] {
    require_ready(c);
    check_n(n);
    (void)source_of(method);
    run_dist_impl(c, d_x, d_y, d_t, n, sims, seed, method, k_out, l_out, upper_l, lower_l,
                  diff_upper, tel);
  });
}

int stk_generate_cstr(stk_ctx* c, uint64_t n, uint64_t seed, double* x, double* y, int64_t* t) {
  return guarded(c, [&] {
    if (!c->have_region) throw StateErr("study region not set (stk_set_region)");
    if (n == 0) return;
    Plan P;
    P.n = n;
    P.R = 1;
    P.bins = 1;
    P.G.cells = 1;
    P.max_items = 1;
    Batch B = alloc_batch(c, P);
    generate(c, B, Source::Csr, 0, 1, seed, nullptr, nullptr, nullptr);
    CK(cudaMemcpyAsync(x, B.x, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(y, B.y, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(t, B.t, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int stk_generate(stk_ctx* c, int method, uint64_t n, const double* ox, const double* oy,
                 const int64_t* ot, uint64_t seed, double* x, double* y, int64_t* t) {
  return guarded(c, [&] {
    if (!c->have_region) throw StateErr("study region not set (stk_set_region)");
    const Source src = source_of(method);
    if (n == 0) {
      if (src != Source::Csr) throw InvalidArg(method == STK_METHOD_BOOTSTRAP
                                                   ? "bootstrap needs n >= 1"
                                                   : "permutation needs n >= 1");
      return;
    }
    if (src != Source::Csr) upload_points(c, ox, oy, ot, n);
    Plan P;
    P.n = n;
    P.R = 1;
    P.bins = 1;
    P.G.cells = 1;
    P.max_items = 1;
    Batch B = alloc_batch(c, P);
    generate(c, B, src, 0, 1, seed, c->sx.p, c->sy.p, c->st.p);
    CK(cudaMemcpyAsync(x, B.x, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(y, B.y, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(t, B.t, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int stk_spatial_weights(stk_ctx* c, const double* cx, const double* cy, const double* d,
                        uint64_t count, double* w_out) {
  return guarded(c, [&] {
    if (!c->have_region) throw StateErr("study region not set (stk_set_region)");
    if (count == 0) return;
    DevBuf<double> b;
    b.ensure(4 * count);
    c->ovf.ensure(1);
    c->bad.ensure(1);
    const unsigned long long init = ~0ULL;
    CK(cudaMemcpyAsync(c->bad.p, &init, 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->ovf.p, 0, sizeof(int), c->stream));
    CK(cudaMemcpyAsync(b.p, cx, 8 * count, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b.p + count, cy, 8 * count, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b.p + 2 * count, d, 8 * count, cudaMemcpyHostToDevice, c->stream));
    const RegionView rv = region_view(c);
    weights_kernel<<<(unsigned)((count + 127) / 128), 128, 0, c->stream>>>(
        b.p, b.p + count, b.p + 2 * count, count, rv, device_region(c, rv), b.p + 3 * count, c->ovf.p,
        c->bad.p);
    CK(cudaGetLastError());
  ++c->launches;
    CK(cudaMemcpyAsync(w_out, b.p + 3 * count, 8 * count, cudaMemcpyDeviceToHost, c->stream));
    unsigned long long bad = 0;
    int ovf = 0;
    CK(cudaMemcpyAsync(&bad, c->bad.p, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&ovf, c->ovf.p, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    b.release();
    if (bad != ~0ULL) throw InvalidArg("weight center outside study region");
    // only spatial_weight_ring (rectangles, <= 8 crossings) can set it: a
    // 64-entry buffer overflow there is an internal error, not a user input
    if (ovf) throw CudaFail("internal error: crossing buffer overflow in the rectangle edge weight");
  });
}

int stk_task_histogram(stk_ctx* c, const double* px, const double* py, const int64_t* pt,
                       const uint32_t* pidx, uint64_t np, const double* cx, const double* cy,
                       const int64_t* ct, const uint32_t* cidx, const double* crad,
                       const int64_t* ctrad, uint64_t nc, double* hist, uint64_t* in_threshold,
                       uint64_t* comparisons) {
  return guarded(c, [&] {
    require_ready(c);
    const uint32_t cs = (uint32_t)c->s_values.size(), ctn = (uint32_t)c->t_values.size();
    const uint32_t bins = cs * ctn;
    // one device block: points (x, y, t, idx), cylinders (x, y, t, idx, r, tr), sums
    const uint64_t pbytes = np * 28, cbytes = nc * 44, hbytes = 3ull * bins * 8 + 64;
    DevBuf<unsigned char> buf;
    buf.ensure(pbytes + cbytes + hbytes + 256);
    unsigned char* q = buf.p;
    auto put = [&](const void* src, size_t bytes, size_t align) {
      q = (unsigned char*)(((uintptr_t)q + align - 1) & ~(uintptr_t)(align - 1));
      if (bytes) CK(cudaMemcpyAsync(q, src, bytes, cudaMemcpyHostToDevice, c->stream));
      unsigned char* at = q;
      q += bytes;
      return at;
    };
    TaskArgs T{};
    T.px = (const double*)put(px, np * 8, 8);
    T.py = (const double*)put(py, np * 8, 8);
    T.pt = (const int64_t*)put(pt, np * 8, 8);
    T.pidx = (const uint32_t*)put(pidx, np * 4, 4);
    T.np = np;
    T.cx = (const double*)put(cx, nc * 8, 8);
    T.cy = (const double*)put(cy, nc * 8, 8);
    T.ct = (const int64_t*)put(ct, nc * 8, 8);
    T.crad = (const double*)put(crad, nc * 8, 8);
    T.ctrad = (const int64_t*)put(ctrad, nc * 8, 8);
    T.cidx = (const uint32_t*)put(cidx, nc * 4, 4);
    T.nc = nc;
    T.s_values = c->d_s.p;
    T.t_values = c->d_T.p;
    T.cs = cs;
    T.ctn = ctn;
    q = (unsigned char*)(((uintptr_t)q + 15) & ~(uintptr_t)15);
    unsigned long long* acc = (unsigned long long*)q;  // h_cnt, h_lo, h_hi, stats[2], bad
    CK(cudaMemsetAsync(acc, 0, (3ull * bins + 2) * 8, c->stream));
    CK(cudaMemsetAsync(acc + 3ull * bins + 2, 0xff, 8, c->stream));
    T.h_cnt = acc;
    T.h_lo = acc + bins;
    T.h_hi = acc + 2ull * bins;
    T.stats = acc + 3ull * bins;
    T.bad = acc + 3ull * bins + 2;
    c->ovf.ensure(1);
    CK(cudaMemsetAsync(c->ovf.p, 0, sizeof(int), c->stream));
    T.overflow = c->ovf.p;
    const RegionView rv = region_view(c);
    if (nc && np) {
      const uint64_t work = nc * np;
      const unsigned blocks =
          (unsigned)std::min<uint64_t>((work + 127) / 128, (uint64_t)c->num_sms * 64);
      task_kernel<<<blocks, 128, 0, c->stream>>>(T, rv, device_region(c, rv));
      CK(cudaGetLastError());
      ++c->launches;
    }
    std::vector<unsigned long long> h(3ull * bins + 3);
    CK(cudaMemcpyAsync(h.data(), acc, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    buf.release();
    if (h[3ull * bins + 2] != ~0ULL) throw InvalidArg("weight center outside study region");
    for (uint32_t b = 0; b < bins; ++b) {
      const unsigned long long raw = h[b], lo = h[bins + b], hi = h[2ull * bins + b];
      const unsigned long long cnt = raw >> 1;  // ordered pairs of the bin
      const unsigned __int128 v = ((unsigned __int128)hi << 64 | lo) +
                                  ((unsigned __int128)cnt << kFixedFracBits);
      if (hist) hist[b] = (raw & 1ULL) ? std::nan("") : fixed_or_nan(v);
    }
    if (in_threshold) *in_threshold = h[3ull * bins];
    if (comparisons) *comparisons = h[3ull * bins + 1];
  });
}

int stk_set_rng(stk_ctx* c, int rng) {
  return guarded(c, [&] {
    if (rng != STK_RNG_MT19937_64 && rng != STK_RNG_PHILOX) throw InvalidArg("unknown rng");
    c->rng = rng;
    drop_graph(c);
  });
}

int stk_philox4x32(stk_ctx* c, const uint32_t* ctr, const uint32_t* key, uint32_t n,
                   uint32_t* out) {
  return guarded(c, [&] {
    if (n == 0) return;
    DevBuf<uint32_t> b;
    b.ensure(10ull * n);
    CK(cudaMemcpyAsync(b.p, ctr, 16ull * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(b.p + 4ull * n, key, 8ull * n, cudaMemcpyHostToDevice, c->stream));
    philox_kat_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(b.p, b.p + 4ull * n, n,
                                                               b.p + 6ull * n);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, b.p + 6ull * n, 16ull * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    b.release();
  });
}

int stk_measure_fp64_peak(stk_ctx* c, double* instr_per_s) {
  return guarded(c, [&] {
    DevBuf<double> o;
    o.ensure(1);
    c->evnext = 0;
    const int blocks = c->num_sms * 8, threads = 256, iters = 2048;
    cudaEvent_t a = c->ev(), b = c->ev();
    dfma_peak_kernel<<<blocks, threads, 0, c->stream>>>(o.p, 64, 1.0000001, 1e-9);  // warm-up
    CK(cudaEventRecord(a, c->stream));
    dfma_peak_kernel<<<blocks, threads, 0, c->stream>>>(o.p, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(b, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    o.release();
    *instr_per_s = (double)blocks * threads * (double)iters * 16.0 * 8.0 / (ms * 1e-3);
  });
}

}  // extern "C"
