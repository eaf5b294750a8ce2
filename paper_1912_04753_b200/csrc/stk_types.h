// stk_types.h — plain structs shared by the host runtime and the kernels.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace stk {

constexpr int kItemCenters = 32;    // centers per warp work item (one per lane)
#ifndef STK_PART_CELLS
#define STK_PART_CELLS 4096
#endif
constexpr int kPartCells = STK_PART_CELLS;    // a cell this populous splits items into parts (>= 2)
constexpr int kMaxParts = 32;       // ... up to this many parts per item
#ifndef STK_TAIL_PARTS
#define STK_TAIL_PARTS 3
#endif
constexpr int kTailParts = STK_TAIL_PARTS;  // slices of each of a task's last kTailItems items
#ifndef STK_TAIL_ITEMS
#define STK_TAIL_ITEMS 32  // two per warp of a 16-warp CTA (16: C4 +0.7%, 48 with 3 slices: same as 32)
#endif
constexpr int kTailItems = STK_TAIL_ITEMS;
constexpr int kTaskMinItems = 4;    // warp items per CTA task: adaptive in [min, max] so the
#ifndef STK_TASKS_PER_CTA
#define STK_TASKS_PER_CTA 8  // adaptive task size: about this many tasks per resident CTA
#endif
#ifndef STK_TASK_MAX
#define STK_TASK_MAX 256
#endif
constexpr int kTaskMaxItems = STK_TASK_MAX;  // batch has ~8 tasks per resident CTA
#ifndef STK_PAIR_WARPS
#define STK_PAIR_WARPS 16
#endif
constexpr int kPairWarps = STK_PAIR_WARPS;  // warps per pair-kernel CTA
constexpr int kBucketTable = 1024;  // time bucket table size for bin guesses
constexpr int kQBuckets = 512;      // distance (q) bucket table size
constexpr int kAngleSlots = 16;    // per-lane crossing scratch: 2 doubles x 8 crossings
constexpr int kRingSmem = 32;      // ring vertices staged in shared memory (bitmask path)
#ifndef STK_ARC_CHUNK
#define STK_ARC_CHUNK 32
#endif
constexpr int kArcChunk = STK_ARC_CHUNK;        // candidate steps between arc drains
constexpr int kFixedFracBits = 53;  // fixed-point weighted sums: value * 2^53
#ifndef STK_ARC_RING
#define STK_ARC_RING 4096
#endif
constexpr int kArcRing = STK_ARC_RING;  // per-warp arc ring entries (> 63 + kArcChunk * 64)
static_assert(kArcRing > 63 + kArcChunk * 64, "the arc ring must hold a chunk's entries");
constexpr int kCplxRing = 128;      // per-warp ring of entries deferred to the general weight (> 31 + 64)

// Study region on the device (geom::StudyRegion, geometry.hpp:95-120).
struct RegionView {
  const double2* ring;  // open ring, nv vertices
  uint32_t nv;
  int64_t p0, p1;       // study period (inclusive)
  double xmin, xmax, ymin, ymax;
  double maxabs;        // max |coordinate| over the ring
  int rect;             // 4-vertex axis-aligned rectangle (exact fast paths apply)
  double box_m;         // rect: on_segment is impossible farther than this outside the box
  double2 rv[4];        // rect: the ring's vertices (kernel-parameter copy)
  // rect sides in the order x = xmin, x = xmax, y = ymin, y = ymax: the
  // reference's segment (A -> B) on that side has A's along-side coordinate
  // sd_start and B - A = sd_len (computed as the reference does)
  double sd_start[4], sd_len[4];
  double sw_dmin;       // rect single-edge closed form: smallest radius it accepts
  double sw_margin;     // ... and smallest d - h (outside midpoint clear of the boundary)
  double sw_q_min;      // q-form of sw_dmin: q >= sw_q_min implies RN(sqrt(q)) >= sw_dmin
  // General polygons.  Horizontal slabs: slab s lists every
  // edge k (ring[k] -> ring[k+1]) whose y-range, widened by the on_segment
  // tolerance, meets the slab; point_in_polygon of a probe then visits only
  // its slab's edges.  Valid for probes with |x|, |y| <= pip_lim.
  const uint32_t* slab_start;  // [nslab + 1]
  const uint32_t* slab_edge;
  uint32_t nslab;
  double slab_y0, slab_inv_h, pip_lim, pip_ylo, pip_yhi;
  // Edge cells: cell (ix, iy) of width 1/ec_inv_w lists every segment i
  // (ring[i-1] -> ring[i]) within ec_reach of the cell; a circle of radius
  // d <= ec_dmax around any point of the cell crosses no other segment
  // (the reference rejects them).  ec_start == nullptr: not built.
  const uint32_t* ec_start;    // [ec_nx * ec_ny + 1]
  const uint32_t* ec_edge;
  const float* ec_dmin;        // per list entry: lower bound of its distance to the cell (ascending)
  const float* ec_far;         // ... and upper bound of its farthest point from the cell
  double ec_abs;               // absolute margin of the reach test (1e-9 S)
  int ec_nx, ec_ny;
  double ec_x0, ec_y0, ec_inv_w, ec_dmax, ec_reach;
  int no_safe;  // debugging (STK_NO_SAFE_RADIUS): every pair takes the exact path
};

// Distance grid in the forms the kernels consume.
// Bucket entries: the lowest bin a bucket can hold and that bin's threshold,
// so one shared-memory load and one compare resolve a single-step bucket.
struct QBucket {           // on q = d^2, indexed by the float bits of q (log scale)
  double thr;              // Q[bin]
  uint32_t bin;
  uint32_t pad;
};
template <typename TT>
struct TBucket {           // on u, linear
  TT thr;                  // T[bin] (clamped to TT)
  uint32_t bin;
};

struct BinView {
  const double* Q;         // Q[k] = largest q with RN(sqrt(q)) <= s_values[k]
  const int64_t* T;        // t_values
  const QBucket* q_tab;    // kQBuckets entries
  const TBucket<int64_t>* t_tab;  // kBucketTable entries (device converts to TT)
  uint32_t cs, ct;
  double Qmax;
  int64_t Tmax;
  int q_shift, q_base;     // bucket = clamp((hi32(q) >> q_shift) - q_base): log-spaced
  int t_shift;             // time bucket = min(u >> t_shift, kBucketTable - 1)
  int single_step;         // every bucket straddles <= 1 threshold: one compare finds the bin
  // Evenly spaced time thresholds T_k = T_0 + k D (32-bit lags): the t bin is
  // ceil(max(u - T_0, 0) / D) = floor(x / D), x = max(u + t_add, t_lo) with
  // t_add = D - 1 - T_0, t_lo = D - 1, by one multiply-high: (x * t_magic) >> 32
  // >> t_sh (host-verified exact at every bin boundary of the lag range).
  int t_uni;
  int32_t t_add, t_lo;
  uint32_t t_magic;
  int t_sh;
};

// Uniform space-time cell grid (replaces the STR R-tree, st_index.cpp:54-130).
struct GridGeom {
  double x0, y0;   // origin of cell (0,0)
  double inv_w;    // 1 / spatial cell width (width >= s_max)
  int64_t t0;      // period start
  int64_t tw;      // temporal cell width (>= t_max)
  double inv_tw;
  int32_t nx, ny, nt;
  uint32_t cells;  // nx*ny*nt
  int32_t rs, rt;  // stencil radius in cells (space, time): cell >= s_max/rs, >= t_max/rt
};

#ifndef STK_MAX_AXIS
#define STK_MAX_AXIS 512
#endif
constexpr int kMaxAxis = STK_MAX_AXIS;  // max bins per axis (smem-resident thresholds)

// Per sorted point: time relative to the period start, the temporal-weight
// threshold (v == 1 iff u <= vt, edge_correction.cpp:81-86), the squared
// radius below which omega == 1 exactly (rounded DOWN to float: still a
// conservative bound), and the input index.  Replaces the reference's
// weight cache (weight_cache.hpp:39-129) with a per-point memo.
template <typename TT>
struct PtMeta {
  TT t;
  TT vt;
  uint32_t sqh;  // high word of a lower bound of the safe q: hi32(q) < sqh => omega == 1
  uint32_t idx;
};

// One batch of R point patterns of n points each, laid out [R][n].
struct Batch {
  int R;
  uint64_t n;
  // unsorted input points
  double* x;
  double* y;
  int64_t* t;
  // grid-sorted layout: interleaved coordinates + one meta record per point
  double2* pxy;   // (x, y)
  double2* parc;  // rectangles: per sorted point rect_arc_record (h, q interval), else null
  void* pmeta;    // PtMeta<int32_t> (16 B) or PtMeta<int64_t> (24 B) when `wide`
  int wide;       // study period >= 2^31 time units: 64-bit relative times
  uint32_t* key;  // cell key per unsorted point
  uint32_t* rank; // rank within the cell per unsorted point
  uint32_t* perm; // input index per sorted position (counting sort pass 2)
  uint32_t* cell_count;  // [R][cells]
  uint32_t* cell_start;  // [R][cells+1]
  uint32_t* item_start;  // [R][cells+1] exclusive scan of ceil(count/32)
  uint2* items;          // [R][max_items]: (cell, first sorted position)
  uint32_t max_items;
  // center selection (patterns [0, n_sel) only): a sorted point is a center
  // iff its input index i satisfies c0 <= i < c1 and i % nshards == shard.
  // The selected SET is independent of the (arbitrary) order within a cell,
  // so shards of one pattern computed by separate calls partition its pairs.
  int n_sel;
  uint32_t shard, nshards;
  uint64_t c0, c1;
  uint32_t* sel_start;   // [n_sel][cells+1] exclusive scan of selected per cell
  uint32_t* center_pos;  // [n_sel][n] sorted positions of selected centers, by cell
  uint32_t* task_start;  // [R+1] exclusive scan of ceil(items_r / task_items)
  uint32_t* task_counter;  // [0] dynamic task counter, [1] task_items, [2] parts per item
  // exact histograms [R][bins]
  unsigned long long* h_cnt;   // in-threshold pairs
  unsigned long long* h_half;  // ordered pairs with v = 1/2 (each adds 1 more; arc terms are (1/omega - 1) / v)
  unsigned long long* h_lo;    // arc-path sum of (1/omega - 1) / v, signed 128-bit fixed 53
  unsigned long long* h_hi;
  double* K;  // [R][bins]
  double* L;  // [R][bins]
  unsigned long long* stats;   // [0] in_threshold [1] candidates [2] exact_path [3] overflow [4] arc (omega != 1)
  int* flags;                  // [R] generator fallback flags
  uint4* arcq;                 // [grid CTAs][warps][kArcRing + kCplxRing] arc-path rings
};

}  // namespace stk
