/*
 * stk.h — C ABI of the B200-native space-time K pair path (libstk.so).
 *
 * Drop-in boundary for the reference's hot path (paths relative to
 * /root/reference/proj).  Each entry point names the reference interface it
 * replaces; INTEGRATION.md shows the reference-side binding.  No C++ or torch
 * types cross this boundary: plain pointers and sizes, caller-owned host
 * buffers, row-major [s][t] surfaces of cs*ct doubles.
 *
 * Error convention: 0 = success; STK_EINVAL mirrors the reference's
 * std::invalid_argument (same message in stk_last_error); STK_EUNSUPPORTED
 * for features outside the hot path (nonzero cache tolerances); STK_ECUDA for
 * device failures.  A context is single-threaded (the reference's WeightCache
 * single-writer contract, core/include/stripley/weight_cache.hpp:34-38); calls
 * block until results are on the host.
 */
#ifndef STK_H_
#define STK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STK_OK 0
#define STK_EINVAL 1       /* reference: std::invalid_argument            */
#define STK_EUNSUPPORTED 2 /* outside the path (cache tolerance != 0 ...) */
#define STK_ECUDA 3        /* device / driver failure                     */
#define STK_ESTATE 4       /* region or grid not set                      */
#define STK_ENCCL 5        /* NCCL unavailable or a collective failed     */

#define STK_METHOD_CSR 0         /* sim::Method::Cstr        */
#define STK_METHOD_BOOTSTRAP 1   /* sim::Method::Bootstrap   */
#define STK_METHOD_PERMUTATION 2 /* sim::Method::Permutation */

#define STK_RNG_MT19937_64 0 /* the reference's rng::Engine stream: bit-exact realisations */
#define STK_RNG_PHILOX 1     /* opt-in Philox4x32-10, counter-based: statistical parity only */

typedef struct stk_ctx stk_ctx;

/* Superset of est::EstimatorTelemetry (core/include/stripley/estimator.hpp:47-51)
 * and the pair counters of rt::RunTelemetry (core/include/stripley/runtime.hpp:59-72).
 * Accumulated with += like the reference (estimator.cpp:180-184). */
typedef struct {
  uint64_t in_threshold_pairs; /* == reference in_threshold_pairs (index-invariant)  */
  uint64_t candidate_pairs;    /* grid-stencil candidate tests (cf. pair_comparisons) */
  uint64_t exact_path_pairs;   /* pairs whose weight went through the arc path       */
  uint64_t patterns;           /* point patterns processed (observed + realisations) */
  double gen_ms;               /* device time: CSR generation                        */
  double grid_ms;              /* device time: grid build (key, scan, scatter)       */
  double pair_ms;              /* device time: pair kernel                           */
  double finalize_ms;          /* device time: prefix/scale/L/envelopes              */
  double total_ms;             /* device time of the whole call                      */
  uint64_t kernel_launches;    /* libstk kernels launched by the call                */
  uint64_t arc_pairs;          /* in-threshold ordered pairs with omega != 1          */
  uint64_t batches;            /* pattern batches the call ran (memory budget)       */
} stk_telemetry;

/* ---- context-free validation (no device needed) ------------------------- */
/* The geom::StudyRegion constructor checks (core/src/geometry.cpp:110-136);
 * writes area and duration.  On STK_EINVAL, msg receives the reference's
 * std::invalid_argument message. */
int stk_check_region(const double* ring_xy, uint32_t nv, int64_t period_start,
                     int64_t period_end, double* area, int64_t* duration, char* msg,
                     size_t msglen);
/* est::DistanceGrid::validate (core/src/estimator.cpp:14-22). */
int stk_check_grid(const double* s_values, uint32_t cs, const int64_t* t_values, uint32_t ct,
                   char* msg, size_t msglen);

/* ---- context ---------------------------------------------------------- */
int stk_create(stk_ctx** out, int device);
void stk_destroy(stk_ctx* ctx);
const char* stk_last_error(const stk_ctx* ctx);
const char* stk_version(void);
/* cudaStream_t the context launches on (for event timing by callers). */
void* stk_stream(stk_ctx* ctx);
/* Upper bound of device bytes for per-batch pattern buffers (default: 40% of the device
 * memory free at stk_create, clamped to [4 GiB, 64 GiB]). */
int stk_set_memory_budget(stk_ctx* ctx, uint64_t bytes);

/* ---- configuration ---------------------------------------------------- */
/* geom::StudyRegion(ring, period_start, period_end)
 * (core/include/stripley/geometry.hpp:95-120, core/src/geometry.cpp:110-136):
 * closed rings accepted and stored open; rejects < 3 vertices, non-finite
 * vertices, self-intersection, zero area, duration <= 0 (same messages). */
int stk_set_region(stk_ctx* ctx, const double* ring_xy, uint32_t nv, int64_t period_start,
                   int64_t period_end);
/* est::DistanceGrid{s_values, t_values}.validate() (core/src/estimator.cpp:14-22). */
int stk_set_grid(stk_ctx* ctx, const double* s_values, uint32_t cs, const int64_t* t_values,
                 uint32_t ct);
/* est::EstimatorOptions (core/include/stripley/estimator.hpp:39-45).  use_index and
 * use_cache never change results in the reference (tests/test_estimator.cpp:91-114,
 * 130-151); the device path always uses its grid index and per-center memo.
 * Nonzero tolerances are order-dependent in the reference and return
 * STK_EUNSUPPORTED. */
int stk_set_options(stk_ctx* ctx, int use_index, int use_cache, double coord_tolerance,
                    double dist_tolerance);

/* Realisation generator for CSR and bootstrap (default STK_RNG_MT19937_64,
 * the reference's std::mt19937_64 stream of rng.hpp:39 and simulation.cpp:10-35,
 * bit for bit).  STK_RNG_PHILOX: Philox4x32-10 keyed by the realisation seed,
 * one counter per point -- fully parallel generation, same distributions and
 * seed ladder, results that agree with the reference statistically
 * (calibration), not bitwise.  Permutation stays on the sequential stream
 * (STK_EUNSUPPORTED with Philox). */
int stk_set_rng(stk_ctx* ctx, int rng);

/* ---- the hot path ----------------------------------------------------- */
/* est::estimate_surface (core/include/stripley/estimator.hpp:107-111,
 * core/src/estimator.cpp:116-186): K surface (cumulative, x A*D/n^2). */
int stk_estimate_surface(stk_ctx* ctx, const double* x, const double* y, const int64_t* t,
                         uint64_t n, double* k_out, stk_telemetry* tel);

/* Per-bin (pre-cumulative) histogram of est::PairHistogram
 * (core/include/stripley/estimator.hpp:55-81) plus exact per-bin counts.
 * hist[b] is the exact sum of 1/(omega*v) rounded once; sum_hi/sum_lo (may
 * be NULL) give it as 128-bit fixed point with 53 fractional bits.  A bin
 * that received 1/0 (omega == 0: the reference adds +inf and its Kahan sum
 * becomes NaN) has hist[b] = NaN and 2^120 added to its fixed-point sum: real
 * sums stay below 2^110, so sums of up to 255 shard partials keep the mark,
 * and stk_finalize turns any sum >= 2^119 into NaN.
 * Shards: the pair work of the pattern is split into nshards disjoint slices;
 * shard s computes only its slice (counts/sums add exactly across shards —
 * the single-huge-pattern multi-GPU path).  nshards = 1 for the whole. */
int stk_pair_histogram(stk_ctx* ctx, const double* x, const double* y, const int64_t* t,
                       uint64_t n, uint32_t shard, uint32_t nshards, uint64_t* counts,
                       uint64_t* sum_hi, uint64_t* sum_lo, double* hist, stk_telemetry* tel);

/* est::finalize_surface + est::to_l (core/src/estimator.cpp:94-114, 51-57, 71-82)
 * from exact (possibly shard-summed) 128-bit sums, in the reference's
 * operation order. */
int stk_finalize(stk_ctx* ctx, uint64_t n, const uint64_t* sum_hi, const uint64_t* sum_lo,
                 double* k_out, double* l_out);

/* sim::run_simulations (core/include/stripley/simulation.hpp:38-43,
 * core/src/simulation.cpp:67-84) restricted to realisations r in [r_begin, r_end)
 * of the seed ladder base_seed + r: their L surfaces ((r_end-r_begin)*cs*ct,
 * may be NULL) and the pointwise max/min over them (sim::envelopes,
 * simulation.cpp:86-102; may be NULL).  Observed points are needed for
 * bootstrap/permutation (pass NULL for CSR). */
int stk_simulate(stk_ctx* ctx, const double* x, const double* y, const int64_t* t, uint64_t n,
                 int method, uint64_t base_seed, uint32_t r_begin, uint32_t r_end,
                 double* l_all, double* upper_l, double* lower_l, stk_telemetry* tel);

/* rt::run_job (core/include/stripley/runtime.hpp:151-153, core/src/runtime.cpp:190-249)
 * minus planning: estimate (K, L) then sims realisations, envelopes and
 * diff_upper (estimator.cpp:188-202).  upper/lower/diff only when sims > 0. */
int stk_run_job(stk_ctx* ctx, const double* x, const double* y, const int64_t* t, uint64_t n,
                uint32_t sims, uint64_t seed, int method, double* k_out, double* l_out,
                double* upper_l, double* lower_l, double* diff_upper, stk_telemetry* tel);

/* Same as stk_run_job with the observed pattern already resident on the
 * context's device (d_x, d_y, d_t device pointers); outputs are host buffers.
 * Used to time the device pipeline with inputs in HBM. */
int stk_run_job_device(stk_ctx* ctx, const double* d_x, const double* d_y, const int64_t* d_t,
                       uint64_t n, uint32_t sims, uint64_t seed, int method, double* k_out,
                       double* l_out, double* upper_l, double* lower_l, double* diff_upper,
                       stk_telemetry* tel);

/* One rank's share of rt::run_job for multi-GPU (one process per GPU): the
 * exact pre-cumulative sums of slice obs_shard of obs_nshards of the observed
 * pattern's pair work (obs_counts, obs_sum_hi/lo: cs*ct each; they add exactly
 * across shards -> all-reduce SUM, then stk_finalize), and the partial
 * envelopes over realisations [r_begin, r_end) (-> all-reduce MAX / MIN).
 * upper/lower are left untouched when r_begin == r_end. */
int stk_run_job_shard(stk_ctx* ctx, const double* x, const double* y, const int64_t* t,
                      uint64_t n, uint32_t obs_shard, uint32_t obs_nshards, uint32_t r_begin,
                      uint32_t r_end, uint64_t seed, int method, uint64_t* obs_counts,
                      uint64_t* obs_sum_hi, uint64_t* obs_sum_lo, double* upper_l,
                      double* lower_l, stk_telemetry* tel);
/* Same with the observed pattern resident on the device. */
int stk_run_job_shard_device(stk_ctx* ctx, const double* d_x, const double* d_y,
                             const int64_t* d_t, uint64_t n, uint32_t obs_shard,
                             uint32_t obs_nshards, uint32_t r_begin, uint32_t r_end,
                             uint64_t seed, int method, uint64_t* obs_counts,
                             uint64_t* obs_sum_hi, uint64_t* obs_sum_lo, double* upper_l,
                             double* lower_l, stk_telemetry* tel);

/* ---- multi-GPU: one process (or thread) per GPU, NCCL inside the context --
 * Replaces the reference's DistributedExecutor + TCP workers
 * (core/src/distributed.cpp:116-245, core/include/stripley/distributed.hpp):
 * rank 0 creates an id with stk_comm_unique_id, every rank receives it by any
 * out-of-band means and calls stk_comm_init on its own context.  libnccl.so.2
 * is loaded on first use (STK_ENCCL when absent). */
#define STK_NCCL_ID_BYTES 128
int stk_comm_unique_id(unsigned char* id_out /* STK_NCCL_ID_BYTES */);
int stk_comm_init(stk_ctx* ctx, const unsigned char* id, int nranks, int rank);
int stk_comm_destroy(stk_ctx* ctx);
/* Rank and size of the context's communicator (STK_ESTATE and 0 / 1 when none). */
int stk_comm_rank(stk_ctx* ctx, int* rank, int* nranks);

/* rt::run_job as a collective over the context's communicator: every rank
 * passes the same observed points and arguments; rank g computes shard g of
 * the observed pattern's pair work and its contiguous block of the
 * realisations; the exact per-bin partials (integer limbs) are summed and the
 * partial envelopes MAX/MIN-reduced with NCCL on the device, then K, L and
 * diff are finalized on the device.  Every rank receives the full result,
 * bit-identical to stk_run_job's at any number of ranks. */
int stk_run_job_dist(stk_ctx* ctx, const double* x, const double* y, const int64_t* t, uint64_t n,
                     uint32_t sims, uint64_t seed, int method, double* k_out, double* l_out,
                     double* upper_l, double* lower_l, double* diff_upper, stk_telemetry* tel);
/* Same with the observed pattern resident on the context's device. */
int stk_run_job_dist_device(stk_ctx* ctx, const double* d_x, const double* d_y,
                            const int64_t* d_t, uint64_t n, uint32_t sims, uint64_t seed,
                            int method, double* k_out, double* l_out, double* upper_l,
                            double* lower_l, double* diff_upper, stk_telemetry* tel);

/* Raw CSR realisation points of generate_cstr(n, region, seed)
 * (core/src/simulation.cpp:10-24), generated on the device (host outputs). */
int stk_generate_cstr(stk_ctx* ctx, uint64_t n, uint64_t seed, double* x, double* y,
                      int64_t* t);

/* sim::generate (core/src/simulation.cpp:55-65) on the device: CSR
 * (generate_cstr, needs only n), bootstrap or permutation of the observed
 * points (ox, oy, ot; n of them).  Outputs n points (host buffers). */
int stk_generate(stk_ctx* ctx, int method, uint64_t n, const double* ox, const double* oy,
                 const int64_t* ot, uint64_t seed, double* x, double* y, int64_t* t);

/* edge::spatial_isotropic_weight for a batch of (center, d) queries
 * (core/src/edge_correction.cpp:42-79); centers must lie inside the region
 * (STK_EINVAL "weight center outside study region" otherwise). */
int stk_spatial_weights(stk_ctx* ctx, const double* cx, const double* cy, const double* d,
                        uint64_t count, double* w_out);

/* rt::execute_task (core/include/stripley/runtime.hpp:96-99, core/src/runtime.cpp:73-117)
 * for the reference's task interface (rt::Executor::run over TaskData): the
 * pre-cumulative histogram of one task -- every (cylinder, point) candidate of
 * the task, the center's own record skipped, within_cylinder with the
 * cylinder's radii, bin_pair on the grid, 1/pair_weight summed exactly and
 * rounded once per bin (NaN where the reference adds 1/0).  Points: px, py,
 * pt, record index pidx (np of them); cylinders: center cx, cy, ct, center
 * record index cidx, spatial radius crad, temporal radius ctrad (nc of them).
 * A compatibility path (brute force over the task, like the reference's
 * use_index = false branch): rt::run_job runs the fused device pipeline. */
int stk_task_histogram(stk_ctx* ctx, const double* px, const double* py, const int64_t* pt,
                       const uint32_t* pidx, uint64_t np, const double* cx, const double* cy,
                       const int64_t* ct, const uint32_t* cidx, const double* crad,
                       const int64_t* ctrad, uint64_t nc, double* hist, uint64_t* in_threshold,
                       uint64_t* comparisons);

/* ---- instrumentation --------------------------------------------------- */
/* Raw Philox4x32-10 blocks computed on the device (known-answer tests):
 * out[4i..4i+3] = philox(ctr[4i..4i+3], key[2i..2i+1]). */
int stk_philox4x32(stk_ctx* ctx, const uint32_t* ctr, const uint32_t* key, uint32_t n,
                   uint32_t* out);
/* Device-measured FP64 issue peak (DFMA thread-instructions per second) at the
 * current clocks: the denominator of the pair kernel's roofline. */
int stk_measure_fp64_peak(stk_ctx* ctx, double* instr_per_s);

#ifdef __cplusplus
}
#endif
#endif /* STK_H_ */
