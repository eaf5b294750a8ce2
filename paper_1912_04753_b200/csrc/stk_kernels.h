// stk_kernels.h — kernel entry points and launch arguments (internal).
#pragma once
#include <cstddef>
#include <cstdint>

#include "stk_types.h"

namespace stk {

struct PairArgs {
  double* angs_g;   // [CTAs][warps][kAngleSlots][32] crossing scratch of the general weight
  Batch B;
  GridGeom G;
  BinView bins;
  RegionView reg;
  const RegionView* reg_g;  // device-memory copy of reg for the out-of-line fallback weight
  const unsigned long long* abort_flag;  // != ~0 (invalid input point found): skip all work
};

__global__ void validate_kernel(const double* x, const double* y, const int64_t* t, uint64_t n,
                                RegionView reg, unsigned long long* bad);
constexpr int kGenThreads = 160 + 320;  // csr_gen_kernel: twist warps + temper warps
__global__ void csr_gen_kernel(Batch B, int p_first, uint64_t seed0, double xmin, double xmax,
                               double ymin, double ymax);
__global__ void csr_finish_kernel(Batch B, int p_first, RegionView reg, uint64_t ntl,
                                  uint64_t m_recip, uint64_t limit);
__global__ void csr_poly_kernel(Batch B, int p_first, uint64_t seed0, RegionView reg,
                                uint64_t ntl, uint64_t limit);
__global__ void csr_seq_kernel(Batch B, int p_first, int count, uint64_t seed0, RegionView reg,
                               uint64_t ntl, uint64_t limit, int force);
__global__ void csr_philox_kernel(Batch B, int p_first, uint64_t seed0, RegionView reg,
                                  uint64_t ntl);
__global__ void bootstrap_philox_kernel(Batch B, int p_first, uint64_t seed0, const double* ox,
                                        const double* oy, const int64_t* ot);
__global__ void perm_draw_kernel(Batch B, int p_first, uint64_t seed0, uint32_t* J);
__global__ void perm_count_kernel(uint64_t n, const uint32_t* J, uint32_t* cnt, uint32_t* rank);
__global__ void perm_scatter_kernel(uint64_t n, const uint32_t* J, const uint32_t* start,
                                    const uint32_t* rank, uint32_t* list);
__global__ void perm_sort_kernel(uint64_t n, const uint32_t* start, uint32_t* list);
__global__ void perm_final_kernel(Batch B, int p_first, const double* ox, const double* oy,
                                  const int64_t* ot, const uint32_t* J, const uint32_t* start,
                                  const uint32_t* list);
__global__ void philox_kat_kernel(const uint32_t* ctr, const uint32_t* key, uint32_t n,
                                  uint32_t* out);
__global__ void bootstrap_kernel(Batch B, int p_first, uint64_t seed0, const double* ox,
                                 const double* oy, const int64_t* ot, uint64_t limit);
__global__ void resample_seq_kernel(Batch B, int p_first, int count, uint64_t seed0,
                                    const double* ox, const double* oy, const int64_t* ot,
                                    int mode);
__global__ void key_kernel(Batch B, GridGeom G, int p_first);
// Exclusive scans of per-cell counts and item counts for R patterns of `cells`
// cells (multi-CTA; `partial` holds scan_scratch(cells, R) entries); returns
// the number of kernels launched.
size_t scan_scratch(uint32_t cells, unsigned R);
int scan_launch(const uint32_t* counts, uint32_t* start, uint32_t* istart, uint32_t cells,
                unsigned R, unsigned long long* max_cell, uint2* partial, cudaStream_t s);
__global__ void select_count_kernel(Batch B, GridGeom G);
__global__ void select_scatter_kernel(Batch B, GridGeom G);
__global__ void place_kernel(Batch B, GridGeom G, int p_first);
__global__ void gather_kernel(Batch B, RegionView R, int p_first, uint32_t qmax_hi);
__global__ void items_kernel(Batch B, GridGeom G, int p_first);
__global__ void tasks_kernel(Batch B, GridGeom G, uint32_t resident_ctas);
// mode = rect | single_step << 1 (kernel template flags)
cudaError_t pair_kernel_prepare(int wide, int mode, size_t smem, size_t smem_limit, int* per_sm);
void pair_kernel_launch(int wide, int mode, unsigned ctas, size_t smem, cudaStream_t stream,
                        const PairArgs& A);
__global__ void finalize_kernel(Batch B, uint32_t cs, uint32_t ct, const double* s_values,
                                const int64_t* t_values, double area, int64_t duration,
                                int p_first, unsigned long long* obs_raw, double* obs_kl);
__global__ void envelope_kernel(Batch B, uint32_t bins, int p_first, int count, int init,
                                double* upper, double* lower);
__global__ void diff_kernel(const double* est_l, const double* upper, uint32_t bins,
                            double* diff);
__global__ void pack_exact_kernel(const unsigned long long* cnt, const unsigned long long* half,
                                  const unsigned long long* lo, const unsigned long long* hi,
                                  uint32_t bins, unsigned long long* limbs);
__global__ void unpack_exact_kernel(const unsigned long long* limbs, uint32_t bins,
                                    unsigned long long* cnt, unsigned long long* half,
                                    unsigned long long* lo, unsigned long long* hi);
__global__ void fill_kernel(double* p, uint32_t n, double v);
__global__ void copy_points_kernel(double* x, double* y, int64_t* t, const double* ox,
                                   const double* oy, const int64_t* ot, uint64_t n,
                                   RegionView reg, unsigned long long* bad);
__global__ void weights_kernel(const double* cx, const double* cy, const double* d,
                               uint64_t count, RegionView reg, const RegionView* reg_g, double* w, int* overflow,
                               unsigned long long* bad);
// rt::execute_task on the device (the reference's task interface).
struct TaskArgs {
  const double *px, *py;      // task points
  const int64_t* pt;
  const uint32_t* pidx;       // their record indices
  uint64_t np;
  const double *cx, *cy;      // cylinder centers
  const int64_t* ct;
  const uint32_t* cidx;       // center record indices
  const double* crad;         // cylinder spatial radius
  const int64_t* ctrad;       // cylinder temporal radius
  uint64_t nc;
  const double* s_values;
  const int64_t* t_values;
  uint32_t cs, ctn;
  unsigned long long *h_cnt, *h_lo, *h_hi;  // [bins] exact sums (h_cnt: 2 per pair, bit 0 = 1/0)
  unsigned long long* stats;  // [0] in-threshold [1] comparisons
  unsigned long long* bad;    // first cylinder whose center lies outside the region
  int* overflow;
};
__global__ void task_kernel(TaskArgs T, RegionView reg, const RegionView* reg_g);
__global__ void dfma_peak_kernel(double* out, int iters, double a, double b);

size_t pair_kernel_smem(uint32_t bins, int wide);

}  // namespace stk
