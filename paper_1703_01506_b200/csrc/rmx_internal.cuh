// rmx_internal.cuh -- shared definitions of librmx's kernels and host driver.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace rmx {

constexpr int kTileM = 128;  // permutations per tile = TMEM lanes = MMA M
constexpr int kTileV = 128;  // voxels per tile; MMA N = 2 * kTileV (S | Q)
constexpr int kSuspectCap = 1 << 16;
// Relative half-width of the candidate band: every voxel whose tensor-core
// statistic lies within kBandRel * max(|t*|, 1) of the permutation's best is
// re-evaluated in fp64.  The measured |t~ - t| / max(|t|,1) is ~1e-6
// (tests/test_gpu_parity.py::test_tensor_core_error_bound), 100x below this.
constexpr float kBandRel = 1e-4f;

struct ConstInfo {    // voxels constant over all subjects (reference quirks kept)
  double best_t;      // max over such voxels of their exact statistic
  double best_abs;    // max of |t|
  double deg_num;     // mean difference at the first degenerate one
  int32_t best_t_voxel, best_abs_voxel;  // -1 when none is non-zero
  int32_t deg_voxel;  // -1 when none is degenerate
  int32_t count;      // constant voxels whose exact statistic is not 0
};

struct NaiveCounters {
  unsigned long long deg_key;  // (perm << 32) | voxel of the first degenerate entry
  unsigned int susp_count;
  unsigned int overflow_count;
  unsigned int band_candidates;
  unsigned int cvox_count;
  unsigned int pad[2];
  unsigned long long rare_groups;  // epilogue diagnostics (lane max per warp)
  unsigned long long all_groups;
};

// Workspace carve-up for one naive call.
struct NaiveLayout {
  int kpad;           // n rounded up to 16 (MMA K granularity)
  int n_vtiles, n_mtiles, n_chunks, tiles_per_chunk, groups, grid, bk, stages;
  int cg;             // CTAs per MMA tile (tcgen05 cta_group): 1 or 2
  int vt;             // voxels per tile: 256 (S-only, n1 == n2) or 128 (S | Q)
  size_t off_planes, off_cand, off_susp, off_cvox, off_overflow, off_best, off_const,
      off_counters;
  size_t total;
};

NaiveLayout naive_layout(int64_t v, int n, int n1, int64_t L, int sm_count);

struct PrepArgs {
  const double* x;
  int64_t v;
  int n, n1, kpad;
  __half* planes;  // [4][v][kpad]: z_hi, q_hi, z_lo, q_lo (q = z^2)
  int32_t* cvox;   // constant voxels with a non-zero exact statistic
  NaiveCounters* counters;
};

struct TfillArgs {
  const int16_t* orders;  // [L][n]
  int64_t L, v;
  int n, n1, kpad, nk16;
  int n_vtiles, n_mtiles, n_chunks, tiles_per_chunk;
  int stride_full, stride_last;  // tile visiting strides (coprime with the chunk length)
  float alpha, beta, gamma, dthr;
  int4* cand;  // [L][n_chunks * groups][2]: top-4 (t~, voxel) pairs
  int32_t* susp;
  uint32_t* best_t;  // [L] running best t~ per permutation (order-encoded, 0 = none)
  NaiveCounters* counters;
  float* dbg_t;  // [L][v] when debugging
};

struct RefineArgs {
  const double* x;  // v x n
  const int16_t* orders;
  int64_t L, v;
  int n, n1, slots, two_sided;
  const int4* cand;
  const int32_t* susp;
  const ConstInfo* cinfo;
  NaiveCounters* counters;
  int32_t* overflow;  // perms needing the exhaustive path
  double* max_out;
  int32_t* argmax_out;
};

// launchers (exact_kernels.cu)
cudaError_t launch_prep(const PrepArgs& a, cudaStream_t s);
cudaError_t launch_const_reduce(const double* x, int64_t v, int n, int n1, const int32_t* cvox,
                                NaiveCounters* counters, ConstInfo* out, cudaStream_t s);
cudaError_t launch_refine(const RefineArgs& a, cudaStream_t s);
cudaError_t launch_transpose(const double* x, int64_t v, int n, double* xt, cudaStream_t s);
// exact statistic for perms `perm_list` (or all when null) x all voxels;
// writes T (perm-major, ld) and/or per-perm max/argmax; reports degenerate.
cudaError_t launch_exact_rows(const double* xt, int64_t v, int n, int n1,
                             const int16_t* orders, const int32_t* perm_list, int64_t nperm,
                             int two_sided, double* t_out, int64_t ld, double* part_val,
                             int32_t* part_idx, int nvb, NaiveCounters* counters,
                             cudaStream_t s);
cudaError_t launch_exact_reduce(const double* part_val, const int32_t* part_idx, int nvb,
                                const int32_t* perm_list, int64_t nperm, double* max_out,
                                int32_t* argmax_out, cudaStream_t s);
cudaError_t launch_pairs(const double* x, int64_t v, int n, int n1, const int16_t* orders,
                         const int32_t* pairs, int64_t npairs, double* t_out, double* num_out,
                         int32_t* deg_out, cudaStream_t s);

// tfill_tc.cu
cudaError_t launch_tfill_tc(const NaiveLayout& lay, const TfillArgs& a, const __half* planes,
                            int two_sided, cudaStream_t s);

int device_sm_count();

}  // namespace rmx
