// rmx_internal.cuh -- shared definitions of librmx's kernels and host driver.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <cstring>

namespace rmx {

constexpr int kTileM = 128;  // permutations per tile = TMEM lanes = MMA M
constexpr int kTileV = 128;  // voxels per tile; MMA N = 2 * kTileV (S | Q)
constexpr int kSuspectCap = 1 << 16;
constexpr int kInvStage = 4096;  // int8 K1: epilogue staging of per-voxel scales (bytes)
// Relative half-width of the candidate band: every voxel whose tensor-core
// statistic lies within kBandRel * max(|t*|, 1) of the permutation's best is
// re-evaluated in fp64.  The measured |t~ - t| / max(|t|,1) is ~1e-6
// (tests/test_gpu_parity.py::test_tensor_core_error_bound), 100x below this.
constexpr float kBandRel = 1e-4f;

// Candidate band for a permutation whose best tensor-core statistic is t
// (two-sided: |t|).  fp16 path: kBandRel * max(|t|, 1).  int8 path (balanced
// groups, alpha = 0): the quantised Z perturbs every group sum S by at most
// e = max_j sum_i |z_ij - zq_ij / scale_j| (K0 measures it), and t = f(S) =
// S / sqrt(gamma - |beta| S^2) is increasing in S, so a voxel's true statistic
// lies in [f(S~ - e), f(S~ + e)].  The true maximum T >= lower(t~max) and the
// voxel attaining it has t~ >= lower(T) >= lower(lower(t~max)): the band
// t~max - lower(lower(t~max)) (+ the fp32 term) is rigorous.  A band that
// reaches a non-positive pooled variance is infinite (-> exhaustive path).
__device__ __forceinline__ double band_lower(double t, double e, double beta_abs, double gamma) {
  const double d = gamma / (1.0 + beta_abs * t * t);
  const double S = t * sqrt(d) - e;
  const double d2 = gamma - beta_abs * S * S;
  if (d2 <= 0.0) return -HUGE_VAL;
  return S / sqrt(d2);
}
// fp32 version for K1's running floors (t - 2 band): its rounding error is
// far inside the factor 2 of the floor, and a vanishing pooled variance
// gives an infinite band (no floor), so it is only ever conservative.
__device__ __forceinline__ float band_lower_f(float t, float e, float beta_abs, float gamma) {
  const float d = gamma / fmaf(beta_abs * t, t, 1.0f);
  const float S = t * sqrtf(d) - e;
  const float d2 = fmaf(-beta_abs * S, S, gamma);
  if (!(d2 > 1e-6f * gamma)) return -HUGE_VALF;
  return S * rsqrtf(d2);
}
__device__ __forceinline__ float band_abs_fast(float t, float rel, float e, float beta_abs,
                                               float gamma) {
  const float base = rel * fmaxf(fabsf(t), 1.0f);
  if (!(e > 0.0f)) return base;
  const float lo = band_lower_f(band_lower_f(t, e, beta_abs, gamma), e, beta_abs, gamma);
  if (lo == -HUGE_VALF) return HUGE_VALF;
  return base + (t - lo) * 1.01f;
}
__device__ __forceinline__ float band_abs(float t, float rel, float e, float beta_abs,
                                          float gamma) {
  const float base = rel * fmaxf(fabsf(t), 1.0f);
  if (!(e > 0.0f)) return base;
  const double lo = band_lower(band_lower(t, e, beta_abs, gamma), e, beta_abs, gamma);
  if (lo == -HUGE_VAL) return HUGE_VALF;
  return base + (float)((double)t - lo) * 1.001f;
}

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
  unsigned int emax_bits;  // int8 path: max_j sum_i |z - dequantised z| (float bits)
  unsigned int pad;
  unsigned long long rare_groups;  // epilogue diagnostics (lane max per warp)
  unsigned long long all_groups;
};

// Voxel chunks of a permutation tile: n_ramp short leading chunks (tiles
// [ramp_start[c], ramp_start[c+1])) -- a cold unit's top-4 threshold climbs
// from nothing, so the first chunks are kept short and every later unit
// starts from the permutation's best over a growing prefix -- then uniform
// chunks of tpc tiles.
constexpr int kMaxRamp = 3;
__host__ __device__ inline void chunk_tiles(int n_ramp, const int* ramp_start, int tpc,
                                            int n_vtiles, int chunk, int* t0, int* t1) {
  if (chunk < n_ramp) {
    *t0 = ramp_start[chunk];
    *t1 = ramp_start[chunk + 1];
  } else {
    *t0 = ramp_start[n_ramp] + (chunk - n_ramp) * tpc;
    *t1 = *t0 + tpc < n_vtiles ? *t0 + tpc : n_vtiles;
  }
}

// Workspace carve-up for one naive call.
struct NaiveLayout {
  int kpad;           // n rounded up to 16 (MMA K granularity)
  int n_vtiles, n_mtiles, n_chunks, tiles_per_chunk, groups, grid, bk, stages;
  int n_ramp, ramp_start[kMaxRamp + 1];  // leading short chunks (chunk_tiles)
  int cg;             // CTAs per MMA tile (tcgen05 cta_group): 1 or 2
  int i8;             // exact int8 MMA on 16-bit fixed-point Z (balanced groups)
  int vt;             // voxels per tile: 256 (S-only, n1 == n2) or 128 (S | Q)
  int mwords;         // 32-bit words of a group-1 indicator row (kpad bits)
  size_t off_planes, off_scale, off_gmask, off_cand, off_susp, off_cvox, off_overflow, off_best,
      off_const, off_counters;
  size_t total;
};

NaiveLayout naive_layout(int64_t v, int n, int n1, int64_t L, int sm_count);
NaiveLayout complete_layout(int64_t v, int r, int64_t B, int sm_count);
int golden_stride_public(int T);
// chunk / stride fields of TfillArgs from a layout
void fill_chunks(const NaiveLayout& lay, struct TfillArgs* a);

struct PrepArgs {
  const double* x;
  int64_t v;
  int n, n1, kpad;
  __half* planes;  // [4][v][kpad]: z_hi, q_hi, z_lo, q_lo (q = z^2)
  int32_t* cvox;   // constant voxels with a non-zero exact statistic
  NaiveCounters* counters;
  // int8 path (balanced groups): z quantised per voxel, zq = 255 h + l,
  // planes8[v][2 kpad] = [h | l] (s8); S = inv[j] * sum_{group 1} zq
  uint8_t* planes8;
  float* inv_scale;
  int zplanes_only;  // balanced fp16 path: the Z^2 planes are not needed
  int64_t v_begin, v_end;  // voxel rows [v_begin, v_end) (v_end = 0: all)
};

struct TfillArgs {
  // group-1 indicator of every permutation as a bit row ([n_mtiles * tile][mwords]
  // u32, bit k of row p = subject k in orders[p, :n1]; zero rows past L):
  // 52 B per permutation at n = 400 instead of the 800 B order row, so the
  // labels stay L2-resident across the chunk sweep (launch_group_mask)
  const uint32_t* gmask;
  int mwords;
  int64_t L, v;
  int n, n1, kpad, nk16;
  int n_vtiles, n_mtiles, n_chunks, tiles_per_chunk;
  int stride_full, stride_last;  // tile visiting strides (coprime with the chunk length)
  int n_ramp, ramp_start[kMaxRamp + 1], ramp_stride[kMaxRamp];  // leading short chunks
  int chunk_begin, chunk_end;    // voxel chunks [begin, end) of this launch
  float alpha, beta, gamma, dthr;
  float band_rel;          // fp32 part of the refinement band (threshold seeding)
  float beta_abs;          // |beta| (int8 band, see band_abs)
  const float* inv_scale;  // int8 path: per-voxel 1/scale
  int4* cand;  // [L][n_chunks * groups][2]: top-4 (t~, voxel) pairs
  int32_t* susp;
  uint32_t* best_t;  // [L] running best t~ per permutation (order-encoded, 0 = none)
  NaiveCounters* counters;
  float* dbg_t;  // [L][v] when debugging
  // RapidPT completion (MODE 1): A = W rows, max of W U^T + sigma z
  const __half* wA;        // [L][kpad] fp16, row p scaled by 1 / wdescale[p]
  const float* wdescale;   // [L]: power-of-2 descale (incl. the U planes' scale)
  uint32_t* maxenc;        // [L] order-encoded running max
  float sigma;
  uint64_t seed;
  int64_t perm_base;
};

struct RefineArgs {
  const double* x;  // v x n
  const int16_t* orders;
  int64_t L, v;
  int n, n1, slots, two_sided;
  float band_rel, beta_abs, gamma;  // band_abs parameters; e from counters->emax_bits
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
// every statistic of nperm labellings written to t_out (perm-major, ld), rows
// staged per block of voxels (exact_kernels.cu: k_exact_rows_vstage); x row-major
bool exact_rows_vstage_supported(int n);
cudaError_t launch_exact_rows_vstage(const double* x, int64_t v, int n, int n1,
                                     const int16_t* orders, int64_t nperm, double* t_out,
                                     int64_t ld, NaiveCounters* counters, cudaStream_t s);
cudaError_t launch_exact_rows(const double* xt, int64_t v, int n, int n1,
                             const int16_t* orders, const int32_t* perm_list, int64_t nperm,
                             int two_sided, double* t_out, int64_t ld, double* part_val,
                             int32_t* part_idx, int nvb, NaiveCounters* counters,
                             cudaStream_t s, bool transposed = true);
cudaError_t launch_exact_reduce(const double* part_val, const int32_t* part_idx, int nvb,
                                const int32_t* perm_list, int64_t nperm, double* max_out,
                                int32_t* argmax_out, cudaStream_t s);
cudaError_t launch_pairs(const double* x, int64_t v, int n, int n1, const int16_t* orders,
                         const int32_t* pairs, int64_t npairs, double* t_out, double* num_out,
                         int32_t* deg_out, cudaStream_t s);

// tfill_tc.cu
cudaError_t launch_group_mask(const int16_t* orders, int64_t L, int64_t rows, int n, int n1,
                              int mwords, uint32_t* gmask, cudaStream_t s);
cudaError_t launch_tfill_tc(const NaiveLayout& lay, const TfillArgs& a, const __half* planes,
                            int two_sided, cudaStream_t s);
cudaError_t launch_complete_tc(const NaiveLayout& lay, const TfillArgs& a, const __half* planes,
                               int two_sided, cudaStream_t s);
// voxel range [v0, v1) covered by K1 chunk c
void chunk_voxels(const NaiveLayout& lay, int64_t v, int c, int64_t* v0, int64_t* v1);

int device_sm_count();

// rng_kernels.cu: the reference's streams on the device
cudaError_t launch_plan_orders(uint64_t seed, int64_t lo, int64_t count, int n, int16_t* out,
                               cudaStream_t s);
cudaError_t launch_omega_draws(uint64_t seed, uint32_t domain, int64_t lo, int64_t count,
                               int has_extra, uint32_t extra, uint32_t v, int k, int32_t* out,
                               cudaStream_t s);

// A small device-to-host read followed by a stream synchronisation, through a
// page-locked bounce buffer.  cudaMemcpyAsync into pageable memory (a stack
// variable) returns only once the copy is done and holds the context lock
// while it waits for the stream's earlier work, which stalls every other
// thread's CUDA calls for that long (measured: the BASIS_INIT normal stream's
// upload thread blocked for the 284 ms of the training-column kernel).  With a
// page-locked destination the copy is enqueued at once and the wait happens in
// cudaStreamSynchronize, which does not hold the lock.
inline cudaError_t read_small_sync(void* dst, const void* dev, size_t bytes, cudaStream_t s) {
  constexpr size_t kCap = 4096;
  static thread_local void* bounce = nullptr;
  if (bytes > kCap) {
    cudaError_t e = cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToHost, s);
    return e != cudaSuccess ? e : cudaStreamSynchronize(s);
  }
  if (!bounce) {
    cudaError_t e = cudaHostAlloc(&bounce, kCap, cudaHostAllocDefault);  // once per host thread
    if (e != cudaSuccess) {
      bounce = nullptr;
      return e;
    }
  }
  cudaError_t e = cudaMemcpyAsync(bounce, dev, bytes, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  std::memcpy(dst, bounce, bytes);
  return cudaSuccess;
}

// The same read, but the host polls an event instead of sleeping in
// cudaStreamSynchronize: with cudaDeviceScheduleBlockingSync (set so waiting
// threads do not spin beside the serial BASIS_INIT draw) every wake-up costs
// ~50-100 us, which a latency-critical loop (GROUSE's checkpoints, ~360 per
// training) should not pay.
inline cudaError_t read_small_spin(void* dst, const void* dev, size_t bytes, cudaStream_t s) {
  constexpr size_t kCap = 4096;
  static thread_local void* bounce = nullptr;
  static thread_local cudaEvent_t ev = nullptr;
  if (bytes > kCap) return read_small_sync(dst, dev, bytes, s);
  if (!bounce) {
    cudaError_t e = cudaHostAlloc(&bounce, kCap, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      bounce = nullptr;
      return e;
    }
  }
  if (!ev) {
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      ev = nullptr;
      return e;
    }
  }
  cudaError_t e = cudaMemcpyAsync(bounce, dev, bytes, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  e = cudaEventRecord(ev, s);
  if (e != cudaSuccess) return e;
  while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
  }
  if (e != cudaSuccess) return e;
  std::memcpy(dst, bounce, bytes);
  return cudaSuccess;
}

}  // namespace rmx
