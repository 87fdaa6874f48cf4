// rapid_stats.cu -- K2 of RapidPT recovery: the statistic of every
// observed (Omega) row under its permutation, bit-identical to the
// reference's batched _welch_rows (rapid.py:156-170).  Compiled with
// -fmad=false (np_exact.cuh).
#include <cstdint>

#include "np_exact.cuh"
#include "rapid_internal.cuh"

namespace rmx {
namespace {

// ------------------------------------------------------------------ K2
// grid (ceil(k / 256), L): one block per permutation chunk of Omega.
__global__ void k_rapid_stats(const double* __restrict__ x, int n, int n1,
                              const int16_t* __restrict__ orders, const int32_t* __restrict__ omegas,
                              int k, double* __restrict__ t_out, unsigned long long* deg_key) {
  extern __shared__ int16_t ord[];
  const int64_t p = blockIdx.y;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ord[i] = orders[p * n + i];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const int64_t row = omegas[p * k + i];
  const WelchExact r = welch_exact(x + row * n, 1, ord, n1, n - n1);
  t_out[p * k + i] = r.t;
  if (r.degenerate) atomicMin(deg_key, ((unsigned long long)p << 32) | (unsigned long long)i);
}

// Warp per Omega row: rows are double-buffered in shared memory (the next
// row's cp.async is in flight while the current one is evaluated), both
// groups' numpy-pairwise chains share each pass over the row
// (welch_exact_warp2: same bits as welch_exact), and the leaf plans of the
// two group sizes are built once per block.  grid (ceil(k / (8 *
// kRowsPerWarp)), L), 8 warps.
constexpr int kStatWarps = 8;
constexpr int kRowsPerWarp = 8;

__device__ __forceinline__ void cp_async8_row(double* dst, const double* src, int n, int lane) {
  for (int c = lane; c < n; c += 32)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst + c)),
                 "l"(src + c)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(32 * kStatWarps)
    k_rapid_stats_warp(const double* __restrict__ x, int n, int n1,
                       const int16_t* __restrict__ orders, const int32_t* __restrict__ omegas, int k,
                       double* __restrict__ t_out, unsigned long long* deg_key) {
  extern __shared__ __align__(16) unsigned char st_smem[];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  NpLeafPlan* plans = reinterpret_cast<NpLeafPlan*>(st_smem);  // [2]
  double* vals = reinterpret_cast<double*>(plans + 2) + (size_t)w * 2 * NpWarpScratch::kMaxLeaves;
  double* rowbuf = reinterpret_cast<double*>(plans + 2) +
                   (size_t)kStatWarps * 2 * NpWarpScratch::kMaxLeaves + (size_t)w * 2 * n;
  int16_t* ord = reinterpret_cast<int16_t*>(reinterpret_cast<double*>(plans + 2) +
                                            (size_t)kStatWarps * 2 * NpWarpScratch::kMaxLeaves +
                                            (size_t)kStatWarps * 2 * n);
  const int64_t p = blockIdx.y;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ord[i] = orders[p * n + i];
  if (threadIdx.x == 0) np_leaf_plan(n1, &plans[0]);
  if (threadIdx.x == 32) np_leaf_plan(n - n1, &plans[1]);
  __syncthreads();
  const int i0 = (blockIdx.x * kStatWarps + w) * kRowsPerWarp;
  const int i1 = min(k, i0 + kRowsPerWarp);
  if (i0 < i1) cp_async8_row(rowbuf, x + (int64_t)omegas[p * k + i0] * n, n, lane);
  for (int i = i0; i < i1; ++i) {
    double* cur = rowbuf + ((i - i0) & 1) * n;
    if (i + 1 < i1) {
      cp_async8_row(rowbuf + ((i + 1 - i0) & 1) * n, x + (int64_t)omegas[p * k + i + 1] * n, n,
                    lane);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const WelchExact r = welch_exact_warp2(cur, ord, plans[0], plans[1], vals);
    if (lane == 0) {
      t_out[p * k + i] = r.t;
      if (r.degenerate) atomicMin(deg_key, ((unsigned long long)p << 32) | (unsigned long long)i);
    }
    __syncwarp();  // every lane is done with `cur` before it is refilled
  }
}

}  // namespace

cudaError_t launch_rapid_stats(const double* x, int n, int n1, const int16_t* orders,
                               const int32_t* omegas, int64_t L, int k, double* t_out,
                               unsigned long long* deg_key, cudaStream_t s) {
  if (n1 <= NpWarpScratch::kMaxTerms && n - n1 <= NpWarpScratch::kMaxTerms && n <= 2048) {
    const size_t smem = 2 * sizeof(NpLeafPlan) +
                        (size_t)kStatWarps * 2 * NpWarpScratch::kMaxLeaves * sizeof(double) +
                        (size_t)kStatWarps * 2 * n * sizeof(double) + (size_t)n * sizeof(int16_t);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_rapid_stats_warp,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    const int per_block = kStatWarps * kRowsPerWarp;
    for (int64_t base = 0; base < L; base += 65535) {
      const int64_t cnt = L - base < 65535 ? L - base : 65535;
      dim3 grid((unsigned)((k + per_block - 1) / per_block), (unsigned)cnt);
      k_rapid_stats_warp<<<grid, 32 * kStatWarps, smem, s>>>(
          x, n, n1, orders + base * n, omegas + base * k, k, t_out + base * k, deg_key);
    }
    return cudaGetLastError();
  }
  for (int64_t base = 0; base < L; base += 65535) {
    const int64_t cnt = L - base < 65535 ? L - base : 65535;
    dim3 grid((unsigned)((k + 255) / 256), (unsigned)cnt);
    k_rapid_stats<<<grid, 256, n * sizeof(int16_t), s>>>(x, n, n1, orders + base * n,
                                                          omegas + base * k, k, t_out + base * k,
                                                          deg_key);
  }
  return cudaGetLastError();
}

}  // namespace rmx
