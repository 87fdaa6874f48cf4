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

// Warp per Omega row: the warp stages the row in smem and evaluates it with
// the numpy-pairwise chains spread over its lanes (welch_exact_warp: same
// bits as welch_exact).  grid (ceil(k / (8 * kRowsPerWarp)), L), 8 warps.
constexpr int kStatWarps = 8;
constexpr int kRowsPerWarp = 8;

__global__ void __launch_bounds__(32 * kStatWarps)
    k_rapid_stats_warp(const double* __restrict__ x, int n, int n1,
                       const int16_t* __restrict__ orders, const int32_t* __restrict__ omegas, int k,
                       double* __restrict__ t_out, unsigned long long* deg_key) {
  extern __shared__ __align__(16) unsigned char st_smem[];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  NpWarpScratch* sc = reinterpret_cast<NpWarpScratch*>(st_smem) + w;
  double* rowbuf = reinterpret_cast<double*>(st_smem + kStatWarps * sizeof(NpWarpScratch)) +
                   (size_t)w * n;
  int16_t* ord = reinterpret_cast<int16_t*>(st_smem + kStatWarps * sizeof(NpWarpScratch) +
                                            (size_t)kStatWarps * n * sizeof(double));
  const int64_t p = blockIdx.y;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ord[i] = orders[p * n + i];
  __syncthreads();
  const int i0 = (blockIdx.x * kStatWarps + w) * kRowsPerWarp;
  for (int i = i0; i < min(k, i0 + kRowsPerWarp); ++i) {
    const double* row = x + (int64_t)omegas[p * k + i] * n;
    __syncwarp();
    for (int c = lane; c < n; c += 32) rowbuf[c] = row[c];
    __syncwarp();
    const WelchExact r = welch_exact_warp(rowbuf, 1, ord, n1, n - n1, sc);
    if (lane == 0) {
      t_out[p * k + i] = r.t;
      if (r.degenerate) atomicMin(deg_key, ((unsigned long long)p << 32) | (unsigned long long)i);
    }
  }
}

}  // namespace

cudaError_t launch_rapid_stats(const double* x, int n, int n1, const int16_t* orders,
                               const int32_t* omegas, int64_t L, int k, double* t_out,
                               unsigned long long* deg_key, cudaStream_t s) {
  if (n <= 2048) {
    const size_t smem = kStatWarps * sizeof(NpWarpScratch) + (size_t)kStatWarps * n * sizeof(double) +
                        (size_t)n * sizeof(int16_t);
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
