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

}  // namespace

cudaError_t launch_rapid_stats(const double* x, int n, int n1, const int16_t* orders,
                               const int32_t* omegas, int64_t L, int k, double* t_out,
                               unsigned long long* deg_key, cudaStream_t s) {
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
