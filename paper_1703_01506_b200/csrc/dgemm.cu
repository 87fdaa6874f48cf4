// dgemm.cu -- the fp64 products of the M-deferred GROUSE (reference
// lrmc.py:160-193 / 208-268, restructured in rapid_abi.cu): register-tiled
// CUDA-core DGEMM, row-major, C = A B (+ C).  B200 runs fp64 FMA on the CUDA
// cores at the same rate as fp64 DMMA, so this is the plain dense kernel:
//
//   flush (every 64 updates):  T = U X (v x r . r x nt), U += T Y^T
//   per update:                Tk = U_Omega X, U_Omega += Tk Y^T
//
// 64 x 64 output tile per 256-thread CTA (4 x 4 per thread), K in steps of
// 16 through a double-buffered shared-memory stage (the next step's global
// loads are in registers while the current one is multiplied).  The A tile
// is stored transposed so both operands are read as 2-wide vectors.
#include <cstdint>

#include "rapid_internal.cuh"

namespace rmx {
namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kT = 256;

__global__ void __launch_bounds__(kT) k_dgemm_rm(int64_t m, int n, int kk,
                                                 const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int64_t ldb,
                                                 double* __restrict__ C, int64_t ldc, int accum) {
  __shared__ __align__(16) double As[2][kBK][kBM + 2];
  __shared__ __align__(16) double Bs[2][kBK][kBN + 2];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * kBM;
  const int n0 = blockIdx.y * kBN;
  // loader mapping: A tile (kBM x kBK): thread -> row tid / 4, cols 4 (tid % 4) .. +3
  const int ar = tid >> 2, ac = (tid & 3) * 4;
  // B tile (kBK x kBN): thread -> row tid / 16, cols 4 (tid % 16) .. +3
  const int br = tid >> 4, bc = (tid & 15) * 4;
  double ra[4], rb[4];
  auto load = [&](int k0) {
    const int64_t row = m0 + ar;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = k0 + ac + q;
      ra[q] = (row < m && c < kk) ? A[row * lda + c] : 0.0;
    }
    const int krow = k0 + br;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = n0 + bc + q;
      rb[q] = (krow < kk && c < n) ? B[(int64_t)krow * ldb + c] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[buf][ac + q][ar] = ra[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) Bs[buf][br][bc + q] = rb[q];
  };
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int nk = (kk + kBK - 1) / kBK;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * kBK);
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      const double2 a01 = *reinterpret_cast<const double2*>(&As[buf][k][ty * 4]);
      const double2 a23 = *reinterpret_cast<const double2*>(&As[buf][k][ty * 4 + 2]);
      const double2 b01 = *reinterpret_cast<const double2*>(&Bs[buf][k][tx * 4]);
      const double2 b23 = *reinterpret_cast<const double2*>(&Bs[buf][k][tx * 4 + 2]);
      const double a[4] = {a01.x, a01.y, a23.x, a23.y};
      const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + ty * 4 + i;
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c < n) {
        double* p = C + row * ldc + c;
        *p = accum ? *p + acc[i][j] : acc[i][j];
      }
    }
  }
}

}  // namespace

cudaError_t launch_dgemm_rm(int64_t m, int n, int kk, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double* C, int64_t ldc, int accum,
                            cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((m + kBM - 1) / kBM), (unsigned)((n + kBN - 1) / kBN));
  k_dgemm_rm<<<grid, kT, 0, s>>>(m, n, kk, A, lda, B, ldb, C, ldc, accum);
  return cudaGetLastError();
}

}  // namespace rmx
