// dgemm.cu -- the fp64 products of the M-deferred GROUSE (reference
// lrmc.py:160-193 / 208-268, restructured in rapid_abi.cu): register-tiled
// CUDA-core DGEMM / SYRK, row-major.  B200 runs fp64 FMA on the CUDA cores
// at the same rate as fp64 DMMA, so this is the plain dense kernel:
//
//   flush (every 64 updates):  T = U X (v x r . r x nt), U += T Y^T
//   per update:                Tk = U_Omega X, U_Omega += Tk Y^T
//                              G = [U_Omega | t]^T [U_Omega | t]  (SYRK)
//
// 64 x 64 output tile per 256-thread CTA (4 x 4 per thread), K in steps of
// 16 through a double-buffered shared-memory stage (the next step's global
// loads are in registers while the current one is multiplied).  The A tile
// is stored transposed so both operands are read as 2-wide vectors.
//
// The per-update products have few output tiles (SYRK: 28 lower tiles of
// the 401 x 401 Gram; Tk: 29 tiles) but a long K, so the K range is split
// over a thread-block cluster of S CTAs (grid z): each CTA keeps its 64 x 64
// partial in shared memory and, after one cluster barrier, CTA z sums rows
// [z 64/S, (z+1) 64/S) of the tile across the S partials through DSMEM in a
// fixed order (deterministic -- no atomics) and writes them.
#include <algorithm>
#include <cstdint>

#include "rapid_internal.cuh"
#include "sm100.cuh"

namespace rmx {
namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kT = 256;
constexpr int kStage = 2 * 2 * kBK * (kBM + 2);  // doubles: As + Bs, double-buffered
constexpr int kPart = kBM * (kBN + 1);          // doubles: the CTA's partial tile

__device__ __forceinline__ double ld_cluster_f64(const double* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

// SYRK = false: C (m x n) (+)= A (m x kk) B (kk x n).
// SYRK = true:  C (n x n, symmetric, both halves written) = A^T A with A
//               (kk x n) row-major; blockIdx.x enumerates the lower tiles.
template <bool SYRK>
__global__ void __launch_bounds__(kT) k_dgemm_rm(int64_t m, int n, int kk,
                                                 const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int64_t ldb,
                                                 double* __restrict__ C, int64_t ldc, int accum) {
  extern __shared__ __align__(16) double dsm[];
  double (*As)[kBK][kBM + 2] = reinterpret_cast<double (*)[kBK][kBM + 2]>(dsm);
  double (*Bs)[kBK][kBN + 2] = reinterpret_cast<double (*)[kBK][kBN + 2]>(dsm + 2 * kBK * (kBM + 2));
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  int64_t m0;
  int n0;
  if (SYRK) {  // lower-triangle tile index -> (ti, tj), tj <= ti
    int ti = 0, rem = blockIdx.x;
    while (rem > ti) {
      rem -= ti + 1;
      ++ti;
    }
    m0 = (int64_t)ti * kBM;
    n0 = rem * kBN;
  } else {
    m0 = (int64_t)blockIdx.x * kBM;
    n0 = blockIdx.y * kBN;
  }
  // this CTA's K range (split over the cluster in z)
  const int S = gridDim.z, z = blockIdx.z;
  const int kper = ((kk + S - 1) / S + kBK - 1) / kBK * kBK;
  const int kb = min(kk, z * kper), ke = min(kk, kb + kper);
  // loader mapping.  GEMM A tile (kBM x kBK): thread -> row tid / 4, cols
  // 4 (tid % 4) ..; SYRK A^T tile = rows of A: thread -> row tid / 16, cols
  // 4 (tid % 16) .. (coalesced).  B tile (kBK x kBN): row tid / 16, cols 4 (tid % 16) ..
  const int ar = tid >> 2, ac = (tid & 3) * 4;
  const int br = tid >> 4, bc = (tid & 15) * 4;
  double ra[4], rb[4];
  auto load = [&](int k0) {
    if (SYRK) {
      const int krow = k0 + br;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ci = (int)m0 + bc + q, cj = n0 + bc + q;
        const bool rowok = krow < ke;
        ra[q] = (rowok && ci < n) ? A[(int64_t)krow * lda + ci] : 0.0;
        rb[q] = (rowok && cj < n) ? A[(int64_t)krow * lda + cj] : 0.0;
      }
    } else {
      const int64_t row = m0 + ar;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = k0 + ac + q;
        ra[q] = (row < m && c < ke) ? A[row * lda + c] : 0.0;
      }
      const int krow = k0 + br;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = n0 + bc + q;
        rb[q] = (krow < ke && c < n) ? B[(int64_t)krow * ldb + c] : 0.0;
      }
    }
  };
  auto store = [&](int buf) {
    if (SYRK) {
#pragma unroll
      for (int q = 0; q < 4; ++q) As[buf][br][bc + q] = ra[q];
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) As[buf][ac + q][ar] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) Bs[buf][br][bc + q] = rb[q];
  };
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int nk = (ke - kb + kBK - 1) / kBK;
  if (nk > 0) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load(kb + (t + 1) * kBK);
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
  auto put = [&](int64_t row, int c, double val) {
    if (SYRK) {
      if (row < n && c < n && c <= row) {
        C[row * ldc + c] = val;
        if (c != row) C[(int64_t)c * ldc + row] = val;
      }
    } else if (row < m && c < n) {
      double* p = C + row * ldc + c;
      *p = accum ? *p + val : val;
    }
  };
  if (S == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) put(m0 + ty * 4 + i, n0 + tx * 4 + j, acc[i][j]);
    return;
  }
  // cluster split-K: partial tile -> smem, then CTA z reduces its row band
  double* P = dsm + kStage;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) P[(ty * 4 + i) * (kBN + 1) + tx * 4 + j] = acc[i][j];
  cluster_sync();
  const int band = kBM / S;
  for (int e = tid; e < band * kBN; e += kT) {
    const int i = z * band + e / kBN, j = e % kBN;
    double sum = 0.0;
    for (int s = 0; s < S; ++s) sum += ld_cluster_f64(P + i * (kBN + 1) + j, (uint32_t)s);
    put(m0 + i, n0 + j, sum);
  }
  cluster_sync();  // no CTA leaves while a peer still reads its partial
}

// K split for grids that cannot fill the GPU: up to 8 CTAs per tile while
// the grid stays within ~3 CTAs per SM and every CTA keeps >= 16 K rows
int pick_split(int64_t tiles, int kk) {
  int S = 1;
  while (S < 8 && tiles * S * 2 <= 3 * 148 && kk / (2 * S) >= kBK) S *= 2;
  return S;
}

template <bool SYRK>
cudaError_t launch(dim3 grid, int S, int64_t m, int n, int kk, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc, int accum,
                   cudaStream_t s) {
  const size_t smem = (size_t)(kStage + (S > 1 ? kPart : 0)) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_dgemm_rm<SYRK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((kStage + kPart) * sizeof(double)));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  grid.z = S;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = S;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_dgemm_rm<SYRK>, m, n, kk, A, lda, B, ldb, C, ldc, accum);
}

}  // namespace

cudaError_t launch_dgemm_rm(int64_t m, int n, int kk, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double* C, int64_t ldc, int accum,
                            cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((m + kBM - 1) / kBM), (unsigned)((n + kBN - 1) / kBN), 1);
  const int S = pick_split((int64_t)grid.x * grid.y, kk);
  return launch<false>(grid, S, m, n, kk, A, lda, B, ldb, C, ldc, accum, s);
}

cudaError_t launch_dsyrk_rm(int kk, int n, const double* A, int64_t lda, double* C, int64_t ldc,
                            cudaStream_t s) {
  if (kk <= 0 || n <= 0) return cudaSuccess;
  const int nt = (n + kBM - 1) / kBM;
  const dim3 grid((unsigned)(nt * (nt + 1) / 2), 1, 1);
  const int S = pick_split(grid.x, kk);
  return launch<true>(grid, S, n, n, kk, A, lda, nullptr, 0, C, ldc, 0, s);
}

}  // namespace rmx
