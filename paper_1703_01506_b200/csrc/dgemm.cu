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
// 16 through a 4-stage cp.async shared-memory ring.
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
constexpr int kStages = 4;                                   // cp.async ring depth
constexpr int kTileD = kBK * (kBM + 2);                      // doubles per operand tile
constexpr int kStage = kStages * 2 * kTileD;                 // doubles: the A + B ring
constexpr int kPart = kBM * (kBN + 1);                       // doubles: the CTA's partial tile
static_assert(kPart <= kStage, "the partial tile reuses the ring");

__device__ __forceinline__ double ld_cluster_f64(const double* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

__device__ __forceinline__ void cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// SYRK = false: C (m x n) (+)= A (m x kk) B (kk x n).
// SYRK = true:  C (n x n, symmetric, both halves written) = A^T A with A
//               (kk x n) row-major; blockIdx.x enumerates the lower tiles.
// Operand tiles stream through a kStages-deep cp.async ring (8-byte copies:
// any leading dimension), A^T tiles stored [k][m] so both operands are read
// as 2-wide vectors.
template <bool SYRK>
__global__ void __launch_bounds__(kT, 2) k_dgemm_rm(int64_t m, int n, int kk,
                                                    const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ B, int64_t ldb,
                                                    double* __restrict__ C, int64_t ldc, int accum) {
  extern __shared__ __align__(16) double dsm[];
  auto As = [&](int st) { return dsm + (size_t)st * 2 * kTileD; };
  auto Bs = [&](int st) { return dsm + (size_t)st * 2 * kTileD + kTileD; };
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
  const int nk = (ke - kb + kBK - 1) / kBK;
  // stage t: K rows [kb + 16 t, +16).  Element e = tid + 256 q (q < 4) of a
  // 16 x 64 tile.  SYRK: (row e / 64, col e % 64) of A for both operands
  // (coalesced along rows); GEMM: A tile (row e / 16, k e % 16) -> As[k][row],
  // B tile (k e / 64, col e % 64).
  auto issue = [&](int t) {
    const int st = t % kStages, k0 = kb + t * kBK;
    double* as = As(st);
    double* bs = Bs(st);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + kT * q;
      if (SYRK) {
        const int kr = e >> 6, cc = e & 63, krow = k0 + kr;
        const int ci = (int)m0 + cc, cj = n0 + cc;
        double* da = as + kr * (kBM + 2) + cc;
        double* db = bs + kr * (kBN + 2) + cc;
        if (krow < ke && ci < n) cp8(da, A + (int64_t)krow * lda + ci); else *da = 0.0;
        if (krow < ke && cj < n) cp8(db, A + (int64_t)krow * lda + cj); else *db = 0.0;
      } else {
        const int ar = e >> 4, ak = e & 15;
        const int64_t row = m0 + ar;
        const int c = k0 + ak;
        double* da = as + ak * (kBM + 2) + ar;
        if (row < m && c < ke) cp8(da, A + row * lda + c); else *da = 0.0;
        const int br = e >> 6, bc = e & 63, krow = k0 + br, cn = n0 + bc;
        double* db = bs + br * (kBN + 2) + bc;
        if (krow < ke && cn < n) cp8(db, B + (int64_t)krow * ldb + cn); else *db = 0.0;
      }
    }
  };
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll
  for (int t = 0; t < kStages - 1; ++t) {
    if (t < nk) issue(t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = 0; t < nk; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
    __syncthreads();  // stage t landed for every thread; stage t - 1's slot is free
    if (t + kStages - 1 < nk) issue(t + kStages - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* as = As(t % kStages);
    const double* bs = Bs(t % kStages);
    // thread (tx, ty): rows 2 ty + {0, 1, 32, 33}, columns 2 tx + {0, 1, 32,
    // 33}: a warp's B reads are 256 contiguous bytes (2 wavefronts, no bank
    // conflicts) and its A reads two broadcast addresses, so the fp64 FMA
    // pipe, not shared memory, bounds the loop
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      const double2 a01 = *reinterpret_cast<const double2*>(as + k * (kBM + 2) + ty * 2);
      const double2 a23 = *reinterpret_cast<const double2*>(as + k * (kBM + 2) + ty * 2 + 32);
      const double2 b01 = *reinterpret_cast<const double2*>(bs + k * (kBN + 2) + tx * 2);
      const double2 b23 = *reinterpret_cast<const double2*>(bs + k * (kBN + 2) + tx * 2 + 32);
      const double a[4] = {a01.x, a01.y, a23.x, a23.y};
      const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();  // the ring is free (the partial tile reuses it)
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
  auto rof = [&](int i) { return ty * 2 + (i & 1) + (i >> 1) * 32; };  // tile row of acc[i]
  auto cof = [&](int j) { return tx * 2 + (j & 1) + (j >> 1) * 32; };  // tile column of acc[.][j]
  if (S == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) put(m0 + rof(i), n0 + cof(j), acc[i][j]);
    return;
  }
  // cluster split-K: partial tile -> smem, then CTA z reduces its row band
  double* P = dsm;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) P[rof(i) * (kBN + 1) + cof(j)] = acc[i][j];
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
// the grid stays within ~2 waves of 2 CTAs per SM and every CTA keeps >= 32 K rows
int pick_split(int64_t tiles, int kk) {
  int S = 1;
  while (S < 8 && tiles * S * 2 <= 4 * 148 && kk / (2 * S) >= 2 * kBK) S *= 2;
  return S;
}

template <bool SYRK>
cudaError_t launch(dim3 grid, int S, int64_t m, int n, int kk, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc, int accum,
                   cudaStream_t s) {
  const size_t smem = (size_t)kStage * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_dgemm_rm<SYRK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kStage * sizeof(double)));
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
