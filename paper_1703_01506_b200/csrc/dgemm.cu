// dgemm.cu -- the fp64 products of the M-deferred GROUSE (reference
// lrmc.py:160-193 / 208-268, restructured in rapid_abi.cu), row-major, on the
// fp64 tensor cores (DMMA, mma.sync.m8n8k4.f64):
//
//   flush (every 64 updates):  T = U X (v x r . r x nt), U += T Y^T
//   per update:                Tk = U_Omega X, U_Omega += Tk Y^T
//                              G = [U_Omega | t]^T [U_Omega | t]  (SYRK)
//
// 64 x 64 output tile per 128-thread CTA, each warp a 32 x 32 quadrant as
// 4 x 4 DMMA tiles (32 fp64 accumulators per thread).  K in steps of 16
// through a 4-stage cp.async shared-memory ring; both operands are stored
// k-major ([k][m], [k][n]) so a DMMA fragment (lane l: row / column l / 4,
// k = l % 4) is one 8-byte shared load.  A DMMA does 256 multiply-adds per
// warp instruction -- the CUDA-core DFMA version of this kernel was bound
// by shared-memory traffic and issue (mio_throttle), not by the fp64 pipe.
//
// The per-update products have few output tiles (SYRK: 28 lower tiles of
// the 401 x 401 Gram; Tk: 29 tiles) but a long K, so the K range is split
// over a thread-block cluster of S CTAs (grid z): each CTA keeps its 64 x 64
// partial in shared memory and, after one cluster barrier, CTA z sums rows
// [z 64/S, (z+1) 64/S) of the tile across the S partials through DSMEM in a
// fixed order (deterministic -- no atomics) and writes them.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "rapid_internal.cuh"
#include "sm100.cuh"

namespace rmx {
namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kT = 128;
constexpr int kLd = 72;                                      // smem row stride (doubles)
// three stages (54 KB) and <= 128 registers: four CTAs per SM.  The k x r x r
// product of a GROUSE update has 406 CTAs and shares the GPU with the solve's
// 16-SM cluster; at three CTAs per SM (four stages, 162 registers) ten of them
// fell into a second wave (68 us in situ against 47 us alone; now 56 us)
constexpr int kStages = 3;                                   // cp.async ring depth
constexpr int kTileD = kBK * kLd;                            // doubles per operand tile
constexpr int kStage = kStages * 2 * kTileD;                 // doubles: the A + B ring
constexpr int kPart = kBM * (kBN + 1);                       // doubles: the CTA's partial tile
static_assert(kPart <= kStage, "the partial tile reuses the ring");

__device__ __forceinline__ double ld_cluster_f64(const double* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  double v;
  // no memory clobber: ordering comes from the cluster barriers, so the S
  // loads of one output element are all in flight before the first add
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
  return v;
}

__device__ __forceinline__ void cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// SYRK = false: C (m x n) (+)= A (m x kk) B (kk x n).
// SYRK = true:  C (n x n, symmetric, both halves written) = A^T A with A
//               (kk x n) row-major; blockIdx.x enumerates the lower tiles.
template <bool SYRK>
__global__ void __launch_bounds__(kT, 4) k_dgemm_rm(int64_t m, int n, int kk,
                                                 const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int64_t ldb,
                                                 double* __restrict__ C, int64_t ldc, int accum) {
  pdl_wait();
  extern __shared__ __align__(16) double dsm[];
  auto As = [&](int st) { return dsm + (size_t)st * 2 * kTileD; };
  auto Bs = [&](int st) { return dsm + (size_t)st * 2 * kTileD + kTileD; };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
  // 16-byte copies when the rows (and so every even column) are 16-byte aligned
  const bool a16 = SYRK && ((lda & 1) == 0) && lda >= n + (n & 1) &&
                   ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool b16 = !SYRK && ((ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
  // stage t: K rows [kb + 16 t, +16)
  auto issue = [&](int t) {
    const int st = t % kStages, k0 = kb + t * kBK;
    double* as = As(st);
    double* bs = Bs(st);
    if (SYRK) {  // both operands are rows of A: [k][m0 + c] and [k][n0 + c]
      if (a16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // 16 x 32 pairs per operand
          const int e = tid + kT * q, kr = e >> 5, cc = (e & 31) * 2, krow = k0 + kr;
          const int ci = (int)m0 + cc, cj = n0 + cc;
          double* da = as + kr * kLd + cc;
          double* db = bs + kr * kLd + cc;
          // a pair starting at n - 1 reads the (allocated, even-length row)
          // padding column: only output entries of columns >= n see it, and
          // they are never written
          if (krow < ke && ci < n) cp16(da, A + (int64_t)krow * lda + ci); else da[0] = da[1] = 0.0;
          if (krow < ke && cj < n) cp16(db, A + (int64_t)krow * lda + cj); else db[0] = db[1] = 0.0;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = tid + kT * q, kr = e >> 6, cc = e & 63, krow = k0 + kr;
          const int ci = (int)m0 + cc, cj = n0 + cc;
          double* da = as + kr * kLd + cc;
          double* db = bs + kr * kLd + cc;
          if (krow < ke && ci < n) cp8(da, A + (int64_t)krow * lda + ci); else *da = 0.0;
          if (krow < ke && cj < n) cp8(db, A + (int64_t)krow * lda + cj); else *db = 0.0;
        }
      }
    } else {
      // A tile (64 rows x 16 k) -> [k][row]: 8-byte scatter
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = tid + kT * q, ar = e >> 4, ak = e & 15;
        const int64_t row = m0 + ar;
        const int c = k0 + ak;
        double* da = as + ak * kLd + ar;
        if (row < m && c < ke) cp8(da, A + row * lda + c); else *da = 0.0;
      }
      if (b16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = tid + kT * q, br = e >> 5, bc = (e & 31) * 2, krow = k0 + br, cn = n0 + bc;
          double* db = bs + br * kLd + bc;
          if (krow < ke && cn + 1 < n) {
            cp16(db, B + (int64_t)krow * ldb + cn);
          } else {
            db[0] = (krow < ke && cn < n) ? B[(int64_t)krow * ldb + cn] : 0.0;
            db[1] = 0.0;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = tid + kT * q, br = e >> 6, bc = e & 63, krow = k0 + br, cn = n0 + bc;
          double* db = bs + br * kLd + bc;
          if (krow < ke && cn < n) cp8(db, B + (int64_t)krow * ldb + cn); else *db = 0.0;
        }
      }
    }
  };
  // warp quadrant (32 x 32) and this lane's fragment coordinates
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
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
#pragma unroll
    for (int k4 = 0; k4 < kBK; k4 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[(k4 + fk) * kLd + wr + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[(k4 + fk) * kLd + wc + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
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
  // accumulator (i, j, h): tile row wr + 8 i + lane / 4, column wc + 8 j + 2 (lane % 4) + h
  const int cr = lane >> 2, cc2 = (lane & 3) * 2;
  if (S == 1) {
    if (!SYRK && accum) {  // C += : all 32 loads in flight before the first store
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t row = m0 + wr + 8 * i + cr;
            const int c = n0 + wc + 8 * j + cc2 + h;
            acc[i][j][h] += (row < m && c < n) ? C[row * ldc + c] : 0.0;
          }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t row = m0 + wr + 8 * i + cr;
            const int c = n0 + wc + 8 * j + cc2 + h;
            if (row < m && c < n) C[row * ldc + c] = acc[i][j][h];
          }
      return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          put(m0 + wr + 8 * i + cr, n0 + wc + 8 * j + cc2 + h, acc[i][j][h]);
    return;
  }
  // cluster split-K: partial tile -> smem, then CTA z reduces its row band
  double* P = dsm;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        P[(wr + 8 * i + cr) * (kBN + 1) + wc + 8 * j + cc2 + h] = acc[i][j][h];
  cluster_sync();
  const int band = kBM / S;
  for (int e = tid; e < band * kBN; e += kT) {
    const int i = z * band + e / kBN, j = e % kBN;
    double part[8];
#pragma unroll
    for (int s = 0; s < 8; ++s)
      part[s] = s < S ? ld_cluster_f64(P + i * (kBN + 1) + j, (uint32_t)s) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (s < S) sum += part[s];  // fixed order: deterministic
    put(m0 + i, n0 + j, sum);
  }
  cluster_sync();  // no CTA leaves while a peer still reads its partial
}

// K split for grids that cannot fill the GPU: up to 8 CTAs per tile while
// the grid stays within ~4 CTAs per SM and every CTA keeps >= 32 K rows
int pick_split(int64_t tiles, int kk) {
  static const int cap = [] {
    const char* e = getenv("RMX_DGEMM_SPLIT_MAX");  // experiments: cap the cluster split
    return e ? std::max(1, std::min(8, atoi(e))) : 8;
  }();
  static const int64_t lim = [] {
    const char* e = getenv("RMX_DGEMM_SPLIT_CTAS");  // experiments: CTA budget of the split
    return e ? (int64_t)std::max(148, atoi(e)) : (int64_t)4 * 148;
  }();
  int S = 1;
  while (S < cap && tiles * S * 2 <= lim && kk / (2 * S) >= 2 * kBK) S *= 2;
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
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  grid.z = S;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = S;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
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
