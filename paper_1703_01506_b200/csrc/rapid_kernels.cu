// rapid_kernels.cu -- RapidPT on the GPU (reference rapid.py / lrmc.py):
// the least-squares algebra (fp64, FMA contraction allowed) and the
// completion.  The bit-exact Omega-row statistics live in rapid_stats.cu.
//
//   k_gram          K3a: G_b = [U_Omega | t]^T [U_Omega | t] for a batch of
//                   gathered row sets (lrmc.py:136-137: gram and rhs at once)
//   k_chol_solve    K3b: blocked Cholesky of G_b[:r,:r], w = G^-1 rhs, and a
//                   singularity flag (lrmc.py:138-148; see DESIGN.md for the
//                   condition-number deviation)
//   k_cg_solve      K3b for one GROUSE system: cluster CG, Gram in DSMEM
//   k_complete_max  K4 on CUDA cores: max_j (W U^T)[p, j] + sigma z(p, j)
//                   (+ mu) (rapid.py:198-205; the tcgen05 version is
//                   k_tfill_tc<..., MODE 1> in tfill_tc.cu)
//   GROUSE step     M-deferred (lrmc.py:160-193): k_gather_urows + cuBLAS
//                   DGEMM by M, k_sparse_terms, cuBLAS Gram, k_cg_solve
//                   (warm-started), k_resid, k_defer_vec, k_grouse_post_m,
//                   k_h_g_part/_fin, k_defer_apply; flush every 64 updates
#include <cuda_fp16.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "philox.cuh"
#include "rapid_internal.cuh"
#include "sm100.cuh"

namespace rmx {
namespace {

// ------------------------------------------------------------------ K3a
// A_b = [U[idx_b[0..k)] | vals_b]  (k x (r+1)), G_b = A_b^T A_b, full
// (r+1)^2 row-major.  64x64 output tiles over the lower triangle, 64
// threads with 8x8 register tiles (4 FMAs per shared load).  The system's
// row ids are staged in smem once; gathered rows stream through a 3-stage
// cp.async ring of 16-row chunks, so the loads of chunk c+2 are in flight
// while chunk c is multiplied.  Optional split over the rows (K) with atomics.
constexpr int kGT = 64;
constexpr int kGK = 16;
constexpr int kGS = 3;  // ring stages
constexpr int kGThreads = 64;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}

__global__ void __launch_bounds__(kGThreads) k_gram(const double* __restrict__ U, int64_t ldu,
                                                    int r, const int32_t* __restrict__ idx, int k,
                                                    const double* __restrict__ vals,
                                                    double* __restrict__ G, int rows_per_split) {
  extern __shared__ __align__(16) double gsm[];
  double (*As)[kGK][kGT] = reinterpret_cast<double (*)[kGK][kGT]>(gsm);
  double (*Bs)[kGK][kGT] = reinterpret_cast<double (*)[kGK][kGT]>(gsm + kGS * kGK * kGT);
  int32_t* rid = reinterpret_cast<int32_t*>(gsm + 2 * kGS * kGK * kGT);
  const int64_t b = blockIdx.y;
  // lower-triangle tile index -> (ti, tj), tj <= ti
  int ti = 0, rem = blockIdx.x;
  while (rem > ti) {
    rem -= ti + 1;
    ++ti;
  }
  const int tj = rem;
  const bool diag = ti == tj;
  const int i0 = ti * kGT, j0 = tj * kGT;
  const int tid = threadIdx.x;
  const int tx = tid & 7, ty = tid >> 3;
  const int kbeg = blockIdx.z * rows_per_split;
  const int kend = min(k, kbeg + rows_per_split);
  const int nrows = max(0, kend - kbeg);
  if (idx) {  // gathered rows: stage the ids (dense: the row number itself)
    for (int i = tid; i < nrows; i += kGThreads) rid[i] = idx[b * k + kbeg + i];
    __syncthreads();
  }
  const double* vb = vals ? vals + b * k : nullptr;
  // chunk c -> ring slot c % kGS; thread fills column tid of 16 rows (A, B)
  auto issue = [&](int c) {
    const int slot = c % kGS;
    const int ca = i0 + tid, cb = j0 + tid;
#pragma unroll 4
    for (int rr = 0; rr < kGK; ++rr) {
      const int row = c * kGK + rr;  // relative to kbeg
      double* da = &As[slot][rr][tid];
      double* db = &Bs[slot][rr][tid];
      if (row < nrows) {
        const double* urow = U + (int64_t)(idx ? rid[row] : kbeg + row) * ldu;
        if (ca < r) cp_async8(da, urow + ca);
        else *da = (ca == r && vb) ? vb[kbeg + row] : 0.0;
        if (!diag) {
          if (cb < r) cp_async8(db, urow + cb);
          else *db = (cb == r && vb) ? vb[kbeg + row] : 0.0;
        }
      } else {
        *da = 0.0;
        if (!diag) *db = 0.0;
      }
    }
  };
  double acc[8][8];
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[q][u] = 0.0;
  const int nchunks = (nrows + kGK - 1) / kGK;
  for (int c = 0; c < kGS - 1; ++c) {
    if (c < nchunks) issue(c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kGS - 2) : "memory");
    __syncthreads();  // chunk c landed for every thread; slot (c-1) % kGS is free
    if (c + kGS - 1 < nchunks) issue(c + kGS - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int slot = c % kGS;
    const double (*Ap)[kGT] = As[slot];
    const double (*Bp)[kGT] = diag ? As[slot] : Bs[slot];
#pragma unroll 2
    for (int kk = 0; kk < kGK; ++kk) {
      double a[8], bb[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 av = *reinterpret_cast<const double2*>(&Ap[kk][ty * 8 + q]);
        const double2 bv = *reinterpret_cast<const double2*>(&Bp[kk][tx * 8 + q]);
        a[q] = av.x;
        a[q + 1] = av.y;
        bb[q] = bv.x;
        bb[q + 1] = bv.y;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[q][u] = fma(a[q], bb[u], acc[q][u]);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  const int ld = r + 1;
  double* Gb = G + b * (int64_t)ld * ld;
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + ty * 8 + q, j = j0 + tx * 8 + u;
      if (i < ld && j < ld && j <= i) {
        if (gridDim.z == 1) {
          Gb[(int64_t)i * ld + j] = acc[q][u];
          if (i != j) Gb[(int64_t)j * ld + i] = acc[q][u];
        } else {  // split-K partial sums (G zeroed by the launcher)
          atomicAdd(&Gb[(int64_t)i * ld + j], acc[q][u]);
          if (i != j) atomicAdd(&Gb[(int64_t)j * ld + i], acc[q][u]);
        }
      }
    }
}

// ------------------------------------------------------------------ K3b
// One CTA per system.  Right-looking blocked Cholesky on G[:r, :r] in place
// (global memory, L2-resident), panel width 32 (the last panel padded with
// the identity).  Per panel: one warp factors the diagonal block with the
// block held in registers (lane = row, columns broadcast by shuffles); the
// panel below is solved one row per thread with the row in registers and
// L_D broadcast from smem; the trailing lower triangle is updated with 4x4
// register tiles from the smem panel (row stride 33: conflict-free).  The
// substitutions for w run per 32-block on one warp (shuffles), the
// off-diagonal updates on all threads.  flag[b] = 1 when a pivot is not
// positive relative to the largest diagonal (rank-deficient restriction).
constexpr int kPW = 32;
constexpr int kPS = kPW + 1;  // padded smem row stride (doubles)

// Factor the 32x32 SPD block D (smem, lower part used; rows/cols >= w are
// the identity) in place into L_D; rinv[c] = 1 / L_cc.  One warp, lane =
// row, the row in registers.  The column loop is unrolled by template
// recursion (a plain 32 x 31 unrolled loop nest is left rolled by the
// compiler, which then indexes a[] dynamically -- through local memory).
template <typename T, int C>
struct Chol32Step {
  __device__ __forceinline__ static void run(T (&a)[kPW], T* rinv, T tiny, int* bad, int lane) {
    T piv = __shfl_sync(0xffffffffu, a[C], C);
    if (!(piv > tiny)) {
      if (lane == 0) *bad = 1;
      piv = fmax(fabs(piv), 1e-300);
    }
    const T d = sqrt(piv);
    const T inv = T(1) / d;  // fp32: a float division (the serial chain's longest step)
    if (lane == C) a[C] = d;
    if (lane > C) a[C] *= inv;
    if (lane == 0) rinv[C] = inv;
#pragma unroll
    for (int l = C + 1; l < kPW; ++l) {
      const T llc = __shfl_sync(0xffffffffu, a[C], l);
      if (lane >= l) a[l] = fma(-a[C], llc, a[l]);
    }
    Chol32Step<T, C + 1>::run(a, rinv, tiny, bad, lane);
  }
};
template <typename T>
struct Chol32Step<T, kPW> {
  __device__ __forceinline__ static void run(T (&)[kPW], T*, T, int*, int) {}
};

template <typename T>
__device__ __forceinline__ void chol_block32(T* D, T* rinv, T tiny, int* bad) {
  const int lane = threadIdx.x & 31;
  T a[kPW];
#pragma unroll
  for (int l = 0; l < kPW; ++l) a[l] = D[lane * kPS + l];
  if constexpr (sizeof(T) == 4) {
    Chol32Step<T, 0>::run(a, rinv, tiny, bad, lane);
  } else {  // fp64: the loop form spills less under the 2-CTA register cap
#pragma unroll
    for (int c = 0; c < kPW; ++c) {
      T piv = __shfl_sync(0xffffffffu, a[c], c);
      if (!(piv > tiny)) {
        if (lane == 0) *bad = 1;
        piv = fmax(fabs(piv), 1e-300);
      }
      const T d = sqrt(piv);
      const T inv = 1.0 / d;
      if (lane == c) a[c] = d;
      if (lane > c) a[c] *= inv;
      if (lane == 0) rinv[c] = inv;
#pragma unroll
      for (int l = c + 1; l < kPW; ++l) {
        const T llc = __shfl_sync(0xffffffffu, a[c], l);
        if (lane >= l) a[l] = fma(-a[c], llc, a[l]);
      }
    }
  }
#pragma unroll
  for (int l = 0; l < kPW; ++l) D[lane * kPS + l] = (l <= lane) ? a[l] : 0.0;
}

// rows of the panel below the first diagonal block (the largest panel)
__host__ __device__ constexpr int chol_panel_rows(int r) { return r > kPW ? r - kPW : 1; }

template <int NT, typename T = double>
__global__ void __launch_bounds__(NT, NT == 256 ? (sizeof(T) == 4 ? 3 : 2) : 1) k_chol_solve(T* __restrict__ G, int r,
                                                   double* __restrict__ w_out,
                                                   int32_t* flag, double* __restrict__ resid2,
                                                   const int32_t* gate = nullptr,
                                                   const double* __restrict__ rhs_ext = nullptr,
                                                   T* __restrict__ pscratch = nullptr,
                                                   int lookahead = 1) {
  // pscratch: the panel in global memory, so the launch needs only a few KB
  // of shared memory
  // gate: run only when *gate != 0 (Cholesky fallback after a cluster-CG
  // solve that did not converge, decided on the device)
  // rhs_ext (refinement): G already holds the factor L; solve L L^T d =
  // rhs_ext[b], w_out[b] += d, flag[b] = 1 when |d| > 1e-7 |w| (not converged)
  pdl_wait();
  if (gate && *gate == 0) return;
  __syncthreads();  // every thread has read the gate before it is overwritten
  extern __shared__ __align__(16) unsigned char chol_smem[];
  T* sm = reinterpret_cast<T*>(chol_smem);
  T* D = sm;                     // kPW x kPS: block / L_D (lower)
  T* rinv = D + kPW * kPS;       // kPW: 1 / L_cc
  T* after = rinv + kPW;
  T* P = pscratch ? pscratch : after;  // chol_panel_rows(r) x kPS panel (factor only)
  constexpr bool kLookAhead = NT == 256 && sizeof(T) == 4;  // see the factor loop
  T* y = pscratch ? after : (rhs_ext ? P : P + (size_t)chol_panel_rows(r) * kPS);  // r: rhs / solution
  __shared__ int bad;
  __shared__ T dmax;
  const int64_t b = blockIdx.x;
  const int ld = r + 1;
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  T* Gb = G + b * (int64_t)ld * ld;
  if (wid == 0 && !rhs_ext) {
    T m = 0.0;
    for (int i = lane; i < r; i += 32) m = fmax(m, Gb[(int64_t)i * ld + i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      bad = 0;
      dmax = m;
    }
  }
  __syncthreads();
  const T tiny = 1e-24 * dmax;
  auto load_block = [&](int jb, int w) {  // D = G[jb.., jb..] (lower), identity padding
    for (int e = tid; e < kPW * kPW; e += NT) {
      const int i = e / kPW, j = e % kPW;
      T val = (i == j) ? 1.0 : 0.0;
      if (i < w && j < w && j <= i) val = Gb[(int64_t)(jb + i) * ld + jb + j];
      D[i * kPS + j] = val;
    }
  };
  // Look-ahead (the batched fp32 factor of the recovery): warp 0 applies the
  // trailing update to the NEXT diagonal block only and factors it while the
  // other warps update the rest of the trailing matrix, so the serial
  // 32-step diagonal factor no longer idles 7 of 8 warps once per panel
  // (ncu: ~30% of the factor's stall samples were warps waiting for it).
  // Same arithmetic, same order: same bits.
  const bool la = kLookAhead && lookahead && !rhs_ext && !pscratch;
  if (la) {
    T* Dn = y + r;               // the second diagonal-block buffer
    T* rn = Dn + kPW * kPS;
    T* Dc = D;
    T* rc = rinv;
    load_block(0, min(kPW, r));
    __syncthreads();
    if (wid == 0) chol_block32(Dc, rc, tiny, &bad);
    __syncthreads();
    for (int jb = 0; jb < r; jb += kPW) {
      const int w = min(kPW, r - jb);
      for (int e = tid; e < w * w; e += NT) {
        const int i = e / w, j = e % w;
        if (j <= i) Gb[(int64_t)(jb + i) * ld + jb + j] = Dc[i * kPS + j];
      }
      const int rows = r - jb - w;
      for (int i = tid; i < rows; i += NT) {  // panel rows, as below
        T* gi = Gb + (int64_t)(jb + w + i) * ld + jb;
        T pr[kPW];
#pragma unroll
        for (int c = 0; c < kPW; ++c) pr[c] = c < w ? gi[c] : 0.0;
#pragma unroll
        for (int c = 0; c < kPW; ++c) {
          T sacc = pr[c];
#pragma unroll
          for (int l = 0; l < c; ++l) sacc = fma(-pr[l], Dc[c * kPS + l], sacc);
          pr[c] = sacc * rc[c];
        }
        T* prow = P + (size_t)i * kPS;
#pragma unroll
        for (int c = 0; c < kPW; ++c) {
          prow[c] = pr[c];
          if (c < w) gi[c] = pr[c];
        }
      }
      __syncthreads();
      if (rows <= 0) break;
      const int wn = min(kPW, rows);
      if (wid == 0) {
        // next diagonal block = its G entries minus P_i . P_j, row `lane`
        const int i = lane;
        const T* pi = P + (size_t)i * kPS;
        for (int j = 0; j < kPW; ++j) {
          T val = (i == j) ? 1.0 : 0.0;
          if (i < wn && j < wn && j <= i) {
            const T* pj = P + (size_t)j * kPS;
            T acc = 0.0;
#pragma unroll 8
            for (int c = 0; c < kPW; ++c) acc = fma(pi[c], pj[c], acc);
            val = Gb[(int64_t)(jb + w + i) * ld + jb + w + j] - acc;
          }
          Dn[i * kPS + j] = val;
        }
        __syncwarp();
        chol_block32(Dn, rn, tiny, &bad);
      } else {
        // the rest of the trailing lower triangle: 4 x 4 tiles whose rows
        // lie below the next diagonal block (tile rows 4 bi >= wn)
        const int nb = (rows + 3) / 4;
        const int t0 = ((wn + 3) / 4) * ((wn + 3) / 4 + 1) / 2;  // tiles inside the block
        const int ntile = nb * (nb + 1) / 2;
        for (int t = t0 + tid - 32; t < ntile; t += NT - 32) {
          int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
          while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
          while (bi * (bi + 1) / 2 > t) --bi;
          const int bj = t - bi * (bi + 1) / 2;
          T acc[4][4] = {};
          const T* pi = P + (size_t)(4 * bi) * kPS;
          const T* pj = P + (size_t)(4 * bj) * kPS;
#pragma unroll 4
          for (int c = 0; c < kPW; ++c) {
            T a[4], bb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              a[q] = (4 * bi + q < rows) ? pi[q * kPS + c] : 0.0;
              bb[q] = (4 * bj + q < rows) ? pj[q * kPS + c] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int u = 0; u < 4; ++u) acc[q][u] = fma(a[q], bb[u], acc[q][u]);
          }
          // all 16 loads in flight before the first store (the element-wise
          // load-subtract-store chain serialised on the L2 latency)
          T old[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = 4 * bi + q;
            const T* grow = Gb + (int64_t)(jb + w + i) * ld + jb + w;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = 4 * bj + u;
              old[q][u] = (i < rows && j <= i) ? grow[j] : T(0);
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = 4 * bi + q;
            if (i >= rows) continue;
            T* grow = Gb + (int64_t)(jb + w + i) * ld + jb + w;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = 4 * bj + u;
              if (j <= i) grow[j] = old[q][u] - acc[q][u];
            }
          }
        }
      }
      __syncthreads();
      T* tD = Dc;
      Dc = Dn;
      Dn = tD;
      T* tr = rc;
      rc = rn;
      rn = tr;
    }
  }
  for (int jb = 0; jb < ((rhs_ext || la) ? 0 : r); jb += kPW) {
    const int w = min(kPW, r - jb);
    load_block(jb, w);
    __syncthreads();
    if (wid == 0) chol_block32(D, rinv, tiny, &bad);
    __syncthreads();
    for (int e = tid; e < w * w; e += NT) {
      const int i = e / w, j = e % w;
      if (j <= i) Gb[(int64_t)(jb + i) * ld + jb + j] = D[i * kPS + j];
    }
    // panel below: P_i L_D^T = G[i, jb:jb+w], one row per thread (registers)
    const int rows = r - jb - w;
    for (int i = tid; i < rows; i += NT) {
      T* gi = Gb + (int64_t)(jb + w + i) * ld + jb;
      T pr[kPW];
#pragma unroll
      for (int c = 0; c < kPW; ++c) pr[c] = c < w ? gi[c] : 0.0;
#pragma unroll
      for (int c = 0; c < kPW; ++c) {
        T sacc = pr[c];
#pragma unroll
        for (int l = 0; l < c; ++l) sacc = fma(-pr[l], D[c * kPS + l], sacc);
        pr[c] = sacc * rinv[c];
      }
      T* prow = P + (size_t)i * kPS;
#pragma unroll
      for (int c = 0; c < kPW; ++c) {
        prow[c] = pr[c];
        if (c < w) gi[c] = pr[c];
      }
    }
    __syncthreads();
    // trailing update G[i, j] -= P_i . P_j over jb+w <= j <= i < r, 4x4 tiles
    const int nb = (rows + 3) / 4;
    const int ntile = nb * (nb + 1) / 2;
    for (int t = tid; t < ntile; t += NT) {
      int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);  // t -> (bi, bj), bj <= bi
      while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
      while (bi * (bi + 1) / 2 > t) --bi;
      const int bj = t - bi * (bi + 1) / 2;
      T acc[4][4] = {};
      const T* pi = P + (size_t)(4 * bi) * kPS;
      const T* pj = P + (size_t)(4 * bj) * kPS;
#pragma unroll 4
      for (int c = 0; c < kPW; ++c) {
        T a[4], bb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = (4 * bi + q < rows) ? pi[q * kPS + c] : 0.0;
          bb[q] = (4 * bj + q < rows) ? pj[q * kPS + c] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[q][u] = fma(a[q], bb[u], acc[q][u]);
      }
      T old[4][4];  // all loads in flight before the first store
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = 4 * bi + q;
        const T* grow = Gb + (int64_t)(jb + w + i) * ld + jb + w;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * bj + u;
          old[q][u] = (i < rows && j <= i) ? grow[j] : T(0);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = 4 * bi + q;
        if (i >= rows) continue;
        T* grow = Gb + (int64_t)(jb + w + i) * ld + jb + w;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * bj + u;
          if (j <= i) grow[j] = old[q][u] - acc[q][u];
        }
      }
    }
    __syncthreads();
  }
  // solve L L^T w = rhs (rhs = G[r, 0:r], the A^T t row), blocked
  for (int i = tid; i < r; i += NT) y[i] = rhs_ext ? rhs_ext[b * r + i] : Gb[(int64_t)r * ld + i];
  __syncthreads();
  for (int jb = 0; jb < r; jb += kPW) {  // forward: L y = rhs
    const int w = min(kPW, r - jb);
    load_block(jb, w);
    __syncthreads();
    if (wid == 0) {  // lane c holds y[jb + c]; row `lane` of L_D in registers
      T lr[kPW];
#pragma unroll
      for (int c = 0; c < kPW; ++c) lr[c] = D[lane * kPS + c];
      T yb = lane < w ? y[jb + lane] : 0.0;
#pragma unroll
      for (int c = 0; c < kPW; ++c) {
        if (lane == c) yb /= lr[c];
        const T yc = __shfl_sync(0xffffffffu, yb, c);
        if (lane > c) yb = fma(-lr[c], yc, yb);
      }
      if (lane < w) y[jb + lane] = yb;
    }
    __syncthreads();
    for (int i = jb + w + tid; i < r; i += NT) {
      const T* li = Gb + (int64_t)i * ld + jb;
      T sacc = 0.0;
      for (int c = 0; c < w; ++c) sacc = fma(li[c], y[jb + c], sacc);
      y[i] -= sacc;
    }
    __syncthreads();
  }
  for (int jb = ((r - 1) / kPW) * kPW; jb >= 0; jb -= kPW) {  // backward: L^T w = y
    const int w = min(kPW, r - jb);
    load_block(jb, w);
    __syncthreads();
    if (wid == 0) {  // lane c holds y[jb + c]; column `lane` of L_D in registers
      T lc[kPW];
#pragma unroll
      for (int c = 0; c < kPW; ++c) lc[c] = D[c * kPS + lane];
      T yb = lane < w ? y[jb + lane] : 0.0;
#pragma unroll
      for (int c = kPW - 1; c >= 0; --c) {
        if (lane == c) yb /= lc[c];
        const T wc = __shfl_sync(0xffffffffu, yb, c);
        if (lane < c) yb = fma(-lc[c], wc, yb);
      }
      if (lane < w) y[jb + lane] = yb;
    }
    __syncthreads();
    for (int i = tid; i < jb; i += NT) {  // coalesced: row jb+c, columns i
      T sacc = 0.0;
      for (int c = 0; c < w; ++c) sacc = fma(Gb[(int64_t)(jb + c) * ld + i], y[jb + c], sacc);
      y[i] -= sacc;
    }
    __syncthreads();
  }
  if (rhs_ext) {
    if (tid < 32) {
      double dd = 0.0, ww = 0.0;
      for (int i = lane; i < r; i += 32) {
        const double wn = w_out[b * r + i] + (double)y[i];
        w_out[b * r + i] = wn;
        dd += y[i] * y[i];
        ww += wn * wn;
      }
      for (int o = 16; o > 0; o >>= 1) {
        dd += __shfl_xor_sync(0xffffffffu, dd, o);
        ww += __shfl_xor_sync(0xffffffffu, ww, o);
      }
      if (lane == 0 && flag) flag[b] = (dd > 1e-14 * ww) ? 1 : 0;
    }
    return;
  }
  if (tid < 32) {
    if (w_out)
      for (int i = lane; i < r; i += 32) w_out[b * r + i] = y[i];
    if (resid2) {
      // resid2[4b..4b+3] = (t.t - rhs.w, w.w, min L_ii, max L_ii): residual
      // norm^2 by the normal equations, the coefficient norm^2 (GROUSE) and
      // the pivot range (max/min L_ii is a lower bound of cond(U_Omega))
      double rw = 0.0, ww = 0.0, dmn = DBL_MAX, dmx = 0.0;
      for (int i = lane; i < r; i += 32) {
        rw += Gb[(int64_t)r * ld + i] * y[i];
        ww += y[i] * y[i];
        const T dd = Gb[(int64_t)i * ld + i];
        dmn = fmin(dmn, dd);
        dmx = fmax(dmx, dd);
      }
      for (int o = 16; o > 0; o >>= 1) {
        rw += __shfl_xor_sync(0xffffffffu, rw, o);
        ww += __shfl_xor_sync(0xffffffffu, ww, o);
        dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
        dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
      }
      if (lane == 0) {
        resid2[4 * b] = Gb[(int64_t)r * ld + r] - rw;
        resid2[4 * b + 1] = ww;
        resid2[4 * b + 2] = dmn;
        resid2[4 * b + 3] = dmx;
      }
    }
    if (lane == 0 && flag) flag[b] = bad;
  }
}

// ------------------------------------------------------------------ K3b (GROUSE)
// One GROUSE solve (B = 1) on a cluster of kCgCtas CTAs: G[:r, :r] is
// split by rows across the CTAs' shared memory (the whole Gram lives on
// chip, 80 KB per CTA at r = 400) and solved by Jacobi-preconditioned
// conjugate gradients.  The U_Omega Gram of a random row sample is well
// conditioned (kappa ~ (1 + sqrt(r/k))^2 / (1 - sqrt(r/k))^2 ~ 8 at config
// 5), so CG reaches the 1e-13 relative residual in ~40 iterations; each
// iteration is a local 25 x 400 mat-vec plus ONE cluster barrier (pipelined
// CG below).  16 CTAs instead of 8: 0.23 -> 0.18 ms per solve at config 5.
// flag = 1 when it has not converged after r iterations: the caller then
// runs the Cholesky kernel on the same (unmodified) G, whose pivots decide
// the ill-conditioning exactly as before.
constexpr int kCgCtas = 16;  // non-portable cluster size (GPCs hold >= 16 SMs)
constexpr int kCgThreads = 256;

// remote store that signals the destination CTA's mbarrier (complete_tx of
// 8 bytes): the receiver waits on its own barrier, no cluster-wide barrier
__device__ __forceinline__ void st_async_f64(double* local_ptr, uint32_t rank, double v,
                                             uint64_t* local_bar) {
  uint32_t raddr, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_ptr)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
               ::"r"(raddr), "d"(v), "r"(rbar)
               : "memory");
}



// Pipelined preconditioned CG (Ghysels & Vanroose, p-PCG): besides x, r,
// u = M r and w = A u, the recurrences carry m = M w, n = A m, z, q, s, p, so
// an iteration needs ONE matrix-vector product (n = A m) and ONE global
// reduction (r.u, w.u, r.r), and both exchanges -- m's rows for the product
// and the three partial dot products -- are posted to every CTA of the
// cluster before a single cluster barrier (DSMEM, double-buffered by
// iteration parity: a CTA can be at most one barrier ahead of another).  The
// classic PCG needed three barriers per iteration.  The stopping test uses
// the recurrence residual; the result is then checked against the true
// residual b - A x, and flag = 1 (Cholesky fallback) when that check or the
// iteration cap fails.
// RMX_CG_STATS phase clocks (CTA 0, thread 0, per iteration): local partial
// dots, block reduction, post + wait for the peers, matvec, vector updates
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// RMX_GROUSE_TRACE (diagnostics): block 0 of each chain kernel stamps its
// entry, the end of its pdl_wait and its exit with the global timer
constexpr unsigned kTraceCap = 16384;
__device__ unsigned long long g_tr[2 * kTraceCap];
__device__ unsigned int g_tr_n;
__device__ int g_tr_on;
__device__ __forceinline__ void tr(int id, int ph) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && g_tr_on) {
    const unsigned i = atomicAdd(&g_tr_n, 1u);
    if (i < kTraceCap) {
      g_tr[2 * i] = globaltimer_ns();
      g_tr[2 * i + 1] = (unsigned long long)(id * 4 + ph);
    }
  }
}
__device__ unsigned long long g_cg_phase[6];
__device__ unsigned long long g_cg_wall[4];  // ns: load G, setup to the loop, loop, tail
__device__ int g_cg_timing;

__device__ __forceinline__ void cg_block_reduce3(double a, double b, double c, double* wsum,
                                                 double& A, double& B, double& C) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    wsum[3 * wid] = a;
    wsum[3 * wid + 1] = b;
    wsum[3 * wid + 2] = c;
  }
  __syncthreads();
  A = B = C = 0.0;
  for (int w = 0; w < kCgThreads / 32; ++w) {
    A += wsum[3 * w];
    B += wsum[3 * w + 1];
    C += wsum[3 * w + 2];
  }
}

// Post this CTA's rows of `v` (nr values) into every CTA's `full` and this
// CTA's totals (a, b, c) into every CTA's slot row `me`, then one cluster
// barrier; returns the cluster sums (same order, same bits on every CTA).
template <int NC>
__device__ __forceinline__ void cg_exchange(const double* v, int nr, int r0, int rtot, double* full,
                                            double a, double b, double c, double* slots,
                                            double* wsum, uint64_t* bars, int par, uint32_t& xph,
                                            double& A, double& B, double& C) {
  const uint32_t me = cluster_ctarank();
  const bool tm = g_cg_timing && me == 0 && threadIdx.x == 0;
  const long long c0 = tm ? clock64() : 0;
  double ta, tb, tc;
  cg_block_reduce3(a, b, c, wsum, ta, tb, tc);
  const long long c1 = tm ? clock64() : 0;
  const int tid = threadIdx.x;
  uint64_t* bar = bars + par;
  // this CTA receives every CTA's rows (rtot values when v is posted) and
  // NC x 3 partials; the arrival may follow the data (tx-count goes negative)
  if (tid == 0) mbar_expect_tx(bar, (uint32_t)(((v ? rtot : 0) + 3 * NC) * sizeof(double)));
  if (v && tid < 8 * 32) {  // thread (dst = tid / 16 ... ): rows i = lane16, lane16 + 16, ..
    const int dst = tid >> 4, sub = tid & 15;  // 16 threads per destination CTA
    for (int d = dst; d < NC; d += 16)
      for (int i = sub; i < nr; i += 16) st_async_f64(full + r0 + i, d, v[i], bar);
  }
  if (tid < NC) {
    st_async_f64(slots + 3 * me, tid, ta, bar);
    st_async_f64(slots + 3 * me + 1, tid, tb, bar);
    st_async_f64(slots + 3 * me + 2, tid, tc, bar);
  }
  // a sender can be at most one exchange ahead of this CTA: it needs this
  // CTA's next post before its own next-but-one wait, so the two parity
  // buffers/barriers never see data of two exchanges at once
  const long long c2 = tm ? clock64() : 0;
  mbar_wait(bar, (xph >> par) & 1u);
  xph ^= 1u << par;
  if (tm) {
    const long long c3 = clock64();
    atomicAdd(&g_cg_phase[1], (unsigned long long)(c1 - c0));  // block reduction
    atomicAdd(&g_cg_phase[2], (unsigned long long)(c2 - c1));  // posting
    atomicAdd(&g_cg_phase[3], (unsigned long long)(c3 - c2));  // waiting for the peers
  }
  // every warp sums the NC partials with the same shuffle tree: the
  // same bits on every CTA (they all take the same convergence decision)
  static_assert(NC <= 32 && (NC & (NC - 1)) == 0, "power-of-2 cluster");
  const int lane = tid & 31;
  double sa = 0.0, sb = 0.0, sc = 0.0;
  if (lane < NC) {
    sa = slots[3 * lane];
    sb = slots[3 * lane + 1];
    sc = slots[3 * lane + 2];
  }
#pragma unroll
  for (int o = NC / 2; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
  }
  // lanes >= NC summed zeros: every thread takes lane 0's totals
  A = __shfl_sync(0xffffffffu, sa, 0);
  B = __shfl_sync(0xffffffffu, sb, 0);
  C = __shfl_sync(0xffffffffu, sc, 0);
  __syncthreads();  // wsum reusable
}

// The exchange when all of the CTA's rows live in warp 0 (nr <= 32, the
// register-resident variant): lane i computed row i, so warp 0 alone reduces
// the partial dot products (shuffles: no shared memory, no block barrier)
// and posts its rows and totals; every warp then waits on the parity
// mbarrier and sums the NC partials as in cg_exchange (same bits: the block
// reduction added only zeros to warp 0's butterfly).
template <int NC>
__device__ __forceinline__ void cg_exchange_w0(const double* v, int nr, int r0, int rtot,
                                               double* full, double a, double b, double c,
                                               double* slots, uint64_t* bars, int par,
                                               uint32_t& xph, double& A, double& B, double& C,
                                               double vreg = 0.0, bool from_reg = false) {
  const uint32_t me = cluster_ctarank();
  const bool tm = g_cg_timing && me == 0 && threadIdx.x == 0;
  const long long c0 = tm ? clock64() : 0;
  const int tid = threadIdx.x, lane = tid & 31;
  uint64_t* bar = bars + par;
  if (tid < 32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
  }
  const long long c1 = tm ? clock64() : 0;
  if (tid == 0) mbar_expect_tx(bar, (uint32_t)(((v ? rtot : 0) + 3 * NC) * sizeof(double)));
  if (tid < 32) {
    if (v && lane < nr) {
      const double vi = from_reg ? vreg : v[lane];  // the lane's row: register or shared memory
#pragma unroll 4
      for (int d = 0; d < NC; ++d) st_async_f64(full + r0 + lane, d, vi, bar);
    }
    if (lane < NC) {
      st_async_f64(slots + 3 * me, lane, a, bar);
      st_async_f64(slots + 3 * me + 1, lane, b, bar);
      st_async_f64(slots + 3 * me + 2, lane, c, bar);
    }
  }
  const long long c2 = tm ? clock64() : 0;
  mbar_wait(bar, (xph >> par) & 1u);
  xph ^= 1u << par;
  if (tm) {
    const long long c3 = clock64();
    atomicAdd(&g_cg_phase[1], (unsigned long long)(c1 - c0));
    atomicAdd(&g_cg_phase[2], (unsigned long long)(c2 - c1));
    atomicAdd(&g_cg_phase[3], (unsigned long long)(c3 - c2));
  }
  static_assert(NC <= 32 && (NC & (NC - 1)) == 0, "power-of-2 cluster");
  double sa = 0.0, sb = 0.0, sc = 0.0;
  if (lane < NC) {
    sa = slots[3 * lane];
    sb = slots[3 * lane + 1];
    sc = slots[3 * lane + 2];
  }
#pragma unroll
  for (int o = NC / 2; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
  }
  A = __shfl_sync(0xffffffffu, sa, 0);
  B = __shfl_sync(0xffffffffu, sb, 0);
  C = __shfl_sync(0xffffffffu, sc, 0);
}

// out[i] = G_rows[i] . full: warp wid owns rows wid + q W (W warps), four
// rows at a time as independent fma chains (the per-row order -- lane
// strided, then the butterfly -- is unchanged, so are the bits)
__device__ __forceinline__ void cg_matvec(const double* Gs, int nr, int r, const double* full,
                                          double* out) {
  constexpr int W = kCgThreads / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i0 = wid; i0 < nr; i0 += 4 * W) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // warp-uniform trip count (a lane-dependent one left the warp diverged
    // before the butterflies, which then compiled to the slow collective
    // shuffle path: ~2,900 cycles per matvec)
#pragma unroll 4
    for (int j0 = 0; j0 < r; j0 += 32) {
      const int j = j0 + lane;
      const bool in = j < r;
      const double f = in ? full[j] : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (in && i0 + q * W < nr) acc[q] = fma(Gs[(size_t)(i0 + q * W) * r + j], f, acc[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + q * W < nr) out[i0 + q * W] = acc[q];
  }
  __syncthreads();
}

// The same product with the CTA's rows of G held in REGISTERS (warp wid owns
// rows wid + q W, lane l columns l + 32 jj): per iteration only the
// exchanged vector is read from shared memory (the shared-memory version
// re-read 25 x 400 doubles per matvec and was bound by shared-memory
// bandwidth, ~2,600 cycles).  Same per-row order (lane-strided chains, then
// the butterfly): same bits.
template <int RL>
__device__ __forceinline__ void cg_matvec_reg(const double (&g)[4][RL], int nr, int r,
                                              const double* full, double* out) {
  constexpr int W = kCgThreads / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int jj = 0; jj < RL; ++jj) {
    const int j = jj * 32 + lane;
    const double f = j < r ? full[j] : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = fma(g[q][jj], f, acc[q]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (wid + q * W < nr) out[wid + q * W] = acc[q];
  __syncthreads();
}

__device__ unsigned long long g_cg_iters[2];  // (solves, iterations): RMX_CG_STATS diagnostics

// doubles of the solver's shared-memory layout before the look-ahead
// correction vector (2 r + 3 doubles): G rows (shared-memory variant only),
// the exchanged vectors, the local rows, the partial-sum slots, the two mbarriers
__host__ __device__ inline size_t cg_corr_offset(int r, int C, bool reg) {
  const size_t R = (size_t)((r + C - 1) / C);
  return (reg ? 0 : R * (size_t)r) + 2 * (size_t)r + 11 * R + 6 * (size_t)C +
         3 * (size_t)(kCgThreads / 32) + 2;
}

template <int NC, int RL = 0>
__global__ void __launch_bounds__(kCgThreads) k_cg_solve(const double* __restrict__ G, int r,
                                                         double* __restrict__ w_out,
                                                         int32_t* __restrict__ flag,
                                                         double* __restrict__ resid2, double tol,
                                                         double* __restrict__ x0,
                                                         const double* __restrict__ corr,
                                                         const GrouseLook* __restrict__ look,
                                                         const double* __restrict__ av, int kav) {
  tr(5, 0);
  pdl_wait();
  tr(5, 1);
  unsigned long long wall0 = 0;
  if (g_cg_timing && threadIdx.x == 0 && cluster_ctarank() == 0) wall0 = globaltimer_ns();
  extern __shared__ double cs[];
  // look-ahead GROUSE: G was formed from the rows before the previous update's
  // rank-1 term a b^T; that term's contribution is added as the rows are read:
  // G' = G + c b^T + b c^T + |a|^2 b b^T (c = A^T a incl. the t column, b_r = 0)
  const bool con = corr != nullptr && look->applied != 0;
  // staged in shared memory (behind the solver's own buffers, see cg_smem_bytes_c):
  // read from global per element, the correction made the load of G 6x slower
  double* corr_s = cs + cg_corr_offset(r, NC, RL > 0);
  const double* cc = corr_s;
  const double* cb = corr_s + (r + 1);
  auto gfix = [&](int i, int j, double g) -> double {  // i, j < r
    if (!con) return g;
    const double bi = cb[i], bj = cb[j];
    return g + (cc[i] * bj + bi * cc[j]) + corr_s[2 * r + 2] * bi * bj;
  };
  auto rhsfix = [&](int j, double g) -> double { return con ? fma(cc[r], cb[j], g) : g; };
  const int R = (r + NC - 1) / NC;  // rows per CTA
  const uint32_t me = cluster_ctarank();
  const int r0 = (int)me * R, nr = max(0, min(R, r - r0));
  double* Gs = cs;                       // nr x r
  double* full = Gs + (RL > 0 ? 0 : (size_t)R * r);  // 2 x r: exchanged vector, by parity
  double* vec = full + 2 * (size_t)r;    // 11 x R local rows
  double *x = vec, *rv = vec + R, *u = vec + 2 * R, *w = vec + 3 * R, *m = vec + 4 * R,
         *nv = vec + 5 * R, *z = vec + 6 * R, *q = vec + 7 * R, *sv = vec + 8 * R,
         *p = vec + 9 * R, *dinv = vec + 10 * R;
  double* slots = vec + 11 * R;          // 2 x NC x 3 partials, by parity
  double* wsum = slots + 6 * NC;    // 3 x warps
  uint64_t* xbar = reinterpret_cast<uint64_t*>(wsum + 3 * (kCgThreads / 32));  // 2, by parity
  uint32_t xph = 0;                      // phase bit of each exchange barrier
  const int ld = r + 1;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  // c and b from k_late, |av|^2 summed here (fixed order: thread strides, xor
  // tree, warps in order -- every CTA gets the same bits)
  auto stage_corr = [&]() {
    double* avp = wsum;  // free until the first exchange
    for (int e = threadIdx.x; e < 2 * r + 2; e += kCgThreads) corr_s[e] = corr[e];
    double ps = 0.0;
    for (int i = threadIdx.x; i < kav; i += kCgThreads) {
      const double x = av[i];
      ps = fma(x, x, ps);
    }
    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    if ((threadIdx.x & 31) == 0) avp[threadIdx.x >> 5] = ps;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kCgThreads / 32; ++q) t += avp[q];
      corr_s[2 * r + 2] = t;
    }
    __syncthreads();
  };
  if (con && RL == 0) stage_corr();  // (register variant: staged below, behind the loads of G)
  // RL > 0: the CTA's rows of G in registers (r <= 32 RL, at most 4 rows per warp)
  constexpr int kRL = RL > 0 ? RL : 1;
  double greg[4][kRL];
  if constexpr (RL > 0) {
    constexpr int W = kCgThreads / 32;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
      for (int jj = 0; jj < RL; ++jj) {
        const int i = wid + qq * W, j = jj * 32 + lane;
        greg[qq][jj] = (i < nr && j < r) ? G[(int64_t)(r0 + i) * ld + j] : 0.0;
      }
    if (con) {  // the raw rows are in flight while the correction vectors are staged
      stage_corr();
#pragma unroll
      for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int jj = 0; jj < RL; ++jj) {
          const int i = wid + qq * W, j = jj * 32 + lane;
          if (i < nr && j < r) greg[qq][jj] = gfix(r0 + i, j, greg[qq][jj]);
        }
    }
  } else {
    for (int e = tid; e < nr * r; e += kCgThreads) {
      const int i = e / r, j = e % r;
      Gs[(size_t)i * r + j] = gfix(r0 + i, j, G[(int64_t)(r0 + i) * ld + j]);
    }
  }
  auto matvec = [&](const double* fv, double* outv) {
    if constexpr (RL > 0) cg_matvec_reg<kRL>(greg, nr, r, fv, outv);
    else cg_matvec(Gs, nr, r, fv, outv);
  };
  double pb = 0.0;
  for (int i = tid; i < nr; i += kCgThreads) {
    const double di = gfix(r0 + i, r0 + i, G[(int64_t)(r0 + i) * ld + r0 + i]);
    dinv[i] = di > 0.0 ? 1.0 / di : 1.0;
    x[i] = x0 ? x0[r0 + i] : 0.0;
    const double bi = rhsfix(r0 + i, G[(int64_t)r * ld + r0 + i]);
    rv[i] = bi;
    pb += bi * bi;
    z[i] = q[i] = sv[i] = p[i] = 0.0;
  }
  cluster_sync();  // every CTA's exchange barriers are initialised before any st.async
  unsigned long long wall1 = 0;
  if (wall0) wall1 = globaltimer_ns();
  int par = 0;
  auto xchg = [&](const double* vv, double pa, double pb2, double pc, double& A, double& B,
                  double& C) {
    if constexpr (RL > 0)
      cg_exchange_w0<NC>(vv, vv ? nr : 0, r0, r, vv ? full + par * r : nullptr, pa, pb2, pc,
                         slots + par * 3 * NC, xbar, par, xph, A, B, C);
    else
      cg_exchange<NC>(vv, vv ? nr : 0, r0, r, vv ? full + par * r : nullptr, pa, pb2, pc,
                      slots + par * 3 * NC, wsum, xbar, par, xph, A, B, C);
  };
  double BB, d0, d1;
  if (x0) {  // r = b - A x0
    xchg(x, pb, 0.0, 0.0, BB, d0, d1);
    matvec(full + par * r, nv);
    for (int i = tid; i < nr; i += kCgThreads) rv[i] -= nv[i];
    par ^= 1;
    __syncthreads();
  }
  for (int i = tid; i < nr; i += kCgThreads) u[i] = rv[i] * dinv[i];
  __syncthreads();
  // w = A u (and |b|^2 when not yet reduced)
  xchg(u, x0 ? 0.0 : pb, 0.0, 0.0, d0, d1, d1);
  if (!x0) BB = d0;
  matvec(full + par * r, w);
  par ^= 1;
  const double stop = tol * tol * BB;
  int converged = BB == 0.0;
  double gamma_prev = 1.0, alpha_prev = 1.0;
  int it = 0;
  const bool tm = g_cg_timing && cluster_ctarank() == 0 && tid == 0;
  unsigned long long wall2 = 0;
  if (wall0) wall2 = globaltimer_ns();
  if constexpr (RL > 0) {
    // Register variant: nr <= 32, so the CTA's rows of every iteration vector
    // live in warp 0's lanes -- kept in registers across the loop (the shared-
    // memory copies cost ~850 of ~4,000 cycles per iteration in loads, stores
    // and their latencies); only the matvec's output passes through shared
    // memory.  Same recurrences; x is written back for the final check.
    const bool act = tid < nr;
    double xr = 0.0, rr = 0.0, ur = 0.0, wr = 0.0, zr = 0.0, qr = 0.0, sr = 0.0, pp = 0.0,
           dr = 0.0;
    if (act) {
      xr = x[tid];
      rr = rv[tid];
      ur = u[tid];
      wr = w[tid];
      zr = z[tid];
      qr = q[tid];
      sr = sv[tid];
      pp = p[tid];
      dr = dinv[tid];
    }
    for (; it < r && !converged; ++it) {
      const double mr = wr * dr;
      double GAM, DEL, RR;
      cg_exchange_w0<NC>(m, nr, r0, r, full + par * r, rr * ur, wr * ur, rr * rr,
                         slots + par * 3 * NC, xbar, par, xph, GAM, DEL, RR, mr, true);
      const int used = par;
      par ^= 1;
      if (RR <= stop) {
        converged = 1;
        break;
      }
      double alpha, beta;
      if (it == 0) {
        beta = 0.0;
        alpha = DEL != 0.0 ? GAM / DEL : 0.0;
      } else {
        beta = GAM / gamma_prev;
        const double den = DEL - beta * GAM / alpha_prev;
        alpha = den != 0.0 ? GAM / den : 0.0;
      }
      if (!(alpha == alpha) || alpha == 0.0) break;  // breakdown: not converged
      gamma_prev = GAM;
      alpha_prev = alpha;
      const long long m0 = tm ? clock64() : 0;
      matvec(full + used * r, nv);  // n = A m (ends with a block barrier)
      if (tm) atomicAdd(&g_cg_phase[4], (unsigned long long)(clock64() - m0));
      if (act) {
        const double nvr = nv[tid];
        zr = fma(beta, zr, nvr);
        qr = fma(beta, qr, mr);
        sr = fma(beta, sr, wr);
        pp = fma(beta, pp, ur);
        xr = fma(alpha, pp, xr);
        rr = fma(-alpha, sr, rr);
        ur = fma(-alpha, qr, ur);
        wr = fma(-alpha, zr, wr);
      }
      // the next matvec overwrites nv only after every peer's rows have
      // arrived, this CTA's included, and warp 0 posts them after this read
    }
    if (act) x[tid] = xr;
    __syncthreads();
  } else
  for (; it < r && !converged; ++it) {
    const long long d0 = tm ? clock64() : 0;
    double pg = 0.0, pd = 0.0, pr = 0.0;
    for (int i = tid; i < nr; i += kCgThreads) {
      pg += rv[i] * u[i];
      pd += w[i] * u[i];
      pr += rv[i] * rv[i];
      m[i] = w[i] * dinv[i];
    }
    if (tm) atomicAdd(&g_cg_phase[0], (unsigned long long)(clock64() - d0));
    double GAM, DEL, RR;
    xchg(m, pg, pd, pr, GAM, DEL, RR);
    const int used = par;
    par ^= 1;  // every exchange flips the buffers (also on the way out)
    if (RR <= stop) {
      converged = 1;
      break;
    }
    // the step scalars need only the exchanged sums: computed before the
    // matvec so their fp64 divisions overlap its loads (same arithmetic)
    double alpha, beta;
    if (it == 0) {
      beta = 0.0;
      alpha = DEL != 0.0 ? GAM / DEL : 0.0;
    } else {
      beta = GAM / gamma_prev;
      const double den = DEL - beta * GAM / alpha_prev;
      alpha = den != 0.0 ? GAM / den : 0.0;
    }
    if (!(alpha == alpha) || alpha == 0.0) break;  // breakdown: not converged
    gamma_prev = GAM;
    alpha_prev = alpha;
    const long long m0 = tm ? clock64() : 0;
    matvec(full + used * r, nv);  // n = A m
    const long long m1 = tm ? clock64() : 0;
    if (tm) atomicAdd(&g_cg_phase[4], (unsigned long long)(m1 - m0));
    for (int i = tid; i < nr; i += kCgThreads) {
      z[i] = fma(beta, z[i], nv[i]);
      q[i] = fma(beta, q[i], m[i]);
      sv[i] = fma(beta, sv[i], w[i]);
      p[i] = fma(beta, p[i], u[i]);
      x[i] = fma(alpha, p[i], x[i]);
      rv[i] = fma(-alpha, sv[i], rv[i]);
      u[i] = fma(-alpha, q[i], u[i]);
      w[i] = fma(-alpha, z[i], w[i]);
    }
    if (tm) atomicAdd(&g_cg_phase[5], (unsigned long long)(clock64() - m1));
    // no barrier: the next iteration's partial sums read only this thread's
    // rows, and cg_exchange's block reduction syncs before the rows are posted
  }
  unsigned long long wall3 = 0;
  if (wall0) wall3 = globaltimer_ns();
  // true residual check: |b - A x|^2 <= 16 stop (else the Cholesky fallback)
  xchg(x, 0.0, 0.0, 0.0, d0, d1, d1);
  matvec(full + par * r, nv);
  par ^= 1;
  double ptr = 0.0, pw = 0.0, pbw = 0.0;
  for (int i = tid; i < nr; i += kCgThreads) {
    const double bi = rhsfix(r0 + i, G[(int64_t)r * ld + r0 + i]);
    const double ti = bi - nv[i];
    ptr += ti * ti;
    pw += x[i] * x[i];
    pbw += bi * x[i];
    if (w_out) w_out[r0 + i] = x[i];
    if (x0) x0[r0 + i] = x[i];
  }
  double TR, WW, BW;
  xchg(nullptr, ptr, pw, pbw, TR, WW, BW);
  if (me == 0 && tid == 0) {
    if (resid2) {
      resid2[0] = G[(int64_t)r * ld + r] - BW;
      resid2[1] = WW;
      resid2[2] = 1.0;
      resid2[3] = 1.0;
    }
    if (flag) flag[0] = (converged && (BB == 0.0 || TR <= 16.0 * stop)) ? 0 : 1;
    atomicAdd(&g_cg_iters[0], 1ull);
    atomicAdd(&g_cg_iters[1], (unsigned long long)it);
  }
  cluster_sync();  // no CTA exits while others may still write into its smem
  if (wall0) {
    const unsigned long long wall4 = globaltimer_ns();
    atomicAdd(&g_cg_wall[0], wall1 - wall0);
    atomicAdd(&g_cg_wall[1], wall2 - wall1);
    atomicAdd(&g_cg_wall[2], wall3 - wall2);
    atomicAdd(&g_cg_wall[3], wall4 - wall3);
  }
}

// ------------------------------------------------------------------ K4 (tcgen05 operands)
// U (v x r fp32) -> planes [2][v][kpad] fp16: hi = fp16(U 2^14), lo =
// fp16(U 2^14 - hi) (|U| <= 1 for an orthonormal basis, so 2^14 keeps both
// halves in fp16's normal range).  W (B x r fp32) -> [B][kpad] fp16 scaled by
// 2^e_p (max |W_p| in [2^14, 2^15)), descale[p] = 2^(-e_p - 14).
constexpr float kUScale = 16384.0f;

__global__ void k_u_planes(const float* __restrict__ U, int64_t v, int r, int kpad,
                           __half* __restrict__ planes) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v * kpad) return;
  const int64_t j = e / kpad;
  const int c = (int)(e % kpad);
  const float x = c < r ? U[j * r + c] * kUScale : 0.0f;
  const __half h = __float2half_rn(x);
  planes[e] = h;
  planes[v * kpad + e] = __float2half_rn(x - __half2float(h));
}

__global__ void k_w_rows(const float* __restrict__ W, int64_t B, int r, int kpad,
                         __half* __restrict__ wA, float* __restrict__ descale) {
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (p >= B) return;
  float m = 0.0f;
  for (int c = lane; c < r; c += 32) m = fmaxf(m, fabsf(W[p * r + c]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0f) {
    frexpf(m, &e);  // m = f 2^e, f in [0.5, 1)
    e = 15 - e;     // m 2^(15 - e) in [2^14, 2^15)
  }
  const float sc = ldexpf(1.0f, e);
  for (int c = lane; c < kpad; c += 32)
    wA[p * kpad + c] = __float2half_rn(c < r ? W[p * r + c] * sc : 0.0f);
  if (lane == 0) descale[p] = ldexpf(1.0f, -e) / kUScale;
}

__global__ void k_max_finalize(const uint32_t* __restrict__ enc, int64_t B, double mu,
                               double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= B) return;
  const uint32_t e = enc[p];
  const float f = __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
  out[p] = (double)f + mu;
}

// ------------------------------------------------------------------ K4
// Block: 64 permutations x all voxels, 128-voxel tiles, r streamed in chunks
// of 32 through smem; thread micro-tile 4 perms x 8 voxels (fp32 FMA).
constexpr int kCP = 64, kCV = 128, kCR = 32;

// Optional inputs: znoise (B x v, fp32) replaces the Philox draw (used for
// the max-gap shift estimator, whose normals come from the reference's
// SHIFT_GAP streams); base (B x v, fp64) gives val = base - (W U^T) instead
// (residual-sup shift estimator, rapid.py:113-114).
__global__ void __launch_bounds__(256) k_complete_max(
    const float* __restrict__ U, int64_t v, int r, int rpad, const float* __restrict__ W,
    int64_t B, int64_t perm_base, float sigma, double mu, uint64_t seed, int two_sided,
    const float* __restrict__ znoise, const double* __restrict__ base,
    double* __restrict__ max_out, uint32_t* __restrict__ max_enc) {
  // grid.y splits the voxels; with gridDim.y > 1 the per-block maxima meet
  // in max_enc (order-encoded atomicMax, decoded by k_max_finalize)
  __shared__ float Ws[kCR][kCP];
  __shared__ float Us[kCR][kCV + 4];
  __shared__ float red[16][kCP];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * kCP;
  float best[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
  const int64_t vtiles = (v + kCV - 1) / kCV;
  const int64_t tper = (vtiles + gridDim.y - 1) / gridDim.y;
  const int64_t jbeg = (int64_t)blockIdx.y * tper * kCV;
  const int64_t jend = min(v, jbeg + tper * kCV);
  for (int64_t j0 = jbeg; j0 < jend; j0 += kCV) {
    float acc[4][8] = {};
    for (int r0 = 0; r0 < rpad; r0 += kCR) {
      for (int e = threadIdx.x; e < kCR * kCP; e += 256) {
        const int pp = e / kCR, rr = e % kCR;
        const int64_t p = p0 + pp;
        Ws[rr][pp] = (p < B && r0 + rr < r) ? W[p * r + r0 + rr] : 0.0f;
      }
      for (int e = threadIdx.x; e < kCR * kCV; e += 256) {
        const int vv = e / kCR, rr = e % kCR;
        const int64_t j = j0 + vv;
        Us[rr][vv] = (j < v && r0 + rr < r) ? U[j * r + r0 + rr] : 0.0f;
      }
      __syncthreads();
#pragma unroll 8
      for (int rr = 0; rr < kCR; ++rr) {
        float a[4], bb[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = Ws[rr][ty * 4 + q];
#pragma unroll
        for (int s = 0; s < 8; ++s) bb[s] = Us[rr][tx * 8 + s];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int s = 0; s < 8; ++s) acc[q][s] = fmaf(a[q], bb[s], acc[q][s]);
      }
      __syncthreads();
    }
    const int64_t jb = j0 + tx * 8;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t p = p0 + ty * 4 + q;
      float z[8] = {};
      if (sigma != 0.0f && p < B) {
        if (znoise) {
#pragma unroll
          for (int s = 0; s < 8; ++s) z[s] = (jb + s < v) ? znoise[p * v + jb + s] : 0.0f;
        } else {
          normals4(seed, perm_base + p, jb / 4, z);
          normals4(seed, perm_base + p, jb / 4 + 1, z + 4);
        }
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (jb + s < v && p < B) {
          float val = fmaf(sigma, z[s], acc[q][s]);
          if (base) val = (float)(base[p * v + jb + s] - (double)acc[q][s]);
          if (two_sided) val = fabsf(val);
          best[q] = fmaxf(best[q], val);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) red[tx][ty * 4 + q] = best[q];
  __syncthreads();
  if (threadIdx.x < kCP) {
    float m = -FLT_MAX;
    for (int t = 0; t < 16; ++t) m = fmaxf(m, red[t][threadIdx.x]);
    const int64_t p = p0 + threadIdx.x;
    if (p < B) {
      if (max_enc) {
        const uint32_t bits = __float_as_uint(m);
        atomicMax(max_enc + p, (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u));
      } else {
        max_out[p] = (double)m + mu;
      }
    }
  }
}

// ------------------------------------------------------------------ GROUSE
// resid[i] = vals[i] - U[idx[i], :] . w   (k rows, one warp per row)
__device__ __forceinline__ void resid_block(int bid, const double* __restrict__ U, int64_t ldu,
                                            int r, const int32_t* __restrict__ idx, int k,
                                            const double* __restrict__ vals,
                                            const double* __restrict__ w,
                                            double* __restrict__ resid, double* __restrict__ sums,
                                            double* __restrict__ rpart = nullptr,
                                            const double* __restrict__ av = nullptr,
                                            const double* __restrict__ b = nullptr) {
  __shared__ double part[2][8];  // blockDim.x == 256
  const int warp = (bid * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  double ee = 0.0, tt = 0.0;
  if (warp < k) {
    const double* u = U + (int64_t)(idx ? idx[warp] : warp) * ldu;
    double s = 0.0;
    if (av) {
      // look-ahead: the previous update's rank-1 term av b^T goes onto the row
      // here (the rows were gathered before it; k_h_g_part reads them next)
      double* um = const_cast<double*>(u);
      const double a = av[warp];
      for (int c = lane; c < r; c += 32) {
        const double x = fma(a, b[c], um[c]);
        um[c] = x;
        s += x * w[c];
      }
    } else
    for (int c = lane; c < r; c += 32) s += u[c] * w[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double e = vals[warp] - s;
    if (lane == 0) resid[warp] = e;
    ee = e * e;
    tt = vals[warp] * vals[warp];
  }
  if (lane == 0) {
    part[0][threadIdx.x >> 5] = ee;
    part[1][threadIdx.x >> 5] = tt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one pair of atomics per block, not per row
    double a = 0.0, b = 0.0;
    for (int q = 0; q < 8; ++q) {
      a += part[0][q];
      b += part[1][q];
    }
    if (rpart) {  // per-block partials, reduced in a fixed order by the consumer
      rpart[2 * bid] = a;
      rpart[2 * bid + 1] = b;
    } else {
      atomicAdd(&sums[0], a);  // |resid|^2
      atomicAdd(&sums[2], b);  // |t_Omega|^2
    }
  }
}

__global__ void k_resid(const double* __restrict__ U, int64_t ldu, int r,
                        const int32_t* __restrict__ idx, int k,
                        const double* __restrict__ vals, const double* __restrict__ w,
                        double* __restrict__ resid, double* __restrict__ sums) {
  resid_block(blockIdx.x, U, ldu, r, idx, k, vals, w, resid, sums);
}

// pred = U w (v rows, one warp per row), sums[1] += |pred|^2
__global__ void k_pred(const double* __restrict__ U, int64_t v, int r, const double* __restrict__ w,
                       double* __restrict__ pred, double* __restrict__ sums) {
  __shared__ double part[32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x / 32;
  double local = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + wib; row < v;
       row += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const double* u = U + row * r;
    double s = 0.0;
    for (int c = lane; c < r; c += 32) s += u[c] * w[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      pred[row] = s;
      local += s * s;
    }
  }
  if (lane == 0) part[wib] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) t += part[i];
    atomicAdd(&sums[1], t);
  }
}

// H tracking: after k_grouse_post decided update t (a = pend_a p + d, b =
// w/|w|, U the matrix before the update, ug = U[Omega] gathered rows):
//   g = U^T a = pend_a H w + pend_b ug^T resid,
//   |a|^2 = pend_a^2 |p|^2 + 2 pend_a pend_b (ug w).resid + pend_b^2 |resid|^2,
//   H += b g^T + g b^T + |a|^2 b b^T.
// k_h_g_part: partial ug^T resid over row slice blockIdx.y (32 columns x 8
// row lanes per block, coalesced over the gathered rows); k_h_g_fin: g =
// pend_a hw + pend_b sum(partials) and |a|^2 (ug w = vals - resid; |p|^2 in
// st->aa) in g[r].
constexpr int kHgSplit = 16;

__global__ void k_h_g_part(int r, GrouseState* __restrict__ st,
                           const double* __restrict__ ug, int64_t ldu, int k,
                           const double* __restrict__ resid, double* __restrict__ gpart,
                           const double* __restrict__ hw, const double* __restrict__ vals,
                           const double* __restrict__ sums, double* __restrict__ g,
                           const GrouseLook* __restrict__ look) {
  tr(8, 0);
  pdl_wait();
  tr(8, 1);
  // look->applied, not st->pending: this runs beside k_defer_apply (its own
  // stream in look-ahead mode), which clears `pending`
  if (st->halted || !look->applied) return;
  __shared__ double part[8][33];
  __shared__ bool last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  const int rows = (k + kHgSplit - 1) / kHgSplit;
  const int i0 = blockIdx.y * rows, i1 = min(k, i0 + rows);
  double ur = 0.0;
  if (c < r)
#pragma unroll 4
    for (int i = i0 + ty; i < i1; i += 8) ur = fma(ug[(int64_t)i * ldu + c], resid[i], ur);
  part[ty][tx] = ur;
  __syncthreads();
  if (ty == 0 && c < r) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += part[q][tx];
    gpart[(int64_t)blockIdx.y * r + c] = t;
  }
  // the last block to finish forms g (was k_h_g_fin: one launch fewer)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned total = gridDim.x * gridDim.y;
    last = atomicAdd(&st->hg_done, 1u) == total - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double a = st->pend_a, bb = st->pend_b;
  for (int cc = threadIdx.x; cc < r; cc += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kHgSplit; ++q) t += __ldcg(gpart + (int64_t)q * r + cc);
    g[cc] = a * hw[cc] + bb * t;
  }
  __shared__ double kp[32];
  const int lane = threadIdx.x & 31;
  double pr = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) pr = fma(vals[i] - resid[i], resid[i], pr);
  for (int o = 16; o > 0; o >>= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
  if (lane == 0) kp[threadIdx.x >> 5] = pr;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += kp[q];
    g[r] = a * a * st->aa + 2.0 * a * bb * t + bb * bb * sums[0];
    st->hg_done = 0;  // ready for the next update
  }
}


__global__ void k_h_drift(const double* __restrict__ H, int r, double* __restrict__ out) {
  __shared__ double part[32];
  double m = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)r * r; e += blockDim.x) {
    const int i = (int)(e / r), j = (int)(e % r);
    m = fmax(m, fabs(H[e] - (i == j ? 1.0 : 0.0)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t = fmax(t, part[w]);
    *out = t;
  }
}

__global__ void k_h_identity(double* __restrict__ H, int r) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < (int64_t)r * r) H[e] = (e / r == e % r) ? 1.0 : 0.0;
}

// ---- M-deferred GROUSE (no pass over U per update)
// U_t = U_base M_t + sum_s d_s c_s^T: the rotation part of every update
// folds into the r x r matrix M (M <- M (I + a w b^T)), the residual part
// stays a sparse term (d_s = beta_s r_s on Omega_s, c_s its r-vector, itself
// rotated by later updates), and |p| = |U w| comes from the tracked
// H = U^T U.  U_base is rewritten once per 64 updates (a cuBLAS DGEMM by M +
// the sparse terms), instead of a read + write of U every update.

// grid (kDeferCap terms) x (k / 256 pieces of the term's index list): one
// binary search per thread, so the latency is one search, not k / 256 of
// them in sequence (expected hits per term: k^2 / v, ~6 at config 5)
// Deterministic sparse terms on the gathered rows (per-update mode): one
// warp per observed row q (voxel rows_sorted[q]); its lanes binary-search
// the voxel in the terms' sorted index lists (lane l: terms l, l + 32), then
// the hits are added in term order, lanes over the columns -- no atomics, so
// every run adds the same terms in the same order (the block-per-term
// version accumulated colliding rows with atomicAdd in arbitrary order).
__global__ void __launch_bounds__(256) k_sparse_terms_rows(
    double* __restrict__ out, int64_t ldo, int r, const int32_t* __restrict__ rows_sorted, int k,
    const int32_t* __restrict__ d_idx, const double* __restrict__ d_val,
    const double* __restrict__ cmat, const GrouseState* __restrict__ st) {
  tr(3, 0);
  pdl_wait();
  tr(3, 1);
  if (st->halted) return;
  const int nt = st->nterms;
  if (nt <= 0) return;
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (q >= k) return;
  const int32_t vox = __ldg(rows_sorted + q);
  // branch-free lower-bound searches, the lane's two terms interleaved (a
  // fixed number of dependent L2 loads instead of two early-exit loops)
  int pos[2] = {-1, -1};
  const int32_t* di0 = d_idx + (int64_t)lane * k;
  const int32_t* di1 = d_idx + (int64_t)(lane + 32) * k;
  const bool a0 = lane < nt, a1 = lane + 32 < nt;
  int p0 = 0, p1 = 0;  // largest index with di[p] <= vox (0 if none)
  int step = 1;
  while (step * 2 <= k) step *= 2;
  for (; step > 0; step >>= 1) {
    if (a0 && p0 + step < k && __ldg(di0 + p0 + step) <= vox) p0 += step;
    if (a1 && p1 + step < k && __ldg(di1 + p1 + step) <= vox) p1 += step;
  }
  if (a0 && __ldg(di0 + p0) == vox) pos[0] = p0;
  if (a1 && __ldg(di1 + p1) == vox) pos[1] = p1;
  double* o = out + (int64_t)q * ldo;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    unsigned hits = __ballot_sync(0xffffffffu, pos[h] >= 0);
    while (hits) {  // ascending term order
      const int src = __ffs(hits) - 1;
      hits &= hits - 1;
      const int sterm = src + 32 * h;
      const int p = __shfl_sync(0xffffffffu, pos[h], src);
      const double dq = d_val[(int64_t)sterm * k + p];
      const double* cs = cmat + (int64_t)sterm * r;
      for (int c = lane; c < r; c += 32) o[c] += dq * cs[c];
    }
  }
}

// Deterministic dense flush of ONE deferred term: U[d_idx[q], :] += d_q c^T.
// A term's voxels are distinct, so no two threads touch one element; the
// host launches the terms one after another (term order = update order).
__global__ void k_sparse_term_dense(double* __restrict__ out, int64_t ldo, int r,
                                    const int32_t* __restrict__ di, const double* __restrict__ dv,
                                    const double* __restrict__ cs, int k) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)k * r) return;
  const int q = (int)(e / r), c = (int)(e - (int64_t)q * r);
  out[(int64_t)di[q] * ldo + c] += dv[q] * cs[c];
}

// Per-update matrix-vector products, one warp per output (coalesced rows):
// hw = H w (for |p|^2 = w.hw and the H update), mw = M w (the M update) and
// dots[s] = w . c_s for the live terms.
__device__ __forceinline__ void defer_vec_block(int bid, const double* __restrict__ H,
                                                const double* __restrict__ M,
                                                const double* __restrict__ cmat,
                                                const double* __restrict__ w, int r,
                                                const GrouseState* __restrict__ st,
                                                double* __restrict__ hw, double* __restrict__ mw,
                                                double* __restrict__ dots,
                                                const double* __restrict__ NT,
                                                double* __restrict__ nw) {
  const int task = bid * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const double* row;
  double* out;
  if (task < r) {
    row = H + (int64_t)task * r;
    out = hw + task;
  } else if (task < 2 * r) {
    row = M + (int64_t)(task - r) * r;
    out = mw + (task - r);
  } else if (task < 3 * r) {  // nw = M^-T w (NT = (M^-1)^T, tracked for the sparse flush)
    row = NT + (int64_t)(task - 2 * r) * r;
    out = nw + (task - 2 * r);
  } else if (task < 3 * r + st->nterms) {
    row = cmat + (int64_t)(task - 3 * r) * r;
    out = dots + (task - 3 * r);
  } else {
    return;
  }
  double acc = 0.0;
  for (int j = lane; j < r; j += 32) acc = fma(row[j], w[j], acc);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) *out = acc;
}

// one launch for the two independent consumers of the solve: the residual
// on Omega (blocks [0, nres)) and H w, M w, C w (the rest)
__global__ void k_resid_defer_vec(const double* __restrict__ U, int64_t ldu, int r, int k,
                                  const double* __restrict__ vals, const double* __restrict__ w,
                                  double* __restrict__ resid, double* __restrict__ sums,
                                  const double* __restrict__ H, const double* __restrict__ M,
                                  const double* __restrict__ cmat,
                                  const GrouseState* __restrict__ st, double* __restrict__ hw,
                                  double* __restrict__ mw, double* __restrict__ dots, int nres,
                                  double* __restrict__ rpart, const double* __restrict__ NT,
                                  double* __restrict__ nw, const double* __restrict__ av,
                                  const double* __restrict__ b,
                                  const GrouseLook* __restrict__ look) {
  tr(6, 0);
  pdl_wait();
  tr(6, 1);
  if ((int)blockIdx.x < nres)
    resid_block(blockIdx.x, U, ldu, r, nullptr, k, vals, w, resid, sums, rpart,
                (av && look->applied && !st->halted) ? av : nullptr, b);
  else
    defer_vec_block(blockIdx.x - nres, H, M, cmat, w, r, st, hw, mw, dots, NT, nw);
}

// gathered rows of U (k x r at ld ldo) and, from the threads of column 0,
// the statistic column t[Omega] into vals and into column r of the rows
__global__ void k_gather_urows_vals(const double* __restrict__ U, int r,
                                    const int32_t* __restrict__ idx, int k, double* __restrict__ out,
                                    int64_t ldo, const double* __restrict__ t,
                                    double* __restrict__ vals, double* __restrict__ zero8,
                                    double* __restrict__ aug) {
  tr(1, 0);
  pdl_wait();
  tr(1, 1);
  if (zero8 && blockIdx.x == 0 && threadIdx.x < 8) zero8[threadIdx.x] = 0.0;  // the update's sums
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)k * r) return;
  const int i = (int)(e / r), c = (int)(e - (int64_t)i * r);
  const int64_t row = idx[i];
  out[(int64_t)i * ldo + c] = U[row * r + c];
  if (c == 0) {
    const double x = t[row];
    vals[i] = x;
    (aug ? aug : out)[(int64_t)i * ldo + r] = x;  // aug: the rows the product with M fills
  }
}

// decisions as k_grouse_post; the update becomes deferred term nterms
__global__ void __launch_bounds__(1024) k_grouse_post_m(
    GrouseState* __restrict__ st, double* __restrict__ sums, const int32_t* __restrict__ flag,
    double step, int64_t step_index, const int32_t* __restrict__ idx, int k,
    const double* __restrict__ resid, const double* __restrict__ w, int r,
    int32_t* __restrict__ d_idx, double* __restrict__ d_val, double* __restrict__ cmat,
    double* __restrict__ wn, int32_t* __restrict__ final_slot, const double* __restrict__ hw,
    int nres, int cg_mode, GrouseLook* __restrict__ look) {
  tr(7, 0);
  pdl_wait();
  tr(7, 1);
  __shared__ int skip, do_update, slot;
  __shared__ double sb, sinvw, sa, pnorm2;
  __shared__ double part[32];
  __shared__ double part2[32];
  {  // |resid|^2 and |t_Omega|^2 from k_resid_defer_vec's per-block partials
     // (sums + 8), in a fixed order: every run gives the same bits
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nres; i += blockDim.x) {
      a += sums[8 + 2 * i];
      b += sums[8 + 2 * i + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
      part[threadIdx.x / 32] = a;
      part2[threadIdx.x / 32] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double ta = 0.0, tb = 0.0;
      for (int i = 0; i < (int)(blockDim.x / 32); ++i) {
        ta += part[i];
        tb += part2[i];
      }
      sums[0] = ta;
      sums[2] = tb;
    }
    __syncthreads();
  }
  {  // |p|^2 = |U w|^2 = w^T H w
    double acc = 0.0;
    for (int c = threadIdx.x; c < r; c += blockDim.x) acc = fma(w[c], hw[c], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < (int)(blockDim.x / 32); ++i) t += part[i];
      pnorm2 = t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    skip = 0;
    do_update = 0;
    slot = 0;
    sa = 0.0;
    if (st->halted) {
      skip = 1;
    } else if (st->nterms >= kDeferCap) {  // never with a correct host loop
      st->halted = 1;
      st->overflow = 1;
      st->halt_step = (int)step_index;
      skip = 1;
    } else if (*flag) {
      // CG mode: the cluster CG did not converge -> the host re-runs this
      // update with the Cholesky solve; Cholesky mode: a non-positive pivot
      // (ill-conditioned restriction) -> the host redraws Omega
      st->halted = 1;
      st->halt_step = (int)step_index;
      st->cg_fail = cg_mode;
      skip = 1;
    } else {
      const double resid_norm = sqrt(fmax(sums[0], 0.0));
      const double pred_norm = sqrt(fmax(pnorm2, 0.0));
      const double t_norm = sqrt(fmax(sums[2], 0.0));
      const double w_norm = sqrt(fmax(sums[5], 0.0));
      int upd = !(step == 0.0 || resid_norm == 0.0);
      if (upd && (pred_norm == 0.0 || w_norm == 0.0)) upd = 0;
      if (upd && resid_norm <= 1e-14 * fmax(1.0, pred_norm)) upd = 0;
      double a = 0.0, bcoef = 0.0;
      if (upd) {
        const double theta = step * atan(resid_norm / pred_norm);
        a = (cos(theta) - 1.0) / pred_norm;
        bcoef = sin(theta) / resid_norm;
      }
      do_update = upd;
      sa = a;
      sb = bcoef;
      sinvw = upd ? 1.0 / w_norm : 0.0;
      // (I + a w b^T)^-1 = I - g w b^T, g = a / (1 + a |w|)  (b.w = |w|)
      st->pend_g = upd ? a / (1.0 + a * w_norm) : 0.0;
      slot = st->nterms;
      st->aa = pnorm2;  // |p|^2 for the H update
      st->rel_sum += t_norm > 0.0 ? resid_norm / t_norm : 0.0;
    }
    if (look) {  // what the next update's late chain has to add (k_late)
      look->applied = (!skip && do_update) ? 1 : 0;
      look->slot = slot;
      look->a = sa;
    }
  }
  __syncthreads();
  if (skip) return;
  if (do_update) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      d_idx[(int64_t)slot * k + i] = idx[i];
      d_val[(int64_t)slot * k + i] = sb * resid[i];
    }
    for (int c = threadIdx.x; c < r; c += blockDim.x) {
      const double bc = w[c] * sinvw;
      wn[c] = bc;
      cmat[(int64_t)slot * r + c] = bc;
    }
  }
  if (final_slot)
    for (int i = threadIdx.x; i < k; i += blockDim.x) final_slot[i] = idx[i];
  if (threadIdx.x == 0) {
    st->pending = do_update;
    st->pend_a = sa;
    st->pend_b = sb;
  }
}

// after k_grouse_post_m (+ the H update): M <- M + a (M w) b^T and the older
// terms c_s <- c_s + a (w . c_s) b; block row y: M row y (y < r) or term
// y - r; then k_defer_count adds the new term
// H <- H + b g^T + g b^T + |a|^2 b b^T (g[r] = |a|^2), after k_h_g_part; off
// the update's critical path (H is next read by the following update's
// k_resid_defer_vec, after its solve)
__global__ void k_h_apply(double* __restrict__ H, const double* __restrict__ g,
                          const double* __restrict__ b, const GrouseState* __restrict__ st,
                          const GrouseLook* __restrict__ look, int r) {
  pdl_wait();
  if (st->halted || !look->applied) return;
  const int i = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < r) H[(int64_t)i * r + c] += b[i] * g[c] + g[i] * b[c] + g[r] * b[i] * b[c];
}

__global__ void k_defer_apply(double* __restrict__ M, double* __restrict__ NT,
                              double* __restrict__ cmat,
                              GrouseState* __restrict__ st, const double* __restrict__ mw,
                              const double* __restrict__ dots, const double* __restrict__ b,
                              const double* __restrict__ nw, int r) {
  tr(9, 0);
  pdl_wait();
  tr(9, 1);
  if (st->halted || !st->pending) return;
  const int y = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const double a = st->pend_a;
  const int nt = st->nterms;
  if (c < r) {
    if (y < r) {
      M[(int64_t)y * r + c] = fma(a * mw[y], b[c], M[(int64_t)y * r + c]);
    } else if (y < 2 * r) {
      // N = M^-1 <- (I - g w b^T) N (pend_g = a / (1 + a |w|)); stored
      // transposed: NT[i][c] -= g (b^T N)_i w_c = g nw[i] b[c]  (nw = NT w, b = w / |w|)
      const int i = y - r;
      NT[(int64_t)i * r + c] = fma(-st->pend_g * nw[i], b[c], NT[(int64_t)i * r + c]);
    } else if (y - 2 * r < nt) {
      const int sterm = y - 2 * r;
      cmat[(int64_t)sterm * r + c] = fma(a * dots[sterm], b[c], cmat[(int64_t)sterm * r + c]);
    }
  }
  // the last block to finish counts the new term (was k_defer_count: one
  // launch fewer); every block read nterms / pending before its arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned total = gridDim.x * gridDim.y;
    if (atomicAdd(&st->da_done, 1u) == total - 1) {
      st->nterms = nt + 1;
      st->pending = 0;
      st->da_done = 0;
    }
  }
}


// ---- look-ahead GROUSE: the late chain of update h + 1
// The early chain (gather, product with M, sparse terms, Gram) of update
// h + 1 runs on a second stream while update h is solved, from the state
// before update h: A = [U_Omega' | t_Omega'] and G = A^T A without update h's
// term.  Update h is U <- U (I + a w b^T) + d b^T (b = w / |w|, d = pend_b
// resid on Omega_h), so on the rows Omega' of update h + 1
//   A' = A + av b^T,  av = a (A w) + d|Omega',
//   G' = G + c b^T + b c^T + |av|^2 b b^T,  c = A^T av (b_r = 0: the t column).
// Since A^T A = G is already there, c = a (G w) + A^T d|Omega' needs no pass
// over all rows: d|Omega' is non-zero only on Omega' /\ Omega_h (k^2 / v rows
// on average), which the early chain lists (k_isect).  On the critical path
// k_late is one launch without reductions: row warps form av, column warps
// form c; the solve sums |av|^2 itself and adds the correction to G as it
// loads its rows (corr); the rank-1 term goes onto the rows in the residual
// kernel's pass over them (k_resid_defer_vec), before k_h_g_part reads them.

// Early chain: pos[q] = index of Omega'[q] in the sorted Omega_h (or -1) and
// the ascending list of the q that are present.  One block; ordered compaction.
__global__ void __launch_bounds__(1024) k_isect(const int32_t* __restrict__ rows_next,
                                                const int32_t* __restrict__ rows_prev, int k,
                                                int32_t* __restrict__ pos,
                                                int32_t* __restrict__ list,
                                                int32_t* __restrict__ count) {
  pdl_wait();
  __shared__ int wcnt[32];
  __shared__ int base_s;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int top = 1;
  while (top * 2 <= k) top *= 2;
  for (int q0 = 0; q0 < k; q0 += blockDim.x) {
    const int q = q0 + threadIdx.x;
    int found = -1;
    if (q < k) {
      const int32_t vox = __ldg(rows_next + q);
      int p = 0;
      for (int step = top; step > 0; step >>= 1)
        if (p + step < k && __ldg(rows_prev + p + step) <= vox) p += step;
      if (__ldg(rows_prev + p) == vox) found = p;
      pos[q] = found;
    }
    const unsigned m = __ballot_sync(0xffffffffu, found >= 0);
    if (lane == 0) wcnt[wid] = __popc(m);
    __syncthreads();
    int before = base_s;
    for (int ww = 0; ww < wid; ++ww) before += wcnt[ww];
    if (found >= 0) list[before + __popc(m & ((1u << lane) - 1u))] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) t += wcnt[ww];
      base_s += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base_s;
}

// grid: nrb row blocks (8 rows each, warp per row) then column blocks (8
// columns each, warp per column of [U_Omega' | t], r + 1 columns)
__global__ void __launch_bounds__(256) k_late(
    const double* __restrict__ A, int64_t lda, int r, int k, const double* __restrict__ G,
    const double* __restrict__ w, const double* __restrict__ d_val,
    const int32_t* __restrict__ pos, const int32_t* __restrict__ list,
    const int32_t* __restrict__ count, const double* __restrict__ b,
    const GrouseState* __restrict__ st, const GrouseLook* __restrict__ look,
    double* __restrict__ av, double* __restrict__ corr, int nrb) {
  pdl_trigger();  // the solve becomes resident (and claims its cluster's SMs) while this runs
  tr(4, 0);
  pdl_wait();
  tr(4, 1);
  if (st->halted || !look->applied) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double a = look->a;
  const double* dv = d_val + (int64_t)look->slot * k;
  if ((int)blockIdx.x < nrb) {  // av = a (A w) + d|Omega'
    const int q = blockIdx.x * 8 + wid;
    if (q >= k) return;
    const double* row = A + (int64_t)q * lda;
    double sacc = 0.0;
    for (int c = lane; c < r; c += 32) sacc = fma(row[c], w[c], sacc);
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) {
      const int p = pos[q];
      av[q] = fma(a, sacc, p >= 0 ? dv[p] : 0.0);
    }
    return;
  }
  // c_j = a (G w)_j + sum over the common rows of A[q][j] d_q   (j <= r)
  const int j = ((int)blockIdx.x - nrb) * 8 + wid;
  if (j > r) return;
  const double* grow = G + (int64_t)j * (r + 1);
  double gacc = 0.0;
  for (int c = lane; c < r; c += 32) gacc = fma(grow[c], w[c], gacc);
  for (int o = 16; o > 0; o >>= 1) gacc += __shfl_xor_sync(0xffffffffu, gacc, o);
  const int n = *count;
  double sp = 0.0;
  for (int e = lane; e < n; e += 32) {
    const int q = list[e];
    sp = fma(A[(int64_t)q * lda + j], dv[pos[q]], sp);
  }
  // fixed order: lanes hold e = lane, lane + 32, ...; xor tree (deterministic)
  for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
  if (lane == 0) {
    corr[j] = fma(a, gacc, sp);
    if (j < r) corr[r + 1 + j] = b[j];
    else corr[2 * r + 1] = 0.0;  // b_r
  }
}

__global__ void k_force_halt(GrouseState* __restrict__ st, int64_t step) {
  if (st->halted) return;
  st->halted = 1;
  st->halt_step = (int)step;
}

// sparse flush (dense-M GROUSE): the deferred terms fold into the base as
// U_base += d_s (c_s^T M^-1), so that U_base M keeps representing U; ctil[s] =
// NT c_s (one warp per output)
__global__ void k_ctil(const double* __restrict__ NT, const double* __restrict__ cmat, int r,
                       int nterms, double* __restrict__ ctil) {
  const int task = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (task >= nterms * r) return;
  const int sterm = task / r, c = task - sterm * r;
  const double* row = NT + (int64_t)c * r;
  const double* cs = cmat + (int64_t)sterm * r;
  double acc = 0.0;
  for (int j = lane; j < r; j += 32) acc = fma(row[j], cs[j], acc);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) ctil[task] = acc;
}

__global__ void k_reset_terms(GrouseState* __restrict__ st) { st->nterms = 0; }

// X <- X L^{-T} for the lower Cholesky factor L stored in G (ld = r + 1):
// row i solves y L^T = x, i.e. L y^T = x^T (forward substitution).  One
// warp per row, lanes split the dot products.
__global__ void k_trsm_lt(double* __restrict__ X, int64_t v, int r, const double* __restrict__ L) {
  extern __shared__ double rows[];
  const int wib = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + wib;
  if (i >= v) return;
  double* y = rows + (int64_t)wib * r;
  for (int c = lane; c < r; c += 32) y[c] = X[i * r + c];
  __syncwarp();
  const int ld = r + 1;
  for (int c = 0; c < r; ++c) {
    double s = 0.0;
    for (int l = lane; l < c; l += 32) s += L[(int64_t)c * ld + l] * y[l];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[c] = (y[c] - s) / L[(int64_t)c * ld + c];
    __syncwarp();
  }
  for (int c = lane; c < r; c += 32) X[i * r + c] = y[c];
}

// out = max |G[i][j] - delta_ij| over the leading r x r block (ld = r + 1)
__global__ void k_max_dev_identity(const double* __restrict__ G, int r, double* out) {
  __shared__ double part[32];
  double m = 0.0;
  const int ld = r + 1;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)r * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / r), j = (int)(e % r);
    m = fmax(m, fabs(G[(int64_t)i * ld + j] - (i == j ? 1.0 : 0.0)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) t = fmax(t, part[i]);
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(t));
  }
}

// row max (or max |.|) of an (rows x cols) fp64 matrix, one block per row
__global__ void k_row_max(const double* __restrict__ A, int64_t cols, int two_sided,
                          double* __restrict__ out) {
  __shared__ double part[32];
  const int64_t i = blockIdx.x;
  double m = -DBL_MAX;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    double val = A[i * cols + j];
    if (two_sided) val = fabs(val);
    m = fmax(m, val);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = -DBL_MAX;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t = fmax(t, part[w]);
    out[i] = t;
  }
}

// batched residuals on gathered rows: R[b, i] = vals[b, i] - U[idx[b, i]] . W[b]
__global__ void k_resid_batch(const double* __restrict__ U, int r, const int32_t* __restrict__ idx,
                              int k, const double* __restrict__ vals, const double* __restrict__ W,
                              int64_t B, double* __restrict__ R) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (warp >= B * k) return;
  const int64_t b = warp / k;
  const double* u = U + (int64_t)idx[warp] * r;
  const double* w = W + b * r;
  double s = 0.0;
  for (int c = lane; c < r; c += 32) s += u[c] * w[c];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) R[warp] = vals[warp] - s;
}

// out[b, i] = t[b, idx[b, i]]  (B rows of length ldt)
__global__ void k_gather_rows(const double* __restrict__ t, int64_t ldt,
                              const int32_t* __restrict__ idx, int k, int64_t B,
                              double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B * k) return;
  out[e] = t[(e / k) * ldt + idx[e]];
}

// two-pass mean / unbiased variance of a vector (single block)
__global__ void k_mean_var(const double* __restrict__ a, int64_t n, double* out) {
  __shared__ double part[32];
  __shared__ double mean_s;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += a[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += part[w];
    mean_s = t / (double)n;
  }
  __syncthreads();
  const double m = mean_s;
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) q += (a[i] - m) * (a[i] - m);
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += part[w];
    out[0] = m;
    out[1] = n > 1 ? t / (double)(n - 1) : 0.0;
  }
}

__global__ void k_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)a[i];
}

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t launch_gram(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                        const double* vals, double* G, int64_t B, cudaStream_t s) {
  const int nt = (r + 1 + kGT - 1) / kGT;
  const int ntiles = nt * (nt + 1) / 2;
  // split the row (K) dimension when the batch alone cannot fill the GPU
  int splits = 1;
  const int64_t blocks = (int64_t)ntiles * B;
  if (blocks < 6 * 148) {  // 64-thread CTAs: several per SM
    splits = (int)std::min<int64_t>((6 * 148 + blocks - 1) / blocks, std::max(1, k / 64));
    // at most two partial sums per element: 0 + a + b is the same in either
    // order, so the atomics stay deterministic (three or more are not)
    splits = std::max(1, std::min(splits, 2));
  }
  const int rps = ((k + splits - 1) / splits + kGK - 1) / kGK * kGK;
  splits = (k + rps - 1) / rps;
  if (splits > 1) {
    cudaError_t e = cudaMemsetAsync(G, 0, (size_t)B * (r + 1) * (r + 1) * sizeof(double), s);
    if (e != cudaSuccess) return e;
  }
  const size_t smem =
      (size_t)2 * kGS * kGK * kGT * sizeof(double) + (idx ? (size_t)rps * sizeof(int32_t) : 0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  for (int64_t base = 0; base < B; base += 65535) {
    const int64_t cnt = B - base < 65535 ? B - base : 65535;
    k_gram<<<dim3(ntiles, (unsigned)cnt, (unsigned)splits), kGThreads, smem, s>>>(
        U, ldu, r, idx ? idx + base * k : nullptr, k, vals ? vals + base * k : nullptr,
        G + base * (int64_t)(r + 1) * (r + 1), rps);
  }
  return cudaGetLastError();
}

cudaError_t launch_chol_solve(double* G, int r, int64_t B, double* w_out, int32_t* flag,
                              double* resid2, cudaStream_t s) {
  // panel sized to the largest one (r - 32 rows): 109 KB at r = 400, two CTAs per SM
  const size_t smem =
      ((size_t)kPW * kPS + kPW + (size_t)chol_panel_rows(r) * kPS + (size_t)r) * sizeof(double);
  // few systems (GROUSE: one per update): a 512-thread CTA hides more of the
  // L2 latency of the trailing updates; batches: 256 threads, several CTAs / SM
  if (B < 148) {
    cudaError_t e = cudaFuncSetAttribute(k_chol_solve<512>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_chol_solve<512><<<(unsigned)B, 512, smem, s>>>(G, r, w_out, flag, resid2);
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_chol_solve<256>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_chol_solve<256><<<(unsigned)B, 256, smem, s>>>(G, r, w_out, flag, resid2);
  }
  return cudaGetLastError();
}

cudaError_t launch_chol_solve_f32(float* G, int r, int64_t B, double* w_out, int32_t* flag,
                                  cudaStream_t s) {
  // + the look-ahead's second diagonal-block buffer (NT = 256)
  const size_t smem = ((size_t)2 * (kPW * kPS + kPW) + (size_t)chol_panel_rows(r) * kPS +
                       (size_t)r) * sizeof(float);
  // RMX_CHOL_NT=512: one 512-thread CTA per SM (working set of the trailing
  // updates ~148 systems -> L2-resident) instead of three 256-thread CTAs
  const char* ntv = getenv("RMX_CHOL_NT");
  if (ntv && atoi(ntv) == 512) {
    auto kern = k_chol_solve<512, float>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)B, 512, smem, s>>>(G, r, w_out, flag, nullptr, nullptr, nullptr, nullptr, 0);
    return cudaGetLastError();
  }
  auto kern = k_chol_solve<256, float>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)B, 256, smem, s>>>(G, r, w_out, flag, nullptr, nullptr, nullptr, nullptr,
                                      getenv("RMX_CHOL_NOLA") ? 0 : 1);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3b (cluster)
// Batched Cholesky factor of G~ (fp32, the tcgen05 Gram) with the whole
// matrix ON CHIP: one system per cluster of kClC CTAs, its rows dealt out by
// quads (rows 4q..4q+3 -> CTA q % kClC) and stored packed (quad q keeps
// columns 0..4q+3) in that CTA's shared memory, the dimension padded to a
// multiple of 32 with identity rows.  Right-looking, panel width 32:
//   1. every CTA gathers the 32 x 32 diagonal block through DSMEM and
//      factors it redundantly (one warp, chol_block32) -- no broadcast;
//   2. the owners solve their panel rows P_i = G[i, panel] L_D^-T;
//   3. cluster barrier; every CTA copies all panel rows (16-byte DSMEM loads)
//      into a local panel buffer;
//   4. trailing update of the CTA's own rows, 4 x 4 register tiles from the
//      panel buffer (G[i, j] -= P_i . P_j), in place in its storage;
//   5. cluster barrier.
// The factor is then written to G's lower triangle (for the refinement
// resolves), G's row r (the right-hand side A^T t) to rhs_out as fp64 and
// w_out zeroed; flag = non-positive pivot (relative to the largest diagonal).
// Replaces the global-memory right-looking factor, whose trailing matrix
// (1,667 systems x 643 KB) streamed through HBM at every panel.
constexpr int kClC = 4;       // CTAs per system
constexpr int kClT = 256;     // threads per CTA
constexpr int kClPS = 36;     // panel-buffer row stride (floats; 16-byte rows)
constexpr int kClMaxN = 416;  // padded dimension supported (r <= 416)

__host__ __device__ inline int cl_quad_off(int t, int c) {  // floats before own quad t
  return 16 * (kClC * t * (t - 1) / 2 + t * (c + 1));
}

__device__ __forceinline__ uint32_t cl_map(const void* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
// DSMEM loads without a memory clobber (ordering comes from the cluster
// barriers), so a thread's independent remote loads are all in flight
// before the first result is used
__device__ __forceinline__ float cl_ld(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 cl_ld4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__global__ void __cluster_dims__(kClC, 1, 1) __launch_bounds__(kClT, 1)
    k_chol_cluster(float* __restrict__ G, int r, double* __restrict__ rhs_out,
                   double* __restrict__ w_out, int32_t* __restrict__ flag) {
  extern __shared__ __align__(16) float clsm[];
  const uint32_t c = cluster_ctarank();
  const int64_t b = blockIdx.x / kClC;
  const int N = (r + 31) / 32 * 32;
  const int nq = N / 4;
  const int nt = (nq - (int)c + kClC - 1) / kClC;  // own quads: q = t kClC + c
  const int stor = cl_quad_off(nt, (int)c);
  // red and St sit at the same offsets in every CTA of the cluster (peers
  // address them through DSMEM); the rest is local and follows St
  float* red = clsm;                                    // the CTA's diagonal maximum
  float* St = clsm + 4;                                 // packed own rows
  float* D = St + (stor + 3) / 4 * 4;                   // 32 x kPS diagonal block
  float* rinv = D + kPW * kPS;                          // 32
  float* Pf = rinv + 32;                                // panel rows (N x kClPS)
  __shared__ int bad;
  const int tid = threadIdx.x;
  const int ld = r + 1;
  float* Gb = G + b * (int64_t)ld * ld;
  // local address of global row i (owned by this CTA), column 0
  auto row_ptr = [&](float* base, int i, int owner) -> int {  // float offset in owner's St
    const int q = i >> 2, t = q / kClC;
    return cl_quad_off(t, owner) + (i & 3) * (4 * q + 4);
  };
  if (tid == 0) red[0] = 0.f;
  __syncthreads();
  // load own rows (lower part, identity beyond r), the local diagonal maximum
  float dmx = 0.f;
  for (int t = 0; t < nt; ++t) {
    const int q = t * kClC + (int)c, len = 4 * q + 4;
    float* base = St + cl_quad_off(t, (int)c);
    for (int e = tid; e < 4 * len; e += kClT) {
      const int ii = e / len, j = e - ii * len, i = 4 * q + ii;
      float val = 0.f;
      if (i < r && j <= i) val = Gb[(int64_t)i * ld + j];
      else if (i >= r && j == i) val = 1.f;
      base[ii * len + j] = val;
      if (j == i && i < r) dmx = fmaxf(dmx, val);
    }
  }
  for (int o = 16; o > 0; o >>= 1) dmx = fmaxf(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
  if ((tid & 31) == 0) atomicMax(reinterpret_cast<int*>(&red[0]), __float_as_int(dmx));  // dmx >= 0
  if (tid == 0) bad = 0;
  // the right-hand side and the zeroed solution (CTA 0)
  if (c == 0) {
    for (int i = tid; i < r; i += kClT) {
      rhs_out[b * r + i] = (double)Gb[(int64_t)r * ld + i];
      w_out[b * r + i] = 0.0;
    }
  }
  cluster_sync();
  float gmax = 0.f;
  for (uint32_t p = 0; p < kClC; ++p) gmax = fmaxf(gmax, cl_ld(cl_map(&red[0], p)));
  const float tiny = 1e-24f * gmax;
  for (int jb = 0; jb < N; jb += kPW) {
    // 1. diagonal block from its owners (all of a thread's loads issued first)
    {
      float val[kPW * kPW / kClT];
#pragma unroll
      for (int u = 0; u < kPW * kPW / kClT; ++u) {
        const int e = tid + u * kClT, ii = e / kPW, jj = e % kPW, i = jb + ii;
        const int owner = (i >> 2) % kClC;
        val[u] = 0.f;
        if (jj <= ii) val[u] = cl_ld(cl_map(St + row_ptr(St, i, owner) + jb + jj, (uint32_t)owner));
      }
#pragma unroll
      for (int u = 0; u < kPW * kPW / kClT; ++u) {
        const int e = tid + u * kClT;
        D[(e / kPW) * kPS + e % kPW] = val[u];
      }
    }
    __syncthreads();
    if (tid < 32) chol_block32(D, rinv, tiny, &bad);
    __syncthreads();
    // 2. own panel rows (i >= jb + 32): own row k = 4 (t - tp) + ii of the
    // quads from tp on, one per thread (the whole warp solves at once)
    {
      int tp = 0;
      while (tp < nt && 4 * (tp * kClC + (int)c) < jb + kPW) ++tp;
      for (int k = tid; k < 4 * (nt - tp); k += kClT) {
        const int t = tp + (k >> 2), ii = k & 3;
        const int q = t * kClC + (int)c, len = 4 * q + 4;
        {
          float* gi = St + cl_quad_off(t, (int)c) + ii * len + jb;
          float pr[kPW];
#pragma unroll
          for (int cc = 0; cc < kPW; cc += 4) {
            const float4 v = *reinterpret_cast<const float4*>(gi + cc);
            pr[cc] = v.x, pr[cc + 1] = v.y, pr[cc + 2] = v.z, pr[cc + 3] = v.w;
          }
#pragma unroll
          for (int cc = 0; cc < kPW; ++cc) {
            float sacc = pr[cc];
#pragma unroll
            for (int l = 0; l < cc; ++l) sacc = fmaf(-pr[l], D[cc * kPS + l], sacc);
            pr[cc] = sacc * rinv[cc];
          }
#pragma unroll
          for (int cc = 0; cc < kPW; cc += 4)
            *reinterpret_cast<float4*>(gi + cc) = make_float4(pr[cc], pr[cc + 1], pr[cc + 2], pr[cc + 3]);
        }
      }
    }
    cluster_sync();  // every CTA has gathered the diagonal block and solved its panel rows
    // own rows of the diagonal block <- L_D (nobody reads them again)
    for (int t = 0; t < nt; ++t) {
      const int q = t * kClC + (int)c;
      if (4 * q < jb || 4 * q >= jb + kPW) continue;
      float* base = St + cl_quad_off(t, (int)c);
      const int len = 4 * q + 4;
      for (int e = tid; e < 4 * kPW; e += kClT) {
        const int ii = e / kPW, cc = e % kPW, i = 4 * q + ii;
        if (cc <= i - jb) base[ii * len + jb + cc] = D[(i - jb) * kPS + cc];
      }
    }
    // 3. all panel rows -> Pf (row i - jb - 32)
    const int prow0 = jb + kPW, nrows = N - prow0;
    for (int e0 = 0; e0 < nrows * (kPW / 4); e0 += 4 * kClT) {  // 4 loads in flight per thread
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + tid + u * kClT;
        if (e < nrows * (kPW / 4)) {
          const int pr = e / (kPW / 4), c4 = (e % (kPW / 4)) * 4, i = prow0 + pr;
          const int owner = (i >> 2) % kClC;
          v[u] = cl_ld4(cl_map(St + row_ptr(St, i, owner) + jb + c4, (uint32_t)owner));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + tid + u * kClT;
        if (e < nrows * (kPW / 4))
          *reinterpret_cast<float4*>(Pf + (size_t)(e / (kPW / 4)) * kClPS + (e % (kPW / 4)) * 4) = v[u];
      }
    }
    __syncthreads();
    // 4. trailing update of own rows: (own quad Q) x (column quad J), J <= Q
    const int J0 = prow0 / 4;
    int t0 = 0;
    while (t0 < nt && t0 * kClC + (int)c < J0) ++t0;
    const int nown = nt - t0, ncq = nq - J0;
    for (int e = tid; e < nown * ncq; e += kClT) {
      const int tt = t0 + e / ncq, J = J0 + e % ncq;
      const int Q = tt * kClC + (int)c;
      if (J > Q) continue;
      const float* pi = Pf + (size_t)(4 * Q - prow0) * kClPS;
      const float* pj = Pf + (size_t)(4 * J - prow0) * kClPS;
      float acc[4][4] = {};
#pragma unroll 2
      for (int kk = 0; kk < kPW; kk += 4) {
        float4 a[4], bq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = *reinterpret_cast<const float4*>(pi + u * kClPS + kk);
          bq[u] = *reinterpret_cast<const float4*>(pj + u * kClPS + kk);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            acc[u][v] = fmaf(a[u].x, bq[v].x, acc[u][v]);
            acc[u][v] = fmaf(a[u].y, bq[v].y, acc[u][v]);
            acc[u][v] = fmaf(a[u].z, bq[v].z, acc[u][v]);
            acc[u][v] = fmaf(a[u].w, bq[v].w, acc[u][v]);
          }
      }
      float* base = St + cl_quad_off(tt, (int)c);
      const int len = 4 * Q + 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float4* g4 = reinterpret_cast<float4*>(base + u * len + 4 * J);
        float4 gv = *g4;
        gv.x -= acc[u][0];
        gv.y -= acc[u][1];
        gv.z -= acc[u][2];
        gv.w -= acc[u][3];
        *g4 = gv;
      }
    }
    cluster_sync();
  }
  // the factor back to G's lower triangle (the resolves read it there)
  for (int t = 0; t < nt; ++t) {
    const int q = t * kClC + (int)c, len = 4 * q + 4;
    const float* base = St + cl_quad_off(t, (int)c);
    for (int e = tid; e < 4 * len; e += kClT) {
      const int ii = e / len, j = e - ii * len, i = 4 * q + ii;
      if (i < r && j <= i) Gb[(int64_t)i * ld + j] = base[ii * len + j];
    }
  }
  if (c == 0 && tid == 0 && flag) flag[b] = bad;
}

size_t chol_cluster_smem(int r) {
  const int N = (r + 31) / 32 * 32, nq = N / 4;
  int stor = 0;
  for (int c = 0; c < kClC; ++c) {
    const int nt = (nq - c + kClC - 1) / kClC;
    stor = std::max(stor, cl_quad_off(nt, c));
  }
  return (4 + (size_t)(stor + 3) / 4 * 4 + kPW * kPS + 32 + (size_t)N * kClPS) * sizeof(float);
}

bool chol_cluster_supported(int r) {
  const char* e = getenv("RMX_CHOL_CLUSTER");
  return e && atoi(e) == 1 && r >= 1 && r <= kClMaxN && chol_cluster_smem(r) <= 232448;
}

cudaError_t launch_chol_cluster_f32(float* G, int r, int64_t B, double* rhs_out, double* w_out,
                                    int32_t* flag, cudaStream_t s) {
  const size_t smem = chol_cluster_smem(r);
  cudaError_t e = cudaFuncSetAttribute(k_chol_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_chol_cluster<<<(unsigned)(B * kClC), kClT, smem, s>>>(G, r, rhs_out, w_out, flag);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3b'
// Refinement resolve with a factor already in G (lower triangle of the
// row-major (r+1) x (r+1) fp32 G~): L L^T d = rhs_b, w_b += d, nconv_b = 1
// when |d|^2 > 1e-14 |w|^2.  ONE WARP PER SYSTEM (all of a batch's systems
// resident at once, the solves' serial chains overlapped across warps):
//   forward, block jb: lane l owns row i = jb + l; its dot product with the
//     solved y[0:jb] streams the row (16-byte loads, y broadcast from smem),
//     then the 32 x 32 diagonal block is solved by shuffles with the row's
//     32 diagonal-block entries in registers;
//   backward, block jb (descending): lane l owns column j = jb + l; the rows
//     below the block are read as coalesced 128-byte row segments, then the
//     block's transpose is solved by shuffles.
// fp32 arithmetic as the CTA version (the correction needs ~fp32 accuracy).
constexpr int kTrsvWarps = 4;

__global__ void __launch_bounds__(32 * kTrsvWarps) k_trsv_warp(const float* __restrict__ G, int r,
                                                                int64_t B, const double* __restrict__ rhs,
                                                                double* __restrict__ w_inout,
                                                                int32_t* __restrict__ nconv,
                                                                const int32_t* active, double tol2) {
  extern __shared__ __align__(16) float ty[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * kTrsvWarps + wid;
  if (b >= B) return;
  if (active && active[b] == 0) return;  // settled earlier: w and nconv[b] stay
  const int ld = r + 1;
  const int rp = (r + 31) / 32 * 32;
  float* y = ty + (size_t)wid * rp;
  const float* Gb = G + b * (int64_t)ld * ld;
  const double* rb = rhs + b * r;
  for (int jb = 0; jb < r; jb += 32) {  // forward: L y = rhs
    const int i = jb + lane;
    const bool live = i < r;
    const float* li = Gb + (int64_t)(live ? i : jb) * ld;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    if (live) {
      // row i is not 16-byte aligned in general (ld = r + 1): scalar head
      // up to alignment, then 16-byte loads
      int c = 0;
      const int head = (int)((4 - ((reinterpret_cast<uintptr_t>(li) >> 2) & 3)) & 3);
      for (; c < head && c < jb; ++c) s0 = fmaf(li[c], y[c], s0);
      for (; c + 4 <= jb; c += 4) {
        const float4 l4 = *reinterpret_cast<const float4*>(li + c);
        s0 = fmaf(l4.x, y[c], s0);
        s1 = fmaf(l4.y, y[c + 1], s1);
        s2 = fmaf(l4.z, y[c + 2], s2);
        s3 = fmaf(l4.w, y[c + 3], s3);
      }
      for (; c < jb; ++c) s0 = fmaf(li[c], y[c], s0);
    }
    float yb = live ? (float)rb[i] - ((s0 + s1) + (s2 + s3)) : 0.f;
    float lr[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) lr[c] = (live && jb + c <= i) ? li[jb + c] : (c == lane ? 1.f : 0.f);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      if (lane == c) yb /= lr[c];
      const float yc = __shfl_sync(0xffffffffu, yb, c);
      if (lane > c) yb = fmaf(-lr[c], yc, yb);
    }
    if (live) y[i] = yb;
    __syncwarp();
  }
  for (int jb = (r - 1) / 32 * 32; jb >= 0; jb -= 32) {  // backward: L^T d = y
    const int j = jb + lane;
    const bool live = j < r;
    float s0 = 0.f, s1 = 0.f;
    int i = jb + 32;
    for (; i + 1 < r; i += 2) {
      if (live) {
        s0 = fmaf(Gb[(int64_t)i * ld + j], y[i], s0);
        s1 = fmaf(Gb[(int64_t)(i + 1) * ld + j], y[i + 1], s1);
      }
    }
    if (i < r && live) s0 = fmaf(Gb[(int64_t)i * ld + j], y[i], s0);
    float db = live ? y[j] - (s0 + s1) : 0.f;
    float lc[32];  // column j of the diagonal block: L[jb + c][j]
#pragma unroll
    for (int c = 0; c < 32; ++c)
      lc[c] = (live && jb + c < r && jb + c >= j) ? Gb[(int64_t)(jb + c) * ld + j] : (c == lane ? 1.f : 0.f);
#pragma unroll
    for (int c = 31; c >= 0; --c) {
      if (lane == c) db /= lc[c];
      const float dc = __shfl_sync(0xffffffffu, db, c);
      if (lane < c) db = fmaf(-lc[c], dc, db);
    }
    __syncwarp();
    if (live) y[j] = db;
    __syncwarp();
  }
  double dd = 0.0, ww = 0.0;
  for (int i = lane; i < r; i += 32) {
    const double d = (double)y[i];
    const double wn = w_inout[b * r + i] + d;
    w_inout[b * r + i] = wn;
    dd += d * d;
    ww += wn * wn;
  }
  for (int o = 16; o > 0; o >>= 1) {
    dd += __shfl_xor_sync(0xffffffffu, dd, o);
    ww += __shfl_xor_sync(0xffffffffu, ww, o);
  }
  if (lane == 0 && nconv) nconv[b] = (dd > tol2 * ww) ? 1 : 0;
}

cudaError_t launch_chol_resolve_f32(float* G, int r, int64_t B, const double* rhs,
                                    double* w_inout, int32_t* nconv, cudaStream_t s,
                                    const int32_t* active, double tol) {
  if (!getenv("RMX_TRSV_CTA")) {  // one warp per system (RMX_TRSV_CTA=1: the CTA version)
    const int rp = (r + 31) / 32 * 32;
    const size_t smem = (size_t)kTrsvWarps * rp * sizeof(float);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_trsv_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_trsv_warp<<<(unsigned)((B + kTrsvWarps - 1) / kTrsvWarps), 32 * kTrsvWarps, smem, s>>>(
        G, r, B, rhs, w_inout, nconv, active, tol * tol);
    return cudaGetLastError();
  }
  const size_t smem = ((size_t)kPW * kPS + kPW + (size_t)r) * sizeof(float);
  auto kern = k_chol_solve<256, float>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)B, 256, smem, s>>>(G, r, w_inout, nconv, nullptr, nullptr, rhs, nullptr, 0);
  return cudaGetLastError();
}

cudaError_t launch_chol_resolve(double* G, int r, int64_t B, const double* rhs, double* w_inout,
                                int32_t* nconv, cudaStream_t s) {
  const size_t smem = ((size_t)kPW * kPS + kPW + (size_t)r) * sizeof(double);  // no panel
  cudaError_t e = cudaFuncSetAttribute(k_chol_solve<256>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_chol_solve<256><<<(unsigned)B, 256, smem, s>>>(G, r, w_inout, nconv, nullptr, nullptr, rhs);
  return cudaGetLastError();
}

cudaError_t launch_u_planes(const float* U, int64_t v, int r, int kpad, __half* planes,
                            cudaStream_t s) {
  const int64_t n = v * kpad;
  k_u_planes<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(U, v, r, kpad, planes);
  return cudaGetLastError();
}

cudaError_t launch_w_rows(const float* W, int64_t B, int r, int kpad, __half* wA, float* descale,
                          cudaStream_t s) {
  k_w_rows<<<(unsigned)((B + 7) / 8), 256, 0, s>>>(W, B, r, kpad, wA, descale);
  return cudaGetLastError();
}

cudaError_t launch_max_finalize(const uint32_t* enc, int64_t B, double mu, double* out,
                                cudaStream_t s) {
  k_max_finalize<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(enc, B, mu, out);
  return cudaGetLastError();
}

int cg_ctas() {  // cluster size of the GROUSE solve: 16 (default) or 8 (RMX_CG_CTAS=8)
  static const int c = [] {
    const char* e = getenv("RMX_CG_CTAS");
    return (e && atoi(e) == 8) ? 8 : kCgCtas;
  }();
  return c;
}

size_t cg_smem_bytes_c(int r, int C) {  // the shared-memory variant's full layout
  return (cg_corr_offset(r, C, false) + 2 * (size_t)r + 3) * sizeof(double);
}

size_t cg_smem_bytes(int r) { return cg_smem_bytes_c(r, cg_ctas()); }

bool cg_solve_supported(int r) { return cg_smem_bytes(r) <= 200 * 1024; }

template <int C, int RL = 0>
cudaError_t launch_cg_solve_c(const double* G, int r, double* w_out, int32_t* flag,
                              double* resid2, double tol, double* x0, cudaStream_t s,
                              const double* corr, const GrouseLook* look, const double* av,
                              int kav) {
  // the register-resident variant keeps no copy of G in shared memory
  const size_t smem =
      cg_smem_bytes_c(r, C) - (RL > 0 ? (size_t)((r + C - 1) / C) * r * sizeof(double) : 0);
  cudaError_t e = cudaFuncSetAttribute(k_cg_solve<C, RL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(k_cg_solve<C, RL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCgThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_cg_solve<C, RL>, G, r, w_out, flag, resid2, tol, x0, corr,
                            look, av, kav);
}

cudaError_t launch_cg_solve(const double* G, int r, double* w_out, int32_t* flag, double* resid2,
                            double tol, double* x0, cudaStream_t s, const double* corr,
                            const GrouseLook* look, const double* av, int kav) {
  // rows of G in registers when each warp holds at most 4 rows of <= 416
  // columns (RMX_CG_SMEM=1: the shared-memory variant)
  const bool reg = r <= 13 * 32 && (r + kCgCtas - 1) / kCgCtas <= 4 * (kCgThreads / 32) &&
                   !getenv("RMX_CG_SMEM");
  if (cg_ctas() == 8)
    return launch_cg_solve_c<8>(G, r, w_out, flag, resid2, tol, x0, s, corr, look, av, kav);
  if (reg)
    return launch_cg_solve_c<kCgCtas, 13>(G, r, w_out, flag, resid2, tol, x0, s, corr, look, av,
                                          kav);
  return launch_cg_solve_c<kCgCtas>(G, r, w_out, flag, resid2, tol, x0, s, corr, look, av, kav);
}

cudaError_t launch_complete_max(const float* U, int64_t v, int r, const float* W, int64_t B,
                                int64_t perm_base, double sigma, double mu, uint64_t seed,
                                int two_sided, const float* znoise, const double* base,
                                double* max_out, cudaStream_t s) {
  const int rpad = (r + kCR - 1) / kCR * kCR;
  const int64_t bx = (B + kCP - 1) / kCP;
  const int64_t vtiles = (v + kCV - 1) / kCV;
  // few permutation blocks (training's shift estimators: B = ell): split the
  // voxels too so that every SM works
  const int vs = (int)std::min<int64_t>(vtiles, std::max<int64_t>(1, (4 * 148 + bx - 1) / bx));
  uint32_t* enc = nullptr;
  if (vs > 1) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&enc), (size_t)B * 4, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(enc, 0, (size_t)B * 4, s);
    if (e != cudaSuccess) return e;
  }
  k_complete_max<<<dim3((unsigned)bx, (unsigned)vs), 256, 0, s>>>(
      U, v, r, rpad, W, B, perm_base, (float)sigma, mu, seed, two_sided, znoise, base, max_out,
      enc);
  if (enc) {
    k_max_finalize<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(enc, B, mu, max_out);
    cudaFreeAsync(enc, s);
  }
  return cudaGetLastError();
}

cudaError_t launch_resid(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                         const double* vals, const double* w, double* resid, double* sums,
                         cudaStream_t s) {
  k_resid<<<(unsigned)((k * 32 + 255) / 256), 256, 0, s>>>(U, ldu, r, idx, k, vals, w, resid,
                                                          sums);
  return cudaGetLastError();
}

cudaError_t launch_pred(const double* U, int64_t v, int r, const double* w, double* pred,
                        double* sums, cudaStream_t s) {
  int64_t blocks = (v + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_pred<<<(unsigned)blocks, 256, 0, s>>>(U, v, r, w, pred, sums);
  return cudaGetLastError();
}

cudaError_t launch_h_update(double* H, int r, const GrouseState* st, const double* hw,
                            const double* wn, const double* ug, int64_t ldu, int k,
                            const double* vals,
                            const double* resid, const double* sums, double* g, cudaStream_t s,
                            const GrouseLook* look) {
  double* gpart = g + r + 1;  // kHgSplit x r scratch after g[0..r]
  cudaError_t e = launch_pdl(k_h_g_part, dim3((unsigned)((r + 31) / 32), kHgSplit), dim3(256), 0,
                             s, r, const_cast<GrouseState*>(st), ug, ldu, k, resid, gpart, hw, vals,
                             sums, g, look);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_h_apply, dim3((unsigned)((r + 255) / 256), (unsigned)r), dim3(256), 0, s, H,
                    static_cast<const double*>(g), wn, st, look, r);
}

cudaError_t launch_h_drift(const double* H, int r, double* out, cudaStream_t s) {
  k_h_drift<<<1, 1024, 0, s>>>(H, r, out);
  return cudaGetLastError();
}

cudaError_t launch_h_identity(double* H, int r, cudaStream_t s) {
  const int64_t n = (int64_t)r * r;
  k_h_identity<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(H, r);
  return cudaGetLastError();
}

cudaError_t launch_sparse_terms_rows(double* out, int64_t ldo, int r, const int32_t* rows_sorted,
                                     int k, const int32_t* d_idx, const double* d_val,
                                     const double* cmat, const GrouseState* st, cudaStream_t s) {
  return launch_pdl(k_sparse_terms_rows, dim3((unsigned)((k + 7) / 8)), dim3(256), 0, s, out, ldo,
                    r, rows_sorted, k, d_idx, d_val, cmat, st);
}

cudaError_t launch_sparse_terms_dense(double* out, int64_t ldo, int r, int k, const int32_t* d_idx,
                                      const double* d_val, const double* cmat, int nterms,
                                      cudaStream_t s) {
  const int64_t n = (int64_t)k * r;
  for (int t = 0; t < nterms; ++t) {
    cudaError_t e = launch_pdl(k_sparse_term_dense, dim3((unsigned)((n + 255) / 256)), dim3(256), 0,
                               s, out, ldo, r, d_idx + (int64_t)t * k, d_val + (int64_t)t * k,
                               cmat + (int64_t)t * r, k);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_resid_defer_vec(const double* U, int64_t ldu, int r, int k, const double* vals,
                                   const double* w, double* resid, double* sums, const double* H,
                                   const double* M, const double* cmat, const GrouseState* st,
                                   double* hw, double* mw, double* dots, cudaStream_t s,
                                   const double* NT, double* nw, const double* av,
                                   const double* b, const GrouseLook* look) {
  const int nres = (k * 32 + 255) / 256;
  const int ndv = (3 * r + kDeferCap + 7) / 8;
  // sums[0] / sums[2] (|resid|^2, |t_Omega|^2): per-block partials in
  // sums + 8.., reduced in a fixed order by k_grouse_post_m (deterministic)
  return launch_pdl(k_resid_defer_vec, dim3((unsigned)(nres + ndv)), dim3(256), 0, s, U, ldu, r, k,
                    vals, w, resid, sums, H, M, cmat, st, hw, mw, dots, nres, sums + 8, NT, nw, av,
                    b, look);
}

cudaError_t launch_gather_urows_vals(const double* U, int r, const int32_t* idx, int k, double* out,
                                     int64_t ldo, const double* t, double* vals, double* zero8,
                                     cudaStream_t s, double* aug) {
  const int64_t n = (int64_t)k * r;
  cudaError_t e = launch_pdl(k_gather_urows_vals, dim3((unsigned)((n + 255) / 256)), dim3(256), 0,
                             s, U, r, idx, k, out, ldo, t, vals, zero8, aug);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_grouse_post_m(GrouseState* st, double* sums, const int32_t* flag,
                                 double step, int64_t step_index, const int32_t* idx, int k,
                                 const double* resid, const double* w, int r, int32_t* d_idx,
                                 double* d_val, double* cmat, double* wn, int32_t* final_slot,
                                 const double* hw, int cg_mode, cudaStream_t s,
                                 GrouseLook* look) {
  const int nres = (k * 32 + 255) / 256;  // k_resid_defer_vec's residual blocks
  return launch_pdl(k_grouse_post_m, dim3(1), dim3(1024), 0, s, st, sums, flag, step, step_index,
                    idx, k, resid, w, r, d_idx, d_val, cmat, wn, final_slot, hw, nres, cg_mode,
                    look);
}

cudaError_t launch_defer_apply(double* M, double* NT, double* cmat, GrouseState* st,
                               const double* mw, const double* dots, const double* wn,
                               const double* nw, int r, cudaStream_t s) {
  return launch_pdl(k_defer_apply, dim3((unsigned)((r + 255) / 256), (unsigned)(2 * r + kDeferCap)),
                    dim3(256), 0, s, M, NT, cmat, st, mw, dots, wn, nw, r);
}

cudaError_t launch_ctil(const double* NT, const double* cmat, int r, int nterms, double* ctil,
                        cudaStream_t s) {
  if (nterms <= 0) return cudaSuccess;
  const int tasks = nterms * r;
  k_ctil<<<(unsigned)((tasks + 7) / 8), 256, 0, s>>>(NT, cmat, r, nterms, ctil);
  return cudaGetLastError();
}

cudaError_t launch_reset_terms(GrouseState* st, cudaStream_t s) {
  k_reset_terms<<<1, 1, 0, s>>>(st);
  return cudaGetLastError();
}

cudaError_t launch_isect(const int32_t* rows_next, const int32_t* rows_prev, int k, int32_t* pos,
                         int32_t* list, int32_t* count, cudaStream_t s) {
  return launch_pdl(k_isect, dim3(1), dim3(1024), 0, s, rows_next, rows_prev, k, pos, list, count);
}

cudaError_t launch_late_chain(const double* A, int64_t lda, int r, int k, const double* G,
                              const double* w, const double* d_val, const int32_t* pos,
                              const int32_t* list, const int32_t* count, const double* b,
                              const GrouseState* st, const GrouseLook* look, double* av,
                              double* corr, cudaStream_t s) {
  const int nrb = (k + 7) / 8, ncb = (r + 1 + 7) / 8;
  return launch_pdl(k_late, dim3((unsigned)(nrb + ncb)), dim3(256), 0, s, A, lda, r, k, G, w,
                    d_val, pos, list, count, b, st, look, av, corr, nrb);
}

cudaError_t launch_force_halt(GrouseState* st, int64_t step, cudaStream_t s) {
  k_force_halt<<<1, 1, 0, s>>>(st, step);
  return cudaGetLastError();
}

void grouse_trace(int on, const char* dump_path) {
  if (!on && dump_path) {
    unsigned int n = 0;
    cudaMemcpyFromSymbol(&n, g_tr_n, sizeof(n));
    if (n > kTraceCap) n = kTraceCap;
    std::vector<unsigned long long> h(2 * (size_t)n);
    if (n) cudaMemcpyFromSymbol(h.data(), g_tr, h.size() * sizeof(unsigned long long));
    if (FILE* f = fopen(dump_path, "w")) {
      for (unsigned i = 0; i < n; ++i)
        fprintf(f, "%llu %llu %llu\n", h[2 * i], h[2 * i + 1] / 4, h[2 * i + 1] % 4);
      fclose(f);
    }
  }
  unsigned int z = 0;
  if (on) cudaMemcpyToSymbol(g_tr_n, &z, sizeof(z));
  cudaMemcpyToSymbol(g_tr_on, &on, sizeof(int));
}

void cg_stats(unsigned long long out[2]) {
  cudaMemcpyFromSymbol(out, g_cg_iters, sizeof(unsigned long long) * 2);
}

void cg_timing(int on, unsigned long long phase[6]) {
  if (phase) cudaMemcpyFromSymbol(phase, g_cg_phase, sizeof(unsigned long long) * 6);
  if (phase && !on) {
    unsigned long long wl[4];
    cudaMemcpyFromSymbol(wl, g_cg_wall, sizeof(wl));
    unsigned long long cs2[2];
    cudaMemcpyFromSymbol(cs2, g_cg_iters, sizeof(cs2));
    const double n = cs2[0] ? (double)cs2[0] : 1.0;
    fprintf(stderr, "rmx cg wall (us per solve): load G %.2f, setup %.2f, loop %.2f, tail %.2f\n",
            wl[0] / n * 1e-3, wl[1] / n * 1e-3, wl[2] / n * 1e-3, wl[3] / n * 1e-3);
  }
  cudaMemcpyToSymbol(g_cg_timing, &on, sizeof(int));
}


cudaError_t launch_trsm_lt(double* X, int64_t v, int r, const double* L, cudaStream_t s) {
  const int wpb = 4;
  k_trsm_lt<<<(unsigned)((v + wpb - 1) / wpb), 32 * wpb, (size_t)wpb * r * sizeof(double), s>>>(
      X, v, r, L);
  return cudaGetLastError();
}

cudaError_t launch_max_dev_identity(const double* G, int r, double* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  k_max_dev_identity<<<64, 256, 0, s>>>(G, r, out);
  return cudaGetLastError();
}

cudaError_t launch_row_max(const double* A, int64_t rows, int64_t cols, int two_sided,
                           double* out, cudaStream_t s) {
  k_row_max<<<(unsigned)rows, 256, 0, s>>>(A, cols, two_sided, out);
  return cudaGetLastError();
}

cudaError_t launch_resid_batch(const double* U, int r, const int32_t* idx, int k,
                               const double* vals, const double* W, int64_t B, double* R,
                               cudaStream_t s) {
  const int64_t warps = B * k;
  k_resid_batch<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(U, r, idx, k, vals, W, B, R);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* t, int64_t ldt, const int32_t* idx, int k, int64_t B,
                               double* out, cudaStream_t s) {
  const int64_t n = B * k;
  k_gather_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(t, ldt, idx, k, B, out);
  return cudaGetLastError();
}

cudaError_t launch_mean_var(const double* a, int64_t n, double* out, cudaStream_t s) {
  k_mean_var<<<1, 1024, 0, s>>>(a, n, out);
  return cudaGetLastError();
}

cudaError_t launch_to_f32(const double* a, int64_t n, float* out, cudaStream_t s) {
  k_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, n, out);
  return cudaGetLastError();
}

}  // namespace rmx
