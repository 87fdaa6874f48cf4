// rapid_kernels.cu -- RapidPT on the GPU (reference rapid.py / lrmc.py).
// Compiled with -fmad=false: the Omega-row statistics reproduce the
// reference's numpy bits (np_exact.cuh); the least-squares algebra is fp64.
//
//   k_rapid_stats   K2: t_Omega[p, i] = statistic of row omega_p[i] under
//                   perm p (rapid.py:156-170, batched _welch_rows)
//   k_gram          K3a: G_b = [U_Omega | t]^T [U_Omega | t] for a batch of
//                   gathered row sets (lrmc.py:136-137: gram and rhs at once)
//   k_chol_solve    K3b: blocked Cholesky of G_b[:r,:r], w = G^-1 rhs, and a
//                   singularity flag (lrmc.py:138-148; see DESIGN.md for the
//                   condition-number deviation)
//   k_complete_max  K4: max_j (W U^T)[p, j] + sigma z(p, j)  (+ mu), fused
//                   with a counter-based Philox normal (rapid.py:198-205)
//   GROUSE helpers  k_resid, k_pred, k_grouse_update (lrmc.py:160-193)
#include <algorithm>
#include <cfloat>
#include <cmath>
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

// ------------------------------------------------------------------ K3a
// A_b = [U[idx_b[0..k)] | vals_b]  (k x (r+1)), G_b = A_b^T A_b, full
// (r+1)^2 row-major.  64x64 output tiles over the lower triangle, 4x4
// micro-tiles per thread, rows streamed through smem 32 at a time.
constexpr int kGT = 64;
constexpr int kGK = 32;

__device__ __forceinline__ double a_elem(const double* U, int64_t ldu, int r, const int32_t* idx,
                                         const double* vals, int64_t b, int k, int row, int col) {
  if (row >= k || col > r) return 0.0;
  const int64_t g = idx ? (int64_t)idx[b * k + row] : (int64_t)row;
  if (col == r) return vals ? vals[b * k + row] : 0.0;
  return U[g * ldu + col];
}

__global__ void __launch_bounds__(256) k_gram(const double* __restrict__ U, int64_t ldu, int r,
                                              const int32_t* __restrict__ idx, int k,
                                              const double* __restrict__ vals, double* __restrict__ G,
                                              int rows_per_split) {
  __shared__ double As[kGK][kGT + 1];
  __shared__ double Bs[kGK][kGT + 1];
  const int64_t b = blockIdx.y;
  // lower-triangle tile index -> (ti, tj), tj <= ti
  int ti = 0, rem = blockIdx.x;
  while (rem > ti) {
    rem -= ti + 1;
    ++ti;
  }
  const int tj = rem;
  const int i0 = ti * kGT, j0 = tj * kGT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  const int kbeg = blockIdx.z * rows_per_split;
  const int kend = min(k, kbeg + rows_per_split);
  for (int k0 = kbeg; k0 < kend; k0 += kGK) {
    for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
      const int rr = e / kGT, cc = e % kGT;
      const bool in = k0 + rr < kend;
      As[rr][cc] = in ? a_elem(U, ldu, r, idx, vals, b, k, k0 + rr, i0 + cc) : 0.0;
      Bs[rr][cc] = in ? a_elem(U, ldu, r, idx, vals, b, k, k0 + rr, j0 + cc) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kGK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[kk][ty * 4 + q];
        bv[q] = Bs[kk][tx * 4 + q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[q][s] += av[q] * bv[s];
    }
    __syncthreads();
  }
  const int ld = r + 1;
  double* Gb = G + b * (int64_t)ld * ld;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int i = i0 + ty * 4 + q, j = j0 + tx * 4 + s;
      if (i < ld && j < ld && j <= i) {
        if (gridDim.z == 1) {
          Gb[(int64_t)i * ld + j] = acc[q][s];
          if (i != j) Gb[(int64_t)j * ld + i] = acc[q][s];
        } else {  // split-K partial sums (G zeroed by the launcher)
          atomicAdd(&Gb[(int64_t)i * ld + j], acc[q][s]);
          if (i != j) atomicAdd(&Gb[(int64_t)j * ld + i], acc[q][s]);
        }
      }
    }
}

// ------------------------------------------------------------------ K3b
// One CTA per system.  Right-looking blocked Cholesky on G[:r, :r] in place
// (global memory, L2-resident), panel width 32 kept in smem; then a one-warp
// forward/back substitution for w.  flag[b] = 1 when a pivot is not
// positive relative to the largest diagonal (rank-deficient restriction).
constexpr int kPW = 32;

__global__ void __launch_bounds__(256) k_chol_solve(double* __restrict__ G, int r,
                                                    double* __restrict__ w_out,
                                                    int32_t* __restrict__ flag,
                                                    double* __restrict__ resid2) {
  extern __shared__ double sm[];
  double* D = sm;                       // kPW x kPW diagonal block
  double* P = sm + kPW * kPW;           // (r) x kPW panel
  __shared__ int bad;
  __shared__ double dmax;
  const int64_t b = blockIdx.x;
  const int ld = r + 1;
  double* Gb = G + b * (int64_t)ld * ld;
  if (threadIdx.x < 32) {
    double m = 0.0;
    for (int i = threadIdx.x; i < r; i += 32) m = fmax(m, Gb[(int64_t)i * ld + i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) {
      bad = 0;
      dmax = m;
    }
  }
  __syncthreads();
  const double tiny = 1e-24 * dmax;
  for (int jb = 0; jb < r; jb += kPW) {
    const int w = min(kPW, r - jb);
    for (int e = threadIdx.x; e < w * w; e += blockDim.x)
      D[(e / w) * kPW + e % w] = Gb[(int64_t)(jb + e / w) * ld + jb + e % w];
    __syncthreads();
    if (threadIdx.x < 32) {  // factor the diagonal block (one warp)
      const int lane = threadIdx.x;
      for (int c = 0; c < w; ++c) {
        double piv = D[c * kPW + c];
        if (!(piv > tiny)) {
          if (lane == 0) bad = 1;
          piv = fmax(fabs(piv), 1e-300);
        }
        const double d = sqrt(piv);
        __syncwarp();
        if (lane == c) D[c * kPW + c] = d;
        if (lane > c && lane < w) D[lane * kPW + c] /= d;
        __syncwarp();
        if (lane > c && lane < w)
          for (int l = c + 1; l <= lane; ++l) D[lane * kPW + l] -= D[lane * kPW + c] * D[l * kPW + c];
        __syncwarp();
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int i = e / w, j = e % w;
      if (j <= i) Gb[(int64_t)(jb + i) * ld + jb + j] = D[i * kPW + j];
    }
    // panel below: P = G[jb+w:, jb:jb+w] L_D^{-T}, one row per thread
    const int rows = r - jb - w;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      const int64_t gi = (int64_t)(jb + w + i) * ld + jb;
      for (int c = 0; c < w; ++c) {
        double s = Gb[gi + c];
        for (int l = 0; l < c; ++l) s -= P[i * kPW + l] * D[c * kPW + l];
        P[i * kPW + c] = s / D[c * kPW + c];
      }
      for (int c = 0; c < w; ++c) Gb[gi + c] = P[i * kPW + c];
      for (int c = w; c < kPW; ++c) P[i * kPW + c] = 0.0;  // last (narrow) panel
    }
    __syncthreads();
    // trailing update: G[i, j] -= P_i . P_j for jb+w <= j <= i < r
    // (warp per row i, lanes over j <= i)
    {
      const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
      for (int ii = wid; ii < rows; ii += nw) {
        double pi[kPW];
#pragma unroll
        for (int c = 0; c < kPW; ++c) pi[c] = c < w ? P[ii * kPW + c] : 0.0;
        double* grow = Gb + (int64_t)(jb + w + ii) * ld + jb + w;
        for (int jj = lane; jj <= ii; jj += 32) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < kPW; ++c) acc += pi[c] * P[jj * kPW + c];
          grow[jj] -= acc;
        }
      }
    }
    __syncthreads();
  }
  // solve L L^T w = rhs (rhs = G[r, 0:r], the A^T t row), one warp
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double* y = P;  // reuse smem: r doubles
    for (int i = lane; i < r; i += 32) y[i] = Gb[(int64_t)r * ld + i];
    __syncwarp();
    for (int j = 0; j < r; ++j) {
      const double yj = y[j] / Gb[(int64_t)j * ld + j];
      __syncwarp();
      if (lane == 0) y[j] = yj;
      for (int i = j + 1 + lane; i < r; i += 32) y[i] -= Gb[(int64_t)i * ld + j] * yj;
      __syncwarp();
    }
    for (int j = r - 1; j >= 0; --j) {
      const double wj = y[j] / Gb[(int64_t)j * ld + j];
      __syncwarp();
      if (lane == 0) y[j] = wj;
      for (int i = lane; i < j; i += 32) y[i] -= Gb[(int64_t)j * ld + i] * wj;
      __syncwarp();
    }
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
        const double dd = Gb[(int64_t)i * ld + i];
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

// ------------------------------------------------------------------ Philox
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Four N(0,1) draws for (perm, voxels 4q..4q+3), keyed by the run seed:
// counter = (q, perm_lo, perm_hi, RESIDUAL domain), Box-Muller in fp32.
__device__ __forceinline__ void normals4(uint64_t seed, int64_t perm, int64_t q, float z[4]) {
  uint32_t c[4] = {(uint32_t)q, (uint32_t)perm, (uint32_t)((uint64_t)perm >> 32), 4u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const float u0 = ((float)c[0] + 0.5f) * 2.3283064365386963e-10f;
  const float u1 = ((float)c[1] + 0.5f) * 2.3283064365386963e-10f;
  const float u2 = ((float)c[2] + 0.5f) * 2.3283064365386963e-10f;
  const float u3 = ((float)c[3] + 0.5f) * 2.3283064365386963e-10f;
  const float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s0, c0, s1, c1;
  sincospif(2.0f * u1, &s0, &c0);
  sincospif(2.0f * u3, &s1, &c1);
  z[0] = r0 * c0;
  z[1] = r0 * s0;
  z[2] = r1 * c1;
  z[3] = r1 * s1;
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
    double* __restrict__ max_out) {
  __shared__ float Ws[kCR][kCP];
  __shared__ float Us[kCR][kCV + 4];
  __shared__ float red[16][kCP];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * kCP;
  float best[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
  for (int64_t j0 = 0; j0 < v; j0 += kCV) {
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
    if (p < B) max_out[p] = (double)m + mu;
  }
}

// ------------------------------------------------------------------ GROUSE
// resid[i] = vals[i] - U[idx[i], :] . w   (k rows, one warp per row)
__global__ void k_resid(const double* __restrict__ U, int r, const int32_t* __restrict__ idx, int k,
                        const double* __restrict__ vals, const double* __restrict__ w,
                        double* __restrict__ resid, double* __restrict__ sums) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (warp >= k) return;
  const double* u = U + (int64_t)idx[warp] * r;
  double s = 0.0;
  for (int c = lane; c < r; c += 32) s += u[c] * w[c];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const double e = vals[warp] - s;
    resid[warp] = e;
    atomicAdd(&sums[0], e * e);                    // |resid|^2
    atomicAdd(&sums[2], vals[warp] * vals[warp]);  // |t_Omega|^2
  }
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

// U += dir (w/|w|)^T, dir = a * pred + b * scatter(resid over idx)
__global__ void k_grouse_update(double* __restrict__ U, int64_t v, int r,
                                const double* __restrict__ pred, const double* __restrict__ wn,
                                double a, const double* __restrict__ dscatter) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v * r) return;
  const int64_t row = e / r;
  const int c = (int)(e % r);
  U[e] += (a * pred[row] + dscatter[row]) * wn[c];
}

__global__ void k_scatter(const int32_t* __restrict__ idx, int k, const double* __restrict__ resid,
                          double bcoef, double* __restrict__ d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) d[idx[i]] = bcoef * resid[i];
}

__global__ void k_unscatter(const int32_t* __restrict__ idx, int k, double* __restrict__ d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) d[idx[i]] = 0.0;
}

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

__global__ void k_gather_vals(const double* __restrict__ t, const int32_t* __restrict__ idx, int k,
                              double* __restrict__ vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) vals[i] = t[idx[i]];
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

__global__ void k_scale_copy(const double* __restrict__ a, int n, double sc, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * sc;
}

__global__ void k_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)a[i];
}

}  // namespace

// ------------------------------------------------------------------ launchers
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

cudaError_t launch_gram(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                        const double* vals, double* G, int64_t B, cudaStream_t s) {
  const int nt = (r + 1 + kGT - 1) / kGT;
  const int ntiles = nt * (nt + 1) / 2;
  // split the row (K) dimension when the batch alone cannot fill the GPU
  int splits = 1;
  const int64_t blocks = (int64_t)ntiles * B;
  if (blocks < 2 * 148) {
    splits = (int)std::min<int64_t>((2 * 148 + blocks - 1) / blocks, std::max(1, k / 64));
    splits = std::max(1, std::min(splits, 4096));
  }
  const int rps = ((k + splits - 1) / splits + kGK - 1) / kGK * kGK;
  splits = (k + rps - 1) / rps;
  if (splits > 1) {
    cudaError_t e = cudaMemsetAsync(G, 0, (size_t)B * (r + 1) * (r + 1) * sizeof(double), s);
    if (e != cudaSuccess) return e;
  }
  for (int64_t base = 0; base < B; base += 65535) {
    const int64_t cnt = B - base < 65535 ? B - base : 65535;
    k_gram<<<dim3(ntiles, (unsigned)cnt, (unsigned)splits), 256, 0, s>>>(
        U, ldu, r, idx ? idx + base * k : nullptr, k, vals ? vals + base * k : nullptr,
        G + base * (int64_t)(r + 1) * (r + 1), rps);
  }
  return cudaGetLastError();
}

cudaError_t launch_chol_solve(double* G, int r, int64_t B, double* w_out, int32_t* flag,
                              double* resid2, cudaStream_t s) {
  const size_t smem = (size_t)(kPW * kPW + (size_t)(r + kPW) * kPW) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_chol_solve<<<(unsigned)B, 256, smem, s>>>(G, r, w_out, flag, resid2);
  return cudaGetLastError();
}

cudaError_t launch_complete_max(const float* U, int64_t v, int r, const float* W, int64_t B,
                                int64_t perm_base, double sigma, double mu, uint64_t seed,
                                int two_sided, const float* znoise, const double* base,
                                double* max_out, cudaStream_t s) {
  const int rpad = (r + kCR - 1) / kCR * kCR;
  k_complete_max<<<(unsigned)((B + kCP - 1) / kCP), 256, 0, s>>>(
      U, v, r, rpad, W, B, perm_base, (float)sigma, mu, seed, two_sided, znoise, base, max_out);
  return cudaGetLastError();
}

cudaError_t launch_resid(const double* U, int r, const int32_t* idx, int k, const double* vals,
                         const double* w, double* resid, double* sums, cudaStream_t s) {
  k_resid<<<(unsigned)((k * 32 + 255) / 256), 256, 0, s>>>(U, r, idx, k, vals, w, resid, sums);
  return cudaGetLastError();
}

cudaError_t launch_pred(const double* U, int64_t v, int r, const double* w, double* pred,
                        double* sums, cudaStream_t s) {
  int64_t blocks = (v + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_pred<<<(unsigned)blocks, 256, 0, s>>>(U, v, r, w, pred, sums);
  return cudaGetLastError();
}

cudaError_t launch_grouse_update(double* U, int64_t v, int r, const double* pred,
                                 const double* wn, double a, const double* dscatter,
                                 cudaStream_t s) {
  const int64_t total = v * r;
  k_grouse_update<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(U, v, r, pred, wn, a, dscatter);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const int32_t* idx, int k, const double* resid, double bcoef,
                           double* d, cudaStream_t s) {
  k_scatter<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(idx, k, resid, bcoef, d);
  return cudaGetLastError();
}

cudaError_t launch_unscatter(const int32_t* idx, int k, double* d, cudaStream_t s) {
  k_unscatter<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(idx, k, d);
  return cudaGetLastError();
}

cudaError_t launch_trsm_lt(double* X, int64_t v, int r, const double* L, cudaStream_t s) {
  const int wpb = 4;
  k_trsm_lt<<<(unsigned)((v + wpb - 1) / wpb), 32 * wpb, (size_t)wpb * r * sizeof(double), s>>>(
      X, v, r, L);
  return cudaGetLastError();
}

cudaError_t launch_gather_vals(const double* t, const int32_t* idx, int k, double* vals,
                               cudaStream_t s) {
  k_gather_vals<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(t, idx, k, vals);
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

cudaError_t launch_scale_copy(const double* a, int n, double sc, double* out, cudaStream_t s) {
  k_scale_copy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, n, sc, out);
  return cudaGetLastError();
}

cudaError_t launch_to_f32(const double* a, int64_t n, float* out, cudaStream_t s) {
  k_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, n, out);
  return cudaGetLastError();
}

}  // namespace rmx
