// dense_small.cu -- exact condition numbers and a pivoted fallback solve for
// the small symmetric systems of RapidPT (reference lrmc.py:96-104, 127-149).
//
// The reference decides "ill-conditioned" from the exact eigenvalues of the
// normal matrix: cond = sqrt(lambda_max / lambda_min) (inf when lambda_min
// <= 0) against COND_LIMIT = 1e12 (numpy eigvalsh), and solves the accepted
// systems with np.linalg.solve (LU with partial pivoting).  The engine's
// fast path is a Cholesky factor whose pivots only bound the condition
// number from below; for the systems that path flags or finds borderline,
// and for every system of the public solve_block, these kernels evaluate
// the reference's quantities:
//
//   k_sym_extreme_eigs  one CTA per system: Householder tridiagonalisation
//                       of the r x r block (backward stable, like LAPACK's
//                       dsytrd inside eigvalsh: eigenvalue errors ~ eps
//                       |G|), then Sturm-count bisection for the smallest
//                       and largest eigenvalue to full precision.
//   k_lu_solve          one CTA per system: Gaussian elimination with
//                       partial pivoting (np.linalg.solve's algorithm) of
//                       G[:r,:r] w = G[r,:r] for the accepted systems the
//                       Cholesky could not factor.
//
// Rare path: the matrices live in a global-memory workspace (O(r) passes),
// which is fine for the handful of systems that ever get here.
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "rapid_internal.cuh"

namespace rmx {
namespace {

constexpr int kDT = 512;  // threads per system

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// number of eigenvalues of the symmetric tridiagonal (d, e) below x
__device__ int sturm_below(const double* d, const double* e2, int r, double x) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < r; ++i) {
    const double qq = (q == 0.0) ? DBL_EPSILON * (fabs(x) + 1e-300) : q;
    q = d[i] - x - e2[i - 1] / qq;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// G_b: system b's (r+1)^2 (ld r+1) or r^2 (ld r) matrix, read only; A: r x r
// workspace per system.  lam[2b] = lambda_min, lam[2b+1] = lambda_max.
__global__ void __launch_bounds__(kDT) k_sym_extreme_eigs(const double* __restrict__ G,
                                                          int64_t gstride, int ldg, int r,
                                                          const int32_t* __restrict__ sel,
                                                          double* __restrict__ A,
                                                          double* __restrict__ dwork,
                                                          double* __restrict__ lam) {
  __shared__ double red[33];
  __shared__ double s_alpha, s_tau, s_k;
  const int64_t b = sel ? sel[blockIdx.x] : blockIdx.x;
  const double* g = G + b * gstride;
  double* a = A + (int64_t)blockIdx.x * r * r;
  double* d = dwork + (int64_t)blockIdx.x * 4 * r;
  double* e2 = d + r;      // squared off-diagonal
  double* v = d + 2 * r;   // Householder vector
  double* q = d + 3 * r;   // p then q
  for (int64_t t = threadIdx.x; t < (int64_t)r * r; t += blockDim.x) {
    const int i = (int)(t / r), j = (int)(t % r);
    a[t] = g[(int64_t)i * ldg + j];
  }
  __syncthreads();
  for (int j = 0; j + 2 < r; ++j) {
    const int m = r - j - 1;  // length of the column below the diagonal
    double ss = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const double x = a[(int64_t)(j + 1 + i) * r + j];
      ss += x * x;
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) {
      const double x0 = a[(int64_t)(j + 1) * r + j];
      const double nrm = sqrt(ss);
      const double alpha = x0 >= 0.0 ? -nrm : nrm;
      const double vn2 = ss - x0 * x0 + (x0 - alpha) * (x0 - alpha);
      s_alpha = alpha;
      s_tau = vn2 > 0.0 ? 2.0 / vn2 : 0.0;
      d[j] = a[(int64_t)j * r + j];
      e2[j] = ss;  // alpha^2
    }
    __syncthreads();
    const double tau = s_tau;
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      v[i] = a[(int64_t)(j + 1 + i) * r + j] - (i == 0 ? s_alpha : 0.0);
    __syncthreads();
    if (tau == 0.0) continue;  // column already zero below the subdiagonal
    // p = tau A22 v: one warp per row
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = wid; i < m; i += nw) {
      const double* row = a + (int64_t)(j + 1 + i) * r + (j + 1);
      double s = 0.0;
      for (int c = lane; c < m; c += 32) s = fma(row[c], v[c], s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) q[i] = tau * s;
    }
    __syncthreads();
    double vp = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) vp = fma(v[i], q[i], vp);
    vp = block_sum(vp, red);
    if (threadIdx.x == 0) s_k = 0.5 * tau * vp;
    __syncthreads();
    const double K = s_k;
    for (int i = threadIdx.x; i < m; i += blockDim.x) q[i] = fma(-K, v[i], q[i]);
    __syncthreads();
    // A22 -= v q^T + q v^T
    for (int64_t t = threadIdx.x; t < (int64_t)m * m; t += blockDim.x) {
      const int i = (int)(t / m), c = (int)(t % m);
      double* p = a + (int64_t)(j + 1 + i) * r + (j + 1 + c);
      *p = *p - v[i] * q[c] - q[i] * v[c];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (r >= 2) {
      d[r - 2] = a[(int64_t)(r - 2) * r + (r - 2)];
      const double off = a[(int64_t)(r - 1) * r + (r - 2)];
      e2[r - 2] = off * off;
    }
    d[r - 1] = a[(int64_t)(r - 1) * r + (r - 1)];
  }
  __syncthreads();
  // Sturm bisection: thread 0 -> lambda_min, thread 32 -> lambda_max
  if (threadIdx.x == 0 || threadIdx.x == 32) {
    double lo = DBL_MAX, hi = -DBL_MAX;
    for (int i = 0; i < r; ++i) {  // Gershgorin interval
      double rad = 0.0;
      if (i > 0) rad += sqrt(e2[i - 1]);
      if (i + 1 < r) rad += sqrt(e2[i]);
      lo = fmin(lo, d[i] - rad);
      hi = fmax(hi, d[i] + rad);
    }
    const double span = fmax(fabs(lo), fabs(hi));
    lo -= 2.0 * DBL_EPSILON * span + 1e-300;
    hi += 2.0 * DBL_EPSILON * span + 1e-300;
    const int want = threadIdx.x == 0 ? 1 : r;  // count of eigenvalues <= lambda
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      if (sturm_below(d, e2, r, mid) >= want) hi = mid;
      else lo = mid;
    }
    lam[2 * (int64_t)blockIdx.x + (threadIdx.x == 0 ? 0 : 1)] = 0.5 * (lo + hi);
  }
}

// Gaussian elimination with partial pivoting on [G[:r,:r] | G[r,:r]^T]
// (the Gram's augmented row is the right-hand side U_Omega^T t).
__global__ void __launch_bounds__(kDT) k_lu_solve(const double* __restrict__ G, int64_t gstride,
                                                  int ldg, int r, const int32_t* __restrict__ sel,
                                                  double* __restrict__ A, double* __restrict__ w,
                                                  int32_t* __restrict__ singular) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_piv;
  const int64_t b = sel[blockIdx.x];
  const double* g = G + b * gstride;
  const int ld = r + 1;
  double* a = A + (int64_t)blockIdx.x * r * ld;  // r x (r + 1) augmented
  for (int64_t t = threadIdx.x; t < (int64_t)r * ld; t += blockDim.x) {
    const int i = (int)(t / ld), j = (int)(t % ld);
    a[t] = j < r ? g[(int64_t)i * ldg + j] : g[(int64_t)r * ldg + i];
  }
  __syncthreads();
  int sing = 0;
  for (int j = 0; j < r; ++j) {
    double best = -1.0;
    int bi = j;
    for (int i = j + threadIdx.x; i < r; i += blockDim.x) {
      const double x = fabs(a[(int64_t)i * ld + j]);
      if (x > best) {
        best = x;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      red_v[threadIdx.x >> 5] = best;
      red_i[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = red_v[0];
      int ii = red_i[0];
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
        if (red_v[q] > bb || (red_v[q] == bb && red_i[q] < ii)) {
          bb = red_v[q];
          ii = red_i[q];
        }
      s_piv = ii;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != j)
      for (int c = threadIdx.x; c < ld; c += blockDim.x) {
        const double t = a[(int64_t)j * ld + c];
        a[(int64_t)j * ld + c] = a[(int64_t)p * ld + c];
        a[(int64_t)p * ld + c] = t;
      }
    __syncthreads();
    const double piv = a[(int64_t)j * ld + j];
    if (piv == 0.0) {
      sing = 1;
      continue;
    }
    const int rows = r - j - 1, cols = ld - j - 1;
    for (int64_t t = threadIdx.x; t < (int64_t)rows * cols; t += blockDim.x) {
      const int i = j + 1 + (int)(t / cols), c = j + 1 + (int)(t % cols);
      const double f = a[(int64_t)i * ld + j] / piv;
      a[(int64_t)i * ld + c] = fma(-f, a[(int64_t)j * ld + c], a[(int64_t)i * ld + c]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // back substitution
    double* wb = w + b * r;
    for (int i = r - 1; i >= 0; --i) {
      double s = a[(int64_t)i * ld + r];
      for (int c = i + 1; c < r; ++c) s = fma(-a[(int64_t)i * ld + c], wb[c], s);
      wb[i] = s / a[(int64_t)i * ld + i];
    }
    if (singular) singular[b] = sing;
  }
}

// GROUSE direction of one track_update (lrmc.py:185-192):
// d = a pred, d[idx] += b resid, U += d (w / |w|)^T
__global__ void k_track_scale(double* __restrict__ d, int64_t v, double a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < v) d[i] = a * d[i];
}

__global__ void k_track_scatter(double* __restrict__ d, const int32_t* __restrict__ idx, int k,
                                const double* __restrict__ resid, double b) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < k) d[idx[j]] += b * resid[j];
}

__global__ void k_track_rank1(double* __restrict__ U, int64_t v, int r,
                              const double* __restrict__ d, const double* __restrict__ w,
                              double winv) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v * r) return;
  const int64_t i = e / r;
  const int c = (int)(e - i * r);
  U[e] += d[i] * (w[c] * winv);
}

}  // namespace

cudaError_t launch_track_apply(double* U, int64_t v, int r, double* pred, double a,
                               const int32_t* idx, int k, const double* resid, double b,
                               const double* w, double winv, cudaStream_t s) {
  k_track_scale<<<(unsigned)((v + 255) / 256), 256, 0, s>>>(pred, v, a);
  k_track_scatter<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(pred, idx, k, resid, b);
  k_track_rank1<<<(unsigned)((v * r + 255) / 256), 256, 0, s>>>(U, v, r, pred, w, winv);
  return cudaGetLastError();
}

cudaError_t launch_sym_extreme_eigs(const double* G, int64_t gstride, int ldg, int r,
                                    const int32_t* sel, int64_t count, double* work, double* lam,
                                    cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  double* A = work;
  double* dw = work + count * (int64_t)r * r;
  k_sym_extreme_eigs<<<(unsigned)count, kDT, 0, s>>>(G, gstride, ldg, r, sel, A, dw, lam);
  return cudaGetLastError();
}

size_t sym_extreme_eigs_work(int r, int64_t count) {
  return (size_t)count * ((size_t)r * r + 4 * (size_t)r) * sizeof(double);
}

cudaError_t launch_lu_solve(const double* G, int64_t gstride, int ldg, int r, const int32_t* sel,
                            int64_t count, double* work, double* w, int32_t* singular,
                            cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  k_lu_solve<<<(unsigned)count, kDT, 0, s>>>(G, gstride, ldg, r, sel, work, w, singular);
  return cudaGetLastError();
}

size_t lu_solve_work(int r, int64_t count) {
  return (size_t)count * (size_t)r * (r + 1) * sizeof(double);
}

}  // namespace rmx
