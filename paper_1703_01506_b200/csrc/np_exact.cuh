// np_exact.cuh -- float64 two-sample statistic, bit-identical to the
// reference's numpy arithmetic.
//
// The reference evaluates (teststat.py:28-50)
//     m_g  = x_g.mean(axis=-1)             -> add.reduce / n_g
//     s2_g = x_g.var(axis=-1, ddof=1)      -> add.reduce((x - mean)^2) / (n_g - 1)
//     t    = (m1 - m2) / sqrt(s2_1/n1 + s2_2/n2)
// on the fancy-indexed blocks values[:, order[:n1]] / values[:, order[n1:]]
// (model.py:65-69).  numpy's float64 add.reduce over a contiguous axis is the
// pairwise sum of loops_utils.h.src: < 8 terms sequential from 0.0; <= 128
// terms with 8 interleaved accumulators combined as ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)) plus a sequential tail; otherwise split at
// n/2 - (n/2)%8 and recurse.  Reproducing that order with explicitly rounded
// IEEE ops (no FMA contraction) gives the reference's bits exactly.
#pragma once
#include <cstdint>

namespace rmx {

// Subject s of the voxel lives at row[s * stride]: stride 1 for the
// DataMatrix layout (v x n row-major), stride v for the transposed copy.
struct GroupVals {  // a[i] = row[ord[i]]
  const double* row;
  const int16_t* ord;
  int64_t stride;
  __device__ __forceinline__ double operator()(int i) const { return row[ord[i] * stride]; }
};

struct GroupSqDev {  // a[i] = (row[ord[i]] - mean)^2
  const double* row;
  const int16_t* ord;
  int64_t stride;
  double mean;
  __device__ __forceinline__ double operator()(int i) const {
    double d = __dsub_rn(row[ord[i] * stride], mean);
    return __dmul_rn(d, d);
  }
};

template <class G>
__device__ __forceinline__ double np_pw_leaf(const G& g, int lo, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, g(lo + i));
    return res;
  }
  double r0 = g(lo + 0), r1 = g(lo + 1), r2 = g(lo + 2), r3 = g(lo + 3);
  double r4 = g(lo + 4), r5 = g(lo + 5), r6 = g(lo + 6), r7 = g(lo + 7);
  int i = 8;
  const int stop = n - (n % 8);
  for (; i < stop; i += 8) {
    r0 = __dadd_rn(r0, g(lo + i + 0));
    r1 = __dadd_rn(r1, g(lo + i + 1));
    r2 = __dadd_rn(r2, g(lo + i + 2));
    r3 = __dadd_rn(r3, g(lo + i + 3));
    r4 = __dadd_rn(r4, g(lo + i + 4));
    r5 = __dadd_rn(r5, g(lo + i + 5));
    r6 = __dadd_rn(r6, g(lo + i + 6));
    r7 = __dadd_rn(r7, g(lo + i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, g(lo + i));
  return res;
}

// Depth-bounded recursion (D levels of halving => n <= 128 * 2^D).
template <int D>
struct NpPairwise {
  template <class G>
  __device__ __noinline__ static double sum(const G& g, int lo, int n) {
    if (n <= 128) return np_pw_leaf(g, lo, n);
    int h = n / 2;
    h -= h % 8;
    return __dadd_rn(NpPairwise<D - 1>::sum(g, lo, h), NpPairwise<D - 1>::sum(g, lo + h, n - h));
  }
};
template <>
struct NpPairwise<0> {
  template <class G>
  __device__ __noinline__ static double sum(const G& g, int lo, int n) {
    return np_pw_leaf(g, lo, n);
  }
};

template <class G>
__device__ __forceinline__ double np_pw_sum(const G& g, int n) {
  return NpPairwise<8>::sum(g, 0, n);  // n <= 32768 (labels are int16: n <= 32767)
}

struct WelchExact {
  double t;
  double num;       // m1 - m2
  bool degenerate;  // var_term == 0 and num != 0
};

// Statistic of one voxel row (n doubles) under the labelling `ord`
// (ord[0..n1) = group 1 in permutation order, ord[n1..n) = group 2).
__device__ __forceinline__ WelchExact welch_exact(const double* row, int64_t stride,
                                                  const int16_t* ord, int n1, int n2) {
  GroupVals a{row, ord, stride}, b{row, ord + n1, stride};
  const double m1 = __ddiv_rn(np_pw_sum(a, n1), (double)n1);
  const double m2 = __ddiv_rn(np_pw_sum(b, n2), (double)n2);
  GroupSqDev da{row, ord, stride, m1}, db{row, ord + n1, stride, m2};
  const double v1 = __ddiv_rn(np_pw_sum(da, n1), (double)(n1 - 1));
  const double v2 = __ddiv_rn(np_pw_sum(db, n2), (double)(n2 - 1));
  const double var_term = __dadd_rn(__ddiv_rn(v1, (double)n1), __ddiv_rn(v2, (double)n2));
  WelchExact r;
  r.num = __dsub_rn(m1, m2);
  if (var_term == 0.0) {
    r.t = 0.0;
    r.degenerate = (r.num != 0.0);
  } else {
    r.t = __ddiv_rn(r.num, __dsqrt_rn(var_term));
    r.degenerate = false;
  }
  return r;
}

struct ConstVals {
  double c;
  __device__ __forceinline__ double operator()(int) const { return c; }
};
struct ConstSqDev {
  double c, mean;
  __device__ __forceinline__ double operator()(int) const {
    double d = __dsub_rn(c, mean);
    return __dmul_rn(d, d);
  }
};

// A voxel whose n values are all equal to c has the same statistic under
// every labelling; numpy's rounding of the group means can still make it
// non-zero (e.g. c = 0.1, n1 = 3, n2 = 4), so it is evaluated exactly once.
__device__ __forceinline__ WelchExact welch_exact_const(double c, int n1, int n2) {
  const double m1 = __ddiv_rn(np_pw_sum(ConstVals{c}, n1), (double)n1);
  const double m2 = __ddiv_rn(np_pw_sum(ConstVals{c}, n2), (double)n2);
  const double v1 = __ddiv_rn(np_pw_sum(ConstSqDev{c, m1}, n1), (double)(n1 - 1));
  const double v2 = __ddiv_rn(np_pw_sum(ConstSqDev{c, m2}, n2), (double)(n2 - 1));
  const double var_term = __dadd_rn(__ddiv_rn(v1, (double)n1), __ddiv_rn(v2, (double)n2));
  WelchExact r;
  r.num = __dsub_rn(m1, m2);
  if (var_term == 0.0) {
    r.t = 0.0;
    r.degenerate = (r.num != 0.0);
  } else {
    r.t = __ddiv_rn(r.num, __dsqrt_rn(var_term));
    r.degenerate = false;
  }
  return r;
}

// ---------------------------------------------------------------------------
// Warp-parallel evaluation with the same bits.  numpy's pairwise sum is a
// fixed tree: leaves of <= 128 terms (split at n/2 - (n/2)%8), each leaf
// eight interleaved sequential chains combined ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)) plus a sequential tail.  Every chain and every tree node
// is kept -- only the chains run on different lanes (8 lanes per leaf, 4
// leaves per round), so the result is bit-identical to np_pw_sum.
struct NpWarpScratch {  // per warp, in shared memory
  static constexpr int kMaxLeaves = 64;
  // every leaf of a split holds >= 57 terms, so groups of <= 57 * 64 terms fit
  static constexpr int kMaxTerms = 3584;
  int2 leaf[kMaxLeaves];                 // (lo, n) in tree order
  double val[kMaxLeaves];
};

template <int D>
struct NpLeaves {
  __device__ __noinline__ static void list(int lo, int n, int& cnt, int2* out) {
    if (n <= 128) {
      out[cnt++] = make_int2(lo, n);
      return;
    }
    int h = n / 2;
    h -= h % 8;
    NpLeaves<D - 1>::list(lo, h, cnt, out);
    NpLeaves<D - 1>::list(lo + h, n - h, cnt, out);
  }
  __device__ __noinline__ static double combine(int n, int& idx, const double* val) {
    if (n <= 128) return val[idx++];
    int h = n / 2;
    h -= h % 8;
    const double left = NpLeaves<D - 1>::combine(h, idx, val);
    const double right = NpLeaves<D - 1>::combine(n - h, idx, val);
    return __dadd_rn(left, right);
  }
};
template <>
struct NpLeaves<0> {
  __device__ __forceinline__ static void list(int lo, int n, int& cnt, int2* out) {
    out[cnt++] = make_int2(lo, n);
  }
  __device__ __forceinline__ static double combine(int, int& idx, const double* val) {
    return val[idx++];
  }
};

// Sum of g(0..n) in numpy's order, computed by the whole warp (all 32 lanes
// must call; every lane returns the sum).  n <= NpWarpScratch::kMaxTerms.
template <class G>
__device__ __forceinline__ double np_pw_sum_warp(const G& g, int n, NpWarpScratch* sc) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & 7;
  int nleaves = 0;
  if (lane == 0) NpLeaves<8>::list(0, n, nleaves, sc->leaf);
  nleaves = __shfl_sync(0xffffffffu, nleaves, 0);
  __syncwarp();
  for (int base = 0; base < nleaves; base += 4) {
    const int l = base + (lane >> 3);
    const bool act = l < nleaves;
    const int2 lf = act ? sc->leaf[l] : make_int2(0, 0);
    const int lo = lf.x, m = lf.y;
    double r = 0.0;
    if (act && m >= 8) {
      r = g(lo + sub);
      const int stop = m - (m % 8);
      for (int i = 8; i < stop; i += 8) r = __dadd_rn(r, g(lo + i + sub));
    }
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) within each 8-lane group
    double t = __shfl_down_sync(0xffffffffu, r, 1);
    r = __dadd_rn(r, t);  // even lanes: r_k + r_k+1
    t = __shfl_down_sync(0xffffffffu, r, 2);
    r = __dadd_rn(r, t);  // lanes % 4 == 0: (r0+r1)+(r2+r3)
    t = __shfl_down_sync(0xffffffffu, r, 4);
    r = __dadd_rn(r, t);  // lane % 8 == 0: the eight-chain sum
    if (act && sub == 0) {
      double res;
      int i;
      if (m < 8) {
        res = 0.0;
        i = 0;
      } else {
        res = r;
        i = m - (m % 8);
      }
      for (; i < m; ++i) res = __dadd_rn(res, g(lo + i));
      sc->val[l] = res;
    }
  }
  __syncwarp();
  int idx = 0;
  const double total = NpLeaves<8>::combine(n, idx, sc->val);
  __syncwarp();
  return total;
}

// Leaf plan of a group size (numpy's pairwise tree depends on n only), built
// once per block and shared by every row the block evaluates.
struct NpLeafPlan {
  int n, nleaves;
  int2 leaf[NpWarpScratch::kMaxLeaves];
};
__device__ __forceinline__ void np_leaf_plan(int n, NpLeafPlan* p) {  // one thread
  int cnt = 0;
  NpLeaves<8>::list(0, n, cnt, p->leaf);
  p->n = n;
  p->nleaves = cnt;
}

// Both groups of one row in one warp pass: the leaves of group 1 then of
// group 2 are spread over the 4 eight-lane slots of each round, each slot
// running one leaf's eight chains exactly as np_pw_sum_warp does, so the two
// sums carry np_pw_sum's bits.  f(i, grp) = the i-th term of group grp (0/1).
// val: per-warp scratch of P1.nleaves + P2.nleaves doubles.
template <class F>
__device__ __forceinline__ void np_pw_sum2_warp(const F& f, const NpLeafPlan& P1,
                                                const NpLeafPlan& P2, double* val, double& s1,
                                                double& s2) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & 7;
  const int total = P1.nleaves + P2.nleaves;
  for (int base = 0; base < total; base += 4) {
    const int l = base + (lane >> 3);
    const bool act = l < total;
    const int grp = (l < P1.nleaves) ? 0 : 1;
    const int2 lf = !act ? make_int2(0, 0) : (grp == 0 ? P1.leaf[l] : P2.leaf[l - P1.nleaves]);
    const int lo = lf.x, m = lf.y;
    double r = 0.0;
    if (act && m >= 8) {
      r = f(lo + sub, grp);
      const int stop = m - (m % 8);
      for (int i = 8; i < stop; i += 8) r = __dadd_rn(r, f(lo + i + sub, grp));
    }
    double t = __shfl_down_sync(0xffffffffu, r, 1);
    r = __dadd_rn(r, t);
    t = __shfl_down_sync(0xffffffffu, r, 2);
    r = __dadd_rn(r, t);
    t = __shfl_down_sync(0xffffffffu, r, 4);
    r = __dadd_rn(r, t);
    if (act && sub == 0) {
      double res;
      int i;
      if (m < 8) {
        res = 0.0;
        i = 0;
      } else {
        res = r;
        i = m - (m % 8);
      }
      for (; i < m; ++i) res = __dadd_rn(res, f(lo + i, grp));
      val[l] = res;
    }
  }
  __syncwarp();
  double a = 0.0, b = 0.0;
  if (lane == 0) {
    int idx = 0;
    a = NpLeaves<8>::combine(P1.n, idx, val);
    idx = 0;
    b = NpLeaves<8>::combine(P2.n, idx, val + P1.nleaves);
  }
  s1 = __shfl_sync(0xffffffffu, a, 0);
  s2 = __shfl_sync(0xffffffffu, b, 0);
  __syncwarp();
}

// welch_exact of a row staged in shared memory (stride 1), both groups per
// pass with precomputed leaf plans: the bits of welch_exact.
__device__ __forceinline__ WelchExact welch_exact_warp2(const double* row, const int16_t* ord,
                                                        const NpLeafPlan& P1,
                                                        const NpLeafPlan& P2, double* val) {
  const int n1 = P1.n, n2 = P2.n;
  double s1, s2;
  np_pw_sum2_warp([&](int i, int grp) { return row[ord[i + grp * n1]]; }, P1, P2, val, s1, s2);
  const double m1 = __ddiv_rn(s1, (double)n1);
  const double m2 = __ddiv_rn(s2, (double)n2);
  double q1, q2;
  np_pw_sum2_warp(
      [&](int i, int grp) {
        const double d = __dsub_rn(row[ord[i + grp * n1]], grp ? m2 : m1);
        return __dmul_rn(d, d);
      },
      P1, P2, val, q1, q2);
  const double v1 = __ddiv_rn(q1, (double)(n1 - 1));
  const double v2 = __ddiv_rn(q2, (double)(n2 - 1));
  const double var_term = __dadd_rn(__ddiv_rn(v1, (double)n1), __ddiv_rn(v2, (double)n2));
  WelchExact r;
  r.num = __dsub_rn(m1, m2);
  if (var_term == 0.0) {
    r.t = 0.0;
    r.degenerate = (r.num != 0.0);
  } else {
    r.t = __ddiv_rn(r.num, __dsqrt_rn(var_term));
    r.degenerate = false;
  }
  return r;
}

// welch_exact with the warp: identical bits, every lane gets the result.
// Larger groups fall back to lane 0 and a broadcast.
__device__ __forceinline__ WelchExact welch_exact_warp(const double* row, int64_t stride,
                                                       const int16_t* ord, int n1, int n2,
                                                       NpWarpScratch* sc) {
  if (n1 > NpWarpScratch::kMaxTerms || n2 > NpWarpScratch::kMaxTerms) {
    WelchExact r{};
    if ((threadIdx.x & 31) == 0) r = welch_exact(row, stride, ord, n1, n2);
    r.t = __shfl_sync(0xffffffffu, r.t, 0);
    r.num = __shfl_sync(0xffffffffu, r.num, 0);
    r.degenerate = __shfl_sync(0xffffffffu, (int)r.degenerate, 0) != 0;
    return r;
  }
  GroupVals a{row, ord, stride}, b{row, ord + n1, stride};
  const double m1 = __ddiv_rn(np_pw_sum_warp(a, n1, sc), (double)n1);
  const double m2 = __ddiv_rn(np_pw_sum_warp(b, n2, sc), (double)n2);
  GroupSqDev da{row, ord, stride, m1}, db{row, ord + n1, stride, m2};
  const double v1 = __ddiv_rn(np_pw_sum_warp(da, n1, sc), (double)(n1 - 1));
  const double v2 = __ddiv_rn(np_pw_sum_warp(db, n2, sc), (double)(n2 - 1));
  const double var_term = __dadd_rn(__ddiv_rn(v1, (double)n1), __ddiv_rn(v2, (double)n2));
  WelchExact r;
  r.num = __dsub_rn(m1, m2);
  if (var_term == 0.0) {
    r.t = 0.0;
    r.degenerate = (r.num != 0.0);
  } else {
    r.t = __ddiv_rn(r.num, __dsqrt_rn(var_term));
    r.degenerate = false;
  }
  return r;
}

}  // namespace rmx
