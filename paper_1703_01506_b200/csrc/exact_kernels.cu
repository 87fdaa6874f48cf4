// exact_kernels.cu -- the fp64 side of the NaivePT path (compiled with
// -fmad=false: every double op is an individually rounded IEEE op, so the
// statistic reproduces the reference's numpy bits, see np_exact.cuh).
//
//   k_prep          K0: per-voxel standardisation, fp16 hi/lo split planes
//   k_const_reduce  voxels constant over all subjects (exact, perm-invariant)
//   k_refine        K2: fp64 refinement of the tensor-core top-4 candidates
//   k_transpose     X (v x n) -> X^T (n x v) for the coalesced exact kernels
//   k_exact_rows    exhaustive exact statistic (materialised T / fallback)
//   k_exact_reduce  per-permutation max/argmax of k_exact_rows' partials
//   k_pairs         exact statistic at explicit (perm, voxel) pairs
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "np_exact.cuh"
#include "rmx_internal.cuh"
#include "sm100.cuh"

namespace rmx {

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// (value, index) max with the lowest index on ties (np.argmax semantics)
__device__ __forceinline__ void warp_argmax(double& v, int& j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oj = __shfl_xor_sync(0xffffffffu, j, o);
    if (ov > v || (ov == v && oj >= 0 && (j < 0 || oj < j))) {
      v = ov;
      j = oj;
    }
  }
}
__device__ __forceinline__ void note_degenerate(NaiveCounters* c, int64_t perm, int64_t voxel) {
  unsigned long long key = ((unsigned long long)perm << 32) | (unsigned long long)voxel;
  atomicMin(&c->deg_key, key);
}

// ---------------------------------------------------------------- K0
// One warp per voxel row: fp64 mean / sd, z = (x - mean) / sd, then either
// the fp16 hi + lo planes of z (and q = z^2) or the int8 digit planes.  R > 0:
// the row is held in registers (R values per lane, n <= 32 R), so X is read
// once with all loads in flight; R = 0: generic re-reading loop.  Rows
// constant across all subjects get z = 0 (tensor-core t~ = 0) and, if numpy's
// rounding makes their exact statistic non-zero, are listed for
// k_const_reduce.
// One voxel row j held by one warp: R > 0: xr[r] = x[j, lane + 32 r] (0 past
// n); R = 0: re-read from `row`.  err_max: running int8 quantisation bound.
template <int R>
__device__ __forceinline__ void prep_row(const PrepArgs& a, int64_t j, int lane,
                                         const double (&xr)[R > 0 ? R : 1], const double* row,
                                         double& err_max) {
  const int64_t plane = a.v * (int64_t)a.kpad;
  // f(k, x) over this lane's subjects k < n
  auto each = [&](auto&& f) {
    if constexpr (R > 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = lane + 32 * r;
        if (k < a.n) f(k, xr[r]);
      }
    } else {
      for (int k = lane; k < a.n; k += 32) f(k, row[k]);
    }
  };
  // f(k, x) over this lane's padded columns k < kpad (x = 0 past n); kpad <= 32 R
  auto each_pad = [&](auto&& f) {
    if constexpr (R > 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = lane + 32 * r;
        if (k < a.kpad) f(k, xr[r]);
      }
    } else {
      for (int k = lane; k < a.kpad; k += 32) f(k, k < a.n ? row[k] : 0.0);
    }
  };
  double s = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
  each([&](int, double x) {
    s += x;
    mn = fmin(mn, x);
    mx = fmax(mx, x);
  });
  s = warp_sum_d(s);
  mn = warp_min_d(mn);
  mx = warp_max_d(mx);
  const double mean = s / a.n;
  double ss = 0.0;
  each([&](int, double x) {
    const double d = x - mean;
    ss += d * d;
  });
  ss = warp_sum_d(ss);
  const bool constant = (mn == mx);
  const double inv = constant ? 0.0 : 1.0 / sqrt(ss / (a.n - 1));
  if (a.planes8) {
    // int8 path: zq = rint(z * scale) in [-32512, 32512], zq = 255 h + l with
    // h, l in [-127, 127]; row j of planes8 = [h_0 .. h_kpad-1 | l_0 .. l_kpad-1]
    double zmax = 0.0;
    each([&](int, double x) { zmax = fmax(zmax, fabs((x - mean) * inv)); });
    zmax = warp_max_d(zmax);
    const double scale = zmax > 0.0 ? 32512.0 / zmax : 0.0;
    const float inv_f = zmax > 0.0 ? (float)(zmax / 32512.0) : 0.0f;
    int8_t* p8 = reinterpret_cast<int8_t*>(a.planes8) + j * (int64_t)(2 * a.kpad);
    double err = 0.0;  // sum_i |z_i - dequantised z_i|: bounds |S~ - S| for any grouping
    each_pad([&](int k, double x) {
      int zq = 0;  // padded subjects and constant voxels: 0
      if (k < a.n && !constant) {
        const double z = (x - mean) * inv;
        zq = min(32512, max(-32512, (int)rint(z * scale)));
        err += fabs(z - (double)zq * (double)inv_f);
      }
      const int h = zq >= 0 ? (zq + 127) / 255 : -((127 - zq) / 255);  // round(zq / 255)
      p8[k] = (int8_t)h;
      p8[a.kpad + k] = (int8_t)(zq - 255 * h);
    });
    err = warp_sum_d(err);
    err_max = fmax(err_max, err);
    if (lane == 0) a.inv_scale[j] = inv_f;
  } else {
    __half* zh = a.planes + j * a.kpad;
    each_pad([&](int k, double x) {
      const double z = (k < a.n && !constant) ? (x - mean) * inv : 0.0;
      const __half h_z = __double2half(z);
      zh[k] = h_z;
      zh[2 * plane + k] = __double2half(z - (double)__half2float(h_z));
      if (!a.zplanes_only) {
        const double q = z * z;
        const __half h_q = __double2half(q);
        zh[plane + k] = h_q;
        zh[3 * plane + k] = __double2half(q - (double)__half2float(h_q));
      }
    });
  }
  if (constant && lane == 0) {
    const WelchExact w = welch_exact_const(mn, a.n1, a.n - a.n1);
    if (w.t != 0.0 || w.degenerate) {
      unsigned slot = atomicAdd(&a.counters->cvox_count, 1u);
      a.cvox[slot] = (int32_t)j;
    }
  }
}

__device__ __forceinline__ void prep_publish_err(const PrepArgs& a, int lane, double err_max) {
  if (a.planes8 && lane == 0 && err_max > 0.0)
    // rounded up; non-negative floats order like their bit patterns
    atomicMax(&a.counters->emax_bits, __float_as_uint((float)(err_max * (1.0 + 1e-6)) + 1e-30f));
}

// K0, generic: one warp per voxel row, the row read straight from global
// memory into registers (R > 0, n <= 32 R) or re-read (R = 0).
template <int R>
__global__ void __launch_bounds__(256, 2) k_prep(PrepArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  double err_max = 0.0;
  const int64_t jend = a.v_end > 0 ? a.v_end : a.v;
  for (int64_t j = a.v_begin + (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
       j < jend; j += warps) {
    const double* row = a.x + j * a.n;
    double xr[R > 0 ? R : 1];
    if constexpr (R > 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = lane + 32 * r;
        xr[r] = k < a.n ? __ldg(row + k) : 0.0;
      }
    }
    prep_row<R>(a, j, lane, xr, row, err_max);
  }
  prep_publish_err(a, lane, err_max);
}

// K0, streamed (even n): X rows are contiguous, so each CTA pulls tiles of
// kPrepRows consecutive rows (kPrepRows * n * 8 bytes) with 1-D bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a kPrepStages ring; warp w
// standardises row w of the tile from shared memory.  The loads of the next
// kPrepStages - 1 tiles are in flight while a tile is processed, independent
// of the register budget that limits the generic kernel to one row per warp.
constexpr int kPrepRows = 8;  // = warps per CTA
constexpr int kPrepStages = 4;

// One voxel row from shared memory, lane-contiguous mapping: lane owns the
// subjects k = 4 lane + 128 g + e (g < G, e < 4), so the int8 digits (and
// fp16 halves) of four consecutive subjects leave as one packed store.
// Constancy is tested against subject 0's value (one compare per element,
// one vote).  int8 quantisation bound, with tq = z / inv (inv = zmax / 32512
// the exact step, inv_f = fp32(inv) the step the epilogue uses) and
// zq = rint(tq):
//   |z - zq inv_f| <= |tq - zq| inv + |zq| |inv - inv_f|
// so e_j = inv sum_i |tq_i - zq_i| + n 32512 |inv - inv_f| (each with a
// 2^-40 relative margin for the fp64 roundings of z and tq) bounds
// |S~ - S| for every grouping; the first sum is accumulated from the
// rounding residuals tq - rint(tq) (two fp64 ops per element).
template <int G>
__device__ __forceinline__ void prep_row4(const PrepArgs& a, int64_t j, int lane,
                                          const double* srow, double& err_max) {
  double d[G][4];
  double s = 0.0;
  const double x0 = srow[0];
  bool varies = false;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int k0 = 4 * lane + 128 * g;
    if (k0 < a.n) {  // n even and k0 % 4 == 0: pairs are whole
      const double2 p0 = *reinterpret_cast<const double2*>(srow + k0);
      const double2 p1 = k0 + 2 < a.n ? *reinterpret_cast<const double2*>(srow + k0 + 2)
                                      : make_double2(x0, x0);
      d[g][0] = p0.x;
      d[g][1] = p0.y;
      d[g][2] = p1.x;
      d[g][3] = p1.y;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) d[g][e] = x0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      varies |= d[g][e] != x0;
      if (k0 + e < a.n) s += d[g][e];
    }
  }
  s = warp_sum_d(s);
  const bool constant = !__any_sync(0xffffffffu, varies);
  const double mean = s / a.n;
  double ss = 0.0;
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool in = 4 * lane + 128 * g + e < a.n;
      d[g][e] = (in && !constant) ? d[g][e] - mean : 0.0;  // centred; 0 past n
      ss = fma(d[g][e], d[g][e], ss);
    }
  ss = warp_sum_d(ss);
  const double inv = constant ? 0.0 : 1.0 / sqrt(ss / (a.n - 1));
  if (a.planes8) {
    double dmax = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < 4; ++e) dmax = fmax(dmax, fabs(d[g][e]));
    const double zmax = warp_max_d(dmax) * inv;
    const double scale = zmax > 0.0 ? 32512.0 / zmax : 0.0;
    const float inv_f = zmax > 0.0 ? (float)(zmax / 32512.0) : 0.0f;
    const double c = inv * scale;  // zq = rint(d c); |d c| <= 32512 (+ rounding < 0.5)
    int8_t* p8 = reinterpret_cast<int8_t*>(a.planes8) + j * (int64_t)(2 * a.kpad);
    double fr = 0.0;  // sum of |tq - rint(tq)|
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int k0 = 4 * lane + 128 * g;
      if (k0 >= a.kpad) continue;  // kpad % 16 == 0: groups are whole
      uint32_t hw = 0u, lw = 0u;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double tq = d[g][e] * c;
        const double rq = rint(tq);
        fr += fabs(tq - rq);
        const int zq = (int)rq;
        const int h = __float2int_rn((float)zq * (1.0f / 255.0f));  // |zq/255 - h| <= 0.498
        hw |= (uint32_t)(uint8_t)(int8_t)h << (8 * e);
        lw |= (uint32_t)(uint8_t)(int8_t)(zq - 255 * h) << (8 * e);
      }
      *reinterpret_cast<uint32_t*>(p8 + k0) = hw;
      *reinterpret_cast<uint32_t*>(p8 + a.kpad + k0) = lw;
    }
    fr = warp_sum_d(fr);
    if (!constant) {
      const double step = zmax / 32512.0;
      const double e = (step * fr + (double)a.n * 32512.0 * fabs(step - (double)inv_f)) *
                       (1.0 + 0x1p-40);
      err_max = fmax(err_max, e);
    }
    if (lane == 0) a.inv_scale[j] = inv_f;
  } else {
    const int64_t plane = a.v * (int64_t)a.kpad;
    __half* zh = a.planes + j * a.kpad;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int k0 = 4 * lane + 128 * g;
      if (k0 >= a.kpad) continue;
      __half hz[4], lz[4], hq[4], lq[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double z = d[g][e] * inv;
        hz[e] = __double2half(z);
        lz[e] = __double2half(z - (double)__half2float(hz[e]));
        const double q = z * z;
        hq[e] = __double2half(q);
        lq[e] = __double2half(q - (double)__half2float(hq[e]));
      }
      *reinterpret_cast<uint2*>(zh + k0) = *reinterpret_cast<const uint2*>(hz);
      *reinterpret_cast<uint2*>(zh + 2 * plane + k0) = *reinterpret_cast<const uint2*>(lz);
      if (!a.zplanes_only) {
        *reinterpret_cast<uint2*>(zh + plane + k0) = *reinterpret_cast<const uint2*>(hq);
        *reinterpret_cast<uint2*>(zh + 3 * plane + k0) = *reinterpret_cast<const uint2*>(lq);
      }
    }
  }
  if (constant && lane == 0) {
    const WelchExact w = welch_exact_const(x0, a.n1, a.n - a.n1);
    if (w.t != 0.0 || w.degenerate) {
      unsigned slot = atomicAdd(&a.counters->cvox_count, 1u);
      a.cvox[slot] = (int32_t)j;
    }
  }
}

template <int R>  // R = 4-subject groups per lane (kpad <= 128 R)
__global__ void __launch_bounds__(32 * kPrepRows, 2) k_prep_bulk(PrepArgs a) {
  extern __shared__ __align__(128) uint8_t psm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(psm);
  double* tiles = reinterpret_cast<double*>(psm + 128);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t jend = a.v_end > 0 ? a.v_end : a.v;
  const int64_t ntiles = (jend - a.v_begin + kPrepRows - 1) / kPrepRows;
  const int64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t tile_elems = (int64_t)kPrepRows * a.n;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPrepStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t i) {  // thread 0: tile blockIdx.x + i * gridDim.x -> stage i % S
    const int64_t r0 = a.v_begin + (blockIdx.x + i * gridDim.x) * kPrepRows;
    const int64_t nr = min((int64_t)kPrepRows, jend - r0);
    const uint32_t bytes = (uint32_t)(nr * a.n * 8);
    uint64_t* bar = &full[i % kPrepStages];
    mbar_expect_tx(bar, bytes);
    bulk_load(tiles + (i % kPrepStages) * tile_elems, a.x + r0 * a.n, bytes, bar);
  };
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < kPrepStages && i < mine; ++i) issue(i);
  double err_max = 0.0;
  for (int64_t i = 0; i < mine; ++i) {
    mbar_wait(&full[i % kPrepStages], (uint32_t)((i / kPrepStages) & 1));
    const int64_t j = a.v_begin + (blockIdx.x + i * gridDim.x) * kPrepRows + warp;
    if (j < jend) {
      const double* srow = tiles + (i % kPrepStages) * tile_elems + (int64_t)warp * a.n;
      prep_row4<R>(a, j, lane, srow, err_max);
    }
    __syncthreads();  // every warp is done with stage i % S
    if (threadIdx.x == 0 && i + kPrepStages < mine) issue(i + kPrepStages);
  }
  prep_publish_err(a, lane, err_max);
}

__global__ void k_const_reduce(const double* x, int n, int n1, const int32_t* cvox,
                               NaiveCounters* counters, ConstInfo* out) {
  __shared__ double sv[32], sa[32];
  __shared__ int sj[32], sja[32], sd[32];
  const int count = (int)counters->cvox_count;
  double best = -DBL_MAX, best_abs = -DBL_MAX;
  int bj = -1, bja = -1, dj = -1;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int j = cvox[i];
    const WelchExact w = welch_exact_const(x[(int64_t)j * n], n1, n - n1);
    if (w.degenerate) {
      if (dj < 0 || j < dj) dj = j;
      continue;
    }
    if (w.t > best || (w.t == best && j < bj)) best = w.t, bj = j;
    const double at = fabs(w.t);
    if (at > best_abs || (at == best_abs && j < bja)) best_abs = at, bja = j;
  }
  warp_argmax(best, bj);
  warp_argmax(best_abs, bja);
  for (int o = 16; o > 0; o >>= 1) {
    int od = __shfl_xor_sync(0xffffffffu, dj, o);
    if (od >= 0 && (dj < 0 || od < dj)) dj = od;
  }
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (lane == 0) sv[w] = best, sj[w] = bj, sa[w] = best_abs, sja[w] = bja, sd[w] = dj;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    best = lane < nw ? sv[lane] : -DBL_MAX;
    bj = lane < nw ? sj[lane] : -1;
    best_abs = lane < nw ? sa[lane] : -DBL_MAX;
    bja = lane < nw ? sja[lane] : -1;
    dj = lane < nw ? sd[lane] : -1;
    warp_argmax(best, bj);
    warp_argmax(best_abs, bja);
    for (int o = 16; o > 0; o >>= 1) {
      int od = __shfl_xor_sync(0xffffffffu, dj, o);
      if (od >= 0 && (dj < 0 || od < dj)) dj = od;
    }
    if (lane == 0) {
      out->best_t = best;
      out->best_t_voxel = bj;
      out->best_abs = best_abs;
      out->best_abs_voxel = bja;
      out->deg_voxel = dj;
      out->count = count;
      out->deg_num = 0.0;
      if (dj >= 0) {
        const WelchExact wd = welch_exact_const(x[(int64_t)dj * n], n1, n - n1);
        out->deg_num = wd.num;
        note_degenerate(counters, 0, dj);  // every labelling: first perm of the call
      }
    }
  }
}

// ---------------------------------------------------------------- K2
// One warp per permutation: gather the (perm, chunk) top-4 candidates, keep
// every voxel whose t~ lies in the band below the best, evaluate those
// exactly in fp64 (reference arithmetic) and take the max.  A chunk whose
// 4th-best is inside the band might hide a fifth in-band voxel: the
// permutation is then queued for the exhaustive exact path.
constexpr int kRefineWarps = 8;
constexpr int kStageMaxN = 2048;  // rows up to this many subjects are staged in smem

// Evaluating one candidate: the warp copies the voxel's row into its smem
// buffer (coalesced), then evaluates the reference arithmetic with the
// numpy-pairwise chains spread over its lanes (welch_exact_warp: same bits);
// the owning lane keeps the result.
template <bool STAGE>
__global__ void __launch_bounds__(32 * kRefineWarps, 4) k_refine(RefineArgs a) {
  extern __shared__ __align__(16) unsigned char refine_smem[];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  NpWarpScratch* sc = reinterpret_cast<NpWarpScratch*>(refine_smem) + w;
  unsigned char* rest = refine_smem + kRefineWarps * sizeof(NpWarpScratch);
  double* rowbuf = reinterpret_cast<double*>(rest) + (size_t)w * (STAGE ? a.n : 0);
  int16_t* ord = reinterpret_cast<int16_t*>(rest + (STAGE ? (size_t)kRefineWarps * a.n * 8 : 0)) +
                 (size_t)w * a.n;
  // leaf plans of the two group sizes, once per block (welch_exact_warp2)
  unsigned char* tail = rest + (STAGE ? (size_t)kRefineWarps * a.n * 8 : 0) +
                        (size_t)kRefineWarps * a.n * sizeof(int16_t);
  NpLeafPlan* plans = reinterpret_cast<NpLeafPlan*>(
      (reinterpret_cast<uintptr_t>(tail) + 15) & ~uintptr_t(15));
  double* pvals = reinterpret_cast<double*>(plans + 2) + (size_t)w * 2 * NpWarpScratch::kMaxLeaves;
  const int n2 = a.n - a.n1;
  const bool two_pass = a.n1 <= NpWarpScratch::kMaxTerms && n2 <= NpWarpScratch::kMaxTerms;
  if (two_pass) {
    if (threadIdx.x == 0) np_leaf_plan(a.n1, &plans[0]);
    if (threadIdx.x == 32 % blockDim.x) np_leaf_plan(n2, &plans[1]);
  }
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * kRefineWarps + w;
  if (p >= a.L) return;
  for (int i = lane; i < a.n; i += 32) ord[i] = a.orders[p * a.n + i];
  __syncwarp();
  const int4* cp = a.cand + 2 * p * a.slots;

  float tmax = -FLT_MAX;
  for (int c = lane; c < a.slots; c += 32) {
    const int4 e = cp[2 * c];
    if (e.y >= 0) tmax = fmaxf(tmax, __int_as_float(e.x));
  }
  for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
  const float band = band_abs(tmax, a.band_rel, __uint_as_float(a.counters->emax_bits),
                              a.beta_abs, a.gamma);
  const float lo = tmax - band;

  double best = -DBL_MAX;
  int bj = -1;
  bool overflow = false;
  unsigned nref = 0;
  // warp-collective: evaluate voxel j for the lane `owner`
  auto eval = [&](int j, int owner) {
    const double* row = a.x + (int64_t)j * a.n;
    if (STAGE) {
      __syncwarp();
      for (int i = lane; i < a.n; i += 32) rowbuf[i] = row[i];
      __syncwarp();
      row = rowbuf;
    }
    const WelchExact r = two_pass ? welch_exact_warp2(row, ord, plans[0], plans[1], pvals)
                                  : welch_exact_warp(row, 1, ord, a.n1, n2, sc);
    if (lane == owner) {
      ++nref;
      if (r.degenerate) {
        note_degenerate(a.counters, p, j);
      } else {
        const double key = a.two_sided ? fabs(r.t) : r.t;
        if (key > best || (key == best && (bj < 0 || j < bj))) {
          best = key;
          bj = j;
        }
      }
    }
  };
  auto eval_all = [&](int j) {  // each lane's j (< 0: none), one at a time
    unsigned m = __ballot_sync(0xffffffffu, j >= 0);
    while (m) {
      const int owner = __ffs(m) - 1;
      m &= m - 1;
      eval(__shfl_sync(0xffffffffu, j, owner), owner);
    }
  };
  if (tmax > -FLT_MAX) {
    for (int c0 = 0; c0 < a.slots; c0 += 32) {
      const int c = c0 + lane;
      int j0 = -1, j1 = -1, j2 = -1, j3 = -1;
      if (c < a.slots) {
        const int4 e0 = cp[2 * c], e1 = cp[2 * c + 1];
        if (e0.y >= 0 && __int_as_float(e0.x) >= lo) j0 = e0.y;
        if (e0.w >= 0 && __int_as_float(e0.z) >= lo) j1 = e0.w;
        if (e1.y >= 0 && __int_as_float(e1.x) >= lo) j2 = e1.y;
        if (e1.w >= 0 && __int_as_float(e1.z) >= lo) {
          j3 = e1.w;
          overflow = true;  // a 5th in-band voxel of this chunk could be hiding
        }
      }
      eval_all(j0);
      eval_all(j1);
      eval_all(j2);
      eval_all(j3);
    }
  }
  const unsigned scount = a.counters->susp_count;
  if (scount > 0 && scount <= (unsigned)kSuspectCap) {
    for (unsigned i0 = 0; i0 < scount; i0 += 32) {
      const unsigned i = i0 + lane;
      eval_all((i < scount && a.susp[2 * i] == (int)p) ? a.susp[2 * i + 1] : -1);
    }
  }
  warp_argmax(best, bj);
  const unsigned any_over = __ballot_sync(0xffffffffu, overflow);
  for (int o = 16; o > 0; o >>= 1) nref += __shfl_xor_sync(0xffffffffu, nref, o);
  if (lane == 0) {
    // constant voxels: the same exact statistic under every labelling
    const ConstInfo ci = *a.cinfo;
    const double cb = a.two_sided ? ci.best_abs : ci.best_t;
    const int cj = a.two_sided ? ci.best_abs_voxel : ci.best_t_voxel;
    if (cj >= 0 && (cb > best || (cb == best && (bj < 0 || cj < bj)))) {
      best = cb;
      bj = cj;
    }
    a.max_out[p] = best;
    a.argmax_out[p] = bj;
    atomicAdd(&a.counters->band_candidates, nref);
    if (any_over || bj < 0) {
      unsigned slot = atomicAdd(&a.counters->overflow_count, 1u);
      a.overflow[slot] = (int32_t)p;
    }
  }
}

// Exhaustive exact statistic for a few permutations straight from X: one
// warp per voxel stages the row in smem, the warp evaluates it (welch_exact_warp).
// grid (nvb, nperm); per-block (max, argmax) partials as k_exact_rows.
__global__ void __launch_bounds__(32 * kRefineWarps)
    k_exact_rows_staged(const double* __restrict__ x, int64_t v, int n, int n1,
                        const int16_t* __restrict__ orders, const int32_t* perm_list,
                        int64_t perm_offset, int two_sided, double* part_val, int32_t* part_idx,
                        NaiveCounters* counters) {
  extern __shared__ __align__(16) unsigned char ex_smem[];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  NpWarpScratch* sc = reinterpret_cast<NpWarpScratch*>(ex_smem) + w;
  unsigned char* rest = ex_smem + kRefineWarps * sizeof(NpWarpScratch);
  double* rowbuf = reinterpret_cast<double*>(rest) + (size_t)w * n;
  int16_t* ord = reinterpret_cast<int16_t*>(rest + (size_t)kRefineWarps * n * 8);
  const int64_t i = blockIdx.y;
  const int64_t p = perm_list ? perm_list[i] : perm_offset + i;
  for (int k = threadIdx.x; k < n; k += blockDim.x) ord[k] = orders[p * n + k];
  __syncthreads();
  const int64_t per = (v + gridDim.x - 1) / gridDim.x;
  const int64_t jlo = blockIdx.x * per, jhi = min(v, jlo + per);
  double best = -DBL_MAX;
  int bj = -1;
  for (int64_t j = jlo + w; j < jhi; j += kRefineWarps) {
    __syncwarp();
    for (int k = lane; k < n; k += 32) rowbuf[k] = x[j * n + k];
    __syncwarp();
    const WelchExact r = welch_exact_warp(rowbuf, 1, ord, n1, n - n1, sc);
    if (lane == 0) {
      if (r.degenerate) {
        if (counters) note_degenerate(counters, p, j);
      } else {
        const double key = two_sided ? fabs(r.t) : r.t;
        if (key > best || (key == best && (bj < 0 || j < bj))) best = key, bj = (int)j;
      }
    }
  }
  __shared__ double sv[32];
  __shared__ int sj[32];
  warp_argmax(best, bj);
  if (lane == 0) sv[w] = best, sj[w] = bj;
  __syncthreads();
  if (w == 0) {
    best = lane < kRefineWarps ? sv[lane] : -DBL_MAX;
    bj = lane < kRefineWarps ? sj[lane] : -1;
    warp_argmax(best, bj);
    if (lane == 0) {
      part_val[i * gridDim.x + blockIdx.x] = best;
      part_idx[i * gridDim.x + blockIdx.x] = bj;
    }
  }
}

__global__ void k_transpose(const double* __restrict__ x, int64_t v, int n, double* __restrict__ xt) {
  __shared__ double tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r;
    const int k = k0 + threadIdx.x;
    if (j < v && k < n) tile[r][threadIdx.x] = x[j * n + k];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r;
    const int64_t j = j0 + threadIdx.x;
    if (j < v && k < n) xt[(int64_t)k * v + j] = tile[threadIdx.x][r];
  }
}

// grid (nvb, nperm): block (vb, i) evaluates perm list[i] over its voxel
// stripe, thread per voxel.  TRANSPOSED: from X^T (coalesced across voxels,
// for many permutations); else straight from X (v x n rows; no transpose or
// scratch, for the few permutations of the overflow fallback).
template <bool TRANSPOSED>
__global__ void k_exact_rows(const double* __restrict__ xt, int64_t v, int n, int n1,
                             const int16_t* __restrict__ orders, const int32_t* perm_list,
                             int64_t perm_offset, int two_sided, double* t_out, int64_t ld,
                             double* part_val, int32_t* part_idx, NaiveCounters* counters) {
  extern __shared__ int16_t ord[];
  const int64_t i = blockIdx.y;
  const int64_t p = perm_list ? perm_list[i] : perm_offset + i;
  for (int k = threadIdx.x; k < n; k += blockDim.x) ord[k] = orders[p * n + k];
  __syncthreads();
  const int64_t per = (v + gridDim.x - 1) / gridDim.x;
  const int64_t jlo = blockIdx.x * per, jhi = min(v, jlo + per);
  double best = -DBL_MAX;
  int bj = -1;
  for (int64_t j = jlo + threadIdx.x; j < jhi; j += blockDim.x) {
    const WelchExact r = TRANSPOSED ? welch_exact(xt + j, v, ord, n1, n - n1)
                                    : welch_exact(xt + j * n, 1, ord, n1, n - n1);
    if (r.degenerate) {
      if (counters) note_degenerate(counters, p, j);
      continue;
    }
    if (t_out) t_out[i * ld + j] = r.t;
    const double key = two_sided ? fabs(r.t) : r.t;
    if (key > best || (key == best && (bj < 0 || j < bj))) best = key, bj = (int)j;
  }
  if (!part_val) return;
  __shared__ double sv[32];
  __shared__ int sj[32];
  warp_argmax(best, bj);
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (lane == 0) sv[w] = best, sj[w] = bj;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    best = lane < nw ? sv[lane] : -DBL_MAX;
    bj = lane < nw ? sj[lane] : -1;
    warp_argmax(best, bj);
    if (lane == 0) {
      part_val[i * gridDim.x + blockIdx.x] = best;
      part_idx[i * gridDim.x + blockIdx.x] = bj;
    }
  }
}

// Many permutations x all voxels with the statistics written out (the
// training columns of RapidPT, a materialised T): thread per voxel like
// k_exact_rows, but a block first stages its kVsVox voxels' rows in shared
// memory ([subject][voxel]: conflict-free for a common subject index) and then
// walks a chunk of permutations over them, so X is read once per chunk of
// permutations instead of once per permutation (k_exact_rows<true> re-read all
// of X^T, 1.7 GB at config 5, for each of the 400 training permutations: 672 GB).
// Same welch_exact arithmetic, so the same bits.  grid (voxel blocks, chunks).
constexpr int kVsVox = 64;

__global__ void __launch_bounds__(kVsVox) k_exact_rows_vstage(
    const double* __restrict__ x, int64_t v, int n, int n1, const int16_t* __restrict__ orders,
    int64_t nperm, int perms_per_chunk, double* __restrict__ t_out, int64_t ld,
    NaiveCounters* counters) {
  extern __shared__ __align__(16) unsigned char vsm[];
  double* xs = reinterpret_cast<double*>(vsm);                         // [n][kVsVox]
  int16_t* ord = reinterpret_cast<int16_t*>(xs + (size_t)n * kVsVox);  // [n]
  const int64_t j0 = (int64_t)blockIdx.x * kVsVox;
  const int nv = (int)min((int64_t)kVsVox, v - j0);
  const int t = threadIdx.x;
  for (int e = t; e < nv * n; e += kVsVox) {  // rows are contiguous in X: coalesced reads
    const int jj = e / n, k = e - jj * n;
    xs[(size_t)k * kVsVox + jj] = x[(j0 + jj) * n + k];
  }
  const int64_t p0 = (int64_t)blockIdx.y * perms_per_chunk;
  const int64_t p1 = min(nperm, p0 + perms_per_chunk);
  for (int64_t p = p0; p < p1; ++p) {
    __syncthreads();  // the rows are staged / the previous labelling is done with
    for (int k = t; k < n; k += kVsVox) ord[k] = orders[p * n + k];
    __syncthreads();
    if (t < nv) {
      const WelchExact r = welch_exact(xs + t, kVsVox, ord, n1, n - n1);
      if (r.degenerate) {
        if (counters) note_degenerate(counters, p, j0 + t);
      } else {
        t_out[p * ld + j0 + t] = r.t;
      }
    }
  }
}

__global__ void k_exact_reduce(const double* part_val, const int32_t* part_idx, int nvb,
                               const int32_t* perm_list, int64_t nperm, double* max_out,
                               int32_t* argmax_out) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (i >= nperm) return;
  double best = -DBL_MAX;
  int bj = -1;
  for (int b = lane; b < nvb; b += 32) {
    const double val = part_val[i * nvb + b];
    const int j = part_idx[i * nvb + b];
    if (j >= 0 && (val > best || (val == best && (bj < 0 || j < bj)))) best = val, bj = j;
  }
  warp_argmax(best, bj);
  if (lane == 0) {
    const int64_t p = perm_list ? perm_list[i] : i;
    max_out[p] = best;
    argmax_out[p] = bj;
  }
}

__global__ void k_pairs(const double* x, int64_t v, int n, int n1, const int16_t* orders,
                        const int32_t* pairs, int64_t npairs, double* t_out, double* num_out,
                        int32_t* deg_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int64_t p = pairs[2 * i];
  const int64_t j = pairs[2 * i + 1];
  const WelchExact r = welch_exact(x + j * n, 1, orders + p * n, n1, n - n1);
  t_out[i] = r.t;
  if (num_out) num_out[i] = r.num;
  if (deg_out) deg_out[i] = r.degenerate ? 1 : 0;
}

}  // namespace

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t s) {
  const int wpb = 8;
  const int64_t rows = (a.v_end > 0 ? a.v_end : a.v) - a.v_begin;
  if (rows <= 0) return cudaSuccess;
  int64_t blocks = (rows + wpb - 1) / wpb;
  if (blocks > 148 * 64) blocks = 148 * 64;
  // even n (16-byte aligned rows for the bulk copies), n <= 512: streamed
  if (a.n % 2 == 0 && a.kpad <= 512 && a.kpad % 16 == 0 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0) {
    const size_t smem = 128 + (size_t)kPrepStages * kPrepRows * a.n * sizeof(double);
    const int64_t tiles = (rows + kPrepRows - 1) / kPrepRows;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, 2 * 148);
    auto go = [&](auto kern) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<grid, 32 * kPrepRows, smem, s>>>(a);
      return cudaGetLastError();
    };
    if (a.kpad <= 128) return go(k_prep_bulk<1>);
    if (a.kpad <= 256) return go(k_prep_bulk<2>);
    if (a.kpad <= 384) return go(k_prep_bulk<3>);
    return go(k_prep_bulk<4>);
  }
  // rows up to 32 R subjects are read once into registers
  if (a.n <= 128) k_prep<4><<<(unsigned)blocks, 32 * wpb, 0, s>>>(a);
  else if (a.n <= 256) k_prep<8><<<(unsigned)blocks, 32 * wpb, 0, s>>>(a);
  else if (a.n <= 512) k_prep<16><<<(unsigned)blocks, 32 * wpb, 0, s>>>(a);
  else k_prep<0><<<(unsigned)blocks, 32 * wpb, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_const_reduce(const double* x, int64_t, int n, int n1, const int32_t* cvox,
                                NaiveCounters* counters, ConstInfo* out, cudaStream_t s) {
  k_const_reduce<<<1, 256, 0, s>>>(x, n, n1, cvox, counters, out);
  return cudaGetLastError();
}

cudaError_t launch_refine(const RefineArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.L + kRefineWarps - 1) / kRefineWarps;
  // per-warp scratch + leaf plans (2) and per-warp leaf sums (welch_exact_warp2)
  const size_t scratch = kRefineWarps * sizeof(NpWarpScratch) + 16 + 2 * sizeof(NpLeafPlan) +
                         (size_t)kRefineWarps * 2 * NpWarpScratch::kMaxLeaves * sizeof(double);
  if (a.n <= kStageMaxN) {
    const size_t smem = scratch + (size_t)kRefineWarps * a.n * (sizeof(int16_t) + sizeof(double));
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_refine<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_refine<true><<<(unsigned)blocks, 32 * kRefineWarps, smem, s>>>(a);
  } else {
    const size_t smem = scratch + (size_t)kRefineWarps * a.n * sizeof(int16_t);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_refine<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_refine<false><<<(unsigned)blocks, 32 * kRefineWarps, smem, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double* x, int64_t v, int n, double* xt, cudaStream_t s) {
  dim3 grid((unsigned)((v + 31) / 32), (unsigned)((n + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, s>>>(x, v, n, xt);
  return cudaGetLastError();
}

cudaError_t launch_exact_rows_vstage(const double* x, int64_t v, int n, int n1,
                                     const int16_t* orders, int64_t nperm, double* t_out,
                                     int64_t ld, NaiveCounters* counters, cudaStream_t s) {
  if (nperm <= 0) return cudaSuccess;
  const size_t smem = (size_t)n * kVsVox * sizeof(double) + (size_t)n * sizeof(int16_t);
  cudaError_t e = cudaFuncSetAttribute(k_exact_rows_vstage,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t vblocks = (v + kVsVox - 1) / kVsVox;
  // enough chunks to fill the GPU a few times over, at least 16 permutations each
  int chunks = (int)std::max<int64_t>(1, std::min<int64_t>((nperm + 15) / 16, (8 * 148 + vblocks - 1) / vblocks));
  chunks = std::min(chunks, 65535);
  const int ppc = (int)((nperm + chunks - 1) / chunks);
  chunks = (int)((nperm + ppc - 1) / ppc);
  k_exact_rows_vstage<<<dim3((unsigned)vblocks, (unsigned)chunks), kVsVox, smem, s>>>(
      x, v, n, n1, orders, nperm, ppc, t_out, ld, counters);
  return cudaGetLastError();
}

bool exact_rows_vstage_supported(int n) {
  return (size_t)n * kVsVox * sizeof(double) + (size_t)n * sizeof(int16_t) <= 200 * 1024;
}

cudaError_t launch_exact_rows(const double* xt, int64_t v, int n, int n1, const int16_t* orders,
                             const int32_t* perm_list, int64_t nperm, int two_sided,
                             double* t_out, int64_t ld, double* part_val, int32_t* part_idx,
                             int nvb, NaiveCounters* counters, cudaStream_t s, bool transposed) {
  if (nperm <= 0) return cudaSuccess;
  if (!transposed && n <= kStageMaxN && part_val && !t_out) {
    const size_t smem = kRefineWarps * sizeof(NpWarpScratch) + (size_t)kRefineWarps * n * sizeof(double) +
                        (size_t)n * sizeof(int16_t);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_exact_rows_staged,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    for (int64_t base = 0; base < nperm; base += 65535) {
      const int64_t cnt = nperm - base < 65535 ? nperm - base : 65535;
      dim3 grid((unsigned)nvb, (unsigned)cnt);
      k_exact_rows_staged<<<grid, 32 * kRefineWarps, smem, s>>>(
          xt, v, n, n1, orders, perm_list ? perm_list + base : nullptr, base, two_sided,
          part_val + base * nvb, part_idx + base * nvb, counters);
    }
    return cudaGetLastError();
  }
  auto kern = transposed ? k_exact_rows<true> : k_exact_rows<false>;
  for (int64_t base = 0; base < nperm; base += 65535) {
    const int64_t cnt = nperm - base < 65535 ? nperm - base : 65535;
    dim3 grid((unsigned)nvb, (unsigned)cnt);
    kern<<<grid, 256, n * sizeof(int16_t), s>>>(
        xt, v, n, n1, orders, perm_list ? perm_list + base : nullptr, base, two_sided,
        t_out ? t_out + base * ld : nullptr, ld, part_val ? part_val + base * nvb : nullptr,
        part_idx ? part_idx + base * nvb : nullptr, counters);
  }
  return cudaGetLastError();
}

cudaError_t launch_exact_reduce(const double* part_val, const int32_t* part_idx, int nvb,
                                const int32_t* perm_list, int64_t nperm, double* max_out,
                                int32_t* argmax_out, cudaStream_t s) {
  if (nperm <= 0) return cudaSuccess;
  const int wpb = 8;
  k_exact_reduce<<<(unsigned)((nperm + wpb - 1) / wpb), 32 * wpb, 0, s>>>(
      part_val, part_idx, nvb, perm_list, nperm, max_out, argmax_out);
  return cudaGetLastError();
}

cudaError_t launch_pairs(const double* x, int64_t v, int n, int n1, const int16_t* orders,
                         const int32_t* pairs, int64_t npairs, double* t_out, double* num_out,
                         int32_t* deg_out, cudaStream_t s) {
  if (npairs <= 0) return cudaSuccess;
  k_pairs<<<(unsigned)((npairs + 127) / 128), 128, 0, s>>>(x, v, n, n1, orders, pairs, npairs,
                                                          t_out, num_out, deg_out);
  return cudaGetLastError();
}

}  // namespace rmx
