// gram_tc.cu -- K3a on the tensor cores: the batched gathered Gram of
// RapidPT recovery (reference lrmc.py:136-137, solve_block's
// `u_stack.T @ u_stack` and `u_stack.T @ values`) as tcgen05 MMAs.
//
// Per system b (one recovered permutation): A_b = [U[idx_b] | t_b] (k x
// (r+1)), G_b = A_b^T A_b.  U is held as two fp16 planes (U 2^14 = hi + lo,
// |lo| <= 2^-11 |hi|); t_b is split the same way with a per-system power-of-2
// scale.  G~ = hi^T hi + hi^T lo + lo^T hi in fp32 TMEM accumulators: about
// fp32 accuracy, which iterative refinement (lsq_resid: the fp64 residual
// U^T (t - U w) from one gather of the fp64 rows, then a solve with the
// factor already computed) lifts to the fp64 normal-equations solution.
//
// Layout.  The gathered rows are the K dimension of both operands, so the
// tiles are MN-major (idesc bits 15/16): one Omega row contributes 16-byte
// pieces of 8 consecutive basis columns, which land as rows of 128-byte core
// matrices (8 K rows x 8 columns) -- a plain cp.async of the global row, no
// transpose.  Core matrices: K-groups at LBO = 128 B, 8-column groups at
// SBO = BK * 16 B.
//
// Work split.  G is symmetric, so only the upper block triangle is formed:
// 128-row strips m = 0.. of A^T (rows = basis columns 128 m ..), each times
// the columns [128 m, rp).  t sits at Gram index rt = round_up(r, 8), so the
// 16-byte piece that carries it holds no U column and is built in registers
// (rp = rt + 1 rounded up to 32; the epilogue maps rt back to index r).  Strips are packed
// into jobs whose TMEM columns sum(rp - 128 m) fit the 512-column
// accumulator; one CTA runs one (system, job) unit at a time (persistent
// grid).  Roles: warp 0 allocates TMEM and issues the MMAs (one thread),
// warps 4-7 drain the accumulator (TMEM lane quadrants 0-3) into G (fp64,
// written transposed so that each warp store is one coalesced row segment of
// G's lower triangle), warps 8-11 gather rows with cp.async into a
// kGStages-deep ring (the unit's row ids and t halves staged in smem first).
#include <cuda_fp16.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "rapid_internal.cuh"
#include "sm100.cuh"

namespace rmx {
namespace {

constexpr int kGBK = 16;        // gathered rows per ring stage (one MMA K step)
constexpr int kGStages = 7;     // ring depth
constexpr int kGLag = 5;        // stages a producer keeps in flight before publishing
constexpr int kGProd = 128;     // producer threads (warps 8-11)
constexpr int kGThreadsTc = 384;
constexpr int kGMaxJobs = 4;
constexpr float kGUScale = 16384.0f;  // U planes hold U 2^14 (|U| <= 1)

struct GramTcArgs {
  const __half* planes;  // [2][v][kpg]: hi, lo of U 2^14; columns >= r are 0
  int64_t v;
  int r, kpg, rp;         // rp = round_up(rt + 1, 32) = kpg
  int rt;                 // Gram index of t: round_up(r, 8) (its 8-column piece holds no U)
  const int32_t* idx;     // [B][k]
  int k;
  const double* vals;     // [B][k]
  void* G;                // [B][(r+1)^2], lower triangle written (fp64 or fp32)
  int g_f32;
  int64_t B;
  int njobs;
  int job_s0[kGMaxJobs], job_s1[kGMaxJobs];
  int stage_mn;           // columns per stage plane (>= every job's extent)
  uint32_t stage_off;     // byte offset of the per-unit staging (row ids, t halves)
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void cp_async16_cg_u32(uint32_t smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gsrc) : "memory");
}

// power-of-2 scale bringing max |t| into [2^14, 2^15)
__device__ __forceinline__ double t_scale(double m) {
  if (!(m > 0.0)) return 1.0;
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return ldexp(1.0, 15 - e);
}

__device__ __forceinline__ double block_absmax_t(const double* t, int k, int tid, int nthr,
                                                 double* red, int bar_id) {
  double m = 0.0;
  for (int i = tid; i < k; i += nthr) m = fmax(m, fabs(t[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int w = tid >> 5;
  if ((tid & 31) == 0) red[w] = m;
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");
  double r = 0.0;
  for (int i = 0; i < nthr / 32; ++i) r = fmax(r, red[i]);
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");  // red reusable
  return r;
}

__global__ void __launch_bounds__(kGThreadsTc, 1) k_gram_tc(const __grid_constant__ GramTcArgs a) {
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) &
                                           ~uintptr_t(1023));
  const uint32_t plane_bytes = (uint32_t)kGBK * a.stage_mn * 2;
  const uint32_t stage_bytes = 2 * plane_bytes;
  uint8_t* stages = sm;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kGStages * stage_bytes);
  uint64_t* empty = full + kGStages;
  uint64_t* tfull = empty + kGStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  double* red = reinterpret_cast<double*>(tmem_slot + 4);  // 2 x 4 doubles
  int32_t* sidx = reinterpret_cast<int32_t*>(sm + a.stage_off);  // unit's row ids [k]
  __half2* st2 = reinterpret_cast<__half2*>(sidx + ((a.k + 3) & ~3));  // (t hi, t lo) [k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t SBO = kGBK * 16u, LBO = 128u;

  // zero the ring once: columns a job does not gather stay finite (zero)
  for (uint32_t i = threadIdx.x * 16; i < kGStages * stage_bytes; i += kGThreadsTc * 16)
    *reinterpret_cast<uint4*>(stages + i) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], kGProd);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t nunits = a.B * a.njobs;
  const int nst = (a.k + kGBK - 1) / kGBK;  // ring stages per unit
  const int ld = a.r + 1;

  if (warp == 0) {
    // ---------------------------------------------------------- MMA issuer
    int64_t g = 0;  // global stage sequence number
    uint32_t acc_phase = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int job = (int)(u % a.njobs);
      const int s0 = a.job_s0[job], s1 = a.job_s1[job];
      const int col0 = 128 * s0;
      mbar_wait(tempty, acc_phase ^ 1);
      tc_fence_after();
      for (int c = 0; c < nst; ++c, ++g) {
        const int st = (int)(g % kGStages);
        mbar_wait(&full[st], (uint32_t)((g / kGStages) & 1));
        tc_fence_after();
        if (elect_one()) {
          const uint32_t hi = smem_u32(stages + st * stage_bytes), lo = hi + plane_bytes;
#pragma unroll
          for (int ks = 0; ks < kGBK / 16; ++ks) {
            const uint32_t koff = ks * 2 * LBO;  // 16 K rows = 2 core-matrix groups
            uint32_t tcol = 0;
            for (int m = s0; m < s1; ++m) {
              const uint32_t aoff = (uint32_t)((128 * m - col0) / 8) * SBO + koff;
              const uint64_t ahi = smem_desc(hi + aoff, LBO, SBO, 0);
              const uint64_t alo = smem_desc(lo + aoff, LBO, SBO, 0);
              for (int nc = 128 * m; nc < a.rp; nc += 256) {
                const int N = min(256, a.rp - nc);
                const uint32_t idesc = idesc_f16_f32(128, N) | (1u << 15) | (1u << 16);
                const uint32_t boff = (uint32_t)((nc - col0) / 8) * SBO + koff;
                const uint64_t bhi = smem_desc(hi + boff, LBO, SBO, 0);
                const uint64_t blo = smem_desc(lo + boff, LBO, SBO, 0);
                const uint32_t d = tmem + tcol + (uint32_t)(nc - 128 * m);
                const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
                mma_f16_ss(d, ahi, bhi, idesc, acc);
                mma_f16_ss(d, ahi, blo, idesc, 1u);
                mma_f16_ss(d, alo, bhi, idesc, 1u);
              }
              tcol += (uint32_t)(a.rp - 128 * m);
            }
          }
          mma_commit(&empty[st]);
          if (c == nst - 1) mma_commit(tfull);
        }
        __syncwarp();
      }
      acc_phase ^= 1;
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------------- producers
    // per unit: the row ids and the scaled t halves are staged in shared
    // memory once, so a piece costs one smem read + two cp.async (no
    // dependent global load per piece); warp pw gathers rows pw, pw + 4, ..
    // of each stage, lanes over the row's 16-byte pieces (coalesced)
    const int ptid = threadIdx.x - 256, pw = ptid >> 5;
    int64_t g = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t b = u / a.njobs;
      const int job = (int)(u % a.njobs);
      const int col0 = 128 * a.job_s0[job];
      const int ppr = (a.rp - col0) / 8;  // 16-byte pieces per gathered row
      const int tq = (a.rt - col0) / 8;   // the piece holding t (no U columns)
      const int32_t* ib = a.idx + b * a.k;
      const double* tb = a.vals + b * a.k;
      // every producer is done issuing the previous unit (staging reusable)
      asm volatile("bar.sync 1, %0;" ::"n"(kGProd) : "memory");
      const double tsc = t_scale(block_absmax_t(tb, a.k, ptid, kGProd, red, 1));
      for (int i = ptid; i < a.k; i += kGProd) {
        sidx[i] = ib[i];
        const double x = tb[i] * tsc;
        const __half th = __double2half(x);
        st2[i] = __halves2half2(th, __double2half(x - (double)__half2float(th)));
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kGProd) : "memory");
      for (int c = 0; c < nst; ++c, ++g) {
        const int st = (int)(g % kGStages);
        mbar_wait(&empty[st], (uint32_t)(((g / kGStages) & 1) ^ 1));
        const uint32_t hi = smem_u32(stages + st * stage_bytes), lo = hi + plane_bytes;
        const int kk0 = c * kGBK;
        for (int kr = pw; kr < kGBK; kr += kGProd / 32) {
          const int kk = kk0 + kr;
          const uint32_t roff = (uint32_t)(kr >> 3) * LBO + (kr & 7) * 16u;
          if (kk < a.k) {
            const __half* ph = a.planes + (int64_t)sidx[kk] * a.kpg + col0;
            for (int q = lane; q < ppr; q += 32) {
              const uint32_t off = (uint32_t)q * SBO + roff;
              if (q == tq) {  // [t, 0, .., 0]
                const __half2 t2 = st2[kk];
                st_shared_v4(hi + off, make_uint4(__half_as_ushort(__low2half(t2)), 0, 0, 0));
                st_shared_v4(lo + off, make_uint4(__half_as_ushort(__high2half(t2)), 0, 0, 0));
              } else {
                cp_async16_cg_u32(hi + off, ph + 8 * q);
                cp_async16_cg_u32(lo + off, ph + a.v * a.kpg + 8 * q);
              }
            }
          } else {  // rows past k: zero
            for (int q = lane; q < ppr; q += 32) {
              st_shared_v4(hi + (uint32_t)q * SBO + roff, make_uint4(0, 0, 0, 0));
              st_shared_v4(lo + (uint32_t)q * SBO + roff, make_uint4(0, 0, 0, 0));
            }
          }
        }
        cp_async_commit();
        if (g >= kGLag) {  // publish stage g - kGLag once its copies landed
          asm volatile("cp.async.wait_group %0;" ::"n"(kGLag) : "memory");
          fence_proxy_async_smem();
          mbar_arrive(&full[(g - kGLag) % kGStages]);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async_smem();
    for (int64_t q = std::max<int64_t>(0, g - kGLag); q < g; ++q) mbar_arrive(&full[q % kGStages]);
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue
    const int quad = warp - 4;  // TMEM lanes 32 quad .. 32 quad + 31
    const int etid = threadIdx.x - 128;
    uint32_t acc_phase = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t b = u / a.njobs;
      const int job = (int)(u % a.njobs);
      const int s0 = a.job_s0[job], s1 = a.job_s1[job];
      const double tsc = t_scale(block_absmax_t(a.vals + b * a.k, a.k, etid, 128, red + 4, 2));
      const double duu = 1.0 / ((double)kGUScale * kGUScale);
      const double dut = 1.0 / ((double)kGUScale * tsc), dtt = 1.0 / (tsc * tsc);
      double* Gb = static_cast<double*>(a.G) + b * (int64_t)ld * ld;
      float* Gf = static_cast<float*>(a.G) + b * (int64_t)ld * ld;
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
      uint32_t tcol = 0;
      for (int m = s0; m < s1; ++m) {
        // this thread's row of G~: a basis column (< r) or t (rt -> index r)
        const int gi = 128 * m + 32 * quad + lane;
        const bool irow = gi < a.r || gi == a.rt;
        const int i = gi == a.rt ? a.r : gi;
        for (int j0 = 128 * m; j0 < a.rp; j0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(32 * quad) << 16) + tcol + (uint32_t)(j0 - 128 * m), v);
          tmem_ld_wait();
          if (irow) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const int gj = j0 + jj;
              if (gj >= gi && (gj < a.r || gj == a.rt)) {
                const int j = gj == a.rt ? a.r : gj;
                const double sc = (j == a.r) ? (i == a.r ? dtt : dut) : duu;
                const double gv = (double)__uint_as_float(v[jj]) * sc;
                if (a.g_f32) Gf[(int64_t)j * ld + i] = (float)gv;
                else Gb[(int64_t)j * ld + i] = gv;
              }
            }
          }
        }
        tcol += (uint32_t)(a.rp - 128 * m);
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// U (fp64, v x r, row stride ldu) -> [2][v][kpg] fp16 planes of U 2^14
__global__ void k_gram_planes(const double* __restrict__ U, int64_t ldu, int64_t v, int r,
                              int kpg, __half* __restrict__ planes) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v * kpg) return;
  const int64_t j = e / kpg;
  const int c = (int)(e - j * kpg);
  const double x = c < r ? U[j * ldu + c] * (double)kGUScale : 0.0;
  const __half h = __double2half(x);
  planes[e] = h;
  planes[v * kpg + e] = __double2half(x - (double)__half2float(h));
}

// g_b = U_b^T (t_b - U_b w_b), U_b = U[idx_b] (fp64).  One CTA per system,
// warp per gathered row: the row is loaded once (lane-strided, coalesced),
// e = t - u.w by a warp reduction, then g += e u in registers; the warps'
// partial g are summed in shared memory.
constexpr int kRWarps = 8;
template <int RL>  // r <= 32 RL
__global__ void __launch_bounds__(32 * kRWarps, 2) k_lsq_resid(const double* __restrict__ U,
                                                            int64_t ldu, int r,
                                                            const int32_t* __restrict__ idx,
                                                            int k, const double* __restrict__ vals,
                                                            const double* __restrict__ W,
                                                            double* __restrict__ gout,
                                                            const int32_t* __restrict__ active) {
  extern __shared__ double rsm[];  // w[r] | part[kRWarps][r]
  double* w = rsm;
  double* part = rsm + r;
  const int64_t b = blockIdx.x;
  if (active && active[b] == 0) return;  // settled system: no refinement step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < r; i += blockDim.x) w[i] = W[b * r + i];
  __syncthreads();
  double wr[RL], acc[RL];
#pragma unroll
  for (int q = 0; q < RL; ++q) {
    const int c = lane + 32 * q;
    wr[q] = c < r ? w[c] : 0.0;
    acc[q] = 0.0;
  }
  const int32_t* ib = idx + b * k;
  const double* tb = vals + b * k;
  // two rows per warp iteration: both rows' loads are in flight together and
  // their dot-product butterflies interleave (the per-row arithmetic and its
  // order are unchanged: same bits)
  int kk = warp;
  for (; kk + kRWarps < k; kk += 2 * kRWarps) {
    const double* urow1 = U + (int64_t)ib[kk] * ldu;
    const double* urow2 = U + (int64_t)ib[kk + kRWarps] * ldu;
    double u1[RL], u2[RL];
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      const int c = lane + 32 * q;
      u1[q] = c < r ? __ldg(urow1 + c) : 0.0;
      u2[q] = c < r ? __ldg(urow2 + c) : 0.0;
    }
    double dot1 = 0.0, dot2 = 0.0;
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      dot1 = fma(u1[q], wr[q], dot1);
      dot2 = fma(u2[q], wr[q], dot2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dot1 += __shfl_xor_sync(0xffffffffu, dot1, o);
      dot2 += __shfl_xor_sync(0xffffffffu, dot2, o);
    }
    const double e1 = tb[kk] - dot1, e2 = tb[kk + kRWarps] - dot2;
#pragma unroll
    for (int q = 0; q < RL; ++q) acc[q] = fma(e2, u2[q], fma(e1, u1[q], acc[q]));
  }
  for (; kk < k; kk += kRWarps) {
    const double* urow = U + (int64_t)ib[kk] * ldu;
    double u[RL];
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      const int c = lane + 32 * q;
      u[q] = c < r ? __ldg(urow + c) : 0.0;
      dot = fma(u[q], wr[q], dot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const double e = tb[kk] - dot;
#pragma unroll
    for (int q = 0; q < RL; ++q) acc[q] = fma(e, u[q], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < RL; ++q) {
    const int c = lane + 32 * q;
    if (c < r) part[warp * r + c] = acc[q];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    double sacc = 0.0;
    for (int q = 0; q < kRWarps; ++q) sacc += part[q * r + c];
    gout[b * r + c] = sacc;
  }
}

}  // namespace

static int gram_tc_rt(int r) { return (r + 7) / 8 * 8; }
int gram_tc_kpg(int r) { return (gram_tc_rt(r) + 1 + 31) / 32 * 32; }

// strips of 128 basis columns, packed into jobs of <= 512 TMEM columns
static int gram_tc_jobs(int rp, int* s0, int* s1) {
  const int strips = (rp + 127) / 128;
  int nj = 0, cur = 0, used = 0;
  for (int m = 0; m < strips; ++m) {
    const int cols = rp - 128 * m;
    if (used > 0 && used + cols > 512) {
      s0[nj] = cur;
      s1[nj] = m;
      ++nj;
      cur = m;
      used = 0;
    }
    used += cols;
  }
  s0[nj] = cur;
  s1[nj] = strips;
  return nj + 1;
}

bool gram_tc_supported(int r, int k) {
  if (r < 16 || k < 16 || gram_tc_kpg(r) > 512) return false;
  int s0[8], s1[8];
  return gram_tc_jobs(gram_tc_kpg(r), s0, s1) <= kGMaxJobs;
}

cudaError_t launch_gram_planes(const double* U, int64_t ldu, int64_t v, int r, __half* planes,
                               cudaStream_t s) {
  const int kpg = gram_tc_kpg(r);
  const int64_t n = v * kpg;
  k_gram_planes<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(U, ldu, v, r, kpg, planes);
  return cudaGetLastError();
}

cudaError_t launch_gram_tc(const __half* planes, int64_t v, int r, const int32_t* idx, int k,
                           const double* vals, void* G, int g_f32, int64_t B, int sm_count,
                           cudaStream_t s) {
  GramTcArgs a{};
  a.planes = planes;
  a.v = v;
  a.r = r;
  a.kpg = gram_tc_kpg(r);
  a.rp = a.kpg;
  a.idx = idx;
  a.k = k;
  a.vals = vals;
  a.G = G;
  a.g_f32 = g_f32;
  a.B = B;
  int s0[8], s1[8];
  a.njobs = gram_tc_jobs(a.rp, s0, s1);
  if (a.njobs > kGMaxJobs) return cudaErrorInvalidValue;
  int mn = 0;
  for (int j = 0; j < a.njobs; ++j) {
    a.job_s0[j] = s0[j];
    a.job_s1[j] = s1[j];
    mn = std::max(mn, std::max(a.rp - 128 * s0[j], 128 * (s1[j] - s0[j])));
  }
  a.stage_mn = mn;
  a.rt = gram_tc_rt(r);
  a.stage_off = (uint32_t)((size_t)kGStages * 2 * kGBK * mn * 2 + 256);
  const size_t smem = 1024 + a.stage_off + (size_t)((k + 3) & ~3) * 4 + (size_t)k * 4;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_gram_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t units = B * a.njobs;
  const unsigned grid = (unsigned)std::min<int64_t>(units, sm_count > 0 ? sm_count : 148);
  k_gram_tc<<<grid, kGThreadsTc, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lsq_resid(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                             const double* vals, const double* W, int64_t B, double* g,
                             cudaStream_t s, const int32_t* active) {
  const size_t smem = (size_t)(1 + kRWarps) * r * sizeof(double);
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    for (int64_t b0 = 0; b0 < B; b0 += 65535) {
      const int64_t cnt = std::min<int64_t>(65535, B - b0);
      kern<<<(unsigned)cnt, 32 * kRWarps, smem, s>>>(U, ldu, r, idx + b0 * k, k, vals + b0 * k,
                                                      W + b0 * r, g + b0 * r,
                                                      active ? active + b0 : nullptr);
    }
    return cudaGetLastError();
  };
  if (r <= 128) return go(k_lsq_resid<4>);
  if (r <= 256) return go(k_lsq_resid<8>);
  if (r <= 416) return go(k_lsq_resid<13>);
  if (r <= 512) return go(k_lsq_resid<16>);
  return cudaErrorInvalidValue;
}

}  // namespace rmx
