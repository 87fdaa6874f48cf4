// tfill_tc.cu -- K1: the NaivePT permutation-matrix fill on tcgen05 tensor cores.
//
// Replaces the reference's per-permutation loop (naive.py:49-57):
//     x1, x2 = x.group_blocks(plan.shuffle(i))      # model.py:65-69
//     col    = tstat_full(x1, x2)                   # teststat.py:28-61
//     out[i] = column_max(col, two_sided)           # teststat.py:88-90
// for all permutations at once.  With per-voxel standardisation z (K0, fp64;
// t is invariant to a per-voxel affine map) the statistic only needs
//     S1 = sum_{j in G1} z_j,   Q1 = sum_{j in G1} z_j^2
// and for all (perm, voxel) pairs that is the contraction
//     [S1 | Q1] (L x 2v) = G (L x n, 0/1 indicator) . [Z | Z^2] (n x 2v).
// Z and Z^2 are split into fp16 hi + lo planes (residual <= 2^-22 |z|), G is
// exact in fp16, and D += G.B_hi + G.B_lo accumulates in fp32 TMEM.
//
// Tile: M = 128 permutations (TMEM lanes), N = 256 = 128 voxels x {S, Q},
// K = subjects.  Persistent CTAs, one per SM, warp-specialised:
//   warp 0     TMA producer: B tiles (hi and lo boxes) into a STAGES-deep ring
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..  epilogue: tcgen05.ld S,Q -> t~ (division-free compare) ->
//              per-permutation top-4 over the unit's voxel chunk; also build
//              the A tile (G, fp16 0/1) in smem once per unit.
// Two TMEM accumulators (2 x 256 columns) let the epilogue of tile t overlap
// the MMAs of tile t+1.  T never leaves the chip; the only outputs are the
// per-(perm, chunk) top-4 candidates refined in fp64 by K2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <mutex>

#include "philox.cuh"
#include "rmx_internal.cuh"
#include "sm100.cuh"

namespace rmx {

namespace {

constexpr int kNumAcc = 2;
constexpr int kTileN = 2 * kTileV;

// Running top-4 (key, voxel) per permutation row; keys are sign(t) t^2
// (two-sided: t^2).  The common path is one compare against the 4th best
// (u > K3 * d, division-free); only entries entering the top-4 divide.
struct Top4 {
  float k0, k1, k2, k3;
  int j0, j1, j2, j3;
  // Entries below `floor` can never be refinement candidates (see seed_key),
  // so the threshold starts there; unfilled slots keep voxel -1.
  __device__ __forceinline__ void reset(float floor) {
    k0 = k1 = k2 = k3 = floor;
    j0 = j1 = j2 = j3 = -1;
  }
  __device__ __forceinline__ void insert(float key, int j) {
    if (!(key > k3)) return;
    if (key > k1) {
      k3 = k2; j3 = j2;
      k2 = k1; j2 = j1;
      if (key > k0) {
        k1 = k0; j1 = j0;
        k0 = key; j0 = j;
      } else {
        k1 = key; j1 = j;
      }
    } else if (key > k2) {
      k3 = k2; j3 = j2;
      k2 = key; j2 = j;
    } else {
      k3 = key; j3 = j;
    }
  }
};

template <bool TWO_SIDED>
__device__ __forceinline__ void stat_ud(uint32_t sbits, uint32_t qbits, float alpha, float beta,
                                        float gamma, float& u, float& d) {
  const float S = __uint_as_float(sbits);
  const float Q = __uint_as_float(qbits);
  // u = sign(t) t^2 d (two-sided: t^2 d); d = var_term * (n1 n2 / n)^2
  u = TWO_SIDED ? S * S : S * fabsf(S);
  d = fmaf(beta, fabsf(u), fmaf(alpha, Q, gamma));
}

__device__ __forceinline__ uint64_t pack2(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

struct EpiConst {
  uint64_t alpha2, beta2, gamma2;  // packed (x, x)
  float alpha, beta, gamma, dthr;
  float sdeg;  // S-only signed tiles: |S| beyond which d~ may fall below dthr (suspects)
};

// Common path over 32 columns (voxels jbase..jbase+31) of one accumulator
// row, packed f32x2 over column pairs, branch-free:
//     m = S^2 - k3 * d      (d = alpha Q + beta S^2 + gamma)
// m > 0 <=> |t| beats the row's 4th-best key k3 (two-sided exactly; signed:
// a superset, negative t included).  A degenerate voxel (d ~ 0) has S^2 at
// its maximum, so m > 0 there too.  Returns the per-column hit mask, built by
// funnel-shifting the sign bits of m (one SHF per column).
template <bool ALPHA0>
__device__ __forceinline__ uint32_t group_hits(const uint32_t (&s)[32], const uint32_t (&q)[32],
                                               const EpiConst& ec, float k3) {
  // k3 < 0 (signed, fewer than 4 non-negative keys yet): test against 0, so
  // every column hits (superset) and a negative d~ can never hide a suspect
  const float k3h = fmaxf(k3, 0.0f);
  const uint64_t nk3 = pack2(__float_as_uint(-k3h), __float_as_uint(-k3h));
  uint32_t neg = 0;
#pragma unroll
  for (int c = 30; c >= 0; c -= 2) {
    const uint64_t S2 = pack2(s[c], s[c + 1]);
    const uint64_t sq = mul2(S2, S2);
    uint64_t d;
    if (ALPHA0) {
      d = fma2(ec.beta2, sq, ec.gamma2);
    } else {
      d = fma2(ec.alpha2, pack2(q[c], q[c + 1]), ec.gamma2);
      d = fma2(ec.beta2, sq, d);
    }
    const uint64_t m = fma2(nk3, d, sq);
    neg = __funnelshift_l((uint32_t)(m >> 32), neg, 1);  // column c+1
    neg = __funnelshift_l((uint32_t)m, neg, 1);          // column c
  }
  return ~neg;
}

// S-only tiles (alpha = 0): d = beta S^2 + gamma with beta < 0, so
//     m > 0  <=>  S^2 > K,   K = k3' gamma / (1 - k3' beta),  k3' = max(k3, 0)
// (denominator >= 1).  The common path is one packed FMA per column pair
// (S^2 - K) and a 3-input AND of the sign bits: "could any column hit".  A
// degenerate or negative-d~ column has S^2 >= gamma / |beta| > K: always hits.
__device__ __forceinline__ float sonly_thr(float k3, const EpiConst& ec) {
  const float k = fmaxf(k3, 0.0f);
  return k * ec.gamma / fmaf(-k, ec.beta, 1.0f);
}
// Signed (one-sided) S-only tiles, hit mask (only for groups whose S^2 test
// fired): a column can matter only if S > sqrt(K) (t above the row's
// threshold) or S < -sdeg (near-zero d~: a suspected degenerate voxel,
// listed whatever its sign).  The S^2 test alone would also send every
// strongly negative t of the row through the rare path (half of the rare
// groups at config 4).
// K == 0 (the row's top-4 not yet full of non-negative keys): every column.
__device__ __forceinline__ float sonly_signed_thr(float K, const EpiConst& ec) {
  return K > 0.0f ? fminf(sqrtf(K) * (1.0f - 1e-6f), ec.sdeg) : -FLT_MAX;
}

// Common path: S^2 > K, one packed FMA per column pair (for signed tiles a
// superset that also admits strongly negative t; sonly_mask then sorts them
// out before the rare path).
__device__ __forceinline__ bool sonly_any(const uint32_t (&s)[32], float K) {
  const uint64_t nk = pack2(__float_as_uint(-K), __float_as_uint(-K));
  uint32_t all = 0xffffffffu;
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    const uint64_t S2 = pack2(s[c], s[c + 1]);
    const uint64_t m = fma2(S2, S2, nk);
    all &= (uint32_t)m & (uint32_t)(m >> 32);
  }
  return (int)all >= 0;  // some sign bit clear
}
template <bool TWO_SIDED>
__device__ __forceinline__ uint32_t sonly_mask(const uint32_t (&s)[32], float K,
                                               const EpiConst& ec) {
  uint32_t neg = 0;
  if constexpr (TWO_SIDED) {
    const uint64_t nk = pack2(__float_as_uint(-K), __float_as_uint(-K));
#pragma unroll
    for (int c = 30; c >= 0; c -= 2) {
      const uint64_t S2 = pack2(s[c], s[c + 1]);
      const uint64_t m = fma2(S2, S2, nk);
      neg = __funnelshift_l((uint32_t)(m >> 32), neg, 1);
      neg = __funnelshift_l((uint32_t)m, neg, 1);
    }
  } else {
    const float thr = sonly_signed_thr(K, ec);
    const uint64_t one = pack2(__float_as_uint(1.0f), __float_as_uint(1.0f));
    const uint64_t mone = pack2(__float_as_uint(-1.0f), __float_as_uint(-1.0f));
    const uint64_t nt = pack2(__float_as_uint(-thr), __float_as_uint(-thr));
    const uint64_t nd = pack2(__float_as_uint(-ec.sdeg), __float_as_uint(-ec.sdeg));
#pragma unroll
    for (int c = 30; c >= 0; c -= 2) {
      const uint64_t S2 = pack2(s[c], s[c + 1]);
      const uint64_t m = fma2(S2, one, nt) & fma2(S2, mone, nd);
      neg = __funnelshift_l((uint32_t)(m >> 32), neg, 1);
      neg = __funnelshift_l((uint32_t)m, neg, 1);
    }
  }
  return ~neg;
}

// Rare path: the warp walks the union of its lanes' hit columns (uniform
// loop); each column is re-read from TMEM (dynamic column = address, so no
// register-array indexing) and every lane that flagged it re-tests exactly:
// suspect listing for near-zero variance, else top-4 insertion.  (Batching
// all union loads behind one wait measured slower: the typical union is 1-3
// columns and the unrolled batch costs registers.)
// I8 tiles: exact integer accumulator S_q -> fp32 S with the voxel's
// dequantisation scale.
__device__ __forceinline__ uint32_t i8_to_s(uint32_t sq, float inv) {
  return __float_as_uint((float)(int)sq * inv);
}

template <bool TWO_SIDED, bool SONLY, bool I8>
__device__ __forceinline__ void group_rare(uint32_t hits, uint32_t taddr_s, int jbase,
                                           const EpiConst& ec, Top4& top, int64_t p, bool prow,
                                           const TfillArgs& a, const float* ginv,
                                           float kfloor = -FLT_MAX) {
  uint32_t uni = __reduce_or_sync(0xffffffffu, hits);
  while (uni) {
    const int c = __ffs(uni) - 1;
    uni &= uni - 1;
    uint32_t sb, qb = 0u;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(sb) : "r"(taddr_s + c));
    if (!SONLY)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                   : "=r"(qb)
                   : "r"(taddr_s + kTileV + c));
    tmem_ld_wait();
    if (I8) sb = i8_to_s(sb, ginv[c]);
    if ((hits >> c) & 1u) {
      float u, d;
      stat_ud<TWO_SIDED>(sb, qb, ec.alpha, ec.beta, ec.gamma, u, d);
      const int j = jbase + c;
      if (d < ec.dthr) {
        // near-zero pooled variance: exact fp64 re-evaluation in K2
        if (prow) {
          unsigned slot = atomicAdd(&a.counters->susp_count, 1u);
          if (slot < (unsigned)kSuspectCap) {
            a.susp[2 * slot] = (int)p;
            a.susp[2 * slot + 1] = j;
          }
        }
      } else if (u > fmaxf(top.k3, kfloor) * d) {
        top.insert(u / d, j);
      }
    }
  }
}

template <bool TWO_SIDED>
__device__ __forceinline__ void group_debug(const uint32_t (&s)[32], const uint32_t (&q)[32],
                                            int jbase, int valid, const EpiConst& ec, int64_t p,
                                            bool prow, const TfillArgs& a) {
  if (!prow) return;
  for (int c = 0; c < 32 && c < valid; ++c) {
    float u, d;
    stat_ud<TWO_SIDED>(s[c], q[c], ec.alpha, ec.beta, ec.gamma, u, d);
    a.dbg_t[p * a.v + jbase + c] =
        (d < ec.dthr) ? __int_as_float(0x7fc00000) : copysignf(sqrtf(fabsf(u) / d), u);
  }
}

// i-th tile of a unit's chunk in a low-discrepancy (golden-ratio stride)
// order: every permutation's top-4 threshold is close to final after the
// first few percent of the sweep, which keeps the epilogue's rare path rare.
__device__ __forceinline__ int chunk_tile(const TfillArgs& a, int chunk, int t0, int t1, int i) {
  const int T = t1 - t0;
  const int stride = chunk < a.n_ramp ? a.ramp_stride[chunk]
                                      : ((T == a.tiles_per_chunk) ? a.stride_full : a.stride_last);
  return t0 + (int)(((int64_t)i * stride) % T);
}

// Voxel-tile range [t0, t1) of a chunk.
__device__ __forceinline__ void chunk_range(const TfillArgs& a, int chunk, int& t0, int& t1) {
  chunk_tiles(a.n_ramp, a.ramp_start, a.tiles_per_chunk, a.n_vtiles, chunk, &t0, &t1);
}

__device__ __forceinline__ float key_to_t(float key) { return copysignf(sqrtf(fabsf(key)), key); }

// Order-preserving float <-> uint32 map for atomicMax; 0 = "no value yet".
__device__ __forceinline__ uint32_t ord_enc(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord_dec(uint32_t e) {
  return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}

// Threshold seed from the permutation's best t~ over chunks finished so far
// (best_t, written by earlier units).  K2 refines exactly the voxels with
// t~ >= t~max - band(t~max), and t~max >= seed, so nothing below
// seed - 2 band(seed) can matter: starting the top-4 there is exact and
// keeps the epilogue's rare path rare.
template <bool TWO_SIDED>
__device__ __forceinline__ float seed_key(const uint32_t* best_t, int64_t p, bool prow,
                                          const TfillArgs& a, float emax) {
  if (!prow) return -FLT_MAX;
  const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(best_t + p);
  if (e == 0u) return -FLT_MAX;
  const float t = ord_dec(e);
  const float band = band_abs(t, a.band_rel, emax, a.beta_abs, a.gamma);
  if (!(band < 1e30f)) return -FLT_MAX;
  const float lo = t - 2.0f * band;
  if (TWO_SIDED) return lo > 0.0f ? lo * lo : 0.0f;
  return lo * fabsf(lo);
}

// The same floor for a running best t (shared across the CTA's epilogue
// groups within a unit, see the epilogue): nothing below t - 2 band(t) can
// become a refinement candidate.
template <bool TWO_SIDED>
__device__ __forceinline__ float floor_key(float t, const TfillArgs& a, float emax) {
  const float band = band_abs_fast(t, a.band_rel, emax, a.beta_abs, a.gamma);
  if (!(band < 1e30f)) return -FLT_MAX;
  const float lo = t - 2.0f * band;
  if (TWO_SIDED) return lo > 0.0f ? lo * lo : 0.0f;
  return lo * fabsf(lo);
}

// CG = 1: one CTA computes a 128-permutation x 128-voxel tile (M = 128).
// CG = 2: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a
//   256 x 128 tile with M = 256 MMAs issued by the leader CTA: each CTA holds
//   its own 128-permutation A tile and loads HALF of every B tile (rank 0 the
//   Z planes, rank 1 the Z^2 planes), so per-SM B traffic halves and the
//   smem ring gets ~2x deeper.  Each CTA's TMEM receives its own 128 rows x
//   256 columns, so the epilogue is identical.
// ALPHA0 (n1 == n2): the pooled variance no longer depends on Q, so the tile
// holds S only for 256 voxels (N = 256 columns of Z): half the MMA work per
// T entry of the general (S | Q) tile.
//
// I8 (balanced groups): exact integer MMA (kind::i8, u8 A x s8 B -> s32).  Z
// is quantised per voxel to zq = rint(z * scale) in [-32512, 32512] and split
// zq = 255 h + l with h, l in [-127, 127] (s8).  B rows hold [h | l] along K
// (K = 2 kpad), A rows [255 G | G] (u8), so one accumulator receives
// S_q = sum_{group 1} zq exactly and S = inv[j] * S_q: the same S-only tile
// (256 voxels) as fp16, at twice the MMA rate and half the operand bytes.
// The refinement band covers the quantisation rigorously (band_abs).
//
// MODE 1 (RapidPT completion, K4): the same fp16 hi/lo S-only pipeline with
// A = the coefficient rows W (fp16, power-of-2 row scales) and B = the basis
// planes [U_hi | U_lo]; the epilogue adds sigma z (Philox, philox.cuh) to the
// completed column and keeps each permutation's running max.
template <int CG, int BK, int STAGES, int EPI_WARPS, bool TWO_SIDED, bool ALPHA0, bool DEBUG,
          bool I8, int MODE>
__global__ void __launch_bounds__(64 + 32 * EPI_WARPS, 1)
    k_tfill_tc(const __grid_constant__ CUtensorMap pmap, const TfillArgs a) {
  static_assert(!I8 || ALPHA0, "int8 tiles are S-only (balanced groups)");
  static_assert(MODE == 0 || (ALPHA0 && !I8 && !DEBUG), "completion tiles are fp16 S-only");
  constexpr int LO_PLANE = MODE == 1 ? 1 : 2;  // plane index of the lo half
  constexpr bool SONLY = ALPHA0;
  constexpr int TV = SONLY ? 2 * kTileV : kTileV;  // voxels per tile
  constexpr int ELT = I8 ? 1 : 2;                   // operand bytes per element
  constexpr int HALF_BYTES = (kTileN / CG) * BK * ELT;  // this CTA's hi (or lo) box
  constexpr int STAGE_BYTES = I8 ? HALF_BYTES : 2 * HALF_BYTES;
  constexpr int KSTEP = I8 ? 32 : 16;  // K per MMA instruction
  constexpr int KSTEPS = BK / KSTEP;
  constexpr int ROW_BYTES = BK * ELT;
  constexpr uint32_t B_LAYOUT = (ROW_BYTES == 128) ? 2u : 4u;  // 128B : 64B swizzle
  constexpr uint32_t B_SBO = (ROW_BYTES == 128) ? 1024u : 512u;
  constexpr int GROUPS = EPI_WARPS / 4;  // epilogue warps sharing a TMEM lane quadrant
  constexpr int COLGROUPS = TV / 32 / GROUPS;
  constexpr uint32_t IDESC =
      I8 ? idesc_u8s8_s32(kTileM * CG, kTileN) : idesc_f16_f32(kTileM * CG, kTileN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_mem = smem;
  uint8_t* a_mem = smem + STAGES * STAGE_BYTES;
  const int kext = I8 ? 2 * a.kpad : a.kpad;  // K extent (elements) of A rows / B rows
  const int a_bytes = kTileM * kext * ELT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(a_mem + a_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + kNumAcc;
  uint64_t* afull = tempty + kNumAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + 1);
  // int8: per-epilogue-warp staging of its columns' dequantisation scales
  float* inv_smem = reinterpret_cast<float*>(a_mem + a_bytes + 256);
  // per-row running best t~ of the unit, shared by the epilogue groups:
  // (unit index << 32) | order-encoded t~ (a new unit supersedes old tags)
  unsigned long long* rowbest =
      reinterpret_cast<unsigned long long*>(a_mem + a_bytes + 256 + (I8 ? kInvStage : 0));

  const int warp = (int)warp_id();
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < kNumAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPI_WARPS * CG);
    }
    mbar_init(afull, kTileM * CG * (MODE == 1 ? 1 : GROUPS));
    fence_mbar_init();
    tma_prefetch(&pmap);
  }
  if (warp == 1) {
    if (CG == 2) tmem_alloc_2sm(tmem_slot, 512);
    else tmem_alloc(tmem_slot, 512);
  }
  for (int i = threadIdx.x; i < kTileM; i += blockDim.x) rowbest[i] = 0ull;
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // units (m-tile, chunk) of chunks [chunk_begin, chunk_end), chunk-major
  const int n_units = a.n_mtiles * a.chunk_end;
  const int unit0 = a.n_mtiles * a.chunk_begin + blockIdx.x / CG, unit_step = gridDim.x / CG;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        const int chunk = u / a.n_mtiles;
        int t0, t1;
        chunk_range(a, chunk, t0, t1);
        for (int i = 0; i < t1 - t0; ++i) {
          const int t = chunk_tile(a, chunk, t0, t1, i);
          for (int kb = 0; kb < kext; kb += BK) {
            uint8_t* dst = stage_mem + stage * STAGE_BYTES;
            if (I8) {  // one box per stage: this CTA's voxels x 128 K-bytes of [h | l]
              if (CG == 2) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
                tma_load_3d_2sm(dst, &pmap, &full[stage], kb, t * TV + (int)rank * kTileV, 0);
              } else {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_expect_tx(&full[stage], STAGE_BYTES);
                tma_load_3d(dst, &pmap, &full[stage], kb, t * TV, 0);
              }
            } else if (CG == 2) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
              if (SONLY) {  // this CTA's 128 of the tile's 256 voxels, Z planes only
                const int v0 = t * TV + (int)rank * kTileV;
                tma_load_3d_2sm(dst, &pmap, &full[stage], kb, v0, 0);  // z_hi
                tma_load_3d_2sm(dst + HALF_BYTES, &pmap, &full[stage], kb, v0, LO_PLANE);  // z_lo
              } else {
                tma_load_3d_2sm(dst, &pmap, &full[stage], kb, t * TV, (int)rank);  // z_hi | q_hi
                tma_load_3d_2sm(dst + HALF_BYTES, &pmap, &full[stage], kb, t * TV,
                                2 + (int)rank);  // z_lo | q_lo
              }
            } else {
              mbar_wait(&empty[stage], phase ^ 1);
              mbar_expect_tx(&full[stage], STAGE_BYTES);
              tma_load_3d(dst, &pmap, &full[stage], kb, t * TV, 0);  // z_hi(, q_hi)
              tma_load_3d(dst + HALF_BYTES, &pmap, &full[stage], kb, t * TV, LO_PLANE);  // z_lo
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (leader) {
      // Descriptors are built once; per MMA only the 14-bit start-address
      // field moves (A: +256 B per K step, B: +32 B per K step within a
      // stage), so the single issuing thread spends ~3 uniform instructions
      // per MMA -- at the int8 rate (128 cycles per M256 N256 K32 MMA) the
      // descriptor arithmetic otherwise throttles the tensor pipe.
      const uint32_t a_sbo = (uint32_t)kext * 8u * ELT;
      const uint64_t adesc0 = smem_desc(smem_u32(a_mem), 128u, a_sbo, 0u);
      const uint64_t bdesc0 = smem_desc(smem_u32(stage_mem), 16u, B_SBO, B_LAYOUT);
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0, a_phase = 0;
      int acc = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        const int chunk = u / a.n_mtiles;
        int t0, t1;
        chunk_range(a, chunk, t0, t1);
        if (CG == 2) mbar_wait_cluster(afull, a_phase);
        else mbar_wait(afull, a_phase);
        a_phase ^= 1;
        tc_fence_after();
        for (int t = t0; t < t1; ++t) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(acc * kTileN);
          for (int kb = 0; kb < kext; kb += BK) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one()) {
              const int ks0 = kb / KSTEP;
              const int nmma = min(KSTEPS, a.nk16 - ks0);  // last stage may be partial
              const uint64_t bst = bdesc0 + (uint64_t)((stage * STAGE_BYTES) >> 4);
              uint64_t adesc = adesc0 + (uint64_t)(ks0 * 16);  // 256 B per K step
#pragma unroll
              for (int s = 0; s < KSTEPS; ++s) {
                if (s < nmma) {
                  const uint32_t accum = (ks0 + s) > 0 ? 1u : 0u;
                  const uint64_t bh = bst + (uint64_t)(s * 2);  // 32 B per K step
                  if (I8) {
                    if (CG == 2) mma_i8_ss_2sm(d_tmem, adesc, bh, IDESC, accum);
                    else mma_i8_ss(d_tmem, adesc, bh, IDESC, accum);
                  } else {
                    const uint64_t bl = bh + (uint64_t)(HALF_BYTES >> 4);
                    if (CG == 2) {
                      mma_f16_ss_2sm(d_tmem, adesc, bh, IDESC, accum);
                      mma_f16_ss_2sm(d_tmem, adesc, bl, IDESC, 1u);
                    } else {
                      mma_f16_ss(d_tmem, adesc, bh, IDESC, accum);
                      mma_f16_ss(d_tmem, adesc, bl, IDESC, 1u);
                    }
                  }
                  adesc += 16u;
                }
              }
              if (CG == 2) {
                mma_commit_2sm(&empty[stage], 0x3);                       // both smem slots free
                if (kb + BK >= kext) mma_commit_2sm(&tfull[acc], 0x3);  // both accumulators
              } else {
                mma_commit(&empty[stage]);
                if (kb + BK >= kext) mma_commit(&tfull[acc]);
              }
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (++acc == kNumAcc) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int quad = warp & 3;  // TMEM lanes [32*quad, 32*quad + 32) are ours
    const int grp = ew / 4;
    const int row = quad * 32 + lane;
    EpiConst ec;
    ec.alpha = a.alpha;
    ec.beta = a.beta;
    ec.gamma = a.gamma;
    ec.dthr = a.dthr;
    // int8: quantisation error bound (K0); a truly degenerate voxel
    // (|S| = sqrt(gamma/|beta|)) then has d~ <= 2 |beta| sqrt(gamma/|beta|) e
    // fp16 S-only: the a priori bound on |S~ - S| (rmx_abi.cu fp16_sonly_error_bound)
    constexpr bool EBOUND = MODE == 0 && (I8 || SONLY);
    const float emax = EBOUND ? __uint_as_float(a.counters->emax_bits) : 0.0f;
    if (EBOUND)
      ec.dthr = fmaxf(a.dthr, 2.5f * a.beta_abs * sqrtf(a.gamma / a.beta_abs) * emax);
    ec.alpha2 = pack2(__float_as_uint(a.alpha), __float_as_uint(a.alpha));
    ec.beta2 = pack2(__float_as_uint(a.beta), __float_as_uint(a.beta));
    ec.gamma2 = pack2(__float_as_uint(a.gamma), __float_as_uint(a.gamma));
    // d~ = beta S^2 + gamma < dthr  <=>  S^2 > (gamma - dthr) / |beta| (alpha = 0);
    // 1e-4 relative margin for the fp32 rounding of d~
    ec.sdeg = (a.gamma > ec.dthr && a.beta_abs > 0.0f)
                  ? sqrtf((a.gamma - ec.dthr) / a.beta_abs) * (1.0f - 1e-4f)
                  : 0.0f;
    const int slots = a.n_chunks * GROUPS;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      const int mtile = u % a.n_mtiles;
      const int chunk = u / a.n_mtiles;
      int t0, t1;
      chunk_range(a, chunk, t0, t1);
      const int64_t p = ((int64_t)mtile * CG + rank) * kTileM + row;
      const bool prow = p < a.L;
      if (MODE == 1) {
        if (grp == 0) {  // A row = W[p] (fp16, kpad halves = kpad / 8 core-matrix rows)
          uint8_t* rbase = a_mem + (row >> 3) * (kext * 8 * ELT) + (row & 7) * 16;
          const uint4* src = reinterpret_cast<const uint4*>(a.wA + p * (int64_t)a.kpad);
          for (int kc = 0; kc < a.kpad / 8; ++kc)
            *reinterpret_cast<uint4*>(rbase + kc * 128) = prow ? src[kc] : make_uint4(0, 0, 0, 0);
          fence_proxy_async_smem();
          if (CG == 2) mbar_arrive_cluster(afull, 0);
          else mbar_arrive(afull);
        }
      } else {
        // A row `row` from the permutation's indicator bits (gmask; zero rows
        // past L), canonical K-major no-swizzle layout: 8x8 core matrices,
        // LBO = 128 B, SBO = kext*8*ELT; a core-matrix row is 16 bytes = 16
        // u8 / 8 fp16 K-elements.  int8: K runs over [h | l], A row =
        // [255 G | G].  Every epilogue group expands its share of the row's
        // core-matrix columns (kc = grp, grp + GROUPS, ...).
        uint8_t* rbase = a_mem + (row >> 3) * (kext * 8 * ELT) + (row & 7) * 16;
        const uint32_t* mrow = a.gmask + p * (int64_t)a.mwords;
        if (I8) {
          const int nkc = a.kpad / 16;  // 16 indicator bits per core-matrix row
          for (int kc = grp; kc < nkc; kc += GROUPS) {
            const uint32_t bits = (mrow[kc >> 1] >> ((kc & 1) * 16)) & 0xFFFFu;
            uint32_t e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)  // 4 bits -> 4 bytes of 0 / 1
              e[q] = (((bits >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
            *reinterpret_cast<uint4*>(rbase + kc * 128) =
                make_uint4(e[0] * 255u, e[1] * 255u, e[2] * 255u, e[3] * 255u);
            *reinterpret_cast<uint4*>(rbase + (nkc + kc) * 128) = make_uint4(e[0], e[1], e[2], e[3]);
          }
        } else {
          const int nkc = a.kpad / 8;  // 8 indicator bits per core-matrix row
          for (int kc = grp; kc < nkc; kc += GROUPS) {
            const uint32_t bits = (mrow[kc >> 2] >> ((kc & 3) * 8)) & 0xFFu;
            uint32_t e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // 2 bits -> two fp16 0 / 1
              const uint32_t b2 = (bits >> (2 * q)) & 3u;
              e[q] = ((b2 & 1u) | ((b2 & 2u) << 15)) * 0x3C00u;
            }
            *reinterpret_cast<uint4*>(rbase + kc * 128) = make_uint4(e[0], e[1], e[2], e[3]);
          }
        }
        fence_proxy_async_smem();
        if (CG == 2) mbar_arrive_cluster(afull, 0);
        else mbar_arrive(afull);
      }
      Top4 top;
      top.reset(MODE == 1 ? -FLT_MAX : seed_key<TWO_SIDED>(a.best_t, p, prow, a, emax));
      float cmax = -FLT_MAX;  // MODE 1: running max of this row over the unit
      const float wsc = (MODE == 1 && prow) ? a.wdescale[p] : 0.0f;
      float kthr = sonly_thr(top.k3, ec);  // S-only hit threshold on S^2
      uint32_t seen_enc = 0u;              // the row's running best (all groups)
      float kfloor = -FLT_MAX;             // and the key floor it implies
      unsigned rare_groups = 0;
      float* winv = inv_smem + ew * (COLGROUPS * 32);  // this warp's columns
      for (int i = 0; i < t1 - t0; ++i) {
        const int t = chunk_tile(a, chunk, t0, t1, i);
        if (I8) {  // stage the tile's scales for our columns; lands during the MMA wait
          __syncwarp();
          if (lane < COLGROUPS * 8)
            cp_async16(winv + 4 * lane, a.inv_scale + (int64_t)t * TV + grp * COLGROUPS * 32 + 4 * lane);
          cp_async_commit();
        }
        // (commit-multicast arrivals; CTA-scope acquire: no L1 invalidation)
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const int64_t vleft = a.v - (int64_t)t * TV;
        const int valid = vleft < TV ? (int)vleft : TV;
        if (I8) {
          cp_async_wait_all();
          __syncwarp();
        }
        if constexpr (SONLY && MODE == 0) {  // pick up the other groups' best for this row
          const unsigned long long rb = rowbest[row];
          const uint32_t enc = (uint32_t)rb;
          if ((uint32_t)(rb >> 32) == (uint32_t)u && enc > seen_enc) {
            seen_enc = enc;
            kfloor = floor_key<TWO_SIDED>(ord_dec(enc), a, emax);
            kthr = sonly_thr(fmaxf(top.k3, kfloor), ec);
          }
        }
#pragma unroll 1
        for (int g = 0; g < COLGROUPS; ++g) {
          const int gc = (grp * COLGROUPS + g) * 32;
          const uint32_t taddr =
              tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * kTileN + gc);
          const int jbase = t * TV + gc;
          const float* ginv = winv + g * 32;
          uint32_t sv[32], qv[32];
          tmem_ld32(taddr, sv);
          if (SONLY) {
#pragma unroll
            for (int c = 0; c < 32; ++c) qv[c] = 0u;
          } else {
            tmem_ld32(taddr + kTileV, qv);
          }
          tmem_ld_wait();
          const int gvalid = valid - gc;
          if constexpr (MODE == 1) {
            if (gvalid > 0 && prow) {
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                float z[4];
                normals4(a.seed, a.perm_base + p, (jbase >> 2) + q4, z);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int c = 4 * q4 + e;
                  float val = fmaf(a.sigma, z[e], __uint_as_float(sv[c]) * wsc);
                  if (TWO_SIDED) val = fabsf(val);
                  if (c < gvalid) cmax = fmaxf(cmax, val);
                }
              }
            }
            continue;
          }
          if (I8) {  // S_q -> S = S_q * inv (packed; scales: broadcast shared loads)
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const float4 iv = reinterpret_cast<const float4*>(ginv)[c4];
              const uint64_t s01 = mul2(pack2(__float_as_uint((float)(int)sv[4 * c4 + 0]),
                                              __float_as_uint((float)(int)sv[4 * c4 + 1])),
                                        pack2(__float_as_uint(iv.x), __float_as_uint(iv.y)));
              const uint64_t s23 = mul2(pack2(__float_as_uint((float)(int)sv[4 * c4 + 2]),
                                              __float_as_uint((float)(int)sv[4 * c4 + 3])),
                                        pack2(__float_as_uint(iv.z), __float_as_uint(iv.w)));
              sv[4 * c4 + 0] = (uint32_t)s01;
              sv[4 * c4 + 1] = (uint32_t)(s01 >> 32);
              sv[4 * c4 + 2] = (uint32_t)s23;
              sv[4 * c4 + 3] = (uint32_t)(s23 >> 32);
            }
          }
          if (DEBUG) group_debug<TWO_SIDED>(sv, qv, jbase, gvalid, ec, p, prow, a);
          if (gvalid <= 0) continue;
          if constexpr (SONLY) {
            if (!__any_sync(0xffffffffu, sonly_any(sv, kthr))) continue;
            uint32_t hits = sonly_mask<TWO_SIDED>(sv, kthr, ec);
            if (gvalid < 32) hits &= (1u << gvalid) - 1u;
            if (__any_sync(0xffffffffu, hits != 0u)) {
              ++rare_groups;
              group_rare<TWO_SIDED, SONLY, I8>(hits, taddr, jbase, ec, top, p, prow, a, ginv,
                                               kfloor);
              if (prow && top.j0 >= 0) {  // publish a new row best to the other groups
                const uint32_t enc = ord_enc(key_to_t(top.k0));
                if (enc > seen_enc) {
                  seen_enc = enc;
                  kfloor = floor_key<TWO_SIDED>(key_to_t(top.k0), a, emax);
                  atomicMax(&rowbest[row], ((unsigned long long)u << 32) | enc);
                }
              }
              kthr = sonly_thr(fmaxf(top.k3, kfloor), ec);
            }
          } else {
            uint32_t hits = group_hits<ALPHA0>(sv, qv, ec, top.k3);
            if (gvalid < 32) hits &= (1u << gvalid) - 1u;
            if (__any_sync(0xffffffffu, hits != 0u)) {
              ++rare_groups;
              group_rare<TWO_SIDED, SONLY, I8>(hits, taddr, jbase, ec, top, p, prow, a, ginv);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // accumulator drained
          if (CG == 2) mbar_arrive_remote(&tempty[acc], 0);
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == kNumAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if constexpr (MODE == 1) {
        if (prow) atomicMax(a.maxenc + p, ord_enc(cmax));
        continue;
      }
      if (lane == 0) {  // diagnostics: warp-groups that took the rare path / all
        atomicAdd(&a.counters->rare_groups, (unsigned long long)rare_groups);
        atomicAdd(&a.counters->all_groups, (unsigned long long)((t1 - t0) * COLGROUPS));
      }
      if (prow && top.j0 >= 0) atomicMax(a.best_t + p, ord_enc(key_to_t(top.k0)));
      if (prow) {
        int4* dst = a.cand + 2 * (p * slots + chunk * GROUPS + grp);
        dst[0] = make_int4(__float_as_int(top.j0 >= 0 ? key_to_t(top.k0) : -FLT_MAX), top.j0,
                           __float_as_int(top.j1 >= 0 ? key_to_t(top.k1) : -FLT_MAX), top.j1);
        dst[1] = make_int4(__float_as_int(top.j2 >= 0 ? key_to_t(top.k2) : -FLT_MAX), top.j2,
                           __float_as_int(top.j3 >= 0 ? key_to_t(top.k3) : -FLT_MAX), top.j3);
      }
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_2sm(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}

// -------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

size_t smem_bytes_for(int cg, int bk, int stages, int kpad, bool i8) {
  // fp16: hi + lo boxes of bk halves; i8: one box of bk bytes of [h | l].
  // The A tile is kTileM x kpad halves or kTileM x 2 kpad bytes: same size.
  const size_t stage = i8 ? (size_t)(kTileN / cg) * bk : (size_t)2 * (kTileN / cg) * bk * 2;
  size_t bytes = stages * stage + (size_t)kTileM * kpad * 2 + 256 + 1024 + (i8 ? kInvStage : 0) +
                 kTileM * sizeof(unsigned long long);
  // one CTA per SM: TMEM (512 columns) is allocated whole by each CTA
  return bytes < 120 * 1024 ? 120 * 1024 : bytes;
}

template <int CG, int BK, int STAGES, int EPI, bool TS, bool A0, bool DBG, bool I8 = false,
          int MODE = 0>
cudaError_t launch_cfg_e(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                         cudaStream_t s) {
  auto kern = k_tfill_tc<CG, BK, STAGES, EPI, TS, A0, DBG, I8, MODE>;
  const size_t smem = smem_bytes_for(CG, BK, STAGES, lay.kpad, I8);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  // persistent grid, at most one CTA (pair) per unit of this launch's chunks
  const int64_t units = (int64_t)lay.n_mtiles * (a.chunk_end - a.chunk_begin);
  const int grid = (int)std::min<int64_t>(lay.grid, (int64_t)CG * units);
  if (grid <= 0) return cudaSuccess;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(64 + 32 * EPI);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, map, a);
}

// epilogue warps: 16 (four per TMEM lane quadrant) for short-K single-CTA
// tiles, where the epilogue is latency-bound; 8 otherwise
template <int CG, int BK, int STAGES, bool TS, bool A0, bool DBG>
cudaError_t launch_cfg(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                       cudaStream_t s) {
  if constexpr (CG == 1 && A0 && !DBG) {
    if (lay.groups == 4) return launch_cfg_e<CG, BK, STAGES, 16, TS, A0, DBG>(lay, a, map, s);
  }
  return launch_cfg_e<CG, BK, STAGES, 8, TS, A0, DBG>(lay, a, map, s);
}

template <bool TS, bool A0, bool DBG>
cudaError_t dispatch(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                     cudaStream_t s) {
  if (lay.cg == 2) {
    if (lay.bk == 64) {
      if (lay.stages >= 6) return launch_cfg<2, 64, 6, TS, A0, DBG>(lay, a, map, s);
      return launch_cfg<2, 64, 4, TS, A0, DBG>(lay, a, map, s);
    }
    if (lay.stages >= 7) return launch_cfg<2, 32, 7, TS, A0, DBG>(lay, a, map, s);
    return launch_cfg<2, 32, 4, TS, A0, DBG>(lay, a, map, s);
  }
  if (lay.bk == 64) return launch_cfg<1, 64, 3, TS, A0, DBG>(lay, a, map, s);
  if (lay.stages >= 4) return launch_cfg<1, 32, 4, TS, A0, DBG>(lay, a, map, s);
  return launch_cfg<1, 32, 3, TS, A0, DBG>(lay, a, map, s);
}

// integer tiles (balanced groups only): bk = 128 bytes (128B swizzle)
template <int CG, int STAGES, bool TS, bool DBG>
cudaError_t launch_i8(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                      cudaStream_t s) {
  if constexpr (!DBG) {
    if (lay.groups == 4) return launch_cfg_e<CG, 128, STAGES, 16, TS, true, DBG, true>(lay, a, map, s);
  }
  return launch_cfg_e<CG, 128, STAGES, 8, TS, true, DBG, true>(lay, a, map, s);
}
template <bool TS, bool DBG>
cudaError_t dispatch_i8(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                        cudaStream_t s) {
  if (lay.cg == 2) {
    if (lay.stages >= 7) return launch_i8<2, 7, TS, DBG>(lay, a, map, s);
    return launch_i8<2, 4, TS, DBG>(lay, a, map, s);
  }
  if (lay.stages >= 4) return launch_i8<1, 4, TS, DBG>(lay, a, map, s);
  return launch_i8<1, 3, TS, DBG>(lay, a, map, s);
}

template <bool TS>
cudaError_t dispatch_a(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                       cudaStream_t s) {
  if (lay.i8) return a.dbg_t ? dispatch_i8<TS, true>(lay, a, map, s) : dispatch_i8<TS, false>(lay, a, map, s);
  const bool a0 = a.alpha == 0.0f;
  if (a.dbg_t) return a0 ? dispatch<TS, true, true>(lay, a, map, s)
                         : dispatch<TS, false, true>(lay, a, map, s);
  return a0 ? dispatch<TS, true, false>(lay, a, map, s) : dispatch<TS, false, false>(lay, a, map, s);
}

}  // namespace

bool make_planes_map(CUtensorMap* map, const __half* planes, int64_t v, int kpad, int bk,
                     int voxels_per_box, int planes_per_box) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kpad, (cuuint64_t)v, 4};
  cuuint64_t strides[2] = {(cuuint64_t)kpad * 2, (cuuint64_t)v * kpad * 2};
  cuuint32_t box[3] = {(cuuint32_t)bk, (cuuint32_t)voxels_per_box, (cuuint32_t)planes_per_box};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(planes), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void chunk_voxels(const NaiveLayout& lay, int64_t v, int c, int64_t* v0, int64_t* v1) {
  int t0, t1;
  chunk_tiles(lay.n_ramp, lay.ramp_start, lay.tiles_per_chunk, lay.n_vtiles, c, &t0, &t1);
  *v0 = std::min<int64_t>((int64_t)t0 * lay.vt, v);
  *v1 = std::min<int64_t>((int64_t)t1 * lay.vt, v);
}

void fill_chunks(const NaiveLayout& lay, TfillArgs* a) {
  a->n_chunks = lay.n_chunks;
  a->tiles_per_chunk = lay.tiles_per_chunk;
  a->n_ramp = lay.n_ramp;
  for (int i = 0; i <= lay.n_ramp; ++i) a->ramp_start[i] = lay.ramp_start[i];
  for (int i = 0; i < lay.n_ramp; ++i)
    a->ramp_stride[i] = golden_stride_public(lay.ramp_start[i + 1] - lay.ramp_start[i]);
  const int bulk = lay.n_vtiles - lay.ramp_start[lay.n_ramp];
  a->stride_full = golden_stride_public(lay.tiles_per_chunk);
  a->stride_last = golden_stride_public(bulk - (lay.n_chunks - lay.n_ramp - 1) * lay.tiles_per_chunk);
}

// completion tiles: fp16 S-only configurations, 16 epilogue warps
template <bool TS>
cudaError_t dispatch_complete(const NaiveLayout& lay, const TfillArgs& a, const CUtensorMap& map,
                              cudaStream_t s) {
  if (lay.cg == 2) {
    if (lay.bk == 64) {
      if (lay.stages >= 6) return launch_cfg_e<2, 64, 6, 16, TS, true, false, false, 1>(lay, a, map, s);
      return launch_cfg_e<2, 64, 4, 16, TS, true, false, false, 1>(lay, a, map, s);
    }
    if (lay.stages >= 7) return launch_cfg_e<2, 32, 7, 16, TS, true, false, false, 1>(lay, a, map, s);
    return launch_cfg_e<2, 32, 4, 16, TS, true, false, false, 1>(lay, a, map, s);
  }
  if (lay.bk == 64) return launch_cfg_e<1, 64, 3, 16, TS, true, false, false, 1>(lay, a, map, s);
  if (lay.stages >= 4) return launch_cfg_e<1, 32, 4, 16, TS, true, false, false, 1>(lay, a, map, s);
  return launch_cfg_e<1, 32, 3, 16, TS, true, false, false, 1>(lay, a, map, s);
}

bool make_planes8_map(CUtensorMap* map, const uint8_t* planes, int64_t v, int kpad, int cg) {
  auto enc = get_encode();
  if (!enc) return false;
  // rows [h | l] of 2 kpad bytes per voxel; box = 128 K-bytes x 256 / cg voxels
  cuuint64_t dims[3] = {(cuuint64_t)(2 * kpad), (cuuint64_t)v, 1};
  cuuint64_t strides[2] = {(cuuint64_t)(2 * kpad), (cuuint64_t)v * 2 * kpad};
  cuuint32_t box[3] = {128u, (cuuint32_t)(2 * kTileV / cg), 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(planes), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t launch_complete_tc(const NaiveLayout& lay, const TfillArgs& a, const __half* planes,
                               int two_sided, cudaStream_t s) {
  // planes [2][v][kpad]: U_hi, U_lo; boxes of 256 / cg voxels of one plane
  auto enc = get_encode();
  if (!enc) return cudaErrorInvalidValue;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)lay.kpad, (cuuint64_t)a.v, 2};
  cuuint64_t strides[2] = {(cuuint64_t)lay.kpad * 2, (cuuint64_t)a.v * lay.kpad * 2};
  cuuint32_t box[3] = {(cuuint32_t)lay.bk, (cuuint32_t)(2 * kTileV / lay.cg), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(planes), dims, strides, box,
          estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          lay.bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return two_sided ? dispatch_complete<true>(lay, a, map, s) : dispatch_complete<false>(lay, a, map, s);
}

// Group-1 indicator bit rows of the labels (K1's A operand source): one warp
// per permutation row; rows in [L, rows) are zero (the tail of the last
// permutation tile).  Reads the L x n int16 orders once (80 MB at config 4).
__global__ void k_group_mask(const int16_t* __restrict__ orders, int64_t L, int64_t rows, int n,
                             int n1, int mwords, uint32_t* __restrict__ gmask) {
  __shared__ uint32_t words[8][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* my = words[w];
  for (int64_t p = (int64_t)blockIdx.x * 8 + w; p < rows; p += (int64_t)gridDim.x * 8) {
    for (int j = lane; j < mwords; j += 32) my[j] = 0u;
    __syncwarp();
    if (p < L) {
      const int16_t* ord = orders + p * n;
      for (int i = lane; i < n1; i += 32) {
        const int k = ord[i];
        atomicOr(&my[k >> 5], 1u << (k & 31));
      }
    }
    __syncwarp();
    for (int j = lane; j < mwords; j += 32) gmask[p * mwords + j] = my[j];
    __syncwarp();
  }
}

cudaError_t launch_group_mask(const int16_t* orders, int64_t L, int64_t rows, int n, int n1,
                              int mwords, uint32_t* gmask, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (mwords > 32) return cudaErrorInvalidValue;  // n > 1024: never a tensor-core tile
  const int blocks = (int)std::min<int64_t>((rows + 7) / 8, 148 * 16);
  k_group_mask<<<blocks, 256, 0, s>>>(orders, L, rows, n, n1, mwords, gmask);
  return cudaGetLastError();
}

cudaError_t launch_tfill_tc(const NaiveLayout& lay, const TfillArgs& a, const __half* planes,
                            int two_sided, cudaStream_t s) {
  CUtensorMap map;
  if (lay.i8) {
    if (!make_planes8_map(&map, reinterpret_cast<const uint8_t*>(planes), a.v, lay.kpad, lay.cg))
      return cudaErrorInvalidValue;
    return two_sided ? dispatch_a<true>(lay, a, map, s) : dispatch_a<false>(lay, a, map, s);
  }
  // box rows per TMA: S-only tiles load 256 (cg 1) or 128 (cg 2) voxels of one
  // plane; (S | Q) tiles load 128 voxels of 2 (cg 1) or 1 (cg 2) planes
  const bool sonly = a.alpha == 0.0f;
  const int vbox = sonly ? 2 * kTileV / lay.cg : kTileV;
  const int pbox = sonly ? 1 : 2 / lay.cg;
  if (!make_planes_map(&map, planes, a.v, lay.kpad, lay.bk, vbox, pbox))
    return cudaErrorInvalidValue;
  return two_sided ? dispatch_a<true>(lay, a, map, s) : dispatch_a<false>(lay, a, map, s);
}

size_t tfill_smem_bytes(int cg, int bk, int stages, int kpad, bool i8) {
  return smem_bytes_for(cg, bk, stages, kpad, i8);
}

}  // namespace rmx
