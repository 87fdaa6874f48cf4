// rng_kernels.cu -- the reference's random streams on the device, bit-exact.
//
// The reference draws every permutation and observation set from its own
// stream (rmx/streams.py:31-38):
//     Generator(SFC64(SeedSequence(entropy=seed, spawn_key=(domain, i[, p]))))
// and uses them as
//     PermutationPlan.shuffle(i) = stream(seed, SHUFFLE, i).permutation(n)   (model.py:100-105)
//     Omega_i = sort(stream(seed, RECOVER_OMEGA, i).choice(v, k, replace=False)) (rapid.py:158-160)
//     Omega_{i,p} = ... stream(seed, TRAIN_OMEGA, i, p) ...                   (lrmc.py:237-241)
// Generating those on the host costs ~26-30 us per stream (3 s
// for 1e5 permutations).  This file restates numpy 2.x's published
// algorithms -- SeedSequence's hash/mix pool and generate_state, SFC64 with
// its 12 warm-up rounds and 32-bit half buffering, Generator.permutation's
// Fisher-Yates with masked-rejection random_interval, Generator.choice's
// Floyd sampling with the open-addressing set and 32-bit Lemire bounded
// integers -- so each stream is reproduced bit for bit on the GPU (pinned
// against numpy itself by tests/test_gpu_rng.py and tests/golden/shuffles.npz).
#include <cstdint>

#include <cuda_runtime.h>

#include "sfc64.cuh"

namespace rmx {
namespace {

using namespace sfc;

__device__ __forceinline__ uint64_t gen_mask(uint64_t x) {
  x |= x >> 1;
  x |= x >> 2;
  x |= x >> 4;
  x |= x >> 8;
  x |= x >> 16;
  x |= x >> 32;
  return x;
}

// numpy random_interval: masked rejection (Generator.shuffle / permutation)
__device__ __forceinline__ uint32_t random_interval32(Sfc64& g, uint32_t mx) {
  if (mx == 0) return 0;
  const uint32_t mask = (uint32_t)gen_mask(mx);
  uint32_t v;
  while ((v = (g.next32() & mask)) > mx) {
  }
  return v;
}

// numpy random_bounded_uint64(0, rng) for rng < 2^32: 32-bit Lemire
__device__ __forceinline__ uint32_t bounded_lemire32(Sfc64& g, uint32_t rng) {
  if (rng == 0) return 0;
  const uint32_t rng_excl = rng + 1;
  uint64_t m = (uint64_t)g.next32() * rng_excl;
  uint32_t left = (uint32_t)m;
  if (left < rng_excl) {
    const uint32_t thr = (0xFFFFFFFFu - rng) % rng_excl;
    while (left < thr) {
      m = (uint64_t)g.next32() * rng_excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// one thread per permutation: row t = shuffle(lo + t) (identity at index 0),
// Fisher-Yates in place in the output row
__global__ void k_plan_orders(uint64_t seed, int64_t lo, int64_t count, int n, int16_t* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int64_t index = lo + t;
  int16_t* row = out + t * n;
  for (int i = 0; i < n; ++i) row[i] = (int16_t)i;
  if (index == 0) return;
  const uint32_t key[2] = {1u /* SHUFFLE */, (uint32_t)index};
  Sfc64 g;
  sfc64_seed(g, seed, key, 2);
  for (int i = n - 1; i > 0; --i) {
    const int j = (int)random_interval32(g, (uint32_t)i);
    const int16_t tmp = row[i];
    row[i] = row[j];
    row[j] = tmp;
  }
}

// The same with the rows shuffled in shared memory (the swaps of a
// Fisher-Yates pass are dependent, random accesses: in global memory they
// thrash L1 and serialise on L2 latency), then written out coalesced: the
// block's kPlanRows rows are contiguous in `out`.
constexpr int kPlanRows = 64;
__global__ void __launch_bounds__(kPlanRows) k_plan_orders_smem(uint64_t seed, int64_t lo,
                                                                int64_t count, int n,
                                                                int16_t* out) {
  extern __shared__ __align__(16) int16_t prow[];
  const int64_t t0 = (int64_t)blockIdx.x * kPlanRows;
  const int rows = (int)(count - t0 < kPlanRows ? count - t0 : kPlanRows);
  int16_t* row = prow + (size_t)threadIdx.x * n;
  if ((int)threadIdx.x < rows) {
    for (int i = 0; i < n; ++i) row[i] = (int16_t)i;
    const int64_t index = lo + t0 + threadIdx.x;
    if (index != 0) {
      const uint32_t key[2] = {1u /* SHUFFLE */, (uint32_t)index};
      Sfc64 g;
      sfc64_seed(g, seed, key, 2);
      for (int i = n - 1; i > 0; --i) {
        const int j = (int)random_interval32(g, (uint32_t)i);
        const int16_t tmp = row[i];
        row[i] = row[j];
        row[j] = tmp;
      }
    }
  }
  __syncthreads();
  const int64_t elems = (int64_t)rows * n;
  int16_t* dst = out + t0 * n;
  if (((reinterpret_cast<uintptr_t>(dst) | (uintptr_t)(elems * 2)) & 15) == 0) {
    const uint4* src4 = reinterpret_cast<const uint4*>(prow);
    uint4* dst4 = reinterpret_cast<uint4*>(dst);
    for (int64_t e = threadIdx.x; e < elems / 8; e += kPlanRows) dst4[e] = src4[e];
  } else {
    for (int64_t e = threadIdx.x; e < elems; e += kPlanRows) dst[e] = prow[e];
  }
}

// one warp per observation set: lane 0 runs Floyd's sampling with numpy's
// open-addressing set (smem), then the warp bitonic-sorts the k values
constexpr int kOmegaWarps = 4;

__global__ void __launch_bounds__(32 * kOmegaWarps)
    k_omega_draws(uint64_t seed, uint32_t domain, int64_t lo, int64_t count, int has_extra,
                  uint32_t extra, uint32_t v, int k, int set_size, int sort_size, int32_t* out) {
  extern __shared__ uint32_t osm[];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int per_warp = set_size > sort_size ? set_size : sort_size;
  uint32_t* hs = osm + (size_t)w * (per_warp + k);
  uint32_t* idx = hs + per_warp;
  const int64_t t = (int64_t)blockIdx.x * kOmegaWarps + w;
  if (t >= count) return;
  for (int i = lane; i < set_size; i += 32) hs[i] = 0xFFFFFFFFu;
  __syncwarp();
  if (lane == 0) {
    const uint32_t key[3] = {domain, (uint32_t)(lo + t), extra};
    Sfc64 g;
    sfc64_seed(g, seed, key, has_extra ? 3 : 2);
    const uint32_t mask = (uint32_t)set_size - 1u;
    for (uint32_t j = v - (uint32_t)k; j < v; ++j) {
      const uint32_t val = bounded_lemire32(g, j);
      uint32_t loc = val & mask;
      while (hs[loc] != 0xFFFFFFFFu && hs[loc] != val) loc = (loc + 1) & mask;
      if (hs[loc] == 0xFFFFFFFFu) {
        hs[loc] = val;
        idx[j - (v - (uint32_t)k)] = val;
      } else {
        loc = j & mask;
        while (hs[loc] != 0xFFFFFFFFu) loc = (loc + 1) & mask;
        hs[loc] = j;
        idx[j - (v - (uint32_t)k)] = j;
      }
    }
  }
  __syncwarp();
  // sort: copy into the (now free) set area padded to a power of two
  uint32_t* srt = hs;
  for (int i = lane; i < sort_size; i += 32) srt[i] = i < k ? idx[i] : 0xFFFFFFFFu;
  __syncwarp();
  for (int size = 2; size <= sort_size; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < sort_size; i += 32) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const uint32_t a = srt[i], b = srt[j];
          if ((a > b) == up) {
            srt[i] = b;
            srt[j] = a;
          }
        }
      }
      __syncwarp();
    }
  int32_t* o = out + t * k;
  for (int i = lane; i < k; i += 32) o[i] = (int32_t)srt[i];
}

}  // namespace

cudaError_t launch_plan_orders(uint64_t seed, int64_t lo, int64_t count, int n, int16_t* out,
                               cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const size_t smem = (size_t)kPlanRows * n * sizeof(int16_t);
  if (smem <= 160 * 1024) {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_plan_orders_smem,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_plan_orders_smem<<<(unsigned)((count + kPlanRows - 1) / kPlanRows), kPlanRows, smem, s>>>(
        seed, lo, count, n, out);
    return cudaGetLastError();
  }
  k_plan_orders<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(seed, lo, count, n, out);
  return cudaGetLastError();
}

// set_size as numpy: 1 + mask(int(1.2 * k)); the caller guarantees the
// Floyd branch (v <= 10000 or k <= v / 50) and v < 2^32
cudaError_t launch_omega_draws(uint64_t seed, uint32_t domain, int64_t lo, int64_t count,
                               int has_extra, uint32_t extra, uint32_t v, int k, int32_t* out,
                               cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  uint64_t m = (uint64_t)(1.2 * (double)k);
  m |= m >> 1;
  m |= m >> 2;
  m |= m >> 4;
  m |= m >> 8;
  m |= m >> 16;
  m |= m >> 32;
  const int set_size = (int)(m + 1);
  int sort_size = 1;
  while (sort_size < k) sort_size <<= 1;
  const int per_warp = set_size > sort_size ? set_size : sort_size;
  const size_t smem = (size_t)kOmegaWarps * (per_warp + k) * sizeof(uint32_t);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_omega_draws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_omega_draws<<<(unsigned)((count + kOmegaWarps - 1) / kOmegaWarps), 32 * kOmegaWarps, smem, s>>>(
      seed, domain, lo, count, has_extra, extra, v, k, set_size, sort_size, out);
  return cudaGetLastError();
}

}  // namespace rmx
