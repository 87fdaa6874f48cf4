// philox.cuh -- counter-based N(0,1) residual noise of RapidPT recovery
// (replaces numpy's RESIDUAL stream, rapid.py:201).
// Shared by the fp32 completion kernel and the tensor-core one, so both
// draw identical normals for a (seed, permutation, voxel).
#pragma once
#include <cstdint>

namespace rmx {

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

}  // namespace rmx
