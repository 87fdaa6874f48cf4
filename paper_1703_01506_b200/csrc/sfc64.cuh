// sfc64.cuh -- numpy's SeedSequence -> SFC64 bit generator, restated for
// host and device (numpy 2.x published algorithms: SeedSequence's hash/mix
// pool and generate_state; SFC64 with its 12 warm-up rounds and buffered
// 32-bit halves).  Used by rng_kernels.cu (device streams) and normals.cu
// (host standard_normal).  Pinned against numpy by tests/test_gpu_rng.py and
// tests/test_normals.py.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define RMX_HD __host__ __device__ __forceinline__
#else
#define RMX_HD inline
#endif

namespace rmx {
namespace sfc {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kPool = 4;

struct Sfc64 {
  uint64_t a, b, c, w;
  uint32_t u32;
  int has32;

  RMX_HD uint64_t next64() {
    const uint64_t tmp = a + b + w++;
    a = b ^ (b >> 11);
    b = c + (c << 3);
    c = ((c << 24) | (c >> 40)) + tmp;
    return tmp;
  }
  RMX_HD uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t n = next64();
    has32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
};

RMX_HD uint32_t hashmix(uint32_t value, uint32_t& hc) {
  value ^= hc;
  hc *= kMultA;
  value *= hc;
  value ^= value >> 16;
  return value;
}
RMX_HD uint32_t mix32(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// SeedSequence(entropy, spawn_key = key[0..nkey)) -> SFC64, key entries < 2^32
RMX_HD void sfc64_seed(Sfc64& g, uint64_t entropy, const uint32_t* key, int nkey) {
  uint32_t ent[kPool + 4];
  int ne = 0;
  ent[ne++] = (uint32_t)entropy;
  if (entropy >> 32) ent[ne++] = (uint32_t)(entropy >> 32);
  if (nkey > 0)
    while (ne < kPool) ent[ne++] = 0u;  // run entropy padded to the pool size
  for (int i = 0; i < nkey; ++i) ent[ne++] = key[i];
  uint32_t pool[kPool];
  uint32_t hc = kInitA;
  for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u, hc);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = mix32(pool[d], hashmix(pool[s], hc));
  for (int s = kPool; s < ne; ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = mix32(pool[d], hashmix(ent[s], hc));
  uint32_t st[6];
  uint32_t hb = kInitB;
  for (int i = 0; i < 6; ++i) {
    uint32_t dv = pool[i % kPool];
    dv ^= hb;
    hb *= kMultB;
    dv *= hb;
    dv ^= dv >> 16;
    st[i] = dv;
  }
  g.a = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  g.b = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  g.c = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
  g.w = 1;
  g.has32 = 0;
  g.u32 = 0;
  for (int i = 0; i < 12; ++i) g.next64();
}

}  // namespace sfc
}  // namespace rmx
