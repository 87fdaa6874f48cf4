// normals.cpp -- numpy's Generator.standard_normal over the reference's
// SFC64 streams, on host cores, bit for bit.
//
// RapidPT draws two kinds of Gaussian streams:
//   BASIS_INIT   one stream of v x r normals for the initial basis
//                (reference lrmc.py:85-93: stream(seed, 5).standard_normal((v, r)))
//   SHIFT_GAP    ell streams of v normals for the max-gap shift estimator
//                (reference rapid.py:115-121)
// numpy's standard_normal is Marsaglia & Tsang's ziggurat with 256 levels on
// 64-bit words (numpy/random/src/distributions/distributions.c,
// random_standard_normal): r = next_uint64; idx = r & 0xff; the sign is bit
// 8; rabs = bits 9..60; x = rabs * w[idx]; accept if rabs < k[idx] (99.3%);
// else the base strip (idx 0: Marsaglia's tail from r = 3.654...) or the
// wedge test against exp(-x^2 / 2).  The tables (k, w, f) are numpy's own:
// paper_1703_01506_b200/normals.py reads them from numpy at start-up
// (rmx_normal_tables_set) -- they are not restated here.
//
// Why host cores: an SFC64 stream has no jump-ahead (its state update mixes
// by addition), so one stream is one serial dependency chain.  A host core
// steps it in ~1 ns; a GPU thread is several times slower.  The serial part
// is kept minimal (the generator core), and the transform is exact IEEE
// double arithmetic with the same libm calls numpy makes (log1p, exp), so the
// values are identical.  Independent streams (SHIFT_GAP) run on a thread pool.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/rmx.h"
#include "sfc64.cuh"

namespace {

struct ZigTables {
  uint64_t k[256];
  double w[256];
  double f[256];
  bool ready = false;
};
ZigTables g_zig;

// numpy's ziggurat constants for the normal tail (distributions.h)
constexpr double kZigR = 3.6541528853610087963519472518;
constexpr double kZigInvR = 0.27366123732975827203338247596;

inline double next_double(rmx::sfc::Sfc64& g) {
  return (double)(g.next64() >> 11) * (1.0 / 9007199254740992.0);
}

// rabs < 2^52 as a double, exactly (the bits of 2^52 + rabs, minus 2^52):
// numpy's (double)rabs without x86's slow unsigned 64-bit conversion
inline double exact_u52(uint64_t rabs) {
  const uint64_t b = 0x4330000000000000ULL | rabs;
  double d;
  std::memcpy(&d, &b, 8);
  return d - 4503599627370496.0;
}

// The rare paths (idx 0 tail, wedge test), given the first word's parts.
__attribute__((noinline)) double standard_normal_slow(rmx::sfc::Sfc64& g, int idx, uint64_t rabs,
                                                      double x);

// out[0..n) = the stream's next n normals.  The generator state lives in
// registers across the loop and is written back only around the rare path.
void fill_normals(rmx::sfc::Sfc64& g, int64_t n, double* out) {
  uint64_t a = g.a, b = g.b, c = g.c, w = g.w;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t r0 = a + b + w++;  // Sfc64::next64, inlined on locals
    a = b ^ (b >> 11);
    b = c + (c << 3);
    c = ((c << 24) | (c >> 40)) + r0;
    const int idx = (int)(r0 & 0xff);
    const uint64_t r = r0 >> 8;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = exact_u52(rabs) * g_zig.w[idx];
    uint64_t xb;
    std::memcpy(&xb, &x, 8);
    xb ^= (r & 0x1) << 63;
    std::memcpy(&x, &xb, 8);
    if (__builtin_expect(rabs < g_zig.k[idx], 1)) {
      out[i] = x;
      continue;
    }
    g.a = a;
    g.b = b;
    g.c = c;
    g.w = w;
    out[i] = standard_normal_slow(g, idx, rabs, x);
    a = g.a;
    b = g.b;
    c = g.c;
    w = g.w;
  }
  g.a = a;
  g.b = b;
  g.c = c;
  g.w = w;
}

inline double standard_normal(rmx::sfc::Sfc64& g) {
  const uint64_t r0 = g.next64();
  const int idx = (int)(r0 & 0xff);
  const uint64_t r = r0 >> 8;
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  double x = exact_u52(rabs) * g_zig.w[idx];
  uint64_t xb;  // x = -x when the sign bit is set, without a branch (50/50)
  std::memcpy(&xb, &x, 8);
  xb ^= (r & 0x1) << 63;
  std::memcpy(&x, &xb, 8);
  if (__builtin_expect(rabs < g_zig.k[idx], 1)) return x;  // ~99.3%
  return standard_normal_slow(g, idx, rabs, x);
}

double standard_normal_slow(rmx::sfc::Sfc64& g, int idx, uint64_t rabs, double x) {
  for (;;) {
    if (idx == 0) {
      for (;;) {  // 1 - U avoids log(0)
        const double xx = -kZigInvR * std::log1p(-next_double(g));
        const double yy = -std::log1p(-next_double(g));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 0x1) ? -(kZigR + xx) : kZigR + xx;
      }
    } else {
      if (((g_zig.f[idx - 1] - g_zig.f[idx]) * next_double(g) + g_zig.f[idx]) <
          std::exp(-0.5 * x * x))
        return x;
    }
    // rejected: numpy's loop draws a fresh word
    uint64_t r = g.next64();
    idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    rabs = (r >> 1) & 0x000fffffffffffffULL;
    x = exact_u52(rabs) * g_zig.w[idx];
    if (sign & 0x1) x = -x;
    if (rabs < g_zig.k[idx]) return x;
  }
}

void seed_stream(rmx::sfc::Sfc64& g, uint64_t seed, const uint32_t* path, int npath) {
  rmx::sfc::sfc64_seed(g, seed, path, npath);
}

int fail(rmx_status* st, int code, const char* msg) {
  if (st) {
    st->code = code;
    std::snprintf(st->msg, sizeof(st->msg), "%s", msg);
  }
  return code;
}

}  // namespace

extern "C" {

int rmx_normal_tables_set(const uint64_t* k, const double* w, const double* f) {
  std::memcpy(g_zig.k, k, sizeof(g_zig.k));
  std::memcpy(g_zig.w, w, sizeof(g_zig.w));
  std::memcpy(g_zig.f, f, sizeof(g_zig.f));
  g_zig.ready = true;
  return RMX_OK;
}

int rmx_standard_normal(uint64_t seed, const uint32_t* path, int32_t npath, int64_t count,
                        double* out, rmx_status* st) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->perm = st->voxel = -1;
  }
  if (!g_zig.ready) return fail(st, RMX_E_USAGE, "normal tables not set (rmx_normal_tables_set)");
  if (npath < 0 || npath > 3 || count < 0 || (count > 0 && !out))
    return fail(st, RMX_E_USAGE, "bad standard_normal arguments");
  rmx::sfc::Sfc64 g;
  seed_stream(g, seed, path, npath);
  fill_normals(g, count, out);
  return RMX_OK;
}

// A stream that is drawn in consecutive pieces (BASIS_INIT: block by block
// into page-locked staging buffers, each uploaded behind the next draw).
struct rmx_normal_stream {
  rmx::sfc::Sfc64 g;
};

int rmx_normal_stream_open(uint64_t seed, const uint32_t* path, int32_t npath,
                           rmx_normal_stream** out, rmx_status* st) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->perm = st->voxel = -1;
  }
  if (!g_zig.ready) return fail(st, RMX_E_USAGE, "normal tables not set (rmx_normal_tables_set)");
  if (npath < 0 || npath > 3 || !out) return fail(st, RMX_E_USAGE, "bad normal stream arguments");
  auto* h = new rmx_normal_stream;
  seed_stream(h->g, seed, path, npath);
  *out = h;
  return RMX_OK;
}

int rmx_normal_stream_fill(rmx_normal_stream* h, int64_t count, double* out) {
  if (!h || count < 0 || (count > 0 && !out)) return RMX_E_USAGE;
  fill_normals(h->g, count, out);
  return RMX_OK;
}

int rmx_normal_stream_close(rmx_normal_stream* h) {
  delete h;
  return RMX_OK;
}

int rmx_standard_normal_rows(uint64_t seed, uint32_t domain, int64_t lo, int64_t hi,
                             int64_t count, float* out32, double* out64, int32_t threads,
                             rmx_status* st) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->perm = st->voxel = -1;
  }
  if (!g_zig.ready) return fail(st, RMX_E_USAGE, "normal tables not set (rmx_normal_tables_set)");
  if (hi < lo || count < 0 || lo < 0 || hi > 0xffffffffLL || (!out32 && !out64))
    return fail(st, RMX_E_USAGE, "bad standard_normal_rows arguments");
  const int64_t rows = hi - lo;
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > rows) nt = (int)std::max<int64_t>(rows, 1);
  std::atomic<int64_t> next{0};
  auto work = [&]() {
    for (int64_t i; (i = next.fetch_add(1)) < rows;) {
      const uint32_t path[2] = {domain, (uint32_t)(lo + i)};
      rmx::sfc::Sfc64 g;
      seed_stream(g, seed, path, 2);
      if (out64) {
        fill_normals(g, count, out64 + i * count);
      } else {
        float* o = out32 + i * count;
        for (int64_t j = 0; j < count; ++j) o[j] = (float)standard_normal(g);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return RMX_OK;
}

}  // extern "C"
