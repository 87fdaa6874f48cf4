// rmx_abi.cu -- extern "C" entry points of librmx.so (declared in include/rmx.h)
// and the host-side driver logic of the NaivePT path: workspace layout,
// persistent-grid / chunk scheduling, and the decisions that need device
// results (suspect overflow, exhaustive fallback, degenerate reporting).
#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <string>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <unistd.h>

#include "../../include/rmx.h"
#include "rmx_internal.cuh"

namespace rmx {

size_t tfill_smem_bytes(int cg, int bk, int stages, int kpad, bool i8);

namespace {

constexpr size_t kMaxSmem = 232448;  // 227 KB opt-in dynamic smem per CTA on sm_100

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int set_status(rmx_status* st, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
int set_status(rmx_status* st, int code, const char* fmt, ...) {
  if (st) {
    st->code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

void clear_status(rmx_status* st) {
  if (!st) return;
  memset(st, 0, sizeof(*st));
  st->perm = -1;
  st->voxel = -1;
}

#define RMX_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return set_status(st, RMX_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(_e)); \
  } while (0)

int check_dims(int64_t v, int32_t n, int32_t n1, int64_t L, rmx_status* st) {
  if (v < 1) return set_status(st, RMX_E_USAGE, "need at least one voxel, got v=%lld", (long long)v);
  if (n1 < 2 || n - n1 < 2)
    return set_status(st, RMX_E_USAGE,
                      "need at least two subjects per group, got n1=%d, n2=%d", n1, n - n1);
  if (n > 32767) return set_status(st, RMX_E_USAGE, "subject count %d exceeds 32767", n);
  if (L < 1) return set_status(st, RMX_E_USAGE, "permutation count must be >= 1");
  if (v > 0x7fffffffLL) return set_status(st, RMX_E_USAGE, "voxel count exceeds int32 range");
  return RMX_OK;
}

// Stage/BK choice for the tensor-core kernel; returns false when the A tile
// does not fit next to a minimal ring (n > ~640).  Instantiated configs
// (tfill_tc.cu): cg=1 (64,3) (32,4) (32,3); cg=2 (64,6) (64,4) (32,7) (32,4).
bool pick_pipeline(int cg, int kpad, int* bk, int* stages) {
  const size_t a_bytes = (size_t)kTileM * kpad * 2 + 256 + 1024 + kTileM * 8;  // + row bests
  if (a_bytes >= kMaxSmem) return false;
  const size_t avail = kMaxSmem - a_bytes;
  auto fit = [&](int b) { return (int)(avail / ((size_t)2 * (2 * kTileV / cg) * b * 2)); };
  if (cg == 1) {
    if (kpad > 32 && fit(64) >= 3) {
      *bk = 64;
      *stages = 3;
      return true;
    }
    const int s = std::min(fit(32), 4);
    if (s < 3) return false;
    *bk = 32;
    *stages = s;
    return true;
  }
  if (kpad > 32 && fit(64) >= 6) {
    *bk = 64;
    *stages = 6;
    return true;
  }
  const int s32 = fit(32);
  if (s32 >= 7) {
    *bk = 32;
    *stages = 7;
    return true;
  }
  if (kpad > 32 && fit(64) >= 4) {
    *bk = 64;
    *stages = 4;
    return true;
  }
  if (s32 >= 4) {
    *bk = 32;
    *stages = 4;
    return true;
  }
  return false;
}

// int8 tiles: bk = 128 K-bytes per stage (one 128B-swizzled box of
// 256 / cg voxel rows); A = kTileM x 2 kpad bytes.  Instantiated
// (cg, stages): (1, 4) (1, 3) (2, 7) (2, 4)
bool pick_pipeline_i8(int cg, int kpad, int* bk, int* stages) {
  const size_t a_bytes = (size_t)kTileM * kpad * 2 + 256 + 1024 + kInvStage + kTileM * 8;
  if (a_bytes >= kMaxSmem) return false;
  const int fit = (int)((kMaxSmem - a_bytes) / ((size_t)(2 * kTileV / cg) * 128));
  const int want = cg == 2 ? 7 : 4;
  const int s = fit >= want ? want : (fit >= (cg == 2 ? 4 : 3) ? (cg == 2 ? 4 : 3) : 0);
  if (!s) return false;
  *bk = 128;
  *stages = s;
  return true;
}

}  // namespace

int device_sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static NaiveLayout naive_layout_compute(int64_t v, int n, int n1, int64_t L, int sm_count);

// The layout (with its chunk-count makespan search, ~0.1 ms of host time at
// config 4) is needed by every phase call; the last few are memoised, keyed
// by the arguments and the tuning environment variables.
NaiveLayout naive_layout(int64_t v, int n, int n1, int64_t L, int sm_count) {
  std::string key = std::to_string(v) + "," + std::to_string(n) + "," + std::to_string(n1) + "," +
                    std::to_string(L) + "," + std::to_string(sm_count);
  for (const char* name : {"RMX_I8", "RMX_CG", "RMX_CHUNKS_MIN", "RMX_RAMP", "RMX_EPI_GROUPS"}) {
    const char* e = getenv(name);
    key += e ? std::string("|") + e : std::string("|-");
  }
  static std::mutex mu;
  static std::vector<std::pair<std::string, NaiveLayout>> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    for (const auto& kv : cache)
      if (kv.first == key) return kv.second;
  }
  const NaiveLayout lay = naive_layout_compute(v, n, n1, L, sm_count);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() >= 8) cache.erase(cache.begin());
  cache.emplace_back(key, lay);
  return lay;
}

static NaiveLayout naive_layout_compute(int64_t v, int n, int n1, int64_t L, int sm_count) {
  NaiveLayout lay{};
  const bool balanced = 2 * n1 == n;
  // balanced groups: t depends on S only -> 256-voxel S-only tiles.  Default
  // there: exact int8 MMA on fixed-point Z; RMX_I8=0 selects fp16 hi/lo.
  // (short K is epilogue-bound, where the fp16 tiles' cheaper epilogue wins)
  lay.i8 = (balanced && n >= 192) ? 1 : 0;
  if (const char* e = getenv("RMX_I8")) lay.i8 = balanced && atoi(e) != 0;
  // int8: the digit planes [h | l] share one K extent 2 kpad, a multiple of
  // the 32-byte MMA K step whenever kpad is a multiple of 16
  lay.kpad = (n + 15) / 16 * 16;
  lay.vt = balanced ? 2 * kTileV : kTileV;
  lay.n_vtiles = (int)((v + lay.vt - 1) / lay.vt);
  // CTA pairs (cta_group::2) by default; RMX_CG=1 forces single-CTA tiles
  // (pairs halve B traffic per SM and deepen the ring; short-K tiles are
  // epilogue-bound and run better as single CTAs)
  lay.cg = lay.kpad >= 192 ? 2 : 1;
  if (const char* e = getenv("RMX_CG")) lay.cg = atoi(e) == 1 ? 1 : 2;
  auto pick = [&](int cg) {
    return lay.i8 ? pick_pipeline_i8(cg, lay.kpad, &lay.bk, &lay.stages)
                  : pick_pipeline(cg, lay.kpad, &lay.bk, &lay.stages);
  };
  if (!pick(lay.cg)) {
    lay.cg = 1;
    if (!pick(1)) {
      lay.bk = 0;
      lay.stages = 0;
    }
  }
  const int tile_perms = kTileM * lay.cg;
  lay.n_mtiles = (int)((L + tile_perms - 1) / tile_perms);
  const int n_clusters = std::max(1, sm_count / lay.cg);
  // Epilogue warps per TMEM lane quadrant: 4 (16 warps) where the epilogue
  // must keep up with a fast MMA -- short-K single-CTA S-only tiles and int8
  // tiles (twice the MMA rate) -- else 2.  16-warp variants are instantiated
  // for S-only tiles with cg = 1 or int8 only.
  const bool can16 = balanced && (lay.cg == 1 || lay.i8);
  lay.groups = (can16 && (lay.kpad <= 128 || lay.i8)) ? 4 : 2;
  if (const char* g = getenv("RMX_EPI_GROUPS"))
    if (can16) lay.groups = atoi(g) == 4 ? 4 : 2;
  // Voxel chunks per permutation tile: minimise the static round-robin
  // makespan over `sm_count` persistent CTAs (unit = one tile of 128 perms x
  // one chunk of voxel tiles; A-tile rebuild counted as ~1/4 tile).
  double best_cost = 1e300;
  int best_c = 1;
  const int cmax = std::min(lay.n_vtiles, 64);
  // Large X arrives from the host in chunk-sized copies (rmx_naive_maxnull_
  // host*): at least 14 chunks keeps the pipeline tail (K0 + K1 of the last
  // chunk after its copy lands) near 2 ms; measured on config 4 (7 -> 14
  // chunks: e2e 40.0 -> 36.9 ms, device step 33.0 -> 32.8 ms).
  int cmin = (double)v * n * 8.0 >= 512.0 * (1 << 20) ? 14 : 1;
  if (const char* e = getenv("RMX_CHUNKS_MIN")) cmin = atoi(e);
  cmin = std::max(1, std::min(cmax, cmin));
  for (int c = cmin; c <= cmax; ++c) {
    const int tpc = (lay.n_vtiles + c - 1) / c;
    const int nc = (lay.n_vtiles + tpc - 1) / tpc;
    if (nc != c) continue;
    const int64_t units = (int64_t)lay.n_mtiles * nc;
    const int grid = (int)std::min<int64_t>(n_clusters, units);
    double worst = 0;
    for (int b = 0; b < std::min(grid, 8); ++b) {  // CTA 0.. carry the most units
      double w = 0;
      for (int64_t u = b; u < units; u += grid) {
        const int chunk = (int)(u / lay.n_mtiles);
        const int tiles = std::min(tpc, lay.n_vtiles - chunk * tpc);
        w += tiles + 0.25;
      }
      worst = std::max(worst, w);
    }
    const double cost = worst * (1.0 + 0.001 * c);
    if (cost < best_cost) {
      best_cost = cost;
      best_c = c;
    }
  }
  // leading short chunks (8 then 32 tiles): the cold top-4 storm of a unit's
  // first tiles is confined to 8 tiles, and the following chunks start from
  // the permutation's best over 2,048 and then 10,240 voxels (RMX_RAMP=0: off)
  lay.n_ramp = 0;
  lay.ramp_start[0] = 0;
  const char* re = getenv("RMX_RAMP");
  if (lay.n_vtiles >= 512 && best_c >= 4 && !(re && atoi(re) == 0)) {
    lay.n_ramp = 2;
    lay.ramp_start[1] = 8;
    lay.ramp_start[2] = 40;
  }
  const int bulk = lay.n_vtiles - lay.ramp_start[lay.n_ramp];
  lay.tiles_per_chunk = (bulk + best_c - 1) / best_c;
  lay.n_chunks = lay.n_ramp + (bulk + lay.tiles_per_chunk - 1) / lay.tiles_per_chunk;
  lay.grid = lay.cg * (int)std::min<int64_t>(n_clusters, (int64_t)lay.n_mtiles * lay.n_chunks);

  lay.mwords = (lay.kpad + 31) / 32;
  size_t off = 0;
  lay.off_planes = off;
  // fp16: [4][v][kpad] halves (z_hi, q_hi, z_lo, q_lo); int8: [v][2 kpad] bytes
  off = align_up(off + (lay.i8 ? (size_t)2 * v * lay.kpad : (size_t)4 * v * lay.kpad * 2), 1024);
  lay.off_scale = off;  // int8: per-voxel dequantisation scale, padded to whole tiles
  off = align_up(off + (lay.i8 ? (size_t)lay.n_vtiles * lay.vt * 4 : 0), 256);
  lay.off_gmask = off;
  off = align_up(off + (size_t)lay.n_mtiles * tile_perms * lay.mwords * 4, 256);
  lay.off_cand = off;
  off = align_up(off + (size_t)lay.n_mtiles * tile_perms * lay.n_chunks * lay.groups * 32, 256);
  lay.off_susp = off;
  off = align_up(off + (size_t)kSuspectCap * 8, 256);
  lay.off_cvox = off;
  off = align_up(off + (size_t)v * 4, 256);
  lay.off_overflow = off;
  off = align_up(off + (size_t)L * 4, 256);
  lay.off_best = off;
  off = align_up(off + (size_t)L * 4, 256);
  lay.off_const = off;
  off = align_up(off + sizeof(ConstInfo), 256);
  lay.off_counters = off;
  off = align_up(off + sizeof(NaiveCounters), 256);
  lay.total = off;
  return lay;
}

// RapidPT completion tiles (K4 on tcgen05): fp16 S-only pipeline over
// B permutation rows x v voxels with K = r.  Returns stages = 0 when r does
// not fit the resident A tile.
NaiveLayout complete_layout(int64_t v, int r, int64_t B, int sm_count) {
  NaiveLayout lay{};
  lay.kpad = (r + 15) / 16 * 16;
  lay.vt = 2 * kTileV;
  lay.n_vtiles = (int)((v + lay.vt - 1) / lay.vt);
  lay.cg = lay.kpad >= 192 ? 2 : 1;
  if (!pick_pipeline(lay.cg, lay.kpad, &lay.bk, &lay.stages)) {
    lay.cg = 1;
    if (!pick_pipeline(1, lay.kpad, &lay.bk, &lay.stages)) {
      lay.stages = 0;
      return lay;
    }
  }
  lay.groups = 4;
  const int tile_perms = kTileM * lay.cg;
  lay.n_mtiles = (int)((B + tile_perms - 1) / tile_perms);
  const int n_clusters = std::max(1, sm_count / lay.cg);
  // chunks: enough units for the persistent grid to balance (>= 6 per cluster)
  int c = 1;
  while (c < lay.n_vtiles && (int64_t)lay.n_mtiles * c < 6LL * n_clusters) c *= 2;
  lay.n_ramp = 0;
  lay.ramp_start[0] = 0;
  lay.tiles_per_chunk = (lay.n_vtiles + c - 1) / c;
  lay.n_chunks = (lay.n_vtiles + lay.tiles_per_chunk - 1) / lay.tiles_per_chunk;
  lay.grid = lay.cg * (int)std::min<int64_t>(n_clusters, (int64_t)lay.n_mtiles * lay.n_chunks);
  return lay;
}

namespace {

int gcd_i(int x, int y) {
  while (y) {
    const int r = x % y;
    x = y;
    y = r;
  }
  return x;
}

// largest stride <= 0.618 T coprime with T (golden-ratio sweep order)
int golden_stride(int T) {
  if (T <= 2) return 1;
  for (int s = (int)(0.6180339887 * T); s > 1; --s)
    if (gcd_i(s, T) == 1) return s;
  return 1;
}

struct Ws {
  NaiveLayout lay;
  uint8_t* base;
  __half* planes() const { return reinterpret_cast<__half*>(base + lay.off_planes); }
  uint8_t* planes8() const { return base + lay.off_planes; }
  float* scale() const { return reinterpret_cast<float*>(base + lay.off_scale); }
  uint32_t* gmask() const { return reinterpret_cast<uint32_t*>(base + lay.off_gmask); }
  int4* cand() const { return reinterpret_cast<int4*>(base + lay.off_cand); }
  int32_t* susp() const { return reinterpret_cast<int32_t*>(base + lay.off_susp); }
  int32_t* cvox() const { return reinterpret_cast<int32_t*>(base + lay.off_cvox); }
  int32_t* overflow() const { return reinterpret_cast<int32_t*>(base + lay.off_overflow); }
  uint32_t* best() const { return reinterpret_cast<uint32_t*>(base + lay.off_best); }
  ConstInfo* cinfo() const { return reinterpret_cast<ConstInfo*>(base + lay.off_const); }
  NaiveCounters* counters() const { return reinterpret_cast<NaiveCounters*>(base + lay.off_counters); }
};

int get_ws(int64_t v, int32_t n, int32_t n1, int64_t L, void* workspace, size_t bytes, Ws* ws,
           rmx_status* st) {
  ws->lay = naive_layout(v, n, n1, L, device_sm_count());
  ws->base = static_cast<uint8_t*>(workspace);
  if (!workspace || bytes < ws->lay.total)
    return set_status(st, RMX_E_USAGE, "workspace of %zu bytes is smaller than the %zu required",
                      bytes, ws->lay.total);
  return RMX_OK;
}

// exhaustive exact fp64 evaluation of `nperm` perms (list or all) -> max/argmax
int run_exhaustive(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                   const int32_t* perm_list, int64_t nperm, int two_sided, double* max_out,
                   int32_t* argmax_out, NaiveCounters* counters, cudaStream_t s, rmx_status* st) {
  if (nperm <= 0) return RMX_OK;
  double* xt = nullptr;
  double* pv = nullptr;
  int32_t* pi = nullptr;
  // voxel stripes per permutation: enough blocks to fill the GPU even when
  // only a few permutations overflowed (one thread per voxel)
  int64_t nvb64 = std::min<int64_t>(std::max<int64_t>(1, (v + 4095) / 4096), 64);
  const int64_t fill = (16 * (int64_t)device_sm_count() + nperm - 1) / nperm;
  nvb64 = std::max(nvb64, std::min(fill, (v + 255) / 256));
  const int nvb = (int)std::min<int64_t>(nvb64, 65535);
  // few permutations (the usual overflow case): read X rows directly; many:
  // transpose once so the per-voxel reads coalesce
  const bool transposed = nperm > 64;
  if (transposed) {
    RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xt), (size_t)v * n * sizeof(double), s));
    RMX_CUDA(launch_transpose(x, v, n, xt, s));
  }
  RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pv), (size_t)nperm * nvb * sizeof(double), s));
  RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pi), (size_t)nperm * nvb * sizeof(int32_t), s));
  RMX_CUDA(launch_exact_rows(transposed ? xt : x, v, n, n1, orders, perm_list, nperm, two_sided,
                             nullptr, 0, pv, pi, nvb, counters, s, transposed));
  RMX_CUDA(launch_exact_reduce(pv, pi, nvb, perm_list, nperm, max_out, argmax_out, s));
  if (xt) RMX_CUDA(cudaFreeAsync(xt, s));
  RMX_CUDA(cudaFreeAsync(pv, s));
  RMX_CUDA(cudaFreeAsync(pi, s));
  return RMX_OK;
}

// Report the first degenerate (perm, voxel) if any; fills mean_diff.
int report_degenerate(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                      unsigned long long key, cudaStream_t s, rmx_status* st) {
  if (key == ~0ull) return RMX_OK;
  const int32_t perm = (int32_t)(key >> 32), voxel = (int32_t)(key & 0xffffffffu);
  int32_t* dpair = nullptr;
  double* dt = nullptr;
  RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dpair), 8, s));
  RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dt), 16, s));
  const int32_t hp[2] = {perm, voxel};
  RMX_CUDA(cudaMemcpyAsync(dpair, hp, 8, cudaMemcpyHostToDevice, s));
  RMX_CUDA(launch_pairs(x, v, n, n1, orders, dpair, 1, dt, dt + 1, nullptr, s));
  double h[2] = {0, 0};
  RMX_CUDA(cudaMemcpyAsync(h, dt, 16, cudaMemcpyDeviceToHost, s));
  RMX_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(dpair, s);
  cudaFreeAsync(dt, s);
  st->perm = perm;
  st->voxel = voxel;
  st->value = h[1];
  return set_status(st, RMX_E_DEGENERATE,
                    "voxel %d: zero pooled variance with group mean difference %.6g "
                    "(permutation %d); statistic would be infinite",
                    voxel, h[1], perm);
}

}  // namespace
}  // namespace rmx

using namespace rmx;

extern "C" {

int rmx_abi_version(void) { return RMX_ABI_VERSION; }

// Upload of pageable host memory through the caller's page-locked ring
// (two halves): memcpy into one half while the other half's H2D copy is in
// flight.  For one-shot uploads (RapidPT's X) this avoids page-locking the
// caller's array in place, whose cost (0.3-1 s for 839 MB, variable) sat
// on the critical path before GROUSE.  Returns after the last copy.
int rmx_upload_staged(const void* host, size_t bytes, void* dev, void* ring, size_t ring_bytes,
                      void* stream, rmx_status* st) {
  clear_status(st);
  if ((!host || !dev || !ring) && bytes) return set_status(st, RMX_E_USAGE, "null buffer");
  const size_t half = ring_bytes / 2;
  if (half == 0) return set_status(st, RMX_E_USAGE, "staging ring too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev[2];
  RMX_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  RMX_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  bool used[2] = {false, false};
  int rc = RMX_OK;
  for (size_t off = 0, i = 0; off < bytes; off += half, ++i) {
    const int b = (int)(i & 1);
    const size_t n = std::min(half, bytes - off);
    char* buf = static_cast<char*>(ring) + b * half;
    if (used[b] && cudaEventSynchronize(ev[b]) != cudaSuccess) {
      rc = set_status(st, RMX_E_CUDA, "staged upload failed");
      break;
    }
    memcpy(buf, static_cast<const char*>(host) + off, n);
    if (cudaMemcpyAsync(static_cast<char*>(dev) + off, buf, n, cudaMemcpyHostToDevice, s) !=
            cudaSuccess ||
        cudaEventRecord(ev[b], s) != cudaSuccess) {
      rc = set_status(st, RMX_E_CUDA, "staged upload failed");
      break;
    }
    used[b] = true;
  }
  cudaStreamSynchronize(s);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  return rc;
}

// Page-lock / unlock host memory in place.  Called through ctypes, which
// drops the GIL for the call: registering the 839 MB config-4 matrix takes
// a few hundred ms, during which host threads (the BASIS_INIT normals) keep
// running -- torch's cudart binding holds the GIL for the whole call.
int rmx_host_register(void* ptr, size_t bytes) {
  return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? 0 : 1;
}
int rmx_host_unregister(void* ptr) { return cudaHostUnregister(ptr) == cudaSuccess ? 0 : 1; }

int rmx_device_check(int device, int32_t* sm_count, rmx_status* st) {
  clear_status(st);
  int ndev = 0;
  RMX_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return set_status(st, RMX_E_USAGE, "device %d not present (%d devices)", device, ndev);
  cudaDeviceProp prop;
  RMX_CUDA(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (prop.major != 10)
    return set_status(st, RMX_E_USAGE, "librmx is built for sm_100a; device %d is sm_%d%d (%s)",
                      device, prop.major, prop.minor, prop.name);
  // Host threads that wait for the GPU block instead of spinning (RMX_SYNC_SPIN=1
  // keeps CUDA's default): a spinning waiter on a hyperthread sibling halves
  // the speed of the serial BASIS_INIT draw running beside it, which is
  // GROUSE's critical path.  Applies to the (already active) primary context.
  const char* spin = getenv("RMX_SYNC_SPIN");
  if (!(spin && atoi(spin) == 1)) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur == device)
      cudaSetDeviceFlags(cudaDeviceScheduleBlockingSync);
    cudaGetLastError();  // best effort: an unchangeable flag is not an error
  }
  // The engine's scratch comes from the stream-ordered pool (cudaMallocAsync).
  // By default the pool returns unused memory to the driver at every
  // synchronisation, so each call would map its GB-sized buffers again
  // (physical allocation: tens to hundreds of ms, and variable); keep it
  // cached instead (RMX_POOL_TRIM=1 restores the default).
  const char* trim = getenv("RMX_POOL_TRIM");
  if (!(trim && atoi(trim) == 1)) {
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess && pool) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  return RMX_OK;
}

size_t rmx_naive_workspace_bytes(int64_t v, int32_t n, int64_t L) {
  // the larger of the balanced (S-only) and general layouts
  const int sm = device_sm_count();
  return std::max(naive_layout(v, n, n / 2, L, sm).total, naive_layout(v, n, 2, L, sm).total);
}

}  // extern "C"

namespace {

// K0 pieces: counters reset, rows [v0, v1), constant-voxel reduction
// A priori bound on |S~ - S| for the fp16 hi/lo S-only tiles (balanced
// designs on the fp16 path: configs 1-2).  S = sum_{G1} z with
// sum_all z^2 = n - 1, so sum_{G1} |z| <= sqrt(n1 (n - 1)) =: P.
//  * split: z = hi + lo + delta, |delta| <= 2^-22 |z| + 2^-25 (lo subnormal);
//  * products hi * g, lo * g with g in {0, 1} are exact in fp32;
//  * accumulation: each tcgen05.mma (K = 16) adds at most 2^-22 (|C| + sum
//    |products|) <= 2^-22 1.001 P -- four fp32 ulps of the magnitude sum, a
//    model that covers truncated (non-IEEE) alignment inside the tensor core
//    (tests/test_gpu_naive.py::test_fp16_accumulation_model checks it
//    against adversarial inputs);
// so e = 2^-22 P + n1 2^-25 + (2 kpad / 16 + 1) 2^-22 1.001 P.  Fed to the
// same band machinery as the int8 quantisation bound (band_abs): rigorous.
float fp16_sonly_error_bound(int n, int n1, int kpad) {
  const double P = std::sqrt((double)n1 * (double)(n - 1));
  const double u = std::ldexp(1.0, -22);
  const double nmma = 2.0 * kpad / 16.0;
  const double e = u * P + n1 * std::ldexp(1.0, -25) + (nmma + 1.0) * u * 1.001 * P;
  return (float)(e * 1.01);
}

int prep_init(const Ws& ws, int32_t n, int32_t n1, int64_t L, cudaStream_t s, rmx_status* st) {
  RMX_CUDA(cudaMemsetAsync(ws.counters(), 0, sizeof(NaiveCounters), s));
  RMX_CUDA(cudaMemsetAsync(&ws.counters()->deg_key, 0xff, sizeof(unsigned long long), s));
  if (!ws.lay.i8 && 2 * n1 == n) {  // fp16 S-only: the a priori bound (K0 adds nothing)
    static thread_local float e;  // pageable source: staged before the call returns
    e = fp16_sonly_error_bound(n, n1, ws.lay.kpad);
    RMX_CUDA(cudaMemcpyAsync(&ws.counters()->emax_bits, &e, sizeof(float), cudaMemcpyHostToDevice,
                             s));
  }
  RMX_CUDA(cudaMemsetAsync(ws.best(), 0, (size_t)L * 4, s));
  // int8 scale padding (voxels past v) must be finite: those columns are masked
  if (ws.lay.i8)
    RMX_CUDA(cudaMemsetAsync(ws.scale(), 0, (size_t)ws.lay.n_vtiles * ws.lay.vt * 4, s));
  return RMX_OK;
}

int prep_rows(const double* x, int64_t v, int32_t n, int32_t n1, const Ws& ws, int64_t v0,
              int64_t v1, cudaStream_t s, rmx_status* st) {
  PrepArgs pa{x, v, n, n1, ws.lay.kpad, ws.planes(), ws.cvox(), ws.counters()};
  if (ws.lay.i8) {
    pa.planes8 = ws.planes8();
    pa.inv_scale = ws.scale();
  }
  pa.zplanes_only = (2 * n1 == n) ? 1 : 0;
  pa.v_begin = v0;
  pa.v_end = v1;
  RMX_CUDA(launch_prep(pa, s));
  return RMX_OK;
}

int tfill_impl(int64_t v, int32_t n, int32_t n1, const int16_t* orders, int64_t L,
               int32_t two_sided, float* dbg, void* workspace, size_t workspace_bytes,
               void* stream, rmx_status* st, rmx_naive_stats* stats, int chunk_begin = 0,
               int chunk_end = -1, bool mask_ready = false) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, L, st)) return rc;
  Ws ws;
  if (int rc = get_ws(v, n, n1, L, workspace, workspace_bytes, &ws, st)) return rc;
  if (ws.lay.stages == 0)
    return set_status(st, RMX_E_USAGE,
                      "n=%d subjects exceed the tensor-core tile (A tile > smem); "
                      "use the exact path",
                      n);
  const double dn = n, d1 = n1, d2 = n - n1;
  const double c = (d1 * d2 / dn) * (d1 * d2 / dn);
  const double T = dn - 1.0;  // sum of z^2 over all subjects
  const double alpha = c * (1.0 / (d1 * (d1 - 1.0)) - 1.0 / (d2 * (d2 - 1.0)));
  const double beta = -c * (1.0 / (d1 * d1 * (d1 - 1.0)) + 1.0 / (d2 * d2 * (d2 - 1.0)));
  const double gamma = c * T / (d2 * (d2 - 1.0));
  const double bmax = std::fabs(alpha) * T + std::fabs(beta) * d1 * T + gamma;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!mask_ready)
    RMX_CUDA(launch_group_mask(orders, L, (int64_t)ws.lay.n_mtiles * kTileM * ws.lay.cg, n, n1,
                               ws.lay.mwords, ws.gmask(), s));
  TfillArgs a{};
  a.gmask = ws.gmask();
  a.mwords = ws.lay.mwords;
  a.L = L;
  a.v = v;
  a.n = n;
  a.n1 = n1;
  a.kpad = ws.lay.kpad;
  a.nk16 = ws.lay.kpad / 16;  // MMA K-steps (int8: 2 kpad / 32)
  a.n_vtiles = ws.lay.n_vtiles;
  a.n_mtiles = ws.lay.n_mtiles;
  fill_chunks(ws.lay, &a);
  a.chunk_begin = chunk_begin;
  a.chunk_end = chunk_end < 0 ? ws.lay.n_chunks : chunk_end;
  a.alpha = (float)alpha;
  a.beta = (float)beta;
  a.gamma = (float)gamma;
  a.dthr = (float)(1e-4 * bmax);
  a.band_rel = kBandRel;
  a.beta_abs = (float)std::fabs(beta);
  a.inv_scale = ws.lay.i8 ? ws.scale() : nullptr;
  a.cand = ws.cand();
  a.susp = ws.susp();
  a.best_t = ws.best();
  a.counters = ws.counters();
  a.dbg_t = dbg;
  RMX_CUDA(launch_tfill_tc(ws.lay, a, ws.planes(), two_sided, s));
  if (stats) {
    stats->chunks = ws.lay.n_chunks;
    stats->grid = ws.lay.grid;
    stats->stages = ws.lay.stages;
    stats->bk = ws.lay.bk;
    stats->cg = ws.lay.cg;
    stats->i8 = ws.lay.i8;
  }
  return RMX_OK;
}

}  // namespace

extern "C" {

int rmx_naive_prepare(const double* x, int64_t v, int32_t n, int32_t n1, int64_t L,
                      void* workspace, size_t workspace_bytes, void* stream, rmx_status* st) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, L, st)) return rc;
  Ws ws;
  if (int rc = get_ws(v, n, n1, L, workspace, workspace_bytes, &ws, st)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int rc = prep_init(ws, n, n1, L, s, st)) return rc;
  if (int rc = prep_rows(x, v, n, n1, ws, 0, v, s, st)) return rc;
  RMX_CUDA(launch_const_reduce(x, v, n, n1, ws.cvox(), ws.counters(), ws.cinfo(), s));
  return RMX_OK;
}

int rmx_naive_tfill(int64_t v, int32_t n, int32_t n1, const int16_t* orders, int64_t L,
                    int32_t two_sided, void* workspace, size_t workspace_bytes, void* stream,
                    rmx_status* st, rmx_naive_stats* stats) {
  return tfill_impl(v, n, n1, orders, L, two_sided, nullptr, workspace, workspace_bytes, stream,
                    st, stats);
}

int rmx_naive_tfill_debug(int64_t v, int32_t n, int32_t n1, const int16_t* orders, int64_t L,
                          int32_t two_sided, float* t_dbg, void* workspace,
                          size_t workspace_bytes, void* stream, rmx_status* st) {
  if (!t_dbg) return set_status(st, RMX_E_USAGE, "t_dbg must not be null");
  return tfill_impl(v, n, n1, orders, L, two_sided, t_dbg, workspace, workspace_bytes, stream, st,
                    nullptr);
}

int rmx_naive_finish(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                     int64_t L, int32_t two_sided, double* max_out, int32_t* argmax_out,
                     void* workspace, size_t workspace_bytes, void* stream, rmx_status* st,
                     rmx_naive_stats* stats) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, L, st)) return rc;
  Ws ws;
  if (int rc = get_ws(v, n, n1, L, workspace, workspace_bytes, &ws, st)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RefineArgs ra{};
  ra.x = x;
  ra.orders = orders;
  ra.L = L;
  ra.v = v;
  ra.n = n;
  ra.n1 = n1;
  ra.slots = ws.lay.n_chunks * ws.lay.groups;
  ra.two_sided = two_sided;
  {
    const double dn = n, d1 = n1, d2 = n - n1;
    const double c = (d1 * d2 / dn) * (d1 * d2 / dn);
    ra.band_rel = kBandRel;
    ra.beta_abs = (float)(c * (1.0 / (d1 * d1 * (d1 - 1.0)) + 1.0 / (d2 * d2 * (d2 - 1.0))));
    ra.gamma = (float)(c * (dn - 1.0) / (d2 * (d2 - 1.0)));
  }
  ra.cand = ws.cand();
  ra.susp = ws.susp();
  ra.cinfo = ws.cinfo();
  ra.counters = ws.counters();
  ra.overflow = ws.overflow();
  ra.max_out = max_out;
  ra.argmax_out = argmax_out;
  RMX_CUDA(launch_refine(ra, s));
  NaiveCounters hc;
  RMX_CUDA(read_small_sync(&hc, ws.counters(), sizeof(hc), s));
  int64_t overflow_perms = 0;
  if (hc.susp_count > (unsigned)kSuspectCap) {
    // too many near-degenerate entries to list: exact fp64 evaluation of everything
    if (int rc = run_exhaustive(x, v, n, n1, orders, nullptr, L, two_sided, max_out, argmax_out,
                                ws.counters(), s, st))
      return rc;
    overflow_perms = L;
  } else if (hc.overflow_count > 0) {
    if (int rc = run_exhaustive(x, v, n, n1, orders, ws.overflow(), hc.overflow_count, two_sided,
                                max_out, argmax_out, ws.counters(), s, st))
      return rc;
    overflow_perms = hc.overflow_count;
  }
  if (overflow_perms > 0) {
    RMX_CUDA(read_small_sync(&hc, ws.counters(), sizeof(hc), s));
  }
  if (stats) {
    stats->suspects = hc.susp_count;
    stats->band_candidates = hc.band_candidates;
    stats->rare_groups = (int64_t)hc.rare_groups;
    stats->all_groups = (int64_t)hc.all_groups;
    stats->overflow_perms = overflow_perms;
    stats->chunks = ws.lay.n_chunks;
    stats->grid = ws.lay.grid;
    stats->stages = ws.lay.stages;
    stats->bk = ws.lay.bk;
    stats->cg = ws.lay.cg;
    stats->i8 = ws.lay.i8;
  }
  return report_degenerate(x, v, n, n1, orders, hc.deg_key, s, st);
}

int rmx_naive_maxnull(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                      int64_t L, int32_t two_sided, double* max_out, int32_t* argmax_out,
                      void* workspace, size_t workspace_bytes, void* stream, rmx_status* st,
                      rmx_naive_stats* stats) {
  if (int rc = rmx_naive_prepare(x, v, n, n1, L, workspace, workspace_bytes, stream, st)) return rc;
  Ws ws;
  ws.lay = naive_layout(v, n, n1, L, device_sm_count());
  if (ws.lay.stages == 0) {
    // subject count beyond the tensor-core A tile: exhaustive exact path
    // (still on the GPU; fp64 CUDA cores)
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ws.base = static_cast<uint8_t*>(workspace);
    if (int rc = run_exhaustive(x, v, n, n1, orders, nullptr, L, two_sided, max_out, argmax_out,
                                ws.counters(), s, st))
      return rc;
    NaiveCounters hc;
    RMX_CUDA(read_small_sync(&hc, ws.counters(), sizeof(hc), s));
    if (stats) {
      memset(stats, 0, sizeof(*stats));
      stats->overflow_perms = L;
    }
    return report_degenerate(x, v, n, n1, orders, hc.deg_key, s, st);
  }
  if (int rc = rmx_naive_tfill(v, n, n1, orders, L, two_sided, workspace, workspace_bytes, stream,
                               st, stats))
    return rc;
  return rmx_naive_finish(x, v, n, n1, orders, L, two_sided, max_out, argmax_out, workspace,
                          workspace_bytes, stream, st, stats);
}

}  // extern "C"

namespace rmx {
int golden_stride_public(int T) { return golden_stride(T); }

// fp32 host X (x_host32, staged through x32_dev): each chunk is upcast into
// x_dev on the prep stream before K0 sees it.  Exact: every float32 is a
// float64, so the engine computes on the same values as from a float64 host
// matrix holding the upcast (reference model.py:21-24 makes that upcast).
__global__ void k_upcast(const float* __restrict__ a, int64_t count, double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // float4 / double2 path when both sides are 16-byte aligned (chunk offsets
  // v0 * n need not be)
  const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t c4 = vec ? count >> 2 : 0;
  for (int64_t j = i; j < c4; j += stride) {
    float4 f = reinterpret_cast<const float4*>(a)[j];
    double2* o = reinterpret_cast<double2*>(out) + 2 * j;
    o[0] = make_double2(f.x, f.y);
    o[1] = make_double2(f.z, f.w);
  }
  for (int64_t j = 4 * c4 + i; j < count; j += stride) out[j] = a[j];
}

cudaError_t launch_upcast(const float* a, int64_t count, double* out, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((count / 4 + 255) / 256 + 1, 4 * 148);
  k_upcast<<<blocks, 256, 0, s>>>(a, count, out);
  return cudaGetLastError();
}

}  // namespace rmx

extern "C" {

// Host buffers in, host results out, with the 8 B/entry upload of X overlapped
// with the engine: X is copied chunk by chunk (K1's voxel chunks) on a copy
// stream; K0 standardises each chunk as it lands and K1 runs that chunk's
// units on alternating streams (so one launch's tail overlaps the next's
// head).  The int8 quantisation bound is a running max over the chunks K0
// has finished, which is all K1 needs for chunk c.
namespace {

// orders from the host buffer (orders_host), from the plan seed on the
// device (plan_seed, generated on the prep stream while X's first chunk is
// in flight), or already in orders_dev (both null).  X from x_host (fp64) or
// x_host32 (fp32, staged in x32_dev).
// X streamed from a .mat0 file (rmx_naive_maxnull_mat0): rows are read by
// parallel positional reads into a caller-provided page-locked ring of
// `nslots` slots and copied from there; the host reads piece p + 1 while the
// copy engine moves piece p and the GPU standardises / contracts the
// chunks already landed.  A slot is reused only after its copy completed.
struct FileSrc {
  const char* path = nullptr;
  double* ring = nullptr;
  int64_t slot_rows = 0;
  int nslots = 0;
  int threads = 0;
  int64_t* bad_index = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<bool> used;
  int next = 0;
  ~FileSrc() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
  // rows [r0, r1) of the file -> x_dev (row-major, n columns) on stream cp
  int rows_to_device(int64_t r0, int64_t r1, int32_t n, double* x_dev, cudaStream_t cp,
                     rmx_status* st) {
    if (ev.empty()) {
      ev.resize(nslots);
      used.assign(nslots, false);
      for (auto& e : ev) RMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (int64_t a = r0; a < r1; a += slot_rows) {
      const int64_t b = std::min(r1, a + slot_rows);
      const int slot = next;
      next = (next + 1) % nslots;
      if (used[slot]) RMX_CUDA(cudaEventSynchronize(ev[slot]));
      double* buf = ring + (size_t)slot * slot_rows * n;
      if (int rc = rmx_mat0_read_rows(path, n, a, b, buf, threads, bad_index, st)) return rc;
      RMX_CUDA(cudaMemcpyAsync(x_dev + a * n, buf, (size_t)(b - a) * n * 8,
                               cudaMemcpyHostToDevice, cp));
      RMX_CUDA(cudaEventRecord(ev[slot], cp));
      used[slot] = true;
    }
    return RMX_OK;
  }
};

int naive_host_impl(const double* x_host, const float* x_host32, float* x32_dev, FileSrc* fsrc,
                    int64_t v, int32_t n, int32_t n1,
                    const int16_t* orders_host, const uint64_t* plan_seed, int64_t perm_base,
                    int64_t L, int32_t two_sided, double* max_host, int32_t* argmax_host, double* x_dev,
                    int16_t* orders_dev, double* max_dev, int32_t* argmax_dev, void* workspace,
                    size_t workspace_bytes, void* stream, rmx_status* st,
                    rmx_naive_stats* stats) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, L, st)) return rc;
  if (plan_seed && (n > 32767 || perm_base < 0 || perm_base + L > 0xFFFFFFFFLL))
    return set_status(st, RMX_E_USAGE, "plan of %lld permutations of n=%d not representable",
                      (long long)L, n);
  if ((!x_host && !(x_host32 && x32_dev) && !fsrc) || !max_host || !argmax_host || !x_dev ||
      !orders_dev || !max_dev || !argmax_dev)
    return set_status(st, RMX_E_USAGE, "null buffer");
  if ((reinterpret_cast<uintptr_t>(x_host32) | reinterpret_cast<uintptr_t>(x32_dev)) & 15)
    return set_status(st, RMX_E_USAGE, "fp32 X buffers must be 16-byte aligned");
  Ws ws;
  if (int rc = get_ws(v, n, n1, L, workspace, workspace_bytes, &ws, st)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t xbytes = (size_t)v * n * sizeof(double);
  const size_t obytes = (size_t)L * n * sizeof(int16_t);
  auto finish_host = [&]() -> int {
    RMX_CUDA(cudaMemcpyAsync(max_host, max_dev, (size_t)L * 8, cudaMemcpyDeviceToHost, s));
    RMX_CUDA(cudaMemcpyAsync(argmax_host, argmax_dev, (size_t)L * 4, cudaMemcpyDeviceToHost, s));
    RMX_CUDA(cudaStreamSynchronize(s));
    return RMX_OK;
  };
  if (ws.lay.stages == 0) {  // exhaustive exact path: nothing to overlap
    if (fsrc) {
      if (int rc = fsrc->rows_to_device(0, v, n, x_dev, s, st)) {
        cudaStreamSynchronize(s);
        return rc;
      }
    } else if (x_host) {
      RMX_CUDA(cudaMemcpyAsync(x_dev, x_host, xbytes, cudaMemcpyHostToDevice, s));
    } else {
      RMX_CUDA(cudaMemcpyAsync(x32_dev, x_host32, xbytes / 2, cudaMemcpyHostToDevice, s));
      RMX_CUDA(rmx::launch_upcast(x32_dev, v * n, x_dev, s));
    }
    if (orders_host)
      RMX_CUDA(cudaMemcpyAsync(orders_dev, orders_host, obytes, cudaMemcpyHostToDevice, s));
    if (plan_seed) RMX_CUDA(launch_plan_orders(*plan_seed, perm_base, L, n, orders_dev, s));
    if (int rc = rmx_naive_maxnull(x_dev, v, n, n1, orders_dev, L, two_sided, max_dev, argmax_dev,
                                   workspace, workspace_bytes, stream, st, stats))
      return rc;
    return finish_host();
  }
  // The pipeline's streams and events persist per host thread and device
  // (creating 4 streams and ~2 chunks' worth of events cost a noticeable part
  // of a 35 ms end-to-end call).  Reuse is safe: every call ends with the
  // caller's stream waiting on all of them and a synchronisation.
  struct Streams {
    int dev = -1;
    cudaStream_t cp = nullptr, pp = nullptr, k[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    cudaError_t event(cudaEvent_t* e) {
      if (used < ev.size()) {
        *e = ev[used++];
        return cudaSuccess;
      }
      cudaError_t r = cudaEventCreateWithFlags(e, cudaEventDisableTiming);
      if (r == cudaSuccess) {
        ev.push_back(*e);
        ++used;
      }
      return r;
    }
  };
  static thread_local Streams* tl_streams = nullptr;  // never freed (process lifetime)
  int cur_dev = 0;
  RMX_CUDA(cudaGetDevice(&cur_dev));
  if (!tl_streams || tl_streams->dev != cur_dev) {
    tl_streams = new Streams();
    tl_streams->dev = cur_dev;
    for (cudaStream_t* x : {&tl_streams->cp, &tl_streams->pp, &tl_streams->k[0], &tl_streams->k[1]})
      RMX_CUDA(cudaStreamCreateWithFlags(x, cudaStreamNonBlocking));
  }
  Streams& S = *tl_streams;
  S.used = 0;
  const int nc = ws.lay.n_chunks;
  cudaEvent_t e0, e_ord, e_pdone, e_k[2];
  RMX_CUDA(S.event(&e0));
  RMX_CUDA(S.event(&e_ord));
  RMX_CUDA(S.event(&e_pdone));
  RMX_CUDA(S.event(&e_k[0]));
  RMX_CUDA(S.event(&e_k[1]));
  std::vector<cudaEvent_t> e_rows(nc), e_prep(nc);
  for (int c = 0; c < nc; ++c) {
    RMX_CUDA(S.event(&e_rows[c]));
    RMX_CUDA(S.event(&e_prep[c]));
  }
  // everything starts after the caller's prior work on `stream`
  RMX_CUDA(cudaEventRecord(e0, s));
  for (cudaStream_t x : {S.cp, S.pp, S.k[0], S.k[1]}) RMX_CUDA(cudaStreamWaitEvent(x, e0, 0));
  // copies: labels first (K1 needs them), then X chunk by chunk
  // (orders_host == NULL: the caller generated the labels on the device,
  // stream-ordered before this call)
  if (orders_host)
    RMX_CUDA(cudaMemcpyAsync(orders_dev, orders_host, obytes, cudaMemcpyHostToDevice, S.cp));
  if (plan_seed) {
    RMX_CUDA(launch_plan_orders(*plan_seed, perm_base, L, n, orders_dev, S.pp));
    RMX_CUDA(cudaEventRecord(e_ord, S.pp));
  } else {
    RMX_CUDA(cudaEventRecord(e_ord, S.cp));
  }
  if (int rc = prep_init(ws, n, n1, L, S.pp, st)) return rc;
  // the labels' bit rows, once, ahead of every chunk's K1 (both K1 streams)
  RMX_CUDA(cudaStreamWaitEvent(S.k[0], e_ord, 0));
  RMX_CUDA(launch_group_mask(orders_dev, L, (int64_t)ws.lay.n_mtiles * kTileM * ws.lay.cg, n, n1,
                             ws.lay.mwords, ws.gmask(), S.k[0]));
  RMX_CUDA(cudaEventRecord(e_ord, S.k[0]));
  RMX_CUDA(cudaStreamWaitEvent(S.k[1], e_ord, 0));
  // chunk c: its rows' copy (after the host read them, for a file), then K0
  // and K1 on them; enqueued chunk by chunk so a file's reads overlap the
  // copies and the engine work of the chunks before
  for (int c = 0; c < nc; ++c) {
    int64_t v0, v1;
    chunk_voxels(ws.lay, v, c, &v0, &v1);
    if (v1 > v0 && fsrc) {
      if (int rc = fsrc->rows_to_device(v0, v1, n, x_dev, S.cp, st)) {
        for (cudaStream_t x : {S.cp, S.pp, S.k[0], S.k[1]}) cudaStreamSynchronize(x);
        return rc;
      }
    } else if (v1 > v0 && x_host) {
      RMX_CUDA(cudaMemcpyAsync(x_dev + v0 * n, x_host + v0 * n, (size_t)(v1 - v0) * n * 8,
                               cudaMemcpyHostToDevice, S.cp));
    } else if (v1 > v0) {
      RMX_CUDA(cudaMemcpyAsync(x32_dev + v0 * n, x_host32 + v0 * n, (size_t)(v1 - v0) * n * 4,
                               cudaMemcpyHostToDevice, S.cp));
    }
    RMX_CUDA(cudaEventRecord(e_rows[c], S.cp));
    RMX_CUDA(cudaStreamWaitEvent(S.pp, e_rows[c], 0));
    if (!x_host && !fsrc)
      RMX_CUDA(rmx::launch_upcast(x32_dev + v0 * n, (v1 - v0) * n, x_dev + v0 * n, S.pp));
    if (int rc = prep_rows(x_dev, v, n, n1, ws, v0, v1, S.pp, st)) return rc;
    RMX_CUDA(cudaEventRecord(e_prep[c], S.pp));
    cudaStream_t ks = S.k[c & 1];
    RMX_CUDA(cudaStreamWaitEvent(ks, e_prep[c], 0));
    if (int rc = tfill_impl(v, n, n1, orders_dev, L, two_sided, nullptr, workspace,
                            workspace_bytes, ks, st, stats, c, c + 1, /*mask_ready=*/true))
      return rc;
  }
  RMX_CUDA(launch_const_reduce(x_dev, v, n, n1, ws.cvox(), ws.counters(), ws.cinfo(), S.pp));
  RMX_CUDA(cudaEventRecord(e_pdone, S.pp));
  RMX_CUDA(cudaEventRecord(e_k[0], S.k[0]));
  RMX_CUDA(cudaEventRecord(e_k[1], S.k[1]));
  for (cudaEvent_t e : {e_pdone, e_k[0], e_k[1]}) RMX_CUDA(cudaStreamWaitEvent(s, e, 0));
  if (int rc = rmx_naive_finish(x_dev, v, n, n1, orders_dev, L, two_sided, max_dev, argmax_dev,
                                workspace, workspace_bytes, stream, st, stats))
    return rc;
  return finish_host();
}

}  // namespace

int rmx_naive_maxnull_host(const double* x_host, int64_t v, int32_t n, int32_t n1,
                           const int16_t* orders_host, int64_t L, int32_t two_sided,
                           double* max_host, int32_t* argmax_host, double* x_dev,
                           int16_t* orders_dev, double* max_dev, int32_t* argmax_dev,
                           void* workspace, size_t workspace_bytes, void* stream,
                           rmx_status* st, rmx_naive_stats* stats) {
  return naive_host_impl(x_host, nullptr, nullptr, nullptr, v, n, n1, orders_host, nullptr, 0, L, two_sided, max_host,
                         argmax_host, x_dev, orders_dev, max_dev, argmax_dev, workspace,
                         workspace_bytes, stream, st, stats);
}

int rmx_naive_maxnull_host_plan(const double* x_host, int64_t v, int32_t n, int32_t n1,
                                uint64_t plan_seed, int64_t L, int32_t two_sided,
                                double* max_host, int32_t* argmax_host, double* x_dev,
                                int16_t* orders_dev, double* max_dev, int32_t* argmax_dev,
                                void* workspace, size_t workspace_bytes, void* stream,
                                rmx_status* st, rmx_naive_stats* stats) {
  return naive_host_impl(x_host, nullptr, nullptr, nullptr, v, n, n1, nullptr, &plan_seed, 0, L, two_sided, max_host,
                         argmax_host, x_dev, orders_dev, max_dev, argmax_dev, workspace,
                         workspace_bytes, stream, st, stats);
}

int rmx_naive_maxnull_host_f32(const float* x_host, int64_t v, int32_t n, int32_t n1,
                               const int16_t* orders_host, int64_t L, int32_t two_sided,
                               double* max_host, int32_t* argmax_host, float* x32_dev,
                               double* x_dev, int16_t* orders_dev, double* max_dev,
                               int32_t* argmax_dev, void* workspace, size_t workspace_bytes,
                               void* stream, rmx_status* st, rmx_naive_stats* stats) {
  if (!x_host) return set_status(st, RMX_E_USAGE, "null buffer");
  return naive_host_impl(nullptr, x_host, x32_dev, nullptr, v, n, n1, orders_host, nullptr, 0, L, two_sided,
                         max_host, argmax_host, x_dev, orders_dev, max_dev, argmax_dev, workspace,
                         workspace_bytes, stream, st, stats);
}

int rmx_naive_maxnull_host_plan_f32(const float* x_host, int64_t v, int32_t n, int32_t n1,
                                    uint64_t plan_seed, int64_t L, int32_t two_sided,
                                    double* max_host, int32_t* argmax_host, float* x32_dev,
                                    double* x_dev, int16_t* orders_dev, double* max_dev,
                                    int32_t* argmax_dev, void* workspace, size_t workspace_bytes,
                                    void* stream, rmx_status* st, rmx_naive_stats* stats) {
  if (!x_host) return set_status(st, RMX_E_USAGE, "null buffer");
  return naive_host_impl(nullptr, x_host, x32_dev, nullptr, v, n, n1, nullptr, &plan_seed, 0, L, two_sided,
                         max_host, argmax_host, x_dev, orders_dev, max_dev, argmax_dev, workspace,
                         workspace_bytes, stream, st, stats);
}

int rmx_naive_maxnull_host_plan_range(const double* x_host, int64_t v, int32_t n, int32_t n1,
                                      uint64_t plan_seed, int64_t perm_base, int64_t L,
                                      int32_t two_sided, double* max_host, int32_t* argmax_host,
                                      double* x_dev, int16_t* orders_dev, double* max_dev,
                                      int32_t* argmax_dev, void* workspace,
                                      size_t workspace_bytes, void* stream, rmx_status* st,
                                      rmx_naive_stats* stats) {
  return naive_host_impl(x_host, nullptr, nullptr, nullptr, v, n, n1, nullptr, &plan_seed, perm_base, L,
                         two_sided, max_host, argmax_host, x_dev, orders_dev, max_dev, argmax_dev,
                         workspace, workspace_bytes, stream, st, stats);
}

int rmx_naive_maxnull_host_plan_range_f32(const float* x_host, int64_t v, int32_t n, int32_t n1,
                                          uint64_t plan_seed, int64_t perm_base, int64_t L,
                                          int32_t two_sided, double* max_host,
                                          int32_t* argmax_host, float* x32_dev, double* x_dev,
                                          int16_t* orders_dev, double* max_dev,
                                          int32_t* argmax_dev, void* workspace,
                                          size_t workspace_bytes, void* stream, rmx_status* st,
                                          rmx_naive_stats* stats) {
  if (!x_host) return set_status(st, RMX_E_USAGE, "null buffer");
  return naive_host_impl(nullptr, x_host, x32_dev, nullptr, v, n, n1, nullptr, &plan_seed, perm_base, L,
                         two_sided, max_host, argmax_host, x_dev, orders_dev, max_dev, argmax_dev,
                         workspace, workspace_bytes, stream, st, stats);
}

int rmx_naive_maxnull_mat0(const char* path, int64_t v, int32_t n, int32_t n1,
                           uint64_t plan_seed, int64_t perm_base, int64_t L, int32_t two_sided,
                           double* max_host, int32_t* argmax_host, double* ring_host,
                           size_t ring_bytes, int32_t threads, int64_t* bad_index, double* x_dev,
                           int16_t* orders_dev, double* max_dev, int32_t* argmax_dev,
                           void* workspace, size_t workspace_bytes, void* stream,
                           rmx_status* st, rmx_naive_stats* stats) {
  clear_status(st);
  if (bad_index) *bad_index = -1;
  if (!path || !ring_host) return set_status(st, RMX_E_USAGE, "null buffer");
  FileSrc fs;
  fs.path = path;
  fs.ring = ring_host;
  fs.threads = threads;
  fs.bad_index = bad_index;
  const int64_t row_bytes = (int64_t)n * 8;
  fs.nslots = (int64_t)ring_bytes / row_bytes >= 3 * 1024 ? 3 : 2;
  fs.slot_rows = std::min<int64_t>((int64_t)ring_bytes / fs.nslots / std::max<int64_t>(1, row_bytes), v);
  if (n < 1 || fs.slot_rows < 1)
    return set_status(st, RMX_E_USAGE, "staging ring of %zu bytes holds no %d-column row",
                      ring_bytes, n);
  return naive_host_impl(nullptr, nullptr, nullptr, &fs, v, n, n1, nullptr, &plan_seed, perm_base,
                         L, two_sided, max_host, argmax_host, x_dev, orders_dev, max_dev,
                         argmax_dev, workspace, workspace_bytes, stream, st, stats);
}

int rmx_tstat_dump_mat0(const double* x_dev, int64_t v, int32_t n, int32_t n1,
                        const int16_t* orders_dev, int64_t L, const char* path, double* ring_host,
                        size_t ring_bytes, int32_t threads, void* stream, rmx_status* st) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, L, st)) return rc;
  if (!x_dev || !orders_dev || !path || !ring_host)
    return set_status(st, RMX_E_USAGE, "null buffer");
  // voxel slabs of `rows` voxels x all L permutations: one slab is a
  // contiguous run of the (v, L) row-major payload.  Two host slots: the
  // GPU computes + copies slab b while the host writes slab b - 1.
  const int64_t rows = std::min<int64_t>(v, (int64_t)(ring_bytes / 2) / (L * 8));
  if (rows < 1)
    return set_status(st, RMX_E_USAGE,
                      "staging ring of %zu bytes holds no two %lld-permutation voxel rows",
                      ring_bytes, (long long)L);
  if (int rc = rmx_mat0_create(path, v, L, 0, 0, st)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  struct Dev {
    double *xt = nullptr, *tp = nullptr, *tv = nullptr;
    NaiveCounters* c = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t s = nullptr;
    ~Dev() {
      if (s) cudaStreamSynchronize(s);
      for (void* p : {(void*)xt, (void*)tp, (void*)tv, (void*)c})
        if (p) cudaFree(p);
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    }
  } d;
  d.s = s;
  RMX_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.xt), (size_t)rows * n * 8));
  RMX_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.tp), (size_t)rows * L * 8));
  RMX_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.tv), (size_t)rows * L * 8));
  RMX_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.c), sizeof(NaiveCounters)));
  for (auto& e : d.ev) RMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const int64_t nslab = (v + rows - 1) / rows;
  auto write_slab = [&](int64_t b) -> int {
    const int64_t v0 = b * rows, v1 = std::min(v, v0 + rows);
    RMX_CUDA(cudaEventSynchronize(d.ev[b & 1]));
    return rmx_mat0_write_rows(path, L, v0, v1, ring_host + (size_t)(b & 1) * rows * L, threads,
                               st);
  };
  for (int64_t b = 0; b < nslab; ++b) {
    const int64_t v0 = b * rows, v1 = std::min(v, v0 + rows), nv = v1 - v0;
    RMX_CUDA(cudaMemsetAsync(d.c, 0, sizeof(NaiveCounters), s));
    RMX_CUDA(cudaMemsetAsync(&d.c->deg_key, 0xff, sizeof(unsigned long long), s));
    // the slab's X^T (n x nv), its L x nv statistics (k_exact_rows: numpy's
    // pairwise sums, the reference's bits), then (nv x L) for the file
    RMX_CUDA(launch_transpose(x_dev + v0 * n, nv, n, d.xt, s));
    const int nvb = (int)std::max<int64_t>(1, std::min<int64_t>((nv + 1023) / 1024, 1024));
    RMX_CUDA(launch_exact_rows(d.xt, nv, n, n1, orders_dev, nullptr, L, 0, d.tp, nv, nullptr,
                               nullptr, nvb, d.c, s));
    RMX_CUDA(launch_transpose(d.tp, L, (int)nv, d.tv, s));
    RMX_CUDA(cudaMemcpyAsync(ring_host + (size_t)(b & 1) * rows * L, d.tv, (size_t)nv * L * 8,
                             cudaMemcpyDeviceToHost, s));
    unsigned long long key = 0;
    RMX_CUDA(cudaMemcpyAsync(&key, &d.c->deg_key, 8, cudaMemcpyDeviceToHost, s));
    RMX_CUDA(cudaEventRecord(d.ev[b & 1], s));
    if (b > 0)
      if (int rc = write_slab(b - 1)) return rc;
    RMX_CUDA(cudaEventSynchronize(d.ev[b & 1]));
    if (key != ~0ull) {  // a degenerate entry: the reference raises before writing
      const int rc = report_degenerate(x_dev + v0 * n, nv, n, n1, orders_dev, key, s, st);
      st->voxel += v0;
      set_status(st, rc,
                 "voxel %lld: zero pooled variance with group mean difference %.6g "
                 "(permutation %lld); statistic would be infinite",
                 (long long)st->voxel, st->value, (long long)st->perm);
      unlink(path);
      return rc;
    }
  }
  return write_slab(nslab - 1);
}

int rmx_plan_orders(uint64_t seed, int64_t lo, int64_t count, int32_t n, int16_t* out,
                    void* stream, rmx_status* st) {
  clear_status(st);
  if (n < 1 || n > 32767 || lo < 0 || count < 0 || lo + count > 0xFFFFFFFFLL || !out)
    return set_status(st, RMX_E_USAGE, "plan rows [%lld, %lld) of n=%d not representable",
                      (long long)lo, (long long)(lo + count), n);
  RMX_CUDA(launch_plan_orders(seed, lo, count, n, out, static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

int rmx_omega_draws(uint64_t seed, int32_t domain, int64_t lo, int64_t count, int64_t extra,
                    int64_t v, int32_t k, int32_t* out, void* stream, rmx_status* st) {
  clear_status(st);
  if (k < 1 || v < k || v > 0xFFFFFFFFLL || lo < 0 || lo + count > 0xFFFFFFFFLL || extra > 0xFFFFFFFFLL ||
      domain < 0 || !out)
    return set_status(st, RMX_E_USAGE, "observation draws out of range (v=%lld, k=%d)",
                      (long long)v, k);
  if (v > 10000 && k > v / 50)  // numpy's tail-shuffle branch: not on the device
    return set_status(st, RMX_E_USAGE, "k=%d of v=%lld takes numpy's tail-shuffle branch", k,
                      (long long)v);
  RMX_CUDA(launch_omega_draws(seed, (uint32_t)domain, lo, count, extra >= 0 ? 1 : 0,
                              (uint32_t)(extra >= 0 ? extra : 0), (uint32_t)v, k, out,
                              static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

int rmx_tstat_exact(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                    int64_t L, double* t_out, int64_t ld, void* stream, rmx_status* st) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, L, st)) return rc;
  if (!t_out || ld < v) return set_status(st, RMX_E_USAGE, "t_out must hold L rows of ld >= v");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* xt = nullptr;
  NaiveCounters* c = nullptr;
  // many labellings: the voxel-staged kernel reads X once per chunk of
  // labellings (RMX_EXACT_VSTAGE=0: the thread-per-voxel kernel over X^T)
  const char* vs_env = getenv("RMX_EXACT_VSTAGE");
  if (L >= 16 && exact_rows_vstage_supported(n) && !(vs_env && atoi(vs_env) == 0)) {
    RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c), sizeof(NaiveCounters), s));
    RMX_CUDA(cudaMemsetAsync(c, 0, sizeof(NaiveCounters), s));
    RMX_CUDA(cudaMemsetAsync(&c->deg_key, 0xff, sizeof(unsigned long long), s));
    RMX_CUDA(launch_exact_rows_vstage(x, v, n, n1, orders, L, t_out, ld, c, s));
    NaiveCounters hv;
    RMX_CUDA(read_small_sync(&hv, c, sizeof(hv), s));
    cudaFreeAsync(c, s);
    return report_degenerate(x, v, n, n1, orders, hv.deg_key, s, st);
  }
  RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xt), (size_t)v * n * sizeof(double), s));
  RMX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c), sizeof(NaiveCounters), s));
  RMX_CUDA(cudaMemsetAsync(c, 0, sizeof(NaiveCounters), s));
  RMX_CUDA(cudaMemsetAsync(&c->deg_key, 0xff, sizeof(unsigned long long), s));
  RMX_CUDA(launch_transpose(x, v, n, xt, s));
  const int nvb = (int)std::max<int64_t>(1, std::min<int64_t>((v + 1023) / 1024, 1024));
  RMX_CUDA(launch_exact_rows(xt, v, n, n1, orders, nullptr, L, 0, t_out, ld, nullptr, nullptr, nvb,
                             c, s));
  NaiveCounters hc;
  RMX_CUDA(read_small_sync(&hc, c, sizeof(hc), s));
  cudaFreeAsync(xt, s);
  cudaFreeAsync(c, s);
  return report_degenerate(x, v, n, n1, orders, hc.deg_key, s, st);
}

int rmx_tstat_pairs(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                    const int32_t* pairs, int64_t npairs, double* t_out, double* num_out,
                    int32_t* deg_out, void* stream, rmx_status* st) {
  clear_status(st);
  if (int rc = check_dims(v, n, n1, 1, st)) return rc;
  RMX_CUDA(launch_pairs(x, v, n, n1, orders, pairs, npairs, t_out, num_out, deg_out,
                        static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

}  // extern "C"
