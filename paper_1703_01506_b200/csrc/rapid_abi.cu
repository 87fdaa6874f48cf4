// rapid_abi.cu -- extern "C" RapidPT entry points (include/rmx.h) and the
// native GROUSE training loop (reference lrmc.py:208-268).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <vector>

#include "../../include/rmx.h"
#include "rapid_internal.cuh"
#include "rmx_internal.cuh"

namespace rmx {
namespace {

int rset(rmx_status* st, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
int rset(rmx_status* st, int code, const char* fmt, ...) {
  if (st) {
    st->code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

void rclear(rmx_status* st) {
  if (!st) return;
  memset(st, 0, sizeof(*st));
  st->perm = -1;
  st->voxel = -1;
}

#define RCUDA(call)                                                                  \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess)                                                           \
      return rset(st, RMX_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(_e));   \
  } while (0)

constexpr double kCondLimit = 1e12;  // lrmc.py:22 COND_LIMIT

size_t gram_bytes(int r) { return (size_t)(r + 1) * (r + 1) * sizeof(double); }

template <class T>
struct DevBuf {  // stream-ordered scratch
  T* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t st) {
    s = st;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace
}  // namespace rmx

using namespace rmx;

extern "C" {

int rmx_rapid_stats(const double* x, int64_t v, int32_t n, int32_t n1, const int16_t* orders,
                    const int32_t* omegas, int64_t L, int32_t k, double* t_out, void* stream,
                    rmx_status* st) {
  rclear(st);
  if (v < 1 || n1 < 2 || n - n1 < 2 || k < 1 || k > v || L < 1)
    return rset(st, RMX_E_USAGE, "bad dimensions v=%lld n=%d n1=%d k=%d L=%lld", (long long)v, n,
                n1, k, (long long)L);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevBuf<unsigned long long> key;
  RCUDA(key.alloc(1, s));
  RCUDA(cudaMemsetAsync(key.p, 0xff, sizeof(unsigned long long), s));
  RCUDA(launch_rapid_stats(x, n, n1, orders, omegas, L, k, t_out, key.p, s));
  unsigned long long hk = 0;
  RCUDA(read_small_sync(&hk, key.p, sizeof(hk), s));
  if (hk != ~0ull) {
    st->perm = (int64_t)(hk >> 32);
    st->voxel = (int64_t)(hk & 0xffffffffu);  // index into the permutation's Omega
    return rset(st, RMX_E_DEGENERATE, "zero pooled variance at permutation %lld, Omega index %lld",
                (long long)st->perm, (long long)st->voxel);
  }
  return RMX_OK;
}

size_t rmx_lsq_workspace_bytes(int32_t r, int64_t batch) {
  return (size_t)batch * gram_bytes(r) + (size_t)batch * 4 * sizeof(double) + 256;
}

int rmx_lsq_solve(const double* u, int64_t ldu, int32_t r, const int32_t* idx, int32_t k,
                  const double* vals, int64_t B, double* w_out, int32_t* flag_out,
                  double* norms_out, void* workspace, size_t workspace_bytes, void* stream,
                  rmx_status* st) {
  rclear(st);
  if (r < 1 || k < r || B < 1 || !vals || !w_out)
    return rset(st, RMX_E_USAGE, "%d observed rows cannot determine %d coefficients", k, r);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t per = gram_bytes(r);
  int64_t chunk = (int64_t)((workspace_bytes > 256 ? workspace_bytes - 256 : 0) /
                            (per + 4 * sizeof(double)));
  if (chunk < 1) return rset(st, RMX_E_USAGE, "lsq workspace too small");
  chunk = std::min<int64_t>(chunk, B);
  double* G = static_cast<double*>(workspace);
  double* nrm = reinterpret_cast<double*>(static_cast<uint8_t*>(workspace) + chunk * per);
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t cnt = std::min(chunk, B - b0);
    RCUDA(launch_gram(u, ldu, r, idx ? idx + b0 * k : nullptr, k, vals + b0 * k, G, cnt, s));
    RCUDA(launch_chol_solve(G, r, cnt, w_out + b0 * r, flag_out ? flag_out + b0 : nullptr,
                            norms_out ? norms_out + 4 * b0 : nrm, s));
  }
  return RMX_OK;
}

// Reference-semantics batched LS (lrmc.py:127-149 solve_block, and the
// cond > COND_LIMIT test of _gram_fit / fit_coefficients): the fp64 Gram of
// [U_Omega | vals]; cond = sqrt(lambda_max / lambda_min) of its r x r block
// from k_sym_extreme_eigs (inf when lambda_min <= 0); accepted systems are
// solved by Cholesky, or by pivoted LU (np.linalg.solve's algorithm) when
// the Cholesky meets a non-positive pivot; rejected systems (cond > 1e12)
// get w = U_Omega^T vals, the reference's solve against the identity.
}  // extern "C"

namespace {

// Pivot ratio max L_ii / min L_ii of the Gram's Cholesky factor (a lower
// bound of cond(U_Omega)) above which a system's condition number is
// evaluated exactly (the reference's decision needs it only near 1e12; the
// restrictions of a random row sample sit at ~2-10).
constexpr double kBorderRatio = 1e4;

// exact_all: every system's cond exactly (public solve_block semantics);
// else only the Cholesky-flagged or borderline ones (internal fits).
int lsq_exact_impl(const double* u, int64_t ldu, int32_t r, const int32_t* idx, int32_t k,
                   const double* vals, int64_t B, double* w_out, int32_t* flag_out,
                   double* cond_out, bool exact_all, cudaStream_t s, rmx_status* st) {
  const int64_t ld = r + 1;
  const size_t per = gram_bytes(r) + (exact_all ? sym_extreme_eigs_work(r, 1) : 0) +
                     8 * sizeof(double);
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, ((int64_t)1 << 30) / (int64_t)per));
  DevBuf<double> G, work, lam, nrm;
  DevBuf<int32_t> cflag, sel;
  RCUDA(G.alloc((size_t)chunk * ld * ld, s));
  const size_t wbytes = std::max(sym_extreme_eigs_work(r, exact_all ? chunk : 1),
                                 lu_solve_work(r, 1));
  RCUDA(work.alloc(wbytes / 8 + 1, s));
  RCUDA(lam.alloc((size_t)2 * chunk, s));
  RCUDA(nrm.alloc((size_t)4 * chunk, s));
  RCUDA(cflag.alloc((size_t)chunk, s));
  RCUDA(sel.alloc(1, s));
  const int32_t zero = 0;
  RCUDA(cudaMemcpyAsync(sel.p, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  std::vector<double> hl((size_t)2 * chunk), hn((size_t)4 * chunk);
  std::vector<int32_t> hf((size_t)chunk);
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t cnt = std::min(chunk, B - b0);
    const int32_t* ib = idx ? idx + b0 * k : nullptr;
    RCUDA(launch_gram(u, ldu, r, ib, k, vals + b0 * k, G.p, cnt, s));
    if (exact_all)
      RCUDA(launch_sym_extreme_eigs(G.p, ld * ld, (int)ld, r, nullptr, cnt, work.p, lam.p, s));
    RCUDA(launch_chol_solve(G.p, r, cnt, w_out + b0 * r, cflag.p, nrm.p, s));
    if (exact_all)
      RCUDA(cudaMemcpyAsync(hl.data(), lam.p, (size_t)2 * cnt * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    RCUDA(cudaMemcpyAsync(hn.data(), nrm.p, (size_t)4 * cnt * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
    RCUDA(cudaMemcpyAsync(hf.data(), cflag.p, (size_t)cnt * sizeof(int32_t),
                          cudaMemcpyDeviceToHost, s));
    RCUDA(cudaStreamSynchronize(s));
    for (int64_t j = 0; j < cnt; ++j) {
      const int64_t b = b0 + j;
      const double ratio = hn[4 * j + 2] > 0.0 ? hn[4 * j + 3] / hn[4 * j + 2] : INFINITY;
      const bool known = exact_all;
      const bool need = hf[j] != 0 || !(ratio <= kBorderRatio);
      double c = ratio;  // a lower bound, exact below
      bool reform = false;
      if (known) {
        const double lo = hl[2 * j], hi = hl[2 * j + 1];
        c = lo > 0.0 ? std::sqrt(hi / lo) : INFINITY;
      } else if (need) {  // borderline: this system's exact cond (re-form its Gram)
        RCUDA(launch_gram(u, ldu, r, idx ? idx + b * k : nullptr, k, vals + b * k, G.p, 1, s));
        RCUDA(launch_sym_extreme_eigs(G.p, ld * ld, (int)ld, r, sel.p, 1, work.p, lam.p, s));
        double l2[2];
        RCUDA(cudaMemcpyAsync(l2, lam.p, sizeof(l2), cudaMemcpyDeviceToHost, s));
        RCUDA(cudaStreamSynchronize(s));
        c = l2[0] > 0.0 ? std::sqrt(l2[1] / l2[0]) : INFINITY;
        reform = true;
      }
      if (cond_out) cond_out[b] = c;
      const bool bad = !(c <= kCondLimit);
      if (flag_out) flag_out[b] = bad ? 1 : 0;
      if (!bad && hf[j] == 0) continue;
      // rare: LU (accepted, Cholesky failed) or w = rhs (rejected)
      if (!reform)
        RCUDA(launch_gram(u, ldu, r, idx ? idx + b * k : nullptr, k, vals + b * k, G.p, 1, s));
      if (bad) {
        RCUDA(cudaMemcpyAsync(w_out + b * r, G.p + (int64_t)r * ld, (size_t)r * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
      } else {
        RCUDA(launch_lu_solve(G.p, ld * ld, (int)ld, r, sel.p, 1, work.p, w_out + b * r, nullptr,
                              s));
      }
      RCUDA(cudaStreamSynchronize(s));
    }
  }
  return RMX_OK;
}

}  // namespace

extern "C" {

int rmx_lsq_solve_exact(const double* u, int64_t ldu, int32_t r, const int32_t* idx, int32_t k,
                        const double* vals, int64_t B, double* w_out, int32_t* flag_out,
                        double* cond_out, void* stream, rmx_status* st) {
  rclear(st);
  if (r < 1 || k < r || B < 1 || !vals || !w_out)
    return rset(st, RMX_E_USAGE, "%d observed rows cannot determine %d coefficients", k, r);
  return lsq_exact_impl(u, ldu, r, idx, k, vals, B, w_out, flag_out, cond_out, true,
                        static_cast<cudaStream_t>(stream), st);
}

// One GROUSE update (lrmc.py:160-193 track_update) on a device basis U (v x
// r, row-major, updated in place); idx (sorted) / vals: the observed column
// on the device.  *resid_norm = |vals - U_Omega w| before the update.
int rmx_track_update(double* u, int64_t v, int32_t r, const int32_t* idx, int32_t k,
                     const double* vals, double step, double* resid_norm, void* stream,
                     rmx_status* st) {
  rclear(st);
  if (k < r)
    return rset(st, RMX_E_USAGE, "%d observed rows cannot determine %d coefficients", k, r);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevBuf<double> w, resid, pred, sums;
  RCUDA(w.alloc((size_t)r, s));
  RCUDA(resid.alloc((size_t)k, s));
  RCUDA(pred.alloc((size_t)v, s));
  RCUDA(sums.alloc(8, s));
  int32_t bad = 0;
  double cond = 0.0;
  if (int rc = rmx_lsq_solve_exact(u, r, r, idx, k, vals, 1, w.p, &bad, &cond, stream, st))
    return rc;
  if (bad) {
    st->value = cond;
    return rset(st, RMX_E_ILLCOND, "restricted basis condition number %.3e exceeds 1e12", cond);
  }
  RCUDA(cudaMemsetAsync(sums.p, 0, 8 * sizeof(double), s));
  RCUDA(launch_resid(u, r, r, idx, k, vals, w.p, resid.p, sums.p, s));
  double hs[8];
  RCUDA(cudaMemcpyAsync(hs, sums.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
  RCUDA(cudaStreamSynchronize(s));
  const double rn = std::sqrt(std::max(hs[0], 0.0));
  if (resid_norm) *resid_norm = rn;
  if (step == 0.0 || rn == 0.0) return RMX_OK;
  RCUDA(launch_pred(u, v, r, w.p, pred.p, sums.p, s));
  std::vector<double> hw((size_t)r);
  RCUDA(cudaMemcpyAsync(hw.data(), w.p, (size_t)r * sizeof(double), cudaMemcpyDeviceToHost, s));
  RCUDA(cudaMemcpyAsync(hs, sums.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
  RCUDA(cudaStreamSynchronize(s));
  const double pn = std::sqrt(std::max(hs[1], 0.0));
  double ww = 0.0;
  for (int c = 0; c < r; ++c) ww += hw[c] * hw[c];
  const double wn = std::sqrt(ww);
  if (pn == 0.0 || wn == 0.0) return RMX_OK;
  if (rn <= 1e-14 * std::max(1.0, pn)) return RMX_OK;
  const double theta = step * std::atan(rn / pn);
  const double a = (std::cos(theta) - 1.0) / pn, b = std::sin(theta) / rn;
  RCUDA(launch_track_apply(u, v, r, pred.p, a, idx, k, resid.p, b, w.p, 1.0 / wn, s));
  RCUDA(cudaStreamSynchronize(s));
  return RMX_OK;
}

}  // extern "C"

namespace {
int lsq_tc_impl(const double* u, int64_t ldu, int64_t v, int32_t r, const int32_t* idx, int32_t k,
                const double* vals, int64_t B, double* w_out, int32_t* flag_out, void* workspace,
                size_t workspace_bytes, int32_t* stats, double settle_tol, void* stream,
                rmx_status* st) {
  rclear(st);
  if (r < 1 || k < r || B < 1 || !vals || !w_out || !idx || v < 1)
    return rset(st, RMX_E_USAGE, "%d observed rows cannot determine %d coefficients", k, r);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!gram_tc_supported(r, k) || getenv("RMX_GRAM_FP64")) {
    if (stats) stats[0] = stats[1] = 0;
    return rmx_lsq_solve(u, ldu, r, idx, k, vals, B, w_out, flag_out, nullptr, workspace,
                         workspace_bytes, stream, st);
  }
  // G~ in fp32 (its precision is the tensor cores' anyway): half the bytes,
  // a twice-as-fast factor; RMX_GRAM_CHOL64=1 keeps the factor in fp64
  const bool f32 = !getenv("RMX_GRAM_CHOL64");
  const char* rs = getenv("RMX_REFINE_STEPS");
  const bool force2 = settle_tol <= 0.0 || (rs && atoi(rs) >= 2);
  const size_t per = f32 ? gram_bytes(r) / 2 : gram_bytes(r);
  int64_t chunk = (int64_t)((workspace_bytes > 256 ? workspace_bytes - 256 : 0) /
                            (per + 4 * sizeof(double)));
  if (chunk < 1) return rset(st, RMX_E_USAGE, "lsq workspace too small");
  chunk = std::min<int64_t>(chunk, B);
  // RMX_LSQ_STREAMS=2 (experiment): two batches in flight on two side streams
  // (each owns half of the workspace), so the tensor-core Gram of one batch
  // overlaps the latency-bound factor / resolves of the other.  Measured
  // slower at config 5 (0.70 s vs 0.67 s per 99,600 systems: the factor's
  // three CTAs per SM leave the Gram no room), so one batch at a time is the
  // default.
  const char* ls_env = getenv("RMX_LSQ_STREAMS");
  const bool two = f32 && B > chunk / 2 && chunk >= 2 && ls_env && atoi(ls_env) == 2;
  if (two) chunk /= 2;
  struct Side {
    cudaStream_t q[2] = {nullptr, nullptr};
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    ~Side() {
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
      for (cudaStream_t x : q)
        if (x) cudaStreamDestroy(x);
    }
  } side;
  void* Gq[2] = {workspace, static_cast<uint8_t*>(workspace) + (two ? chunk * per : 0)};
  double* G = static_cast<double*>(workspace);
  double* nrm = reinterpret_cast<double*>(static_cast<uint8_t*>(workspace) +
                                          (two ? 2 : 1) * chunk * per);
  DevBuf<__half> planes;
  DevBuf<double> gbuf;
  DevBuf<int32_t> flags, nconv;
  RCUDA(planes.alloc((size_t)2 * v * gram_tc_kpg(r), s));
  RCUDA(gbuf.alloc((size_t)(two ? 2 : 1) * chunk * r, s));
  RCUDA(flags.alloc((size_t)B, s));
  RCUDA(nconv.alloc((size_t)B, s));
  RCUDA(launch_gram_planes(u, ldu, v, r, planes.p, s));
  if (two) {
    int prio = 0;
    RCUDA(cudaStreamGetPriority(s, &prio));
    for (auto& x : side.q) RCUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio));
    for (auto& e : side.ev) RCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    RCUDA(cudaEventRecord(side.ev[2], s));  // planes, scratch and the caller's inputs are ready
    for (auto& x : side.q) RCUDA(cudaStreamWaitEvent(x, side.ev[2], 0));
  }
  cudaStream_t s_caller = s;
  const int sms = device_sm_count();
  int64_t batch_no = 0;
  for (int64_t b0 = 0; b0 < B; b0 += chunk, ++batch_no) {
    const int64_t cnt = std::min(chunk, B - b0);
    const int32_t* ib = idx + b0 * k;
    const double* vb = vals + b0 * k;
    double* wb = w_out + b0 * r;
    const int qi = two ? (int)(batch_no & 1) : 0;
    cudaStream_t s = two ? side.q[qi] : s_caller;  // this batch's stream (shadows the caller's)
    void* Graw = Gq[qi];
    double* gp = gbuf.p + (size_t)qi * chunk * r;
    RCUDA(launch_gram_tc(planes.p, v, r, ib, k, vb, Graw, f32 ? 1 : 0, cnt, sms, s));
    if (f32 && chol_cluster_supported(r)) {
      // factor on chip (4-CTA clusters), then the first solve as a resolve
      // from w = 0 (its convergence flag is overwritten by the refinements)
      RCUDA(launch_chol_cluster_f32(static_cast<float*>(Graw), r, cnt, gp, wb, flags.p + b0, s));
      RCUDA(launch_chol_resolve_f32(static_cast<float*>(Graw), r, cnt, gp, wb, nconv.p + b0, s));
    } else if (f32) {
      RCUDA(launch_chol_solve_f32(static_cast<float*>(Graw), r, cnt, wb, flags.p + b0, s));
    } else {
      RCUDA(launch_chol_solve(G, r, cnt, wb, flags.p + b0, nrm, s));
    }
    // fp64 refinement: step 1 on every system.  settle_tol > 0: a first
    // correction within settle_tol |w| means the fp32 solve's error (and the
    // step's contraction) is about that size, so the refined w is within
    // ~settle_tol^2 |w| of the solution and the system is settled; only the
    // rest take a second step.  settle_tol = 0 (rmx_lsq_solve_tc): two steps
    // on every system (w to ~1e-12).  RMX_REFINE_STEPS=2 forces two steps.
    if (f32) {
      RCUDA(launch_lsq_resid(u, ldu, r, ib, k, vb, wb, cnt, gp, s));
      RCUDA(launch_chol_resolve_f32(static_cast<float*>(Graw), r, cnt, gp, wb, nconv.p + b0, s,
                                    nullptr, force2 ? 0.0 : settle_tol));
      if (getenv("RMX_LSQ_STATS")) {  // diagnostics: systems taking the second step
        std::vector<int32_t> h((size_t)cnt);
        RCUDA(cudaMemcpyAsync(h.data(), nconv.p + b0, (size_t)cnt * 4, cudaMemcpyDeviceToHost, s));
        RCUDA(cudaStreamSynchronize(s));
        int64_t c2 = 0;
        for (int32_t x : h) c2 += x != 0;
        fprintf(stderr, "[lsq_tc] batch of %lld systems: %lld take a second refinement step\n",
                (long long)cnt, (long long)c2);
      }
      RCUDA(launch_lsq_resid(u, ldu, r, ib, k, vb, wb, cnt, gp, s, nconv.p + b0));
      RCUDA(launch_chol_resolve_f32(static_cast<float*>(Graw), r, cnt, gp, wb, nconv.p + b0, s,
                                    nconv.p + b0, 1e-7));
    } else {
      for (int it = 0; it < 2; ++it) {
        RCUDA(launch_lsq_resid(u, ldu, r, ib, k, vb, wb, cnt, gp, s));
        RCUDA(launch_chol_resolve(G, r, cnt, gp, wb, nconv.p + b0, s));
      }
    }
  }
  if (two)
    for (int qi = 0; qi < 2; ++qi) {
      RCUDA(cudaEventRecord(side.ev[qi], side.q[qi]));
      RCUDA(cudaStreamWaitEvent(s, side.ev[qi], 0));
    }
  // systems whose fp32 factor was singular or whose refinement has not
  // settled (rare: cond(U_Omega) >~ 1e3): the reference's decision on the
  // fp64 Gram -- exact cond vs 1e12, Cholesky or pivoted LU, w = rhs when
  // rejected (rmx_lsq_solve_exact), one by one
  std::vector<int32_t> hf((size_t)B), hn((size_t)B);
  RCUDA(cudaMemcpyAsync(hf.data(), flags.p, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
  RCUDA(cudaMemcpyAsync(hn.data(), nconv.p, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
  RCUDA(cudaStreamSynchronize(s));
  (void)G;
  (void)nrm;
  int32_t redo = 0;
  for (int64_t b = 0; b < B; ++b) {
    if (hf[b] == 0 && hn[b] == 0) continue;
    ++redo;
    int32_t bad = 0;
    if (int rc = lsq_exact_impl(u, ldu, r, idx + b * k, k, vals + b * k, 1, w_out + b * r, &bad,
                                nullptr, false, s, st))
      return rc;
    hf[b] = bad;
  }
  if (redo) RCUDA(cudaMemcpyAsync(flags.p, hf.data(), (size_t)B * 4, cudaMemcpyHostToDevice, s));
  if (flag_out) RCUDA(cudaMemcpyAsync(flag_out, flags.p, (size_t)B * 4, cudaMemcpyDeviceToDevice, s));
  if (stats) {
    stats[0] = 1;
    stats[1] = redo;
  }
  RCUDA(cudaStreamSynchronize(s));
  return RMX_OK;
}

}  // namespace

extern "C" {

int rmx_lsq_solve_tc(const double* u, int64_t ldu, int64_t v, int32_t r, const int32_t* idx,
                     int32_t k, const double* vals, int64_t B, double* w_out, int32_t* flag_out,
                     void* workspace, size_t workspace_bytes, int32_t* stats, void* stream,
                     rmx_status* st) {
  return lsq_tc_impl(u, ldu, v, r, idx, k, vals, B, w_out, flag_out, workspace, workspace_bytes,
                     stats, 0.0, stream, st);
}

int rmx_lsq_solve_tc_settle(const double* u, int64_t ldu, int64_t v, int32_t r,
                            const int32_t* idx, int32_t k, const double* vals, int64_t B,
                            double* w_out, int32_t* flag_out, void* workspace,
                            size_t workspace_bytes, int32_t* stats, double settle_tol,
                            void* stream, rmx_status* st) {
  if (!(settle_tol >= 0.0 && settle_tol < 1e-2)) {
    rclear(st);
    return rset(st, RMX_E_USAGE, "settle_tol %g outside [0, 1e-2)", settle_tol);
  }
  return lsq_tc_impl(u, ldu, v, r, idx, k, vals, B, w_out, flag_out, workspace, workspace_bytes,
                     stats, settle_tol, stream, st);
}

int rmx_complete_max(const float* u32, int64_t v, int32_t r, const float* w32, int64_t B,
                     int64_t perm_base, double sigma, double mu, uint64_t seed, int32_t two_sided,
                     const float* znoise, const double* base, double* max_out, void* stream,
                     rmx_status* st) {
  rclear(st);
  if (v < 1 || r < 1 || B < 1) return rset(st, RMX_E_USAGE, "bad completion dimensions");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Philox recovery (sigma > 0, the hot call): W U^T on the tensor cores
  // (fp16 W, split fp16 U: |error| <= ~2^-12 sum |w_i u_i|, far below the
  // sigma-scale noise); sigma = 0 (deterministic parity), znoise / base
  // (training's shift estimators) keep the fp32 CUDA-core kernel.
  NaiveLayout lay{};
  const bool tc = !znoise && !base && sigma > 0.0 && !getenv("RMX_COMPLETE_FP32") &&
                  (lay = complete_layout(v, r, B, device_sm_count())).stages > 0;
  if (!tc) {
    RCUDA(launch_complete_max(u32, v, r, w32, B, perm_base, sigma, mu, seed, two_sided, znoise,
                              base, max_out, s));
    return RMX_OK;
  }
  DevBuf<__half> planes, wA;
  DevBuf<float> desc;
  DevBuf<uint32_t> enc;
  RCUDA(planes.alloc((size_t)2 * v * lay.kpad, s));
  RCUDA(wA.alloc((size_t)B * lay.kpad, s));
  RCUDA(desc.alloc((size_t)B, s));
  RCUDA(enc.alloc((size_t)B, s));
  RCUDA(cudaMemsetAsync(enc.p, 0, (size_t)B * 4, s));
  RCUDA(launch_u_planes(u32, v, r, lay.kpad, planes.p, s));
  RCUDA(launch_w_rows(w32, B, r, lay.kpad, wA.p, desc.p, s));
  TfillArgs a{};
  a.L = B;
  a.v = v;
  a.kpad = lay.kpad;
  a.nk16 = lay.kpad / 16;
  a.n_vtiles = lay.n_vtiles;
  a.n_mtiles = lay.n_mtiles;
  fill_chunks(lay, &a);
  a.chunk_begin = 0;
  a.chunk_end = lay.n_chunks;
  a.wA = wA.p;
  a.wdescale = desc.p;
  a.maxenc = enc.p;
  a.sigma = (float)sigma;
  a.seed = seed;
  a.perm_base = perm_base;
  RCUDA(launch_complete_tc(lay, a, planes.p, two_sided, s));
  RCUDA(launch_max_finalize(enc.p, B, mu, max_out, s));
  return RMX_OK;  // scratch freed stream-ordered (cudaFreeAsync)
}

int rmx_to_f32(const double* a, int64_t n, float* out, void* stream, rmx_status* st) {
  rclear(st);
  RCUDA(launch_to_f32(a, n, out, static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

int rmx_row_max(const double* a, int64_t rows, int64_t cols, int32_t two_sided, double* out,
                void* stream, rmx_status* st) {
  rclear(st);
  RCUDA(launch_row_max(a, rows, cols, two_sided, out, static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

int rmx_resid_batch(const double* u, int32_t r, const int32_t* idx, int32_t k,
                    const double* vals, const double* w, int64_t B, double* resid, void* stream,
                    rmx_status* st) {
  rclear(st);
  RCUDA(launch_resid_batch(u, r, idx, k, vals, w, B, resid, static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

int rmx_gather_rows(const double* t, int64_t ldt, const int32_t* idx, int32_t k, int64_t B,
                    double* out, void* stream, rmx_status* st) {
  rclear(st);
  RCUDA(launch_gather_rows(t, ldt, idx, k, B, out, static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

int rmx_gemv(const double* u, int64_t v, int32_t r, const double* w, double* out, void* stream,
             rmx_status* st) {
  rclear(st);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevBuf<double> sums;
  RCUDA(sums.alloc(4, s));
  RCUDA(launch_pred(u, v, r, w, out, sums.p, s));
  return RMX_OK;
}

int rmx_mean_var(const double* a, int64_t n, double* out2, void* stream, rmx_status* st) {
  rclear(st);
  RCUDA(launch_mean_var(a, n, out2, static_cast<cudaStream_t>(stream)));
  return RMX_OK;
}

// Orthonormalise U (v x r, in place) by CholeskyQR2.  Returns the
// orthonormality error max|U^T U - I| measured BEFORE the call in *drift.
// count normals of an open stream straight into device memory: drawn into
// one half of the page-locked ring while the other half's copy is in
// flight, all inside one call (through ctypes, without the GIL: the
// BASIS_INIT stream is GROUSE's critical path and its Python-side copy
// loop cost as much as the draw).  Returns after the last copy completed.
int rmx_normal_stream_fill_device(rmx_normal_stream* h, int64_t count, double* dev_out,
                                  double* pinned, int64_t pinned_doubles, void* stream,
                                  rmx_status* st) {
  rclear(st);
  if (!h || !dev_out || !pinned || pinned_doubles < 2 || count < 0)
    return rset(st, RMX_E_USAGE, "bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t half = pinned_doubles / 2;
  cudaEvent_t ev[2];
  RCUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  RCUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  bool used[2] = {false, false};
  int rc = RMX_OK;
  const bool trace = getenv("RMX_TRACE_BASIS") != nullptr;  // diagnostics: where the time goes
  double t_wait = 0.0, t_draw = 0.0, t_issue = 0.0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  for (int64_t lo = 0, i = 0; lo < count && rc == RMX_OK; lo += half, ++i) {
    const int b = (int)(i & 1);
    const int64_t n = std::min(half, count - lo);
    double* buf = pinned + (size_t)b * half;
    const auto t0 = now();
    if (used[b] && cudaEventSynchronize(ev[b]) != cudaSuccess) {
      rc = rset(st, RMX_E_CUDA, "normal upload failed");
      break;
    }
    const auto t1 = now();
    if (rmx_normal_stream_fill(h, n, buf) != 0) {
      rc = rset(st, RMX_E_USAGE, "normal stream fill failed");
      break;
    }
    const auto t2 = now();
    if (cudaMemcpyAsync(dev_out + lo, buf, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, s) !=
            cudaSuccess ||
        cudaEventRecord(ev[b], s) != cudaSuccess) {
      rc = rset(st, RMX_E_CUDA, "normal upload failed");
      break;
    }
    used[b] = true;
    if (trace) {
      const double di = secs(t2, now());
      t_wait += secs(t0, t1);
      t_draw += secs(t1, t2);
      t_issue += di;
      if (di > 0.005)
        fprintf(stderr, "[basis-init] block %lld: copy issue took %.1f ms (draw %.1f ms)\n",
                (long long)i, 1e3 * di, 1e3 * secs(t1, t2));
    }
  }
  if (trace)
    fprintf(stderr, "[basis-init] ring waits %.3f s, draws %.3f s, copy issue %.3f s\n", t_wait,
            t_draw, t_issue);
  cudaStreamSynchronize(s);  // the ring is the caller's: no copy may still read it
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  return rc;
}

int rmx_orthonormalize(double* u, int64_t v, int32_t r, int32_t force, double* drift,
                       void* stream, rmx_status* st) {
  rclear(st);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevBuf<double> G, dev;
  RCUDA(G.alloc((size_t)(r + 1) * (r + 1), s));
  RCUDA(dev.alloc(2, s));
  // U^T U on the fp64 tensor cores, cluster split-K with a fixed reduction
  // order (deterministic; the atomics of a split-K k_gram were not); row and
  // column r (the unused right-hand side) stay 0
  RCUDA(cudaMemsetAsync(G.p, 0, (size_t)(r + 1) * (r + 1) * sizeof(double), s));
  if (v > INT32_MAX) return rset(st, RMX_E_USAGE, "basis of %lld rows too tall", (long long)v);
  RCUDA(launch_dsyrk_rm((int)v, r, u, r, G.p, r + 1, s));
  RCUDA(launch_max_dev_identity(G.p, r, dev.p, s));
  double h = 0.0;
  RCUDA(read_small_sync(&h, dev.p, sizeof(double), s));
  if (drift) *drift = h;
  if (!force && h <= 1e-8) return RMX_OK;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass > 0) RCUDA(launch_dsyrk_rm((int)v, r, u, r, G.p, r + 1, s));
    DevBuf<int32_t> flag;
    RCUDA(flag.alloc(1, s));
    RCUDA(launch_chol_solve(G.p, r, 1, nullptr, flag.p, nullptr, s));
    RCUDA(launch_trsm_lt(u, v, r, G.p, s));
  }
  RCUDA(cudaStreamSynchronize(s));
  return RMX_OK;
}

// GROUSE (reference lrmc.py:160-193 track_update + 208-268 train_basis).
// t: (ell x v) training statistics, perm-major.  omegas0: (max_passes x ell x
// k) first-attempt observation sets.  cb supplies resampled sets.
int rmx_grouse_train(const double* t, int64_t v, int32_t ell, int32_t r, int32_t k,
                     const int32_t* omegas0, int32_t max_passes, double tol, double* u,
                     rmx_omega_cb cb, void* user, double* pass_resid, int32_t* passes_out,
                     int32_t* converged_out, int64_t* updates_out, int32_t* final_omegas,
                     void* stream, rmx_status* st) {
  rclear(st);
  if (k < r) return rset(st, RMX_E_USAGE, "%d observed rows per update cannot identify rank %d", k, r);
  if (k > v) return rset(st, RMX_E_USAGE, "observed rows %d exceed voxel count %lld", k, (long long)v);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // sums: 0 |r|^2 1 |p|^2 2 |t|^2 4.. solver (4 resid, 5 |w|^2)
  DevBuf<double> G, w, vals, resid, sums, wn, ug, ualt, M, NT, cmat, ctil, dval, H, hg, hw,
      mw, nw, dots, wprev, ugraw;
  DevBuf<int32_t> flag, idxbuf, didx;
  DevBuf<GrouseState> gst;
  // look-ahead (two-stream) mode double-buffers the early chain's outputs
  // (rows, values, Gram); buffer 0 also serves the serial path
  const size_t gsz = (size_t)(r + 1) * (r + 1);
  RCUDA(G.alloc(2 * gsz, s));
  RCUDA(w.alloc(r, s));
  RCUDA(wn.alloc(r, s));
  RCUDA(vals.alloc(3 * (size_t)k, s));
  RCUDA(resid.alloc(k, s));
  // + the residual blocks' partials (k_resid_defer_vec -> k_grouse_post_m)
  RCUDA(sums.alloc(8 + 2 * (size_t)((k * 32 + 255) / 256), s));
  RCUDA(flag.alloc(1, s));
  RCUDA(idxbuf.alloc(k, s));
  // ug rows: [U_Omega row | t_Omega] (the Gram's operand), padded to an even
  // length (16-byte aligned rows)
  const int64_t lu = (r + 2) / 2 * 2;
  const size_t ugsz = (size_t)k * lu;
  RCUDA(ug.alloc(3 * ugsz, s));
  DevBuf<double> lav, lcorr;
  DevBuf<int32_t> ipos, ilist, icount;  // Omega' /\ Omega_h per rows buffer (k_isect)
  DevBuf<GrouseLook> lookb;
  RCUDA(lav.alloc(k, s));
  RCUDA(ipos.alloc(3 * (size_t)k, s));
  RCUDA(ilist.alloc(3 * (size_t)k, s));
  RCUDA(icount.alloc(4, s));
  RCUDA(lcorr.alloc(2 * (size_t)r + 3, s));
  RCUDA(lookb.alloc(1, s));
  RCUDA(cudaMemsetAsync(lookb.p, 0, sizeof(GrouseLook), s));
  RCUDA(ualt.alloc((size_t)v * r, s));  // the rebase target (U_base M), swapped with U_base
  RCUDA(M.alloc((size_t)r * r, s));
  RCUDA(NT.alloc((size_t)r * r, s));    // (M^-1)^T, tracked for the sparse flush
  RCUDA(ugraw.alloc(2 * ugsz, s));      // gathered rows of U_base before the product with M (x2)
  RCUDA(cmat.alloc((size_t)kDeferCap * r, s));
  RCUDA(ctil.alloc((size_t)kDeferCap * r, s));
  RCUDA(nw.alloc(r, s));
  RCUDA(dval.alloc((size_t)kDeferCap * k, s));
  RCUDA(didx.alloc((size_t)kDeferCap * k, s));
  RCUDA(H.alloc((size_t)r * r, s));
  RCUDA(hg.alloc((size_t)r + 1 + 16 * (size_t)r, s));  // g, |a|^2, k_h_g partials
  RCUDA(hw.alloc(r, s));
  RCUDA(mw.alloc(r, s));
  RCUDA(dots.alloc(kDeferCap, s));
  RCUDA(gst.alloc(1, s));
  // each column's CG solution from the previous pass warm-starts its next
  // solve (same stopping rule |G w - b| <= 1e-13 |b|, far fewer iterations
  // once the basis settles)
  if (getenv("RMX_CG_STATS")) cg_timing(1, nullptr);
  const bool warm = !getenv("RMX_GROUSE_COLD");
  if (warm) {
    RCUDA(wprev.alloc((size_t)ell * r, s));
    RCUDA(cudaMemsetAsync(wprev.p, 0, (size_t)ell * r * sizeof(double), s));
  }
  RCUDA(cudaMemsetAsync(gst.p, 0, sizeof(GrouseState), s));
  RCUDA(launch_h_identity(M.p, r, s));   // M = I
  RCUDA(launch_h_identity(NT.p, r, s));  // M^-1 = I
  RCUDA(launch_h_identity(H.p, r, s));   // the caller hands in an orthonormalised U
  std::vector<int32_t> host_idx(k);
  const double tau = ell * max_passes / 2.0;
  const bool use_cg = cg_solve_supported(r) && !getenv("RMX_GROUSE_CHOL");
  // tests: every CG solve is treated as not converged (the Cholesky fallback runs)
  const bool force_fallback = getenv("RMX_GROUSE_FORCE_FALLBACK") != nullptr;
  // U = ubase M + sum_s d_s c_s^T (rapid_kernels.cu, M-deferred GROUSE): the
  // rotation part of every update folds into the dense r x r matrix M, the
  // residual part stays a sparse term for at most kDeferCap updates.
  //  * flush (every kDeferCap updates): only the sparse terms are folded into
  //    the base, as ubase[Omega_s] += d_s (c_s^T M^-1) -- k rows per term
  //    instead of two DGEMMs over all v rows (M^-1 is tracked, transposed, by
  //    the same rank-1 updates as M);
  //  * rebase (every kRebase = 4,096 updates, before a re-orthonormalisation
  //    and at the end): ubase <- ubase M out of place (one v x r x r DGEMM, 2 v
  //    r^2 flops), M = M^-1 = I, which also bounds the rounding drift of the
  //    tracked inverse (measured max |M M^-1 - I| at config 5: 1e-14 after
  //    1,024 updates, 2e-14 after 4,096, 3e-14 after all 20,000).
  double* ubase = u;
  double* uother = ualt.p;
  const int64_t kRebase = [] {
    const char* e = getenv("RMX_GROUSE_REBASE");
    const long long q = e ? atoll(e) : 4096;
    return (int64_t)std::max<long long>(kDeferCap, q / kDeferCap * kDeferCap);
  }();
  auto flush = [&](int nt) -> int {  // sparse terms -> ubase (M unchanged)
    RCUDA(launch_ctil(NT.p, cmat.p, r, nt, ctil.p, s));
    RCUDA(launch_sparse_terms_dense(ubase, r, r, k, didx.p, dval.p, ctil.p, nt, s));
    RCUDA(launch_reset_terms(gst.p, s));
    return RMX_OK;
  };
  double inv_drift_max = 0.0;  // RMX_GROUSE_HOSTPROF: max |M M^-1 - I| seen at a rebase
  auto rebase = [&]() -> int {  // ubase <- ubase M (no pending terms), M = M^-1 = I
    if (getenv("RMX_GROUSE_HOSTPROF")) {  // diagnostics: how far the tracked inverse drifted
      std::vector<double> hm((size_t)r * r), hn((size_t)r * r);
      RCUDA(cudaMemcpyAsync(hm.data(), M.p, hm.size() * 8, cudaMemcpyDeviceToHost, s));
      RCUDA(cudaMemcpyAsync(hn.data(), NT.p, hn.size() * 8, cudaMemcpyDeviceToHost, s));
      RCUDA(cudaStreamSynchronize(s));
      for (int i = 0; i < r; ++i)
        for (int j = 0; j < r; ++j) {  // (M N)_ij = sum_l M_il N_lj = sum_l M_il NT_jl
          double acc = 0.0;
          for (int l = 0; l < r; ++l) acc += hm[(size_t)i * r + l] * hn[(size_t)j * r + l];
          inv_drift_max = std::max(inv_drift_max, std::fabs(acc - (i == j ? 1.0 : 0.0)));
        }
    }
    RCUDA(launch_dgemm_rm(v, r, r, ubase, r, M.p, r, uother, r, 0, s));
    std::swap(ubase, uother);
    RCUDA(launch_h_identity(M.p, r, s));
    RCUDA(launch_h_identity(NT.p, r, s));
    return RMX_OK;
  };
  // One update, entirely on the device (lrmc.py:160-193): the Omega rows of
  // U (ubase[Omega] M + the sparse terms), Gram, solve (cluster CG; Cholesky
  // on the same G when CG does not converge), residual, |p|^2 from H, and
  // k_grouse_post_m's decisions; the update itself only touches M, the
  // terms and H.  No host round trip: the host syncs every 64 updates.
  // RMX_GROUSE_PROFILE=1 (diagnostics): CUDA events between the phases of
  // updates [128, 192) -> per-phase in-stream time (kernel + any idle gap
  // before it) printed to stderr at the end
  struct PhaseProf {
    enum { kPh = 9, kLo = 128, kN = 64 };
    bool on = getenv("RMX_GROUSE_PROFILE") != nullptr;
    std::vector<cudaEvent_t> ev;
    int64_t cur = -1;
    int slot = 0;
    void mark(cudaStream_t st) {
      if (cur < 0) return;
      cudaEventRecord(ev[(size_t)(cur - kLo) * kPh + slot++], st);
    }
    ~PhaseProf() {
      for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
  } prof;
  if (prof.on) {
    prof.ev.resize((size_t)PhaseProf::kPh * PhaseProf::kN);
    for (auto& e : prof.ev) RCUDA(cudaEventCreate(&e));
  }
  bool m_identity = true;  // no update applied since the last rebase (M = I exactly)
  // b encodes the buffers of an update: rows / values b >> 1 (of 3), Gram b & 1.
  // the raw rows of U_base on Omega (and t[Omega] into column r of the product's
  // rows): depends only on U_base, so the look-ahead loop issues it one update
  // further ahead than the rest of the early chain
  auto enqueue_gather = [&](int i, const int32_t* idx, int b, cudaStream_t se, bool marks) -> int {
    const double* trow = t + (int64_t)i * v;
    const int bu = b >> 1, bg = b & 1;
    RCUDA(launch_gather_urows_vals(ubase, r, idx, k, ugraw.p + (size_t)bg * ugsz, lu, trow,
                                   vals.p + (size_t)bu * k, marks ? sums.p : nullptr, se,
                                   ug.p + (size_t)bu * ugsz));
    return RMX_OK;
  };
  // early chain of an update (everything before the solve) on stream `se`: the
  // rows of U on Omega (product with M, deferred sparse terms) and their Gram;
  // idx_prev (look-ahead): the previous update's Omega, for k_isect; gathered:
  // the raw rows were issued ahead (enqueue_gather)
  auto enqueue_early = [&](int i, const int32_t* idx, int b, cudaStream_t se, bool marks,
                           const int32_t* idx_prev = nullptr, bool gathered = false) -> int {
    const double* trow = t + (int64_t)i * v;
    const int bu = b >> 1, bg = b & 1;  // rows / values buffer (of 3), Gram buffer (of 2)
    double* ugb = ug.p + (size_t)bu * ugsz;
    // U_Omega = ubase[Omega] M: the raw rows, then one k x r x r DGEMM; right
    // after a rebase M = I and the rows are gathered in place
    if (m_identity && !gathered) {
      RCUDA(launch_gather_urows_vals(ubase, r, idx, k, ugb, lu, trow, vals.p + (size_t)bu * k,
                                     marks ? sums.p : nullptr, se));
      if (marks) prof.mark(se);
    } else {
      if (!gathered)
        if (int rc = enqueue_gather(i, idx, b, se, marks)) return rc;
      if (marks) prof.mark(se);
      RCUDA(launch_dgemm_rm(k, r, r, ugraw.p + (size_t)bg * ugsz, lu, M.p, r, ugb, lu, 0, se));
    }
    if (marks) prof.mark(se);
    RCUDA(launch_sparse_terms_rows(ugb, lu, r, idx, k, didx.p, dval.p, cmat.p, gst.p, se));
    if (marks) prof.mark(se);
    // Gram of [U_Omega | t_Omega] (column r of ug is vals): the full (r+1)^2
    RCUDA(launch_dsyrk_rm(k, r + 1, ugb, lu, G.p + (size_t)bg * gsz, r + 1, se));
    if (marks) prof.mark(se);
    // look-ahead: the rows this update shares with the previous one (the late
    // chain adds the previous update's sparse term on them)
    if (idx_prev && !gathered)  // (issued with the rows when they were gathered ahead)
      RCUDA(launch_isect(idx, idx_prev, k, ipos.p + (size_t)bu * k, ilist.p + (size_t)bu * k,
                         icount.p + bu, se));
    return RMX_OK;
  };
  // the rest of the update on the main stream: (late chain,) solve, residual,
  // decisions, H, M.  corr: the look-ahead correction is applied by the solve.
  // before_apply (optional): an event the M / term update must wait for (the
  // next update's early chain reads M's factors and the terms)
  bool prof_la_mark = false;  // set below: look-ahead profiling marks the late chain's end
  auto enqueue_main = [&](int i, const int32_t* idx, int64_t tglob, bool chol, int b, bool late,
                          cudaEvent_t before_apply, cudaStream_t sh = nullptr,
                          cudaEvent_t h_prev = nullptr, cudaEvent_t post_done = nullptr,
                          cudaEvent_t h_done = nullptr) -> int {
    const double step = 1.0 / (1.0 + (double)tglob / tau);
    const int bu = b >> 1, bg = b & 1;
    double* ugb = ug.p + (size_t)bu * ugsz;
    double* valsb = vals.p + (size_t)bu * k;
    double* Gb = G.p + (size_t)bg * gsz;
    if (late) {
      RCUDA(launch_late_chain(ugb, lu, r, k, Gb, w.p, dval.p, ipos.p + (size_t)bu * k,
                              ilist.p + (size_t)bu * k, icount.p + bu, wn.p, gst.p, lookb.p,
                              lav.p, lcorr.p, s));
    }
    if (prof_la_mark) prof.mark(s);
    const bool cg = use_cg && !chol;
    if (cg) {
      RCUDA(launch_cg_solve(Gb, r, w.p, flag.p, sums.p + 4, 1e-13,
                            warm ? wprev.p + (int64_t)i * r : nullptr, s,
                            late ? lcorr.p : nullptr, late ? lookb.p : nullptr,
                            late ? lav.p : nullptr, late ? k : 0));
      prof.mark(s);
      if (force_fallback) RCUDA(cudaMemsetAsync(flag.p, 0x01, 1, s));  // tests: flag = 1
    } else {
      RCUDA(launch_chol_solve(Gb, r, 1, w.p, flag.p, sums.p + 4, s));
      prof.mark(s);
    }
    prof.mark(s);
    // sh (look-ahead): the H update runs on its own stream beside the next
    // update's late chain and solve; H is read again here (hw = H w)
    if (h_prev) RCUDA(cudaStreamWaitEvent(s, h_prev, 0));
    RCUDA(launch_resid_defer_vec(ugb, lu, r, k, valsb, w.p, resid.p, sums.p, H.p, M.p, cmat.p,
                                 gst.p, hw.p, mw.p, dots.p, s, NT.p, nw.p, late ? lav.p : nullptr,
                                 wn.p, lookb.p));
    prof.mark(s);
    RCUDA(launch_grouse_post_m(gst.p, sums.p, flag.p, step, tglob, idx, k, resid.p, w.p, r,
                               didx.p, dval.p, cmat.p, wn.p,
                               final_omegas ? final_omegas + (int64_t)i * k : nullptr, hw.p,
                               cg ? 1 : 0, s, lookb.p));
    if (sh) {
      RCUDA(cudaEventRecord(post_done, s));
      RCUDA(cudaStreamWaitEvent(sh, post_done, 0));
    }
    RCUDA(launch_h_update(H.p, r, gst.p, hw.p, wn.p, ugb, lu, k, valsb, resid.p, sums.p, hg.p,
                          sh ? sh : s, lookb.p));
    if (sh) RCUDA(cudaEventRecord(h_done, sh));
    if (before_apply) RCUDA(cudaStreamWaitEvent(s, before_apply, 0));
    RCUDA(launch_defer_apply(M.p, NT.p, cmat.p, gst.p, mw.p, dots.p, wn.p, nw.p, r, s));
    m_identity = false;
    prof.mark(s);
    return RMX_OK;
  };
  // chol: solve with the batched Cholesky (a retry after the cluster CG did
  // not converge, and the redraws of an ill-conditioned restriction); else
  // the cluster CG, whose non-convergence halts the update for that retry --
  // no gated fallback kernel in every update's chain
  auto enqueue = [&](int p, int i, const int32_t* idx, int64_t tglob, bool chol) -> int {
    prof.cur = (prof.on && tglob >= PhaseProf::kLo && tglob < PhaseProf::kLo + PhaseProf::kN)
                   ? tglob : -1;
    prof.slot = 0;
    prof.mark(s);
    if (int rc = enqueue_early(i, idx, 0, s, true)) return rc;
    (void)p;
    return enqueue_main(i, idx, tglob, chol, 0, false, nullptr);
  };
  double hdrift_host = 0.0;
  // RMX_GROUSE_HOSTPROF=1 (diagnostics): host time spent enqueueing vs
  // waiting at the checkpoints (a wait near zero = the host is the bound)
  const bool hostprof = getenv("RMX_GROUSE_HOSTPROF") != nullptr;
  double host_wait_s = 0.0;
  int reorth_count = 0;
  const auto host_t0 = std::chrono::steady_clock::now();
  auto read_state = [&](GrouseState* h) -> int {
    const auto w0 = std::chrono::steady_clock::now();
    struct Acc {
      double& a;
      std::chrono::steady_clock::time_point t;
      ~Acc() { a += std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count(); }
    } acc{host_wait_s, w0};
    // one read (the drift lands in the state struct), polled rather than slept on
    RCUDA(launch_h_drift(H.p, r, &gst.p->hdrift, s));
    RCUDA(read_small_spin(h, gst.p, sizeof(GrouseState), s));
    hdrift_host = h->hdrift;
    return RMX_OK;
  };
  int passes = 0, converged = 0;
  const int64_t total = (int64_t)max_passes * ell;
  int64_t tglob = 0;
  // a checkpoint follows update tglob - 1 when tglob is a flush point (every
  // kDeferCap updates) or a pass end; the host reads the device state there
  auto is_checkpoint = [&](int64_t tg) { return tg % kDeferCap == 0 || tg % ell == 0; };
  const bool force_halt = getenv("RMX_GROUSE_TEST_HALT") != nullptr;  // tests: halt at these steps
  std::vector<int64_t> halt_at;
  if (force_halt) {
    for (const char* c = getenv("RMX_GROUSE_TEST_HALT"); *c;) {
      char* e = nullptr;
      const long long hv = strtoll(c, &e, 10);
      if (e == c) break;
      halt_at.push_back(hv);
      c = (*e == ',') ? e + 1 : e;
    }
  }
  std::vector<char> halt_used(halt_at.size(), 0);
  // Look-ahead mode (default with the cluster CG; RMX_GROUSE_LOOKAHEAD=0 or
  // the phase profiler select the serial chain): update h + 1's early chain
  // runs on a second stream from the state before update h while update h is
  // solved; its late chain then adds update h's rank-1 term (k_late /
  // the solve's corr).  Ordering: early(h + 1) starts after update
  // h - 1 is fully applied (evD) and must finish (evE) before update h's term
  // is written into M's factors and the term list, which it reads.  The first
  // update after a checkpoint starts cold (its early chain sees every term).
  const char* la_env = getenv("RMX_GROUSE_LOOKAHEAD");
  // RMX_GROUSE_PROFILE=2: marks on the main stream of the look-ahead chain
  const bool prof_la = prof.on && atoi(getenv("RMX_GROUSE_PROFILE")) == 2;
  const bool lookahead = use_cg && (!prof.on || prof_la) && !(la_env && atoi(la_env) == 0);
  struct LookStreams {
    cudaStream_t s2 = nullptr, s3 = nullptr;
    cudaEvent_t evE[2] = {nullptr, nullptr}, evD = nullptr, evP = nullptr;
    cudaEvent_t evH[2] = {nullptr, nullptr};
    ~LookStreams() {
      for (cudaEvent_t e : evE)
        if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : evH)
        if (e) cudaEventDestroy(e);
      if (evD) cudaEventDestroy(evD);
      if (evP) cudaEventDestroy(evP);
      if (s2) cudaStreamDestroy(s2);
      if (s3) cudaStreamDestroy(s3);
    }
  } ls;
  if (lookahead) {
    int prio = 0;
    RCUDA(cudaStreamGetPriority(s, &prio));
    // one notch below the main stream: the solve's cluster is placed before
    // the early chain's pending blocks when SMs free up
    int plo = 0, phi = 0;
    RCUDA(cudaDeviceGetStreamPriorityRange(&plo, &phi));  // (least, greatest), numerically plo >= phi
    RCUDA(cudaStreamCreateWithPriority(&ls.s2, cudaStreamNonBlocking, std::min(plo, prio + 1)));
    RCUDA(cudaStreamCreateWithPriority(&ls.s3, cudaStreamNonBlocking, std::min(plo, prio + 1)));
    for (auto& e : ls.evE) RCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ls.evH) RCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    RCUDA(cudaEventCreateWithFlags(&ls.evD, cudaEventDisableTiming));
    RCUDA(cudaEventCreateWithFlags(&ls.evP, cudaEventDisableTiming));
  }
  prof_la_mark = prof_la;
  int64_t h_last = -1;                 // the last update whose H update went to s3
  int64_t pregathered = -1;            // update whose raw rows are already gathered (s2)
  bool have_early = false;  // update tglob's early chain is already in flight on s2
  auto early_on_s2 = [&](int64_t h) -> int {  // after everything enqueued on s so far
    const int hp = (int)(h / ell), hi = (int)(h % ell);
    RCUDA(cudaEventRecord(ls.evD, s));
    RCUDA(cudaStreamWaitEvent(ls.s2, ls.evD, 0));
    // rows / values are triple-buffered: buffer h % 3 was last read by update
    // h - 3, whose H update (stream s3) completed before update h - 2's
    // residual kernel, so only evD orders this chain
    // the chain sees the terms of the updates applied so far: all but update
    // h - 1's when that update is in flight (its term comes with the late
    // chain), every term when cold
    const int64_t hm = h - 1;  // the update in flight whose term the late chain will add
    const int32_t* idx_prev = have_early ? omegas0 + hm * k : nullptr;
    const bool gathered = pregathered == h;
    if (!have_early) pregathered = -1;  // cold start: nothing issued ahead survives
    if (int rc = enqueue_early(hi, omegas0 + ((int64_t)hp * ell + hi) * k,
                               (int)((h % 3) * 2 + (h & 1)), ls.s2, false, idx_prev,
                               have_early && gathered))
      return rc;
    RCUDA(cudaEventRecord(ls.evE[h & 1], ls.s2));
    // the gather of update h + 1 behind this chain (it only needs U_base, which
    // changes at checkpoints), so it runs beside the current solve's iterations
    // instead of beside the next solve's load of G.  Its buffers (h + 1) % 3
    // were last read by update h - 2, H update included (evH).
    const int64_t g = h + 1;
    if (have_early && g < total && !is_checkpoint(g) && h_last >= 0 && h_last == h - 2) {
      RCUDA(cudaStreamWaitEvent(ls.s2, ls.evH[h_last & 1], 0));
      if (int rc = enqueue_gather((int)(g % ell), omegas0 + g * k, (int)((g % 3) * 2 + (g & 1)),
                                  ls.s2, false))
        return rc;
      // and the rows it shares with update h (static Omega lists): off both chains
      RCUDA(launch_isect(omegas0 + g * k, omegas0 + h * k, k, ipos.p + (size_t)(g % 3) * k,
                         ilist.p + (size_t)(g % 3) * k, icount.p + (g % 3), ls.s2));
      pregathered = g;
    }
    return RMX_OK;
  };
  while (tglob < total) {
    const int p = (int)(tglob / ell), i = (int)(tglob % ell);
    for (size_t q = 0; q < halt_at.size(); ++q)
      if (halt_at[q] == tglob && !halt_used[q]) {  // test hook: as if this solve flagged
        halt_used[q] = 1;
        RCUDA(launch_force_halt(gst.p, tglob, s));
      }
    if (!lookahead) {
      if (int rc = enqueue(p, i, omegas0 + ((int64_t)p * ell + i) * k, tglob, false)) return rc;
    } else {
      const int64_t h = tglob;
      const bool cold = !have_early;
      if (cold)
        if (int rc = early_on_s2(h)) return rc;
      RCUDA(cudaStreamWaitEvent(s, ls.evE[h & 1], 0));
      prof.cur = (prof.on && h >= PhaseProf::kLo && h < PhaseProf::kLo + PhaseProf::kN) ? h : -1;
      prof.slot = 0;
      prof.mark(s);
      // the next update's early chain, unless a checkpoint follows this update
      const bool next = h + 1 < total && !is_checkpoint(h + 1);
      if (next) {
        have_early = true;
        if (int rc = early_on_s2(h + 1)) return rc;
      }
      if (int rc = enqueue_main(i, omegas0 + ((int64_t)p * ell + i) * k, h, false,
                                (int)((h % 3) * 2 + (h & 1)),
                                !cold, next ? ls.evE[(h + 1) & 1] : nullptr, ls.s3,
                                h_last >= 0 ? ls.evH[h_last & 1] : nullptr, ls.evP,
                                ls.evH[h & 1]))
        return rc;
      h_last = h;
      while (prof.cur >= 0 && prof.slot < PhaseProf::kPh) prof.mark(s);
      have_early = next;
    }
    ++tglob;
    bool stop = false;
    // Process the checkpoint at tglob.  After a halt is resolved by a redraw,
    // the updates after the halted one are replayed from h + 1 -- and when h
    // + 1 is itself a checkpoint, it is processed here before any further
    // update is enqueued (so at most kDeferCap terms are ever pending, and no
    // pass end is skipped).
    while (is_checkpoint(tglob)) {
      GrouseState hs;
      if (lookahead && h_last >= 0) RCUDA(cudaStreamWaitEvent(s, ls.evH[h_last & 1], 0));
      if (int rc = read_state(&hs)) return rc;
      if (const char* tp = getenv("RMX_GROUSE_TRACE")) {  // one flush block's timeline
        if (tglob == 2048) grouse_trace(1, nullptr);
        if (tglob == 2176) grouse_trace(0, tp);  // two flush blocks: the checkpoint gap is visible
      }
      if (hs.overflow)
        return rset(st, RMX_E_CUDA, "GROUSE: more than %d deferred updates between flushes",
                    kDeferCap);
      if (hs.halted && hs.cg_fail) {
        // the cluster CG of update h did not converge: the same Omega again
        // with the Cholesky solve (the updates after h were no-ops)
        const int64_t h = hs.halt_step;
        const int hp = (int)(h / ell), hi = (int)(h % ell);
        GrouseState z{};
        RCUDA(cudaMemcpyAsync(&gst.p->halted, &z.halted, sizeof(int), cudaMemcpyHostToDevice, s));
        RCUDA(cudaMemcpyAsync(&gst.p->cg_fail, &z.cg_fail, sizeof(int), cudaMemcpyHostToDevice, s));
        if (int rc = enqueue(hp, hi, omegas0 + ((int64_t)hp * ell + hi) * k, h, true)) return rc;
        if (int rc = read_state(&hs)) return rc;
        if (!hs.halted) {
          tglob = h + 1;  // replay the skipped updates
          continue;
        }
        // else: the Cholesky solve flagged the restriction -> redraw below
      }
      if (hs.halted) {
        // ill-conditioned restriction at update h: redraw its Omega from the same
        // stream (lrmc.py:240-250); updates after h were no-ops and are replayed
        const int64_t h = hs.halt_step;
        const int hp = (int)(h / ell), hi = (int)(h % ell);
        bool ok = false;
        for (int attempt = 1; attempt < 5 && cb; ++attempt) {
          if (cb(user, hi, hp, attempt, host_idx.data()) != 0)
            return rset(st, RMX_E_USAGE, "omega callback failed");
          RCUDA(cudaMemcpyAsync(idxbuf.p, host_idx.data(), k * sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
          RCUDA(cudaMemsetAsync(gst.p, 0, sizeof(int), s));  // clear `halted`
          if (int rc = enqueue(hp, hi, idxbuf.p, h, true)) return rc;
          if (int rc = read_state(&hs)) return rc;
          if (!hs.halted) {
            ok = true;
            break;
          }
        }
        if (!ok)
          return rset(st, RMX_E_ILLCOND,
                      "training column %d pass %d: restricted basis stayed ill-conditioned", hi,
                      hp);
        tglob = h + 1;  // replay the skipped updates (checkpoint at h + 1 first, if any)
        continue;
      }
      const int pc = (int)((tglob - 1) / ell);  // pass of the update before the checkpoint
      if (tglob % kDeferCap == 0) {  // at most kDeferCap deferred terms: rewrite U
        if (int rc = flush(hs.nterms)) return rc;
        const bool reorth = hdrift_host > 1e-8;  // lrmc.py:258-259 every 64 updates, from the tracked H
        if (reorth || tglob % kRebase == 0) {
          if (int rc = rebase()) return rc;
          m_identity = true;
        }
        if (reorth) {
          ++reorth_count;
          double drift = 0.0;
          if (int rc = rmx_orthonormalize(ubase, v, r, 1, &drift, stream, st)) return rc;
          RCUDA(launch_h_identity(H.p, r, s));
        }
      }
      if (tglob % ell == 0) {
        const double rel = hs.rel_sum / ell;
        if (pass_resid) pass_resid[pc] = rel;
        passes = pc + 1;
        RCUDA(cudaMemsetAsync(&gst.p->rel_sum, 0, sizeof(double), s));
        if (rel < tol) {
          converged = 1;
          stop = true;
        }
      }
      break;
    }
    if (stop) break;
  }
  if (prof.on && tglob >= PhaseProf::kLo + PhaseProf::kN) {
    RCUDA(cudaStreamSynchronize(s));
    static const char* names_serial[PhaseProf::kPh - 1] = {
        "gather", "deferred_dgemms", "sparse_terms", "syrk+memset", "cg", "chol_gate", "resid",
        "post+h_update+defer"};
    static const char* names_la[PhaseProf::kPh - 1] = {
        "late_chain", "cg", "gate", "resid", "post+h_update+wait_early+defer", "-", "-", "-"};
    const char* const* names = lookahead ? names_la : names_serial;
    double tot[PhaseProf::kPh - 1] = {};
    for (int u = 0; u < PhaseProf::kN; ++u)
      for (int q = 0; q + 1 < PhaseProf::kPh; ++q) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, prof.ev[(size_t)u * PhaseProf::kPh + q],
                             prof.ev[(size_t)u * PhaseProf::kPh + q + 1]);
        tot[q] += ms;
      }
    fprintf(stderr, "{\"grouse_phase_us_per_update\": {");
    for (int q = 0; q + 1 < PhaseProf::kPh; ++q)
      fprintf(stderr, "%s\"%s\": %.2f", q ? ", " : "", names[q], 1e3 * tot[q] / PhaseProf::kN);
    fprintf(stderr, "}}\n");
  }
  {
    GrouseState hs;
    RCUDA(read_small_sync(&hs, gst.p, sizeof(GrouseState), s));
    if (int rc = flush(hs.nterms)) return rc;
    if (int rc = rebase()) return rc;
    if (ubase != u) {  // an odd number of rebases: the result belongs in the caller's buffer
      RCUDA(cudaMemcpyAsync(u, ubase, (size_t)v * r * sizeof(double), cudaMemcpyDeviceToDevice, s));
      ubase = u;
    }
  }
  if (hostprof)
    fprintf(stderr,
            "{\"grouse_host\": {\"loop_s\": %.3f, \"checkpoint_wait_s\": %.3f, \"lookahead\": %d, "
            "\"reorthonormalisations\": %d, \"max_inverse_drift_at_rebase\": %.3g}}\n",
            std::chrono::duration<double>(std::chrono::steady_clock::now() - host_t0).count(),
            host_wait_s, lookahead ? 1 : 0, reorth_count, inv_drift_max);
  if (getenv("RMX_CG_STATS")) {
    unsigned long long cs[2] = {0, 0}, ph[6] = {0, 0, 0, 0, 0, 0};
    cudaStreamSynchronize(s);
    cg_stats(cs);
    cg_timing(0, ph);
    const double it = cs[1] ? (double)cs[1] : 1.0;
    fprintf(stderr,
            "rmx cg: %llu solves, %llu iterations (%.1f per solve); CTA 0 cycles per iteration: "
            "local dots %.0f, block reduce %.0f, post %.0f, wait for peers %.0f, matvec %.0f, "
            "scalars + vector updates %.0f\n",
            cs[0], cs[1], cs[0] ? (double)cs[1] / (double)cs[0] : 0.0, ph[0] / it, ph[1] / it,
            ph[2] / it, ph[3] / it, ph[4] / it, ph[5] / it);
  }
  double drift = 0.0;
  if (int rc = rmx_orthonormalize(ubase, v, r, 0, &drift, stream, st)) return rc;
  const int64_t tcount = (int64_t)passes * ell;
  if (passes_out) *passes_out = passes;
  if (converged_out) *converged_out = converged;
  if (updates_out) *updates_out = tcount;
  RCUDA(cudaStreamSynchronize(s));
  return RMX_OK;
}

}  // extern "C"
