// rapid_internal.cuh -- launchers of rapid_kernels.cu (RapidPT on the GPU).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

namespace rmx {

// Programmatic dependent launch for the GROUSE per-update kernel chain
// (RMX_PDL=0 turns it off): a kernel launched with the attribute may be
// scheduled as soon as its predecessor's blocks have exited, and every chain
// kernel starts with griddepcontrol.wait (pdl_wait, sm100.cuh) before it
// touches memory, so the dependent-launch latency overlaps the tail of the
// previous kernel instead of following its completion.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RMX_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

cudaError_t launch_rapid_stats(const double* x, int n, int n1, const int16_t* orders,
                               const int32_t* omegas, int64_t L, int k, double* t_out,
                               unsigned long long* deg_key, cudaStream_t s);
// G_b = [U[idx_b] | vals_b]^T [U[idx_b] | vals_b], (r+1)^2 each; idx = null -> all rows
cudaError_t launch_gram(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                        const double* vals, double* G, int64_t B, cudaStream_t s);
// in-place Cholesky of G_b[:r,:r]; w_b = G^-1 G_b[r, :r]; resid2[4b..] =
// (t.t - rhs.w, w.w, min L_ii, max L_ii); flag_b = 1 on a non-positive pivot
cudaError_t launch_chol_solve(double* G, int r, int64_t B, double* w_out, int32_t* flag,
                              double* resid2, cudaStream_t s);
// refinement solve with the factor k_chol_solve left in G: w_b += (L L^T)^-1 rhs_b;
// nconv_b = 1 when the correction exceeds 1e-7 |w_b|
cudaError_t launch_chol_resolve(double* G, int r, int64_t B, const double* rhs, double* w_inout,
                                int32_t* nconv, cudaStream_t s);
// the same on an fp32 G (the tensor-core Gram's precision; the fp64
// refinement restores the solution's accuracy)
// K3b on chip: one system per 4-CTA cluster (r <= 416); writes L into G's
// lower triangle, rhs_out (B x r) = G row r, w_out = 0, flag = bad pivot
bool chol_cluster_supported(int r);
cudaError_t launch_chol_cluster_f32(float* G, int r, int64_t B, double* rhs_out, double* w_out,
                                    int32_t* flag, cudaStream_t s);
cudaError_t launch_chol_solve_f32(float* G, int r, int64_t B, double* w_out, int32_t* flag,
                                  cudaStream_t s);
// w += (L L^T)^-1 rhs; nconv[b] = |correction| > tol |w|.  active (optional):
// only systems with active[b] != 0 are touched.
cudaError_t launch_chol_resolve_f32(float* G, int r, int64_t B, const double* rhs,
                                    double* w_inout, int32_t* nconv, cudaStream_t s,
                                    const int32_t* active = nullptr, double tol = 1e-7);
// Tensor-core Gram (gram_tc.cu): G_b ~ [U[idx_b] | vals_b]^T [U[idx_b] | vals_b]
// (lower triangle, (r+1)^2 each) from fp16 hi/lo planes of U (gram_planes),
// fp32-accurate; refined to fp64 accuracy by lsq_resid + launch_chol_resolve
bool gram_tc_supported(int r, int k);
int gram_tc_kpg(int r);  // plane row pitch (halves)
cudaError_t launch_gram_planes(const double* U, int64_t ldu, int64_t v, int r, __half* planes,
                               cudaStream_t s);
// G: fp64 (g_f32 = 0) or fp32 (g_f32 = 1) (r+1)^2 per system
cudaError_t launch_gram_tc(const __half* planes, int64_t v, int r, const int32_t* idx, int k,
                           const double* vals, void* G, int g_f32, int64_t B, int sm_count,
                           cudaStream_t s);
// g_b = U_Omega^T (t - U_Omega w_b) in fp64 (one gather of the rows)
cudaError_t launch_lsq_resid(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                             const double* vals, const double* W, int64_t B, double* g,
                             cudaStream_t s, const int32_t* active = nullptr);
// GROUSE step state kept on the device, so the update loop runs without a
// host round trip per update (decisions by k_grouse_post_m).
struct GrouseState {
  int halted;      // a solve flagged ill-conditioning: later step kernels no-op
  int halt_step;   // global update index that halted
  int pending;     // this step's update (pend_a, pend_b, wn) is still to be folded into M/H
  int overflow;    // a term would have exceeded kDeferCap (host bug guard): halted, error
  double pend_a;
  double rel_sum;  // sum over the pass of |r| / |t_Omega|
  double pend_b;   // beta of the pending update (d = beta r on Omega)
  double aa;       // |p|^2 = w^T H w of the pending update
  int nterms;      // deferred sparse terms since the last flush (M-deferred GROUSE)
  int cg_fail;     // the halt came from a cluster CG that did not converge (retry: Cholesky)
  unsigned int hg_done;  // blocks of k_h_g_part finished (last-block reduction)
  unsigned int da_done;  // blocks of k_defer_apply finished (last block counts the term)
  double pend_g;   // the pending update's inverse factor: (I + a w b^T)^-1 = I - pend_g w b^T
  double hdrift;   // max |H - I| (k_h_drift at a checkpoint; read with the rest of the state)
};
// look-ahead GROUSE: what update h decided, for the late chain of update h + 1
// (written by k_grouse_post_m, read by k_late / k_cg_solve)
struct GrouseLook {
  int applied;        // update h added a term (not halted, not degenerate)
  int slot;           // its deferred-term slot (d_idx / d_val row)
  unsigned int done;  // (unused)
  int pad;
  double a;           // pend_a of the update
};
// M-deferred GROUSE: U = U_base M + sum_s d_s c_s^T (d_s sparse on Omega_s)
constexpr int kDeferCap = 64;  // terms between flushes (the host flushes every 64 updates)
// deterministic variants (no atomics): per-update rows / per-term dense flush
cudaError_t launch_sparse_terms_rows(double* out, int64_t ldo, int r, const int32_t* rows_sorted,
                                     int k, const int32_t* d_idx, const double* d_val,
                                     const double* cmat, const GrouseState* st, cudaStream_t s);
cudaError_t launch_sparse_terms_dense(double* out, int64_t ldo, int r, int k, const int32_t* d_idx,
                                      const double* d_val, const double* cmat, int nterms,
                                      cudaStream_t s);
cudaError_t launch_resid_defer_vec(const double* U, int64_t ldu, int r, int k, const double* vals,
                                   const double* w, double* resid, double* sums, const double* H,
                                   const double* M, const double* cmat, const GrouseState* st,
                                   double* hw, double* mw, double* dots, cudaStream_t s,
                                   const double* NT, double* nw, const double* av = nullptr,
                                   const double* b = nullptr, const GrouseLook* look = nullptr);
cudaError_t launch_gather_urows_vals(const double* U, int r, const int32_t* idx, int k, double* out,
                                     int64_t ldo, const double* t, double* vals, double* zero8,
                                     cudaStream_t s, double* aug = nullptr);
cudaError_t launch_grouse_post_m(GrouseState* st, double* sums, const int32_t* flag,
                                 double step, int64_t step_index, const int32_t* idx, int k,
                                 const double* resid, const double* w, int r, int32_t* d_idx,
                                 double* d_val, double* cmat, double* wn, int32_t* final_slot,
                                 const double* hw, int cg_mode, cudaStream_t s,
                                 GrouseLook* look = nullptr);
// look-ahead update (rapid_kernels.cu): k_isect (early chain: Omega' /\ Omega_h),
// k_late (av and corr = (c[0..r], b[0..r], -)); the rank-1 term A += av b^T is
// applied by k_resid_defer_vec's pass over the rows
cudaError_t launch_isect(const int32_t* rows_next, const int32_t* rows_prev, int k, int32_t* pos,
                         int32_t* list, int32_t* count, cudaStream_t s);
cudaError_t launch_late_chain(const double* A, int64_t lda, int r, int k, const double* G,
                              const double* w, const double* d_val, const int32_t* pos,
                              const int32_t* list, const int32_t* count, const double* b,
                              const GrouseState* st, const GrouseLook* look, double* av,
                              double* corr, cudaStream_t s);
// M += a (M w) b^T, its inverse (transposed, NT) likewise, and the older
// terms' c_s (H: launch_h_update)
cudaError_t launch_defer_apply(double* M, double* NT, double* cmat, GrouseState* st,
                               const double* mw, const double* dots, const double* wn,
                               const double* nw, int r, cudaStream_t s);
// sparse flush: ctil[s] = M^-T c_s (the terms expressed against U_base M)
cudaError_t launch_ctil(const double* NT, const double* cmat, int r, int nterms, double* ctil,
                        cudaStream_t s);
cudaError_t launch_reset_terms(GrouseState* st, cudaStream_t s);
// test hook: mark update `step` as halted (ill-conditioned) before it runs
cudaError_t launch_force_halt(GrouseState* st, int64_t step, cudaStream_t s);
// H = U^T U tracked through the rank-1 updates (the every-64-updates drift
// check of lrmc.py:258-259 without a 168 GFLOP Gram)
cudaError_t launch_h_update(double* H, int r, const GrouseState* st, const double* hw,
                            const double* wn, const double* ug, int64_t ldu, int k,
                            const double* vals, const double* resid, const double* sums, double* g,
                            cudaStream_t s, const GrouseLook* look);
cudaError_t launch_h_drift(const double* H, int r, double* out, cudaStream_t s);
cudaError_t launch_h_identity(double* H, int r, cudaStream_t s);
void cg_timing(int on, unsigned long long phase[6]);
// diagnostics: start (on = 1) / stop and dump (on = 0) the chain kernels' timeline
void grouse_trace(int on, const char* dump_path);
void cg_stats(unsigned long long out[2]);  // k_cg_solve (solves, iterations) so far
// K4 on tcgen05: operand preparation and the max decode
cudaError_t launch_u_planes(const float* U, int64_t v, int r, int kpad, __half* planes,
                            cudaStream_t s);
cudaError_t launch_w_rows(const float* W, int64_t B, int r, int kpad, __half* wA, float* descale,
                          cudaStream_t s);
cudaError_t launch_max_finalize(const uint32_t* enc, int64_t B, double mu, double* out,
                                cudaStream_t s);
// one well-conditioned system (GROUSE) by cluster CG; flag = not converged;
// x0 (optional, in/out): starting point, overwritten with the solution
bool cg_solve_supported(int r);
cudaError_t launch_cg_solve(const double* G, int r, double* w_out, int32_t* flag, double* resid2,
                            double tol, double* x0, cudaStream_t s, const double* corr = nullptr,
                            const GrouseLook* look = nullptr, const double* av = nullptr,
                            int kav = 0);
cudaError_t launch_complete_max(const float* U, int64_t v, int r, const float* W, int64_t B,
                                int64_t perm_base, double sigma, double mu, uint64_t seed,
                                int two_sided, const float* znoise, const double* base,
                                double* max_out, cudaStream_t s);
cudaError_t launch_resid(const double* U, int64_t ldu, int r, const int32_t* idx, int k,
                         const double* vals, const double* w, double* resid, double* sums,
                         cudaStream_t s);
cudaError_t launch_pred(const double* U, int64_t v, int r, const double* w, double* pred,
                        double* sums, cudaStream_t s);
cudaError_t launch_trsm_lt(double* X, int64_t v, int r, const double* L, cudaStream_t s);
cudaError_t launch_max_dev_identity(const double* G, int r, double* out, cudaStream_t s);
cudaError_t launch_row_max(const double* A, int64_t rows, int64_t cols, int two_sided,
                           double* out, cudaStream_t s);
cudaError_t launch_resid_batch(const double* U, int r, const int32_t* idx, int k,
                               const double* vals, const double* W, int64_t B, double* R,
                               cudaStream_t s);
cudaError_t launch_to_f32(const double* a, int64_t n, float* out, cudaStream_t s);
cudaError_t launch_gather_rows(const double* t, int64_t ldt, const int32_t* idx, int k, int64_t B,
                               double* out, cudaStream_t s);
// dense_small.cu: exact condition numbers (Householder tridiagonalisation +
// Sturm bisection) and a pivoted LU fallback solve, one CTA per system.
// G: systems at stride gstride, leading dimension ldg; sel: system ids
// (nullable for sym_extreme_eigs = 0..count-1); lam: (min, max) per entry
cudaError_t launch_sym_extreme_eigs(const double* G, int64_t gstride, int ldg, int r,
                                    const int32_t* sel, int64_t count, double* work, double* lam,
                                    cudaStream_t s);
size_t sym_extreme_eigs_work(int r, int64_t count);
cudaError_t launch_lu_solve(const double* G, int64_t gstride, int ldg, int r, const int32_t* sel,
                            int64_t count, double* work, double* w, int32_t* singular,
                            cudaStream_t s);
size_t lu_solve_work(int r, int64_t count);
// track_update's rotation: d = a pred, d[idx] += b resid, U += d (w winv)^T
cudaError_t launch_track_apply(double* U, int64_t v, int r, double* pred, double a,
                               const int32_t* idx, int k, const double* resid, double b,
                               const double* w, double winv, cudaStream_t s);
// dgemm.cu: C (m x n, ldc) = A (m x kk, lda) B (kk x n, ldb) (+ C when accum), row-major fp64
cudaError_t launch_dgemm_rm(int64_t m, int n, int kk, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double* C, int64_t ldc, int accum,
                            cudaStream_t s);
// G (n x n, both halves) = A^T A, A (kk x n) row-major (dgemm.cu)
cudaError_t launch_dsyrk_rm(int kk, int n, const double* A, int64_t lda, double* C, int64_t ldc,
                            cudaStream_t s);
cudaError_t launch_mean_var(const double* a, int64_t n, double* out, cudaStream_t s);
}  // namespace rmx
