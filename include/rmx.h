/*
 * rmx.h -- C ABI of librmx.so, the B200 (sm_100a) max-null engine.
 *
 * The reference (rapidmaxnull 0.1.0, pure Python) has no FFI; its boundary is
 * the Python module API.  Each entry point below replaces the numerical work
 * behind one reference function and is bound by
 * paper_1703_01506_b200/_native.py (ctypes).  INTEGRATION.md shows the
 * binding a reference maintainer would add.
 *
 * Conventions
 *   - Every array pointer is a DEVICE pointer owned by the caller (allocated
 *     e.g. as a torch tensor on the current device).  Host pointers are only
 *     the rmx_status out-parameter and scalar arguments.
 *   - `stream` is a cudaStream_t (passed as void*); all work is stream-
 *     ordered.  Entry points that must decide on device results (fallback
 *     paths, error detection) synchronise that stream before returning.
 *   - Layouts follow the reference: x is the DataMatrix.values layout
 *     (v x n row-major float64, reference model.py:27-34); orders[p] is
 *     PermutationPlan.shuffle(p) as int16 (reference model.py:100-105);
 *     T is StatMatrix.values (v x L row-major, reference naive.py:25-34).
 *   - Return value = rmx_status.code.  Error codes map onto the reference
 *     exception hierarchy (reference errors.py:8-43):
 *        RMX_OK 0, RMX_E_USAGE 1 -> UsageError,
 *        RMX_E_DEGENERATE 2 -> DegenerateVoxelError(voxel, value = mean_diff),
 *        RMX_E_ILLCOND 3 -> IllConditionedBasisError(value = cond),
 *        RMX_E_CUDA 4 / RMX_E_NUMERIC 5 -> NumericalError,
 *        RMX_E_FORMAT 6 -> DataFormatError, RMX_E_IO 7 -> OSError.
 */
#ifndef RMX_H_
#define RMX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RMX_OK 0
#define RMX_E_USAGE 1
#define RMX_E_DEGENERATE 2
#define RMX_E_ILLCOND 3
#define RMX_E_CUDA 4
#define RMX_E_NUMERIC 5
#define RMX_E_FORMAT 6 /* -> DataFormatError (a malformed .mat0 payload) */
#define RMX_E_IO 7     /* -> OSError (open / read / write failed) */

#define RMX_ABI_VERSION 1

typedef struct rmx_status {
  int32_t code;
  int32_t _pad;
  int64_t perm;  /* permutation index of the failure (global), or -1 */
  int64_t voxel; /* voxel index of the failure, or -1 */
  double value;  /* mean_diff (DEGENERATE) / condition number (ILLCOND) */
  char msg[256];
} rmx_status;

/* Diagnostics / counters for the last naive call (host struct). */
typedef struct rmx_naive_stats {
  int64_t suspects;        /* near-zero-variance entries re-evaluated exactly */
  int64_t band_candidates; /* fp64 refinements performed */
  int64_t overflow_perms;  /* permutations re-run by the exhaustive fp64 path */
  int32_t chunks;          /* voxel chunks per permutation tile */
  int32_t grid;            /* persistent CTAs of the tensor-core kernel */
  int32_t stages;          /* smem pipeline depth */
  int32_t bk;              /* K elements per stage */
  int64_t rare_groups;     /* epilogue: 32-column groups that took the exact path */
  int64_t all_groups;      /* epilogue: all 32-column groups (per warp) */
  int32_t cg;              /* CTAs per MMA tile (tcgen05 cta_group 1 or 2) */
  int32_t i8;              /* 1: exact int8 MMA on 16-bit fixed-point z (balanced groups) */
} rmx_naive_stats;

int rmx_abi_version(void);

/* Device capability probe: returns RMX_OK on an sm_100 device, fills SM count. */
int rmx_device_check(int device, int32_t *sm_count, rmx_status *st);
/* cudaHostRegister / cudaHostUnregister of caller memory (page-locking the
 * reference's host arrays in place for the overlapped uploads); 0 = ok.
 * Through ctypes these calls release the Python GIL. */
int rmx_host_register(void *ptr, size_t bytes);
int rmx_host_unregister(void *ptr);
/* bytes of pageable host memory -> dev through the caller's page-locked
 * ring (two halves: memcpy into one while the other's copy is in flight),
 * for one-shot uploads; returns after the last copy. */
int rmx_upload_staged(const void *host, size_t bytes, void *dev, void *ring, size_t ring_bytes,
                      void *stream, rmx_status *st);

/* ---------------------------------------------------------------- NaivePT
 * Replaces reference naive.py:60-109 run_naive (the _max_block loop 49-57:
 * group_blocks model.py:65-69 + _welch_rows teststat.py:28-50 + column_max
 * teststat.py:88-90) for permutations [0, L) of `orders`.
 *
 * max_out[p]    = max_j t_pj (or max_j |t_pj| when two_sided), float64,
 *                 bit-identical to the reference (fp64 refinement of the
 *                 tensor-core candidates);
 * argmax_out[p] = the voxel attaining it (lowest index on exact ties).
 * Degenerate voxel (zero pooled variance, unequal means) in any permutation:
 *   returns RMX_E_DEGENERATE with the first (perm, voxel) in permutation order.
 */
size_t rmx_naive_workspace_bytes(int64_t v, int32_t n, int64_t L);

int rmx_naive_maxnull(const double *x, int64_t v, int32_t n, int32_t n1,
                      const int16_t *orders, int64_t L, int32_t two_sided,
                      double *max_out, int32_t *argmax_out, void *workspace,
                      size_t workspace_bytes, void *stream, rmx_status *st,
                      rmx_naive_stats *stats);

/* The same call split in its three stream-ordered phases so a caller can
 * time the tensor-core contraction alone (bench.py):
 *   prepare: K0 -- standardise each voxel in fp64, split Z and Z^2 into
 *            fp16 hi/lo planes (4 x v x kpad), exact constant-voxel handling;
 *   tfill:   K1 -- tcgen05 contraction G.[Z|Z^2] with the fused t / top-2
 *            epilogue (T never leaves TMEM/registers);
 *   finish:  K2 -- fp64 refinement of the band candidates, suspects and
 *            fallbacks; synchronises `stream`.  */
int rmx_naive_prepare(const double *x, int64_t v, int32_t n, int32_t n1, int64_t L,
                      void *workspace, size_t workspace_bytes, void *stream,
                      rmx_status *st);
int rmx_naive_tfill(int64_t v, int32_t n, int32_t n1, const int16_t *orders, int64_t L,
                    int32_t two_sided, void *workspace, size_t workspace_bytes,
                    void *stream, rmx_status *st, rmx_naive_stats *stats);
int rmx_naive_finish(const double *x, int64_t v, int32_t n, int32_t n1,
                     const int16_t *orders, int64_t L, int32_t two_sided,
                     double *max_out, int32_t *argmax_out, void *workspace,
                     size_t workspace_bytes, void *stream, rmx_status *st,
                     rmx_naive_stats *stats);

/* Debug/validation: the tensor-core statistic t~ for every entry, written
 * as t_dbg[p * v + j] (float32).  Same kernel as tfill with the epilogue's
 * store path enabled; used by the parity tests to bound |t~ - t|. */
int rmx_naive_tfill_debug(int64_t v, int32_t n, int32_t n1, const int16_t *orders,
                          int64_t L, int32_t two_sided, float *t_dbg, void *workspace,
                          size_t workspace_bytes, void *stream, rmx_status *st);

/* NaivePT from HOST buffers (the reference-facing call: DataMatrix.values
 * and the plan's label matrix live in host memory): copies X (v x n fp64) and
 * the labels into the caller's device buffers, overlapping the X upload with
 * K0/K1 chunk by chunk, runs the engine and copies max/argmax back into
 * max_host/argmax_host.  Synchronous.  Results and errors as
 * rmx_naive_maxnull.  Host buffers should be page-locked (cudaHostRegister)
 * for the overlap; pageable buffers work but serialise the copies.
 * orders_host may be NULL when orders_dev already holds the labels (e.g.
 * from rmx_plan_orders on the same stream). 
 * Replaces reference naive.py:60-109 run_naive end to end. */
int rmx_naive_maxnull_host(const double *x_host, int64_t v, int32_t n, int32_t n1,
                           const int16_t *orders_host, int64_t L, int32_t two_sided,
                           double *max_host, int32_t *argmax_host, double *x_dev,
                           int16_t *orders_dev, double *max_dev, int32_t *argmax_dev,
                           void *workspace, size_t workspace_bytes, void *stream,
                           rmx_status *st, rmx_naive_stats *stats);

/* rmx_naive_maxnull_host with the plan given by its seed, as the reference's
 * PermutationPlan(seed, L, n) (model.py:76-105): the L x n labels are
 * generated into orders_dev on the device (rmx_plan_orders' streams,
 * bit-identical to numpy) while the first X chunk is in flight.
 * Replaces reference naive.py:60-109 run_naive (plan shuffles included). */
int rmx_naive_maxnull_host_plan(const double *x_host, int64_t v, int32_t n, int32_t n1,
                                uint64_t plan_seed, int64_t L, int32_t two_sided,
                                double *max_host, int32_t *argmax_host, double *x_dev,
                                int16_t *orders_dev, double *max_dev, int32_t *argmax_dev,
                                void *workspace, size_t workspace_bytes, void *stream,
                                rmx_status *st, rmx_naive_stats *stats);

/* rmx_naive_maxnull_host / _host_plan with X given as float32 on the host
 * (v x n row-major; the BASELINE.json configs' data type): half the upload
 * bytes.  Each chunk lands in x32_dev (v x n fp32 device buffer, 16-byte
 * aligned) and is upcast into x_dev (v x n fp64) before K0 sees it, so the
 * results are those of rmx_naive_maxnull_host on the float64 upcast -- the
 * matrix the reference's DataMatrix holds (model.py:21-24, np.float64).
 * Replaces reference naive.py:60-109 run_naive end to end. */
int rmx_naive_maxnull_host_f32(const float *x_host, int64_t v, int32_t n, int32_t n1,
                               const int16_t *orders_host, int64_t L, int32_t two_sided,
                               double *max_host, int32_t *argmax_host, float *x32_dev,
                               double *x_dev, int16_t *orders_dev, double *max_dev,
                               int32_t *argmax_dev, void *workspace, size_t workspace_bytes,
                               void *stream, rmx_status *st, rmx_naive_stats *stats);
int rmx_naive_maxnull_host_plan_f32(const float *x_host, int64_t v, int32_t n, int32_t n1,
                                    uint64_t plan_seed, int64_t L, int32_t two_sided,
                                    double *max_host, int32_t *argmax_host, float *x32_dev,
                                    double *x_dev, int16_t *orders_dev, double *max_dev,
                                    int32_t *argmax_dev, void *workspace, size_t workspace_bytes,
                                    void *stream, rmx_status *st, rmx_naive_stats *stats);

/* _host_plan(_f32) over the permutation range [perm_base, perm_base + L) of
 * the plan: one rank's shard of a multi-GPU run, the labels of
 * the global indices generated on the device, X uploaded and overlapped as
 * above; max_host/argmax_host get the L local entries.  The statistic of a
 * permutation depends only on its labels, so every shard reproduces its
 * slice of the single-GPU result bit for bit.  Replaces the per-range body
 * of reference naive.py:49-57 (_max_block over [lo, hi)) for a process
 * that owns that range. */
int rmx_naive_maxnull_host_plan_range(const double *x_host, int64_t v, int32_t n, int32_t n1,
                                      uint64_t plan_seed, int64_t perm_base, int64_t L,
                                      int32_t two_sided, double *max_host, int32_t *argmax_host,
                                      double *x_dev, int16_t *orders_dev, double *max_dev,
                                      int32_t *argmax_dev, void *workspace,
                                      size_t workspace_bytes, void *stream, rmx_status *st,
                                      rmx_naive_stats *stats);
int rmx_naive_maxnull_host_plan_range_f32(const float *x_host, int64_t v, int32_t n, int32_t n1,
                                          uint64_t plan_seed, int64_t perm_base, int64_t L,
                                          int32_t two_sided, double *max_host,
                                          int32_t *argmax_host, float *x32_dev, double *x_dev,
                                          int16_t *orders_dev, double *max_dev,
                                          int32_t *argmax_dev, void *workspace,
                                          size_t workspace_bytes, void *stream, rmx_status *st,
                                          rmx_naive_stats *stats);

/* NaivePT straight from a .mat0 data file (the reference CLI
 * path cli.py:70-116 = read_matrix -> run_naive -> [write_array of T]):
 * the v x n float64 payload is streamed file -> ring_host (page-locked,
 * ring_bytes, 2-3 slots) -> device in pieces by parallel positional reads,
 * each chunk standardised (K0) and contracted (K1) as it lands while the
 * host reads the next; labels of plan rows [perm_base, perm_base + L) are
 * generated on the device.  Non-finite payload entries: RMX_E_FORMAT with
 * *bad_index = the flat element index (the reference's read_array check).
 * Header validation and n1/n2 are the caller's (matio.py messages).
 * x_dev (v x n fp64) keeps the data for a follow-up rmx_tstat_dump_mat0. */
int rmx_naive_maxnull_mat0(const char *path, int64_t v, int32_t n, int32_t n1,
                           uint64_t plan_seed, int64_t perm_base, int64_t L, int32_t two_sided,
                           double *max_host, int32_t *argmax_host, double *ring_host,
                           size_t ring_bytes, int32_t threads, int64_t *bad_index, double *x_dev,
                           int16_t *orders_dev, double *max_dev, int32_t *argmax_dev,
                           void *workspace, size_t workspace_bytes, void *stream,
                           rmx_status *st, rmx_naive_stats *stats);
/* The streamed --dump-T writer (reference naive.py:79-87 materialize=True +
 * cli.py:114-116 write_array(mat.values)): the (v, L) float64 statistic
 * matrix T[j, i] = tstat(perm i, voxel j) -- the reference's exact bits
 * (k_exact_rows) -- written to `path` as a bare .mat0 (n1 = n2 = 0) in voxel
 * slabs: slab b computed, transposed and copied to one half of ring_host
 * while the host writes slab b - 1.  Never holds T on the host; no memory
 * cap.  A degenerate (perm, voxel) raises RMX_E_DEGENERATE and removes the
 * file. */
int rmx_tstat_dump_mat0(const double *x_dev, int64_t v, int32_t n, int32_t n1,
                        const int16_t *orders_dev, int64_t L, const char *path, double *ring_host,
                        size_t ring_bytes, int32_t threads, void *stream, rmx_status *st);

/* ---------------------------------------------------------------- .mat0 I/O
 * The reference's binary matrix format (matio.py:23-91): 44-byte header
 * "<8sIQQQQ" = magic "RMXMAT0\0", u32 version (1), u64 rows, cols, n1, n2;
 * then rows x cols little-endian float64, row-major.  Host-side only. */
typedef struct rmx_mat0_info {
  char magic[8];
  uint32_t version;
  uint32_t _pad;
  int64_t rows, cols, n1, n2;
  int64_t header_bytes; /* bytes of header present (< 44: truncated) */
  int64_t file_bytes;
} rmx_mat0_info;
/* Raw header fields and file size (validation and the reference's messages
 * are the caller's: matio.py).  Replaces reference matio.py:40-57. */
int rmx_mat0_header(const char *path, rmx_mat0_info *info, rmx_status *st);
/* rows x cols payload -> out (any host buffer, e.g. page-locked), read by
 * `threads` parallel positional reads, scanned for non-finite values in the
 * same pass: RMX_E_FORMAT with *bad_index = first non-finite element (flat
 * index).  Replaces reference matio.py:58-72. */
int rmx_mat0_read(const char *path, int64_t rows, int64_t cols, double *out, int32_t threads,
                  int64_t *bad_index, rmx_status *st);
/* Rows [row0, row1) of a cols-wide payload -> out (same checks as
 * rmx_mat0_read; *bad_index is a flat index of the whole file).  The piece
 * reader of the streamed engine entry rmx_naive_maxnull_mat0.  Replaces the
 * payload read of reference matio.py:58-72 for a row range. */
int rmx_mat0_read_rows(const char *path, int64_t cols, int64_t row0, int64_t row1, double *out,
                       int32_t threads, int64_t *bad_index, rmx_status *st);
/* Create (truncate) a .mat0 file: header + a rows x cols payload to be
 * filled by rmx_mat0_write_rows (the streamed --dump-T writer). */
int rmx_mat0_create(const char *path, int64_t rows, int64_t cols, int64_t n1, int64_t n2,
                    rmx_status *st);
/* Rows [row0, row1) of the payload from a (row1 - row0) x cols host buffer,
 * parallel positional writes. */
int rmx_mat0_write_rows(const char *path, int64_t cols, int64_t row0, int64_t row1,
                        const double *a, int32_t threads, rmx_status *st);
/* Header + payload.  Replaces reference matio.py:30-37 write_array. */
int rmx_mat0_write(const char *path, const double *a, int64_t rows, int64_t cols, int64_t n1,
                   int64_t n2, rmx_status *st);

/* The reference's random streams on the device, bit-identical to numpy:
 * row t of out (count x n, int16) = PermutationPlan(seed, ., n).shuffle(lo + t)
 * (model.py:100-105: stream(seed, SHUFFLE, i).permutation(n), identity at 0). */
int rmx_plan_orders(uint64_t seed, int64_t lo, int64_t count, int32_t n, int16_t *out,
                    void *stream, rmx_status *st);
/* row t of out (count x k, int32) = sort(stream(seed, domain, lo + t[, extra])
 * .choice(v, k, replace=False)) (rapid.py:158-160, lrmc.py:237-241; extra < 0:
 * no third key).  RMX_E_USAGE when numpy would take its tail-shuffle branch
 * (v > 10000 and k > v / 50): the caller draws those on the host. */
int rmx_omega_draws(uint64_t seed, int32_t domain, int64_t lo, int64_t count, int64_t extra,
                    int64_t v, int32_t k, int32_t *out, void *stream, rmx_status *st);

/* ---------------------------------------------------------------- exact fp64
 * Bit-exact statistic matrix (reference _welch_rows arithmetic):
 *   t_out[p * ld + j] = t(perm p, voxel j), p < L, j < v  (perm-major; the
 *   caller transposes into StatMatrix's v x L layout).
 * Replaces the `store[:, i] = col` path (naive.py:55-56) and RapidPT's
 * training columns (rapid.py:64-69).  Degenerate -> RMX_E_DEGENERATE. */
int rmx_tstat_exact(const double *x, int64_t v, int32_t n, int32_t n1,
                    const int16_t *orders, int64_t L, double *t_out, int64_t ld,
                    void *stream, rmx_status *st);

/* Exact statistic at explicit (perm, voxel) pairs: pairs[2i] = perm row of
 * `orders`, pairs[2i+1] = voxel.  Outputs t, mean difference and a
 * degenerate flag per pair.  Replaces tstat_subset (teststat.py:64-77). */
int rmx_tstat_pairs(const double *x, int64_t v, int32_t n, int32_t n1,
                    const int16_t *orders, const int32_t *pairs, int64_t npairs,
                    double *t_out, double *num_out, int32_t *deg_out, void *stream,
                    rmx_status *st);

/* ---------------------------------------------------------------- RapidPT
 * Replaces reference rapid.py:138-206 (_recover_block), lrmc.py:127-157
 * (solve_block / fit_coefficients / complete_column) and lrmc.py:160-268
 * (track_update / train_basis).  Observation sets (Omega) and labels are
 * drawn host-side with the reference's own streams and passed in, so they
 * are bit-identical; the Gaussian residuals of the recovery are drawn on the
 * device from a counter-based Philox stream keyed by (seed, permutation)
 * ("RapidPT noise").
 *
 * rmx_rapid_stats: t_out[p*k + i] = statistic of voxel omegas[p*k + i] under
 *   orders[p] (bit-identical to the reference's batched _welch_rows).
 *   Degenerate -> RMX_E_DEGENERATE with perm = p, voxel = i (Omega index). */
int rmx_rapid_stats(const double *x, int64_t v, int32_t n, int32_t n1,
                    const int16_t *orders, const int32_t *omegas, int64_t L, int32_t k,
                    double *t_out, void *stream, rmx_status *st);

/* Batched least squares on gathered rows (solve_block semantics):
 *   w_b = argmin |U[idx_b] w - vals_b|  via G = A^T A, A = [U[idx_b] | vals_b],
 *   Cholesky in fp64.  idx = NULL uses rows 0..k-1.  flag_out[b] = 1 for a
 *   rank-deficient restriction (caller resamples, rapid.py:173-196).
 *   norms_out[4b..4b+3] = (|resid|^2 by the normal equations, |w|^2,
 *   min L_ii, max L_ii) -- max/min L_ii is a lower bound of the reference's
 *   condition number sqrt(lambda_max / lambda_min) of U_Omega. */
size_t rmx_lsq_workspace_bytes(int32_t r, int64_t batch);
int rmx_lsq_solve(const double *u, int64_t ldu, int32_t r, const int32_t *idx, int32_t k,
                  const double *vals, int64_t B, double *w_out, int32_t *flag_out,
                  double *norms_out, void *workspace, size_t workspace_bytes, void *stream,
                  rmx_status *st);

/* Reference-semantics batched least squares (replaces lrmc.py:127-149
 * solve_block and the condition test of lrmc.py:96-104 _gram_fit /
 * lrmc.py:107-124 fit_coefficients): G = [U[idx_b] | vals_b]^T [..] in fp64;
 * cond_b = sqrt(lambda_max / lambda_min) of G's r x r block (Householder
 * tridiagonalisation + bisection on the device; inf when lambda_min <= 0);
 * flag_b = cond_b > 1e12 (COND_LIMIT, lrmc.py:22).  Accepted systems: w by
 * Cholesky, or by pivoted LU when the Cholesky meets a non-positive pivot;
 * rejected: w = U_Omega^T vals (the reference's solve against the identity).
 * u, idx, vals, w_out: device; flag_out, cond_out: HOST arrays (nullable). */
int rmx_lsq_solve_exact(const double *u, int64_t ldu, int32_t r, const int32_t *idx, int32_t k,
                        const double *vals, int64_t B, double *w_out, int32_t *flag_out,
                        double *cond_out, void *stream, rmx_status *st);

/* One GROUSE update in place (replaces lrmc.py:160-193 track_update): u
 * (v x r, device, row-major), idx (sorted, device), vals (device).  Returns
 * RMX_E_ILLCOND (st->value = cond) when the restricted basis is rejected;
 * *resid_norm (host) = |vals - U_Omega w| before the update. */
int rmx_track_update(double *u, int64_t v, int32_t r, const int32_t *idx, int32_t k,
                     const double *vals, double step, double *resid_norm, void *stream,
                     rmx_status *st);

/* numpy's Generator.standard_normal over the reference's streams, bit for
 * bit, on host cores (replaces the normal draws of lrmc.py:85-93 BASIS_INIT
 * and rapid.py:115-121 SHIFT_GAP).  rmx_normal_tables_set installs numpy's
 * ziggurat tables (k, w, f: 256 entries each; normals.py reads them from the
 * installed numpy).  rmx_standard_normal: stream(seed, *path) (npath <= 3)
 * -> out[0..count) (host).  rmx_standard_normal_rows: rows i in [lo, hi) of
 * stream(seed, domain, i), count each, into out32 (float, as numpy's float64
 * cast) or out64, on `threads` host threads (0 = all). */
int rmx_normal_tables_set(const uint64_t *k, const double *w, const double *f);
int rmx_standard_normal(uint64_t seed, const uint32_t *path, int32_t npath, int64_t count,
                        double *out, rmx_status *st);
int rmx_standard_normal_rows(uint64_t seed, uint32_t domain, int64_t lo, int64_t hi,
                             int64_t count, float *out32, double *out64, int32_t threads,
                             rmx_status *st);
/* The same stream drawn in consecutive pieces (open / fill* / close). */
typedef struct rmx_normal_stream rmx_normal_stream;
int rmx_normal_stream_open(uint64_t seed, const uint32_t *path, int32_t npath,
                           rmx_normal_stream **out, rmx_status *st);
int rmx_normal_stream_fill(rmx_normal_stream *h, int64_t count, double *out);
int rmx_normal_stream_close(rmx_normal_stream *h);
/* count normals of the stream into device memory (dev_out), drawn through
 * the caller's page-locked ring (pinned_doubles doubles, two halves) with
 * each half's upload on `stream` overlapping the next half's draw; returns
 * after the last copy.  Replaces the init_basis draw + transfer of
 * lrmc.py:85-93 (the reference draws into host memory). */
int rmx_normal_stream_fill_device(rmx_normal_stream *h, int64_t count, double *dev_out,
                                  double *pinned, int64_t pinned_doubles, void *stream,
                                  rmx_status *st);

/* rmx_lsq_solve with the Gram on the tensor cores (v = rows of U): G~ =
 * [U_Omega | vals]^T [U_Omega | vals] from fp16 hi/lo planes (tcgen05,
 * fp32-accurate), Cholesky of G~ in fp64, then two steps of iterative
 * refinement with the fp64 residual U_Omega^T (vals - U_Omega w): the result
 * is the fp64 normal-equations solution (relative difference ~1e-12 at the
 * well-conditioned restrictions of random Omega).  Systems whose factor is
 * singular (flag_out, as rmx_lsq_solve) or whose refinement has not settled
 * are re-solved with the fp64 Gram.  stats (optional, 2 ints): [tensor path
 * used, systems re-solved in fp64].  Falls back to rmx_lsq_solve for shapes
 * the tensor path does not take (r + 1 > 512) or when RMX_GRAM_FP64 is set.
 * Replaces reference lrmc.py:127-149 solve_block (batched). */
int rmx_lsq_solve_tc(const double *u, int64_t ldu, int64_t v, int32_t r, const int32_t *idx,
                     int32_t k, const double *vals, int64_t B, double *w_out, int32_t *flag_out,
                     void *workspace, size_t workspace_bytes, int32_t *stats, void *stream,
                     rmx_status *st);

/* rmx_lsq_solve_tc with an adaptive second refinement step (RapidPT
 * recovery, rapid.py:198-205): every system takes one fp64 refinement step;
 * a system whose first correction is within settle_tol |w| is settled (its w
 * is within ~settle_tol^2 |w| of the normal-equations solution: 1e-8 at the
 * engine's 1e-4), the others take the second step and, if still unsettled,
 * the fp64 Gram path.  settle_tol = 0 is rmx_lsq_solve_tc. */
int rmx_lsq_solve_tc_settle(const double *u, int64_t ldu, int64_t v, int32_t r,
                            const int32_t *idx, int32_t k, const double *vals, int64_t B,
                            double *w_out, int32_t *flag_out, void *workspace,
                            size_t workspace_bytes, int32_t *stats, double settle_tol,
                            void *stream, rmx_status *st);

/* Completion + residual + max (rapid.py:198-205): for each of B columns,
 *   max_out[b] = max_j op(W[b] . U[j] + sigma * z(perm_base + b, j)) + mu,
 * op = |.| when two_sided.  z is Philox N(0,1) unless znoise (B x v fp32) is
 * given; base (B x v fp64) switches to op(base - W[b].U[j]) (residual-sup). */
int rmx_complete_max(const float *u32, int64_t v, int32_t r, const float *w32, int64_t B,
                     int64_t perm_base, double sigma, double mu, uint64_t seed,
                     int32_t two_sided, const float *znoise, const double *base,
                     double *max_out, void *stream, rmx_status *st);

/* Small helpers used by the host orchestration. */
int rmx_to_f32(const double *a, int64_t n, float *out, void *stream, rmx_status *st);
int rmx_row_max(const double *a, int64_t rows, int64_t cols, int32_t two_sided, double *out,
                void *stream, rmx_status *st);
int rmx_resid_batch(const double *u, int32_t r, const int32_t *idx, int32_t k,
                    const double *vals, const double *w, int64_t B, double *resid,
                    void *stream, rmx_status *st);
int rmx_gather_rows(const double *t, int64_t ldt, const int32_t *idx, int32_t k, int64_t B,
                    double *out, void *stream, rmx_status *st);
int rmx_gemv(const double *u, int64_t v, int32_t r, const double *w, double *out, void *stream,
             rmx_status *st);
int rmx_mean_var(const double *a, int64_t n, double *out2, void *stream, rmx_status *st);
/* CholeskyQR2 re-orthonormalisation of U (v x r) when max|U^T U - I| > 1e-8
 * (or always with force); *drift receives the error before the call. */
int rmx_orthonormalize(double *u, int64_t v, int32_t r, int32_t force, double *drift,
                       void *stream, rmx_status *st);

/* GROUSE training (train_basis): t is ell x v (training statistics,
 * perm-major), omegas0 max_passes x ell x k first-attempt observation sets,
 * u (v x r) the initial orthonormal basis, updated in place.  cb draws the
 * next observation set of (col, pass) on an ill-conditioned restriction. */
typedef int (*rmx_omega_cb)(void *user, int32_t col, int32_t pass, int32_t attempt,
                            int32_t *omega_out);
int rmx_grouse_train(const double *t, int64_t v, int32_t ell, int32_t r, int32_t k,
                     const int32_t *omegas0, int32_t max_passes, double tol, double *u,
                     rmx_omega_cb cb, void *user, double *pass_resid, int32_t *passes_out,
                     int32_t *converged_out, int64_t *updates_out, int32_t *final_omegas,
                     void *stream, rmx_status *st);

#ifdef __cplusplus
}
#endif

#endif /* RMX_H_ */
