/*
 * rmx_oracle.c -- CPU restatement of the reference NaivePT statistic path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path never links it.
 *
 * What it restates (reference = /root/reference/pkg/src/rapidmaxnull):
 *   - numpy's float64 add.reduce along a contiguous axis (pairwise summation,
 *     8 accumulators, block 128) -- the arithmetic under x.mean()/x.var()
 *     used by _welch_rows (teststat.py:36-40);
 *   - _welch_rows (teststat.py:28-50): t = (m1-m2)/sqrt(s1^2/n1 + s2^2/n2),
 *     two-pass unbiased variance, var_term == 0 rule (num == 0 -> t = 0,
 *     else DegenerateVoxelError(first voxel, mean_diff));
 *   - DataMatrix.group_blocks (model.py:65-69): group 1 = order[:n1] in
 *     permutation order, group 2 = order[n1:];
 *   - column_max (teststat.py:88-90) and the _max_block loop of run_naive
 *     (naive.py:49-57), plus the argmax (first index on ties, np.argmax).
 *
 * The restatement is bit-exact against the reference: every operation is a
 * single IEEE-754 double op in the same order numpy performs it (build with
 * -O2 -ffp-contract=off; see oracle/Makefile).  tests/test_oracle_golden.py
 * pins it against vectors produced by the reference itself.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PW_BLOCK 128

/* numpy pairwise sum (loops_utils.h.src, @TYPE@_pairwise_sum): the value
 * a[i] is produced on the fly by `get(ctx, i)` so gathers and the squared
 * deviations of the variance pass need no temporaries. */
typedef double (*getter_fn)(const void *ctx, long i);

static double pw_sum(getter_fn get, const void *ctx, long lo, long n)
{
    if (n < 8) {
        double res = 0.0;
        for (long i = 0; i < n; i++) res += get(ctx, lo + i);
        return res;
    }
    if (n <= PW_BLOCK) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = get(ctx, lo + j);
        long i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += get(ctx, lo + i + j);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += get(ctx, lo + i);
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(get, ctx, lo, n2) + pw_sum(get, ctx, lo + n2, n - n2);
}

typedef struct {
    const double *row;     /* one voxel row, n subjects */
    const int64_t *idx;    /* subject indices of the group, in order */
    double mean;
} group_ctx;

static double get_val(const void *c, long i)
{
    const group_ctx *g = (const group_ctx *)c;
    return g->row[g->idx[i]];
}

static double get_sqdev(const void *c, long i)
{
    const group_ctx *g = (const group_ctx *)c;
    double d = g->row[g->idx[i]] - g->mean;
    return d * d;
}

/* _welch_rows for one voxel row under one labelling.
 * Returns 0 on success, 1 when var_term == 0 and num != 0 (degenerate);
 * *num_out always receives m1 - m2. */
int rmx_oracle_welch(const double *row, const int64_t *order, int n1, int n2,
                     double *t_out, double *num_out)
{
    group_ctx g1 = {row, order, 0.0};
    group_ctx g2 = {row, order + n1, 0.0};
    double m1 = pw_sum(get_val, &g1, 0, n1) / (double)n1;
    double m2 = pw_sum(get_val, &g2, 0, n2) / (double)n2;
    g1.mean = pw_sum(get_val, &g1, 0, n1) / (double)n1;   /* var() recomputes its mean */
    g2.mean = pw_sum(get_val, &g2, 0, n2) / (double)n2;
    double v1 = pw_sum(get_sqdev, &g1, 0, n1) / (double)(n1 - 1);
    double v2 = pw_sum(get_sqdev, &g2, 0, n2) / (double)(n2 - 1);
    double var_term = v1 / (double)n1 + v2 / (double)n2;
    double num = m1 - m2;
    *num_out = num;
    if (var_term == 0.0) {
        *t_out = 0.0;
        return num != 0.0 ? 1 : 0;
    }
    *t_out = num / sqrt(var_term);
    return 0;
}

/* run_naive restated (naive.py:60-109 / _max_block 49-57).
 *   x      : v x n row-major float64 (DataMatrix.values)
 *   orders : L x n int64, row i = PermutationPlan.shuffle(i)
 *   t_out  : NULL or v x L row-major (StatMatrix.values layout)
 * On a degenerate voxel returns 1 and reports the first (perm, voxel) in
 * permutation order with its mean difference, as the reference raises. */
int rmx_oracle_naive(const double *x, int64_t v, int n, int n1,
                     const int64_t *orders, int64_t L, int two_sided,
                     double *max_out, int64_t *argmax_out, double *t_out,
                     int64_t *deg_perm, int64_t *deg_voxel, double *deg_num)
{
    int n2 = n - n1;
    for (int64_t p = 0; p < L; p++) {
        const int64_t *ord = orders + p * (int64_t)n;
        double best = 0.0;
        int64_t arg = -1;
        for (int64_t j = 0; j < v; j++) {
            double t, num;
            if (rmx_oracle_welch(x + j * (int64_t)n, ord, n1, n2, &t, &num)) {
                *deg_perm = p;
                *deg_voxel = j;
                *deg_num = num;
                return 1;
            }
            if (t_out) t_out[j * L + p] = t;
            double key = two_sided ? fabs(t) : t;
            if (arg < 0 || key > best) {
                best = key;
                arg = j;
            }
        }
        max_out[p] = best;
        argmax_out[p] = arg;
    }
    return 0;
}

/* numpy mean of a contiguous vector (add.reduce / n) -- exposed so tests can
 * pin the pairwise restatement directly against np.sum / np.mean. */
double rmx_oracle_np_sum(const double *a, int64_t n)
{
    group_ctx g;
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; i++) idx[i] = i;
    g.row = a;
    g.idx = idx;
    g.mean = 0.0;
    double s = pw_sum(get_val, &g, 0, n);
    free(idx);
    return s;
}
