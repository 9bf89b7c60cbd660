/*
 * flexconv_oracle.c -- CPU restatement of the reference flex-convolution hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing here is on the product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this library,
 * and only as the checker.  The product (paper_1803_07289_b200/) never links it.
 *
 * Every routine restates the reference algorithm in plain C, fp64 arithmetic,
 * int64 neighbour indices, point-major layouts, exactly as the reference does:
 *   /root/reference/pkg/src/flexconv/_native.pyx   (Cython kernels, KERNEL_VERSION 1)
 *   /root/reference/pkg/src/flexconv/neighborhood.py (brute-force kNN oracle)
 * Parity of this restatement is PINNED against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py -> tests/golden/*.npz) and
 * against the compiled reference (oracle/_ref/_native*.so) in tests/test_oracle.py.
 *
 * Summation order follows the reference loops statement by statement, with
 * separately rounded multiply and add (compile with -ffp-contract=off), so the
 * forward, pool and kNN results are bitwise identical to _native.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define NBR(i, s) nbr[(int64_t)(i) * k + (s)]

/* _native.pyx:25-66 -- moments X[c,t] = sum_s f[j,c]*(l_i - l_j)_t, X[c,d] = sum_s f[j,c],
 * then out[i,c'] = sum_c (sum_t theta[c',c,t] X[c,t]) + theta_b[c',c] X[c,d]. */
void fco_conv_forward(int64_t n, int64_t C, int64_t d, int64_t k, int64_t cout,
                      const double *feat, const double *loc, const int64_t *nbr,
                      const double *theta, const double *theta_b, double *out,
                      int num_threads)
{
    int nt = num_threads > 0 ? num_threads : 1;
#pragma omp parallel num_threads(nt)
    {
        double *X = (double *)malloc(sizeof(double) * C * (d + 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            for (int64_t q = 0; q < C * (d + 1); ++q) X[q] = 0.0;
            for (int64_t s = 0; s < k; ++s) {
                int64_t j = NBR(i, s);
                for (int64_t t = 0; t < d; ++t) {
                    double ot = loc[i * d + t] - loc[j * d + t];
                    for (int64_t c = 0; c < C; ++c)
                        X[c * (d + 1) + t] += feat[j * C + c] * ot;
                }
                for (int64_t c = 0; c < C; ++c)
                    X[c * (d + 1) + d] += feat[j * C + c];
            }
            for (int64_t cp = 0; cp < cout; ++cp) {
                double acc = 0.0;
                for (int64_t c = 0; c < C; ++c) {
                    for (int64_t t = 0; t < d; ++t)
                        acc = acc + theta[(cp * C + c) * d + t] * X[c * (d + 1) + t];
                    acc = acc + theta_b[cp * C + c] * X[c * (d + 1) + d];
                }
                out[i * cout + cp] = acc;
            }
        }
        free(X);
    }
}

/* _native.pyx:69-127 -- exact gradients, single-threaded fixed i-order.
 * Outputs are ACCUMULATED (callers zero-fill, as flexops.py:123-126 does).
 * d_loc may be NULL when with_locations == 0. */
void fco_conv_backward(int64_t n, int64_t C, int64_t d, int64_t k, int64_t cout,
                       const double *up, const double *feat, const double *loc,
                       const int64_t *nbr, const double *theta, const double *theta_b,
                       double *d_feat, double *d_loc, double *d_theta, double *d_theta_b,
                       int with_locations)
{
    double *X = (double *)malloc(sizeof(double) * C * (d + 1));
    double *W = (double *)malloc(sizeof(double) * C * (d + 1));
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t q = 0; q < C * (d + 1); ++q) { X[q] = 0.0; W[q] = 0.0; }
        for (int64_t s = 0; s < k; ++s) {
            int64_t j = NBR(i, s);
            for (int64_t t = 0; t < d; ++t) {
                double ot = loc[i * d + t] - loc[j * d + t];
                for (int64_t c = 0; c < C; ++c)
                    X[c * (d + 1) + t] += feat[j * C + c] * ot;
            }
            for (int64_t c = 0; c < C; ++c)
                X[c * (d + 1) + d] += feat[j * C + c];
        }
        for (int64_t cp = 0; cp < cout; ++cp) {
            double gi = up[i * cout + cp];
            for (int64_t c = 0; c < C; ++c) {
                for (int64_t t = 0; t < d; ++t) {
                    d_theta[(cp * C + c) * d + t] += gi * X[c * (d + 1) + t];
                    W[c * (d + 1) + t] += gi * theta[(cp * C + c) * d + t];
                }
                d_theta_b[cp * C + c] += gi * X[c * (d + 1) + d];
                W[c * (d + 1) + d] += gi * theta_b[cp * C + c];
            }
        }
        for (int64_t s = 0; s < k; ++s) {
            int64_t j = NBR(i, s);
            for (int64_t c = 0; c < C; ++c) {
                double acc = W[c * (d + 1) + d];
                for (int64_t t = 0; t < d; ++t)
                    acc = acc + W[c * (d + 1) + t] * (loc[i * d + t] - loc[j * d + t]);
                d_feat[j * C + c] += acc;
            }
            if (with_locations) {
                for (int64_t t = 0; t < d; ++t) {
                    double dt = 0.0;
                    for (int64_t c = 0; c < C; ++c)
                        dt = dt + feat[j * C + c] * W[c * (d + 1) + t];
                    d_loc[i * d + t] += dt;
                    d_loc[j * d + t] -= dt;
                }
            }
        }
    }
    free(X);
    free(W);
}

/* flex_deconv = the adjoint A(theta)^T x of flex_conv (no reference function; the
 * reference's exact equivalent is flex_conv_backward(...).d_features, which does not
 * depend on `features`: _native.pyx:106-120).  y[j,c] += sum_{i: j in N(i)} w_ij(c),
 * w_ij(c) = W_i[c,d] + sum_t W_i[c,t](l_i-l_j)_t, W_i = x_i^T [theta;theta_b].
 * Accumulates into y (callers zero-fill). */
void fco_deconv_forward(int64_t n, int64_t C, int64_t d, int64_t k, int64_t cout,
                        const double *x, const double *loc, const int64_t *nbr,
                        const double *theta, const double *theta_b, double *y)
{
    double *W = (double *)malloc(sizeof(double) * C * (d + 1));
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t q = 0; q < C * (d + 1); ++q) W[q] = 0.0;
        for (int64_t cp = 0; cp < cout; ++cp) {
            double gi = x[i * cout + cp];
            for (int64_t c = 0; c < C; ++c) {
                for (int64_t t = 0; t < d; ++t)
                    W[c * (d + 1) + t] += gi * theta[(cp * C + c) * d + t];
                W[c * (d + 1) + d] += gi * theta_b[cp * C + c];
            }
        }
        for (int64_t s = 0; s < k; ++s) {
            int64_t j = NBR(i, s);
            for (int64_t c = 0; c < C; ++c) {
                double acc = W[c * (d + 1) + d];
                for (int64_t t = 0; t < d; ++t)
                    acc = acc + W[c * (d + 1) + t] * (loc[i * d + t] - loc[j * d + t]);
                y[j * C + c] += acc;
            }
        }
    }
    free(W);
}

/* _native.pyx:130-155 -- per-point per-channel max; ties -> lowest global index. */
void fco_pool_forward(int64_t n, int64_t C, int64_t k, const double *feat,
                      const int64_t *nbr, double *out, int64_t *argmax, int num_threads)
{
    int nt = num_threads > 0 ? num_threads : 1;
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t c = 0; c < C; ++c) {
            int64_t bj = NBR(i, 0);
            double bv = feat[bj * C + c];
            for (int64_t s = 1; s < k; ++s) {
                int64_t j = NBR(i, s);
                double v = feat[j * C + c];
                if (v > bv || (v == bv && j < bj)) { bv = v; bj = j; }
            }
            out[i * C + c] = bv;
            argmax[i * C + c] = bj;
        }
    }
}

/* _native.pyx:158-168 -- scatter-add upstream to the recorded winner, fixed i-order.
 * Accumulates into d_feat (callers zero-fill, flexops.py:163). */
void fco_pool_backward(int64_t n, int64_t C, const double *up, const int64_t *argmax,
                       double *d_feat)
{
    for (int64_t i = 0; i < n; ++i)
        for (int64_t c = 0; c < C; ++c)
            d_feat[argmax[i * C + c] * C + c] += up[i * C + c];
}

/* neighborhood.py:171-187 (knn_brute_force) -- row i = [i, the k-1 nearest OTHER points
 * ordered by (squared distance, index)].  The reference takes a stable argsort of the
 * d^2 row and drops i; a bounded insertion list over ascending j gives the same rows.
 * d^2 = sum_t (p_i,t - p_j,t)^2 accumulated left to right (numpy's
 * ((a-b)**2).sum(-1) and _native.pyx:218-221 agree on this order). */
void fco_knn_brute(int64_t n, int64_t d, int64_t k, const double *pts, int64_t *out,
                   int num_threads)
{
    int nt = num_threads > 0 ? num_threads : 1;
    int64_t kk = k - 1;
#pragma omp parallel num_threads(nt)
    {
        double *bd = (double *)malloc(sizeof(double) * (kk > 0 ? kk : 1));
        int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (kk > 0 ? kk : 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            out[i * k] = i;
            int64_t cnt = 0;
            for (int64_t j = 0; j < n && kk > 0; ++j) {
                if (j == i) continue;
                double dist = 0.0;
                for (int64_t t = 0; t < d; ++t) {
                    double dv = pts[i * d + t] - pts[j * d + t];
                    dist = dist + dv * dv;
                }
                int64_t m;
                if (cnt == kk) {
                    /* j ascending: an equal distance never beats an earlier index */
                    if (!(dist < bd[kk - 1])) continue;
                    m = kk - 1;
                } else {
                    m = cnt;
                }
                int64_t q = m;
                while (q > 0 && bd[q - 1] > dist) { bd[q] = bd[q - 1]; bi[q] = bi[q - 1]; --q; }
                bd[q] = dist;
                bi[q] = j;
                if (cnt < kk) ++cnt;
            }
            for (int64_t p = 0; p < kk; ++p) out[i * k + 1 + p] = bi[p];
        }
        free(bd);
        free(bi);
    }
}

/* Same contract as fco_knn_brute, for a subset of query rows only (large-n spot checks):
 * out[r*k..] = the row of point rows[r]. */
void fco_knn_rows(int64_t n, int64_t d, int64_t k, const double *pts, const int64_t *rows,
                  int64_t nrows, int64_t *out, int num_threads)
{
    int nt = num_threads > 0 ? num_threads : 1;
    int64_t kk = k - 1;
#pragma omp parallel num_threads(nt)
    {
        double *bd = (double *)malloc(sizeof(double) * (kk > 0 ? kk : 1));
        int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (kk > 0 ? kk : 1));
#pragma omp for schedule(static)
        for (int64_t r = 0; r < nrows; ++r) {
            int64_t i = rows[r];
            out[r * k] = i;
            int64_t cnt = 0;
            for (int64_t j = 0; j < n && kk > 0; ++j) {
                if (j == i) continue;
                double dist = 0.0;
                for (int64_t t = 0; t < d; ++t) {
                    double dv = pts[i * d + t] - pts[j * d + t];
                    dist = dist + dv * dv;
                }
                int64_t m;
                if (cnt == kk) {
                    if (!(dist < bd[kk - 1])) continue;
                    m = kk - 1;
                } else {
                    m = cnt;
                }
                int64_t q = m;
                while (q > 0 && bd[q - 1] > dist) { bd[q] = bd[q - 1]; bi[q] = bi[q - 1]; --q; }
                bd[q] = dist;
                bi[q] = j;
                if (cnt < kk) ++cnt;
            }
            for (int64_t p = 0; p < kk; ++p) out[r * k + 1 + p] = bi[p];
        }
        free(bd);
        free(bi);
    }
}

/* ---------------------------------------------------------------------------------------
 * Large-n checkers (row subsets and a parallel parameter-gradient reduction).  Same
 * arithmetic as the full routines above; used where the serial reference loop would take
 * minutes (1M / 7M-point clouds).  TEST INFRASTRUCTURE ONLY, like everything in this file.
 * ------------------------------------------------------------------------------------- */

/* _native.pyx:46-66 restricted to query rows: out[r, :] = forward row of point rows[r]
 * (the same statement order as fco_conv_forward, hence bitwise equal to it). */
void fco_conv_forward_rows(int64_t n, int64_t C, int64_t d, int64_t k, int64_t cout,
                           const double *feat, const double *loc, const int64_t *nbr,
                           const double *theta, const double *theta_b,
                           const int64_t *rows, int64_t nrows, double *out, int num_threads)
{
    (void)n;
    int nt = num_threads > 0 ? num_threads : 1;
#pragma omp parallel num_threads(nt)
    {
        double *X = (double *)malloc(sizeof(double) * C * (d + 1));
#pragma omp for schedule(static)
        for (int64_t r = 0; r < nrows; ++r) {
            int64_t i = rows[r];
            for (int64_t q = 0; q < C * (d + 1); ++q) X[q] = 0.0;
            for (int64_t s = 0; s < k; ++s) {
                int64_t j = NBR(i, s);
                for (int64_t t = 0; t < d; ++t) {
                    double ot = loc[i * d + t] - loc[j * d + t];
                    for (int64_t c = 0; c < C; ++c)
                        X[c * (d + 1) + t] += feat[j * C + c] * ot;
                }
                for (int64_t c = 0; c < C; ++c)
                    X[c * (d + 1) + d] += feat[j * C + c];
            }
            for (int64_t cp = 0; cp < cout; ++cp) {
                double acc = 0.0;
                for (int64_t c = 0; c < C; ++c) {
                    for (int64_t t = 0; t < d; ++t)
                        acc = acc + theta[(cp * C + c) * d + t] * X[c * (d + 1) + t];
                    acc = acc + theta_b[cp * C + c] * X[c * (d + 1) + d];
                }
                out[r * cout + cp] = acc;
            }
        }
        free(X);
    }
}

/* W_i[c, t] = sum_c' g_i[c'] theta[c', c, t], W_i[c, d] = sum_c' g_i[c'] theta_b[c', c]
 * in the statement order of _native.pyx:104-113. */
static void oracle_weights(int64_t i, int64_t C, int64_t d, int64_t cout, const double *up,
                           const double *theta, const double *theta_b, double *W)
{
    for (int64_t q = 0; q < C * (d + 1); ++q) W[q] = 0.0;
    for (int64_t cp = 0; cp < cout; ++cp) {
        double gi = up[i * cout + cp];
        for (int64_t c = 0; c < C; ++c) {
            for (int64_t t = 0; t < d; ++t)
                W[c * (d + 1) + t] += gi * theta[(cp * C + c) * d + t];
            W[c * (d + 1) + d] += gi * theta_b[cp * C + c];
        }
    }
}

/* d_features and d_locations of _native.pyx:69-127 at query rows only.  Row j receives
 *   d_f[j]  += w_ij            for every slot (i, s) with nbr[i, s] == j,
 *   d_l[j]  += dt(j, s)        for every slot s of its own row (centre role),
 *   d_l[j]  -= dt(i, s)        for every slot (i, s) with nbr[i, s] == j (neighbour role),
 * and the reference adds these in ascending i, then s -- so the contributing rows i (the
 * reverse list of j plus j itself) are visited in ascending order with the reference's
 * per-slot statement order, which makes each requested row bitwise equal to the serial
 * reference.  Reverse lists are found by one scan of the neighbour table. */
void fco_conv_backward_rows(int64_t n, int64_t C, int64_t d, int64_t k, int64_t cout,
                            const double *up, const double *feat, const double *loc,
                            const int64_t *nbr, const double *theta, const double *theta_b,
                            const int64_t *rows, int64_t nrows, double *d_feat_rows,
                            double *d_loc_rows, int num_threads)
{
    int nt = num_threads > 0 ? num_threads : 1;
    /* slot of each requested row (-1 elsewhere); duplicates in `rows` map to the last */
    int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * n);
    for (int64_t q = 0; q < n; ++q) slot[q] = -1;
    for (int64_t r = 0; r < nrows; ++r) slot[rows[r]] = r;
    /* reverse lists of the requested rows: count, scan, fill (ascending i by construction) */
    int64_t *cnt = (int64_t *)calloc(nrows + 1, sizeof(int64_t));
    for (int64_t e = 0; e < n * k; ++e) {
        int64_t r = slot[nbr[e]];
        if (r >= 0) cnt[r + 1]++;
    }
    for (int64_t r = 0; r < nrows; ++r) cnt[r + 1] += cnt[r];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nrows + 1));
    memcpy(fill, cnt, sizeof(int64_t) * (nrows + 1));
    int64_t *rev = (int64_t *)malloc(sizeof(int64_t) * (cnt[nrows] > 0 ? cnt[nrows] : 1));
    for (int64_t e = 0; e < n * k; ++e) {
        int64_t r = slot[nbr[e]];
        if (r >= 0) rev[fill[r]++] = e / k;
    }
#pragma omp parallel num_threads(nt)
    {
        double *W = (double *)malloc(sizeof(double) * C * (d + 1));
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < nrows; ++r) {
            int64_t j = rows[r];
            double *df = d_feat_rows + r * C;
            double *dl = d_loc_rows ? d_loc_rows + r * d : NULL;
            for (int64_t c = 0; c < C; ++c) df[c] = 0.0;
            if (dl) for (int64_t t = 0; t < d; ++t) dl[t] = 0.0;
            int64_t a = cnt[r], b = cnt[r + 1];
            int own_done = 0;
            int64_t prev = -1;
            /* visit the distinct contributing rows i in ascending order: rev[a..b) is
             * ascending (with repeats when j occurs twice in a row); j itself is merged in */
            while (a < b || !own_done) {
                int64_t i;
                if (a < b && (own_done || rev[a] <= j)) {
                    i = rev[a];
                } else {
                    i = j;
                }
                if (i == j) own_done = 1;
                /* skip repeats of the same i (its slots are all handled in one visit) */
                while (a < b && rev[a] == i) ++a;
                if (i == prev) continue;
                prev = i;
                oracle_weights(i, C, d, cout, up, theta, theta_b, W);
                for (int64_t s = 0; s < k; ++s) {
                    int64_t jj = NBR(i, s);
                    if (jj == j) {
                        for (int64_t c = 0; c < C; ++c) {
                            double acc = W[c * (d + 1) + d];
                            for (int64_t t = 0; t < d; ++t)
                                acc = acc + W[c * (d + 1) + t] * (loc[i * d + t] - loc[jj * d + t]);
                            df[c] += acc;
                        }
                    }
                    if (dl && (i == j || jj == j)) {
                        for (int64_t t = 0; t < d; ++t) {
                            double dt = 0.0;
                            for (int64_t c = 0; c < C; ++c)
                                dt = dt + feat[jj * C + c] * W[c * (d + 1) + t];
                            if (i == j) dl[t] += dt;
                            if (jj == j) dl[t] -= dt;
                        }
                    }
                }
            }
        }
        free(W);
    }
    free(slot);
    free(cnt);
    free(fill);
    free(rev);
}

/* d_theta and d_theta_b of _native.pyx:104-111 over ALL points, fp64, in parallel: each
 * thread accumulates a static block of points in i order into its own buffer, and the
 * buffers are added in thread order.  The result differs from the serial reference only
 * by fp64 regrouping (~1e-13 relative); it is the full-N checker for the GPU reductions. */
void fco_conv_param_grads(int64_t n, int64_t C, int64_t d, int64_t k, int64_t cout,
                          const double *up, const double *feat, const double *loc,
                          const int64_t *nbr, double *d_theta, double *d_theta_b,
                          int num_threads)
{
    int nt = num_threads > 0 ? num_threads : 1;
    int64_t P = cout * C * (d + 1);
    double *part = (double *)calloc((size_t)nt * P, sizeof(double));
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *acc = part + (int64_t)tid * P; /* [cout][C][d+1] */
        double *X = (double *)malloc(sizeof(double) * C * (d + 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            for (int64_t q = 0; q < C * (d + 1); ++q) X[q] = 0.0;
            for (int64_t s = 0; s < k; ++s) {
                int64_t j = NBR(i, s);
                for (int64_t t = 0; t < d; ++t) {
                    double ot = loc[i * d + t] - loc[j * d + t];
                    for (int64_t c = 0; c < C; ++c)
                        X[c * (d + 1) + t] += feat[j * C + c] * ot;
                }
                for (int64_t c = 0; c < C; ++c)
                    X[c * (d + 1) + d] += feat[j * C + c];
            }
            for (int64_t cp = 0; cp < cout; ++cp) {
                double gi = up[i * cout + cp];
                double *a = acc + cp * C * (d + 1);
                for (int64_t q = 0; q < C * (d + 1); ++q) a[q] += gi * X[q];
            }
        }
        free(X);
    }
    for (int64_t cp = 0; cp < cout; ++cp)
        for (int64_t c = 0; c < C; ++c) {
            for (int64_t t = 0; t <= d; ++t) {
                double v = 0.0;
                for (int q = 0; q < nt; ++q) v += part[(int64_t)q * P + (cp * C + c) * (d + 1) + t];
                if (t < d) d_theta[(cp * C + c) * d + t] = v;
                else d_theta_b[cp * C + c] = v;
            }
        }
    free(part);
}

int fco_version(void) { return 2; }
