/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's RaPP table path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * The product path (paper_2505_01968_b200/) never links or calls this file.
 *
 * Every function cites the reference (paths relative to /root/reference,
 * hs/ = pkg/src/hybridscale/).  Arithmetic is IEEE binary64, each operation
 * rounded individually, evaluated left to right exactly as the reference
 * writes it.  Build with -ffp-contract=off (see oracle/Makefile) so gcc never
 * fuses a multiply-add: the reference's Cython C is compiled at -O2 for
 * x86-64 without FMA (hs/_kernels/_grid_cy.pyx:4-5).
 *
 * Parity pin: tests/test_oracle.py checks this file against the golden
 * vectors in tests/golden/ (produced by the real reference, see
 * tests/golden/gen_golden.py) and, where oracle/_ref is built, against the
 * reference's own compiled _grid_cy extension on random inputs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* hs/_kernels/_grid_cy.pyx:9-33 (twin _grid_py.py:11-34).  Clamped binary
 * search; a node hit returns t == 0.0 exactly; NaN falls through to
 * (0,1,NaN) when n >= 2. */
void or_locate(const double *axis, int64_t n, double x,
               int64_t *lo_out, int64_t *hi_out, double *t_out)
{
    int64_t last = n - 1, lo, hi, mid;
    if (x <= axis[0]) { *lo_out = 0; *hi_out = 0; *t_out = 0.0; return; }
    if (x >= axis[last]) { *lo_out = last; *hi_out = last; *t_out = 0.0; return; }
    lo = 0;
    hi = last;
    while (hi - lo > 1) {
        mid = (lo + hi) >> 1;
        if (axis[mid] <= x) lo = mid; else hi = mid;
    }
    if (axis[lo] == x) { *lo_out = lo; *hi_out = lo; *t_out = 0.0; return; }
    *lo_out = lo;
    *hi_out = hi;
    *t_out = (x - axis[lo]) / (axis[hi] - axis[lo]);
}

/* hs/_kernels/_grid_cy.pyx:36-51: quota lerps, then sm, then batch. */
double or_interp3(const double *b_axis, int64_t nb, const double *s_axis, int64_t ns,
                  const double *q_axis, int64_t nq, const double *v,
                  double b, double s, double q)
{
    int64_t i0, i1, j0, j1, k0, k1;
    double tb, ts, tq, c00, c01, c10, c11, c0, c1;
    or_locate(b_axis, nb, b, &i0, &i1, &tb);
    or_locate(s_axis, ns, s, &j0, &j1, &ts);
    or_locate(q_axis, nq, q, &k0, &k1, &tq);
#define V(i, j, k) v[((i) * ns + (j)) * nq + (k)]
    c00 = V(i0, j0, k0) + (V(i0, j0, k1) - V(i0, j0, k0)) * tq;
    c01 = V(i0, j1, k0) + (V(i0, j1, k1) - V(i0, j1, k0)) * tq;
    c10 = V(i1, j0, k0) + (V(i1, j0, k1) - V(i1, j0, k0)) * tq;
    c11 = V(i1, j1, k0) + (V(i1, j1, k1) - V(i1, j1, k0)) * tq;
#undef V
    c0 = c00 + (c01 - c00) * ts;
    c1 = c10 + (c11 - c10) * ts;
    return c0 + (c1 - c0) * tb;
}

/* hs/_kernels/_grid_cy.pyx:67-74: map over coords[n,3] into out[n]. */
void or_interp3_many(const double *b_axis, int64_t nb, const double *s_axis, int64_t ns,
                     const double *q_axis, int64_t nq, const double *v,
                     const double *coords, int64_t n, double *out)
{
    for (int64_t i = 0; i < n; ++i)
        out[i] = or_interp3(b_axis, nb, s_axis, ns, q_axis, nq, v,
                            coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]);
}

/* hs/perf.py:95-98: batch / (latency_ms / 1000.0). */
double or_throughput_from_latency(double batch, double latency_ms)
{
    return batch / (latency_ms / 1000.0);
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* hs/perf.py:140-145 (_batch_lattice): sorted unique allowed batches inside
 * [batches[0], batches[-1]]; None or empty -> all table batches.
 * Returns the count written to out (capacity >= max(nallowed, nb)). */
int64_t or_batch_lattice(const double *b_axis, int64_t nb, const int64_t *allowed,
                         int64_t nallowed, int64_t *out)
{
    int64_t m = 0;
    if (allowed != NULL && nallowed >= 0) {
        double lo = b_axis[0], hi = b_axis[nb - 1];
        for (int64_t i = 0; i < nallowed; ++i) {
            double bd = (double)allowed[i];
            if (lo <= bd && bd <= hi) out[m++] = allowed[i];
        }
        if (m > 0) {
            qsort(out, (size_t)m, sizeof(int64_t), cmp_i64);
            int64_t u = 1;
            for (int64_t i = 1; i < m; ++i)
                if (out[i] != out[u - 1]) out[u++] = out[i];
            return u;
        }
    }
    for (int64_t i = 0; i < nb; ++i) out[i] = (int64_t)b_axis[i];
    return nb;
}

/* hs/perf.py:104-138 (most_efficient_config).  Lattice batch x table sms x
 * range(step, 101, step); meet key (s*q, s, q, b) over rps >= target,
 * fallback key (-rps, s*q, s, q, b).  Returns 0, or -1 for the ValueError
 * branches at perf.py:114-117.  `allowed == NULL` means batches=None.
 * Strict-< updates in loop order == argmin of a total key. */
int or_most_efficient_config(const double *b_axis, int64_t nb, const double *s_axis,
                             int64_t ns, const double *q_axis, int64_t nq,
                             const double *v, double target, int64_t step,
                             const int64_t *allowed, int64_t nallowed,
                             int64_t out_bsq[3])
{
    if (!(target > 0.0)) {
        /* `target_rps <= 0` raises; NaN passes that test in Python, so
         * only reject what the reference rejects. */
        if (target <= 0.0) return -1;
    }
    if (step < 1 || step > 100) return -1;
    int64_t cap = nallowed > nb ? nallowed : nb;
    int64_t *bl = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
    int64_t m = or_batch_lattice(b_axis, nb, allowed, nallowed, bl);
    int have_meet = 0, have_all = 0;
    int64_t mk[4] = {0}, mc[3] = {0}, ac[3] = {0};
    double a_nrps = 0.0;
    int64_t ak[4] = {0};
    for (int64_t bi = 0; bi < m; ++bi) {
        int64_t b = bl[bi];
        for (int64_t si = 0; si < ns; ++si) {
            int64_t s = (int64_t)s_axis[si];
            for (int64_t q = step; q <= 100; q += step) {
                double lat = or_interp3(b_axis, nb, s_axis, ns, q_axis, nq, v,
                                        (double)b, (double)s, (double)q);
                double rps = or_throughput_from_latency((double)b, lat);
                int64_t cost = s * q;
                double nrps = -rps;
                int64_t k[4] = {cost, s, q, b};
                int better_all = !have_all;
                if (have_all) {
                    if (nrps < a_nrps) better_all = 1;
                    else if (nrps == a_nrps) {
                        for (int c = 0; c < 4; ++c) {
                            if (k[c] < ak[c]) { better_all = 1; break; }
                            if (k[c] > ak[c]) break;
                        }
                    }
                }
                if (better_all) {
                    have_all = 1; a_nrps = nrps; memcpy(ak, k, sizeof k);
                    ac[0] = b; ac[1] = s; ac[2] = q;
                }
                if (rps >= target) {
                    int better = !have_meet;
                    if (have_meet) {
                        for (int c = 0; c < 4; ++c) {
                            if (k[c] < mk[c]) { better = 1; break; }
                            if (k[c] > mk[c]) break;
                        }
                    }
                    if (better) {
                        have_meet = 1; memcpy(mk, k, sizeof k);
                        mc[0] = b; mc[1] = s; mc[2] = q;
                    }
                }
            }
        }
    }
    free(bl);
    if (have_meet) memcpy(out_bsq, mc, sizeof mc);
    else memcpy(out_bsq, ac, sizeof ac);
    return 0;
}

/* Batched form used as the CPU baseline / checker of the lattice kernel:
 * one most_efficient_config per function (table id per function). */
int or_most_efficient_config_batch(int64_t nfn, const int64_t *table_of_fn,
                                   const int64_t *nb, const int64_t *ns, const int64_t *nq,
                                   const double *const *b_axes, const double *const *s_axes,
                                   const double *const *q_axes, const double *const *values,
                                   const double *targets, int64_t step,
                                   const int64_t *allowed, int64_t nallowed,
                                   int64_t *out_bsq)
{
    for (int64_t f = 0; f < nfn; ++f) {
        int64_t t = table_of_fn[f];
        int rc = or_most_efficient_config(b_axes[t], nb[t], s_axes[t], ns[t], q_axes[t],
                                          nq[t], values[t], targets[f], step, allowed,
                                          nallowed, out_bsq + 3 * f);
        if (rc) return rc;
    }
    return 0;
}
