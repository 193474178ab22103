/*
 * cocg_oracle.c -- CPU restatement of the REXI step for 2D/3D pencils,
 * where the reference itself cannot run (its factorize() falls back to a
 * dense LU, solvers.py:108-115).  TEST / BASELINE INFRASTRUCTURE ONLY:
 * loaded by tests/ and by bench.py's cpu_baseline / --impl reference legs.
 *
 * Semantics follow the reference step (integrate.py:171, 203-213, 59-68,
 * 224): S_j formed entrywise with the reference rounding, rhs = 1j*(B@u),
 * terms fl(beta_j * x_j), Kahan sum in ascending j.  The per-shift solver
 * is Jacobi-preconditioned COCG (complex-symmetric CG with unconjugated
 * inner products), optionally followed by rounds of residual refinement
 * with a double-double residual -- the same algorithm as the GPU path.
 * Shifts run in parallel with OpenMP; the reduction is serial.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct { double re, im; } c128;
static inline c128 cmk(double r, double i) { c128 z = {r, i}; return z; }
static inline c128 cadd(c128 a, c128 b) { return cmk(a.re + b.re, a.im + b.im); }
static inline c128 csub(c128 a, c128 b) { return cmk(a.re - b.re, a.im - b.im); }
static inline c128 cmul(c128 a, c128 b) {
    return cmk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
static inline c128 cdivz(c128 a, c128 b) {
    double den = b.re * b.re + b.im * b.im;
    return cmk((a.re * b.re + a.im * b.im) / den, (a.im * b.re - a.re * b.im) / den);
}
typedef struct { double hi, lo; } dd;
static inline dd two_sum(double a, double b) {
    double s = a + b, bb = s - a;
    dd r = {s, (a - (s - bb)) + (b - bb)};
    return r;
}
static inline dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
    s.lo += t.hi; s = two_sum(s.hi, s.lo); s.lo += t.lo;
    return two_sum(s.hi, s.lo);
}
static inline dd two_prod(double a, double b) { double p = a * b; dd r = {p, fma(a, b, -p)}; return r; }
static inline dd dd_neg(dd a) { dd r = {-a.hi, -a.lo}; return r; }

static inline c128 form_entry(double tau, double a, double b, c128 s) {
    return cmk(tau * a + s.im * b, -(s.re * b));
}

typedef struct {
    int64_t n;
    const int32_t *indptr, *indices;
    const double *a, *b;
    double tau;
    c128 s;
} shifted;

static void spmv(const shifted *S, const c128 *x, c128 *y) {
    for (int64_t r = 0; r < S->n; ++r) {
        c128 acc = {0.0, 0.0};
        for (int32_t q = S->indptr[r]; q < S->indptr[r + 1]; ++q)
            acc = cadd(acc, cmul(form_entry(S->tau, S->a[q], S->b[q], S->s), x[S->indices[q]]));
        y[r] = acc;
    }
}

static void residual_dd(const shifted *S, const c128 *b, const c128 *x, c128 *res) {
    for (int64_t r = 0; r < S->n; ++r) {
        dd re = {b[r].re, 0.0}, im = {b[r].im, 0.0};
        for (int32_t q = S->indptr[r]; q < S->indptr[r + 1]; ++q) {
            c128 e = form_entry(S->tau, S->a[q], S->b[q], S->s);
            c128 v = x[S->indices[q]];
            re = dd_add(re, dd_neg(dd_add(two_prod(e.re, v.re), dd_neg(two_prod(e.im, v.im)))));
            im = dd_add(im, dd_neg(dd_add(two_prod(e.re, v.im), two_prod(e.im, v.re))));
        }
        res[r] = cmk(re.hi + re.lo, im.hi + im.lo);
    }
}

static double nrm2(const c128 *v, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i].re * v[i].re + v[i].im * v[i].im;
    return sqrt(s);
}

/* Jacobi-COCG from x = 0; returns iterations, -1 on breakdown, -2 no convergence. */
static int cocg(const shifted *S, const c128 *dinv, const c128 *b, c128 *x, double tol,
                int maxit, c128 *r, c128 *p, c128 *q) {
    const int64_t n = S->n;
    double nb = nrm2(b, n);
    for (int64_t i = 0; i < n; ++i) { x[i] = cmk(0.0, 0.0); r[i] = b[i]; }
    if (nb == 0.0) return 0;
    c128 rho = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i) {
        p[i] = cmul(dinv[i], r[i]);
        rho = cadd(rho, cmul(r[i], p[i]));
    }
    for (int it = 1; it <= maxit; ++it) {
        spmv(S, p, q);
        c128 mu = {0.0, 0.0};
        for (int64_t i = 0; i < n; ++i) mu = cadd(mu, cmul(p[i], q[i]));
        if (mu.re == 0.0 && mu.im == 0.0) return -1;
        c128 alpha = cdivz(rho, mu);
        double rr = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            x[i] = cadd(x[i], cmul(alpha, p[i]));
            r[i] = csub(r[i], cmul(alpha, q[i]));
            rr += r[i].re * r[i].re + r[i].im * r[i].im;
        }
        if (sqrt(rr) <= tol * nb) return it;
        c128 rho2 = {0.0, 0.0};
        for (int64_t i = 0; i < n; ++i) rho2 = cadd(rho2, cmul(r[i], cmul(dinv[i], r[i])));
        if (rho.re == 0.0 && rho.im == 0.0) return -1;
        c128 beta = cdivz(rho2, rho);
        for (int64_t i = 0; i < n; ++i) p[i] = cadd(cmul(dinv[i], r[i]), cmul(beta, p[i]));
        rho = rho2;
    }
    return -2;
}

/*
 * One REXI step with per-shift COCG.  iters (k ints, optional) receives the
 * total COCG iterations per shift; returns 0, or 10+j on failure of shift j.
 */
int orc_cocg_step(int64_t n, const int32_t *indptr, const int32_t *indices, const double *a,
                  const double *bv, int32_t k, const c128 *shifts, const c128 *weights,
                  double tau, const c128 *u_in, c128 *u_out, double tol, int32_t maxit,
                  int32_t refine, double tol_refine, int32_t nthreads, int32_t *iters) {
    c128 *rhs = malloc(sizeof(c128) * n);
    for (int64_t r = 0; r < n; ++r) {
        double sr = 0.0, si = 0.0;
        for (int32_t q = indptr[r]; q < indptr[r + 1]; ++q) {
            sr += bv[q] * u_in[indices[q]].re;
            si += bv[q] * u_in[indices[q]].im;
        }
        rhs[r] = cmk(-si, sr);
    }
    c128 *work = malloc(sizeof(c128) * (size_t)k * n);
    int failed = -1;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    #pragma omp parallel for schedule(dynamic) num_threads(nthreads)
    for (int j = 0; j < k; ++j) {
        shifted S = {n, indptr, indices, a, bv, tau, shifts[j]};
        c128 *dinv = malloc(sizeof(c128) * n), *r = malloc(sizeof(c128) * n);
        c128 *p = malloc(sizeof(c128) * n), *q = malloc(sizeof(c128) * n);
        c128 *d = malloc(sizeof(c128) * n), *res = malloc(sizeof(c128) * n);
        for (int64_t i = 0; i < n; ++i) {
            c128 diag = {0.0, 0.0};
            for (int32_t t = indptr[i]; t < indptr[i + 1]; ++t)
                if (indices[t] == i) diag = form_entry(tau, a[t], bv[t], shifts[j]);
            dinv[i] = cdivz(cmk(1.0, 0.0), diag);
        }
        c128 *x = work + (size_t)j * n;
        int it = cocg(&S, dinv, rhs, x, tol, maxit, r, p, q);
        int total = it;
        for (int rr = 0; rr < refine && it >= 0; ++rr) {
            residual_dd(&S, rhs, x, res);
            it = cocg(&S, dinv, res, d, tol_refine, maxit, r, p, q);
            if (it >= 0) {
                for (int64_t i = 0; i < n; ++i) x[i] = cadd(x[i], d[i]);
                total += it;
            }
        }
        if (iters) iters[j] = it < 0 ? it : total;
        if (it < 0) {
            #pragma omp critical
            { if (failed < 0 || j < failed) failed = j; }
        }
        free(dinv); free(r); free(p); free(q); free(d); free(res);
    }
    for (int64_t i = 0; i < n; ++i) {
        c128 acc = {0.0, 0.0}, comp = {0.0, 0.0};
        for (int j = 0; j < k; ++j) {
            c128 row = cmul(weights[j], work[(size_t)j * n + i]);
            c128 y = csub(row, comp);
            c128 t = cadd(acc, y);
            comp = csub(csub(t, acc), y);
            acc = t;
        }
        u_out[i] = acc;
    }
    free(rhs); free(work);
    return failed < 0 ? 0 : 10 + failed;
}

/* dd residual res = b - S (xh + xl), x in double-double (exact products) */
static void residual_dd2(const shifted *S, const c128 *b, const c128 *xh, const c128 *xl,
                         c128 *res) {
    for (int64_t r = 0; r < S->n; ++r) {
        dd re = {b[r].re, 0.0}, im = {b[r].im, 0.0};
        for (int32_t q = S->indptr[r]; q < S->indptr[r + 1]; ++q) {
            c128 e = form_entry(S->tau, S->a[q], S->b[q], S->s);
            int64_t c = S->indices[q];
            /* (e.re + i e.im) * ((xh.re + xl.re) + i (xh.im + xl.im)), each
             * product split exactly: two_prod on the high word, fma-rounded
             * low-word products (|xl| <= ulp(xh), below the dd floor) */
            dd pr = dd_add(two_prod(e.re, xh[c].re), dd_neg(two_prod(e.im, xh[c].im)));
            dd pi = dd_add(two_prod(e.re, xh[c].im), two_prod(e.im, xh[c].re));
            pr = dd_add(pr, two_sum(e.re * xl[c].re, -(e.im * xl[c].im)));
            pi = dd_add(pi, two_sum(e.re * xl[c].im, e.im * xl[c].re));
            re = dd_add(re, dd_neg(pr));
            im = dd_add(im, dd_neg(pi));
        }
        res[r] = cmk(re.hi + re.lo, im.hi + im.lo);
    }
}

/*
 * Truth-level REXI step for 2D/3D pencils (TEST INFRASTRUCTURE): the same
 * rhs = 1j*(B@u) as the reference (integrate.py:203-206), each shift solved
 * by Jacobi-COCG to tol and then refined against a double-double residual
 * with x kept in double-double until the correction is below 1e-22 of x
 * (at most `rounds` rounds, correction solves to tol_refine), and the sum
 * sum_j beta_j x_j taken with exact products in double-double -- the 2D/3D
 * counterpart of rexi_oracle.c's mode 1, free of the fp64 floor that the
 * reference's own Kahan sum of fl(beta_j x_j) carries.
 * iters[j] = total COCG iterations of shift j; corr[j] = last relative
 * correction.  Returns 0, or 10+j if shift j broke down / did not converge.
 */
int orc_cocg_truth_step(int64_t n, const int32_t *indptr, const int32_t *indices, const double *a,
                        const double *bv, int32_t k, const c128 *shifts, const c128 *weights,
                        double tau, const c128 *u_in, c128 *u_out, double tol, int32_t maxit,
                        int32_t rounds, double tol_refine, int32_t nthreads, int32_t *iters,
                        double *corr, c128 *xs_out) {
    c128 *rhs = malloc(sizeof(c128) * (n ? n : 1));
    for (int64_t r = 0; r < n; ++r) {
        double sr = 0.0, si = 0.0;
        for (int32_t q = indptr[r]; q < indptr[r + 1]; ++q) {
            sr += bv[q] * u_in[indices[q]].re;
            si += bv[q] * u_in[indices[q]].im;
        }
        rhs[r] = cmk(-si, sr);
    }
    c128 *work = malloc(sizeof(c128) * (size_t)k * (n ? n : 1));
    c128 *work_lo = calloc((size_t)k * (n ? n : 1), sizeof(c128));
    int failed = -1;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    #pragma omp parallel for schedule(dynamic) num_threads(nthreads)
    for (int j = 0; j < k; ++j) {
        shifted S = {n, indptr, indices, a, bv, tau, shifts[j]};
        c128 *dinv = malloc(sizeof(c128) * n), *r = malloc(sizeof(c128) * n);
        c128 *p = malloc(sizeof(c128) * n), *q = malloc(sizeof(c128) * n);
        c128 *d = malloc(sizeof(c128) * n), *res = malloc(sizeof(c128) * n);
        for (int64_t i = 0; i < n; ++i) {
            c128 diag = {0.0, 0.0};
            for (int32_t t = indptr[i]; t < indptr[i + 1]; ++t)
                if (indices[t] == i) diag = form_entry(tau, a[t], bv[t], shifts[j]);
            dinv[i] = cdivz(cmk(1.0, 0.0), diag);
        }
        c128 *x = work + (size_t)j * n, *xl = work_lo + (size_t)j * n;
        int it = cocg(&S, dinv, rhs, x, tol, maxit, r, p, q);
        int total = it;
        double rel = 1.0;
        for (int rr = 0; rr < rounds && it >= 0; ++rr) {
            residual_dd2(&S, rhs, x, xl, res);
            it = cocg(&S, dinv, res, d, tol_refine, maxit, r, p, q);
            if (it < 0) break;
            total += it;
            double nd = 0.0, nx = 0.0;
            for (int64_t i = 0; i < n; ++i) {
                dd sr = dd_add(two_sum(x[i].re, xl[i].re), two_sum(d[i].re, 0.0));
                dd si = dd_add(two_sum(x[i].im, xl[i].im), two_sum(d[i].im, 0.0));
                x[i] = cmk(sr.hi, si.hi);
                xl[i] = cmk(sr.lo, si.lo);
                nd += d[i].re * d[i].re + d[i].im * d[i].im;
                nx += x[i].re * x[i].re + x[i].im * x[i].im;
            }
            rel = nx > 0 ? sqrt(nd / nx) : 0.0;
            if (rel < 1e-22) break;
        }
        if (iters) iters[j] = it < 0 ? it : total;
        if (corr) corr[j] = rel;
        if (it < 0) {
            #pragma omp critical
            { if (failed < 0 || j < failed) failed = j; }
        }
        free(dinv); free(r); free(p); free(q); free(d); free(res);
    }
    if (xs_out) memcpy(xs_out, work, sizeof(c128) * (size_t)k * n);
    #pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        dd sre = {0.0, 0.0}, sim = {0.0, 0.0};
        for (int j = 0; j < k; ++j) {
            c128 bw = weights[j];
            c128 xh = work[(size_t)j * n + i], xlo = work_lo[(size_t)j * n + i];
            dd pr = dd_add(two_prod(xh.re, bw.re), dd_neg(two_prod(xh.im, bw.im)));
            dd pi = dd_add(two_prod(xh.im, bw.re), two_prod(xh.re, bw.im));
            pr = dd_add(pr, two_sum(xlo.re * bw.re, -(xlo.im * bw.im)));
            pi = dd_add(pi, two_sum(xlo.im * bw.re, xlo.re * bw.im));
            sre = dd_add(sre, pr);
            sim = dd_add(sim, pi);
        }
        u_out[i] = cmk(sre.hi + sre.lo, sim.hi + sim.lo);
    }
    free(rhs); free(work); free(work_lo);
    return failed < 0 ? 0 : 10 + failed;
}

/* ||b - S x|| / ||b|| for the CSR pencil, residual in double-double,
 * parallel over rows (a full-size check of one shift's solution). */
double orc_csr_rel_residual(int64_t n, const int32_t *indptr, const int32_t *indices,
                            const double *a, const double *bv, double tau, c128 sigma,
                            const c128 *b, const c128 *x, int32_t nthreads) {
    shifted S = {n, indptr, indices, a, bv, tau, sigma};
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    double nr = 0.0, nb = 0.0;
    #pragma omp parallel for schedule(static) num_threads(nthreads) reduction(+:nr, nb)
    for (int64_t r = 0; r < n; ++r) {
        dd re = {b[r].re, 0.0}, im = {b[r].im, 0.0};
        for (int32_t q = indptr[r]; q < indptr[r + 1]; ++q) {
            c128 e = form_entry(tau, a[q], bv[q], S.s);
            c128 v = x[indices[q]];
            re = dd_add(re, dd_neg(dd_add(two_prod(e.re, v.re), dd_neg(two_prod(e.im, v.im)))));
            im = dd_add(im, dd_neg(dd_add(two_prod(e.re, v.im), two_prod(e.im, v.re))));
        }
        double rr = re.hi + re.lo, ri = im.hi + im.lo;
        nr += rr * rr + ri * ri;
        nb += b[r].re * b[r].re + b[r].im * b[r].im;
    }
    return nb > 0 ? sqrt(nr / nb) : sqrt(nr);
}
