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
