/*
 * rexi_oracle.c -- CPU ORACLE for the REXI step.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline -- never as part of the product path.
 *
 * What it restates (reference = rexiprop 0.1.0 under /root/reference/pkg):
 *   - operator formation  S_j = tau*A - (1j*sigma_j)*B     integrate.py:171
 *       re = fl(fl(tau*a) + fl(Im(sigma)*b)), im = -fl(Re(sigma)*b)
 *   - rhs = 1j * (B @ u), CSR row order                    integrate.py:203-206
 *   - factorize -> BandedFactorization: LAPACK zgbtrf      solvers.py:42-69, 108-115
 *       (restated: zgbtf2 partial pivoting with IZAMAX on |re|+|im|),
 *       singular if a zero pivot or min|U_ii| < 1e-14 max|U_ii|
 *   - solve -> LAPACK zgbtrs (L with row interchanges, then ztbsv upper)
 *                                                          solvers.py:76-80
 *   - terms work[j] = weights[j] * x_j                     integrate.py:208-213
 *   - _kahan_rows: compensated sum over j ascending        integrate.py:59-68, 224
 * The LAPACK routines are third-party (scipy 1.18.1 / scipy-openblas
 * 0.3.30 in the build container); this file restates the published
 * reference-LAPACK algorithms, so agreement with the reference is to
 * rounding, not bitwise.
 *
 * "Truth" mode: each per-shift solution is refined
 * against a residual evaluated in double-double (error-free products via
 * fma) and kept as a double-double; terms beta_j*x_j are formed exactly
 * and summed in double-double.  This is the fp64-floor-free target that
 * both the reference and the GPU path are measured against.
 *
 * Shifts are processed in parallel with OpenMP (schedule dynamic); the
 * reduction is always serial in ascending j, so results do not depend on
 * the thread count.
 */
#include <math.h>
#include <stdio.h>
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
static inline double cabs1(c128 a) { return fabs(a.re) + fabs(a.im); }
/* Smith's algorithm (the range-reduced complex division Fortran uses). */
static inline c128 cdiv(c128 a, c128 b) {
    if (fabs(b.re) >= fabs(b.im)) {
        double r = b.im / b.re, den = b.re + r * b.im;
        return cmk((a.re + a.im * r) / den, (a.im - a.re * r) / den);
    } else {
        double r = b.re / b.im, den = b.im + r * b.re;
        return cmk((a.re * r + a.im) / den, (a.im * r - a.re) / den);
    }
}

/* ---- double-double helpers (error-free transforms) ---- */
typedef struct { double hi, lo; } dd;
static inline dd two_sum(double a, double b) {
    double s = a + b, bb = s - a;
    dd r = {s, (a - (s - bb)) + (b - bb)};
    return r;
}
static inline dd two_prod(double a, double b) {
    double p = a * b;
    dd r = {p, fma(a, b, -p)};
    return r;
}
static inline dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return two_sum(s.hi, s.lo);
}
static inline dd dd_add_d(dd a, double b) {
    dd s = two_sum(a.hi, b);
    s.lo += a.lo;
    return two_sum(s.hi, s.lo);
}
static inline dd dd_neg(dd a) { dd r = {-a.hi, -a.lo}; return r; }
/* (a_hi + a_lo) * b exactly enough: error-free prod of hi plus lo*b */
static inline dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo += a.lo * b;
    return two_sum(p.hi, p.lo);
}
typedef struct { dd re, im; } cdd;

/* ------------------------------------------------------------------ */
typedef struct {
    int64_t n, nnz;
    int32_t *indptr, *indices;
    double *a, *b;                  /* values on the shared pattern */
    int32_t k;
    c128 *shifts, *weights;
    double tau;
    int32_t kl, ku, ldab;           /* band extents, ldab = 2kl+ku+1 */
    c128 *ab;                       /* k * ldab * n, column-major per shift */
    int32_t *ipiv;                  /* k * n */
    int32_t nthreads;
    int32_t bad_shift;              /* index of the singular shift, -1 if none */
    double *umin, *umax;            /* per shift: extremes of |U_ii| (solvers.py:59-69) */
    int32_t *uinfo;                 /* per shift: zgbtf2 info */
    char msg[256];
} orc_plan;

#define AB(p, j, row, col) ((p)->ab[(size_t)(j) * (p)->ldab * (p)->n + (size_t)(col) * (p)->ldab + (row)])

static inline c128 form_entry(double tau, double a, double b, c128 s) {
    /* scipy: (tau*A - (1j*sigma)*B); see header */
    double re = tau * a + s.im * b;   /* fl(fl(tau a) + fl(Im s * b)) with contraction off */
    double im = -(s.re * b);
    return cmk(re, im);
}

/* zgbtf2 restated (0-based). returns info (0 ok, >0 = 1-based zero pivot). */
static int gbtf2(orc_plan *p, int j) {
    const int64_t n = p->n;
    const int kl = p->kl, ku = p->ku, kv = kl + ku;
    int info = 0;
    int64_t ju = 0;
    for (int64_t col = 0; col < n; ++col) {
        if (col + kv < n)
            for (int i = 0; i < kl; ++i) AB(p, j, i, col + kv) = cmk(0.0, 0.0);
        int64_t km = kl < (n - 1 - col) ? kl : (n - 1 - col);
        /* izamax over AB(kv .. kv+km, col) */
        int64_t jp = 0;
        double best = cabs1(AB(p, j, kv, col));
        for (int64_t i = 1; i <= km; ++i) {
            double v = cabs1(AB(p, j, kv + i, col));
            if (v > best) { best = v; jp = i; }
        }
        p->ipiv[(size_t)j * n + col] = (int32_t)(jp + col);
        c128 piv = AB(p, j, kv + jp, col);
        if (piv.re != 0.0 || piv.im != 0.0) {
            int64_t cand = col + ku + jp;
            if (cand > n - 1) cand = n - 1;
            if (cand > ju) ju = cand;
            if (jp != 0) {
                for (int64_t c = col; c <= ju; ++c) {
                    /* element (row col+jp, c) at band row kv+jp-(c-col); (row col, c) at kv-(c-col) */
                    int64_t r1 = kv + jp - (c - col), r0 = kv - (c - col);
                    c128 t = AB(p, j, r1, c);
                    AB(p, j, r1, c) = AB(p, j, r0, c);
                    AB(p, j, r0, c) = t;
                }
            }
            if (km > 0) {
                c128 rp = cdiv(cmk(1.0, 0.0), AB(p, j, kv, col));
                for (int64_t i = 1; i <= km; ++i) AB(p, j, kv + i, col) = cmul(rp, AB(p, j, kv + i, col));
                for (int64_t c = col + 1; c <= ju; ++c) {
                    c128 y = AB(p, j, kv - (c - col), c);       /* row col, column c */
                    if (y.re == 0.0 && y.im == 0.0) continue;
                    for (int64_t i = 1; i <= km; ++i) {
                        int64_t r = kv + i - (c - col);         /* row col+i, column c */
                        AB(p, j, r, c) = csub(AB(p, j, r, c), cmul(AB(p, j, kv + i, col), y));
                    }
                }
            }
        } else if (info == 0) {
            info = (int)(col + 1);
        }
    }
    return info;
}

/* zgbtrs restated, no transpose, one rhs in place */
static void gbtrs(const orc_plan *p, int j, c128 *x) {
    const int64_t n = p->n;
    const int kl = p->kl, ku = p->ku, kv = kl + ku;
    if (kl > 0) {
        for (int64_t col = 0; col < n - 1; ++col) {
            int64_t lm = kl < (n - 1 - col) ? kl : (n - 1 - col);
            int64_t l = p->ipiv[(size_t)j * n + col];
            if (l != col) { c128 t = x[l]; x[l] = x[col]; x[col] = t; }
            c128 xc = x[col];
            for (int64_t i = 1; i <= lm; ++i)
                x[col + i] = csub(x[col + i], cmul(AB(p, j, kv + i, col), xc));
        }
    }
    /* ztbsv upper, non-unit, k = kl+ku superdiagonals, column oriented */
    for (int64_t col = n - 1; col >= 0; --col) {
        if (x[col].re != 0.0 || x[col].im != 0.0) {
            x[col] = cdiv(x[col], AB(p, j, kv, col));
            c128 t = x[col];
            int64_t i0 = col - kv > 0 ? col - kv : 0;
            for (int64_t i = i0; i < col; ++i)
                x[i] = csub(x[i], cmul(t, AB(p, j, kv + i - col, col)));
        }
    }
}

/* ---------------- public API (extern "C" style) ---------------- */

orc_plan *orc_create(int64_t n, int64_t nnz, const int32_t *indptr, const int32_t *indices,
                     const double *a, const double *b, int32_t k, const c128 *shifts,
                     const c128 *weights, double tau, int32_t nthreads, int32_t *status) {
    orc_plan *p = (orc_plan *)calloc(1, sizeof(orc_plan));
    p->n = n; p->nnz = nnz; p->k = k; p->tau = tau; p->bad_shift = -1;
    p->nthreads = nthreads > 0 ? nthreads : omp_get_max_threads();
    p->indptr = malloc(sizeof(int32_t) * (n + 1));
    p->indices = malloc(sizeof(int32_t) * (nnz ? nnz : 1));
    p->a = malloc(sizeof(double) * (nnz ? nnz : 1));
    p->b = malloc(sizeof(double) * (nnz ? nnz : 1));
    memcpy(p->indptr, indptr, sizeof(int32_t) * (n + 1));
    memcpy(p->indices, indices, sizeof(int32_t) * nnz);
    memcpy(p->a, a, sizeof(double) * nnz);
    memcpy(p->b, b, sizeof(double) * nnz);
    p->shifts = malloc(sizeof(c128) * k);
    p->weights = malloc(sizeof(c128) * k);
    memcpy(p->shifts, shifts, sizeof(c128) * k);
    memcpy(p->weights, weights, sizeof(c128) * k);
    /* _band_extents (solvers.py:30-36) */
    int kl = 0, ku = 0;
    for (int64_t r = 0; r < n; ++r)
        for (int32_t q = indptr[r]; q < indptr[r + 1]; ++q) {
            int64_t d = (int64_t)indices[q] - r;
            if (-d > kl) kl = (int)(-d);
            if (d > ku) ku = (int)d;
        }
    p->kl = kl; p->ku = ku; p->ldab = 2 * kl + ku + 1;
    p->ab = calloc((size_t)k * p->ldab * n, sizeof(c128));
    p->ipiv = calloc((size_t)k * n, sizeof(int32_t));
    p->umin = calloc((size_t)(k ? k : 1), sizeof(double));
    p->umax = calloc((size_t)(k ? k : 1), sizeof(double));
    p->uinfo = calloc((size_t)(k ? k : 1), sizeof(int32_t));
    if (!p->ab || !p->ipiv) { *status = 7; snprintf(p->msg, sizeof p->msg, "out of memory"); return p; }
    int bad = -1;
    #pragma omp parallel for schedule(dynamic) num_threads(p->nthreads)
    for (int j = 0; j < k; ++j) {
        const int kv = p->kl + p->ku;
        for (int64_t r = 0; r < n; ++r)
            for (int32_t q = indptr[r]; q < indptr[r + 1]; ++q) {
                int64_t c = indices[q];
                AB(p, j, kv + r - c, c) = cadd(AB(p, j, kv + r - c, c),
                                               form_entry(tau, a[q], b[q], shifts[j]));
            }
        int info = gbtf2(p, j);
        int singular = info > 0;
        double umin = INFINITY, umax = 0.0;
        for (int64_t c = 0; c < n; ++c) {
            c128 u = AB(p, j, kv, c);
            double v = hypot(u.re, u.im);
            if (v < umin) umin = v;
            if (v > umax) umax = v;
        }
        p->umin[j] = umin;
        p->umax[j] = umax;
        p->uinfo[j] = info;
        if (!singular && n > 0) {
            if (!(umin > 0.0) || umin < 1e-14 * umax) singular = 1;
        }
        if (singular) {
            #pragma omp critical
            { if (bad < 0 || j < bad) bad = j; }
        }
    }
    p->bad_shift = bad;
    *status = bad >= 0 ? 2 : 0;
    if (bad >= 0) snprintf(p->msg, sizeof p->msg, "shift j = %d is singular", bad);
    return p;
}

int32_t orc_bad_shift(const orc_plan *p) { return p->bad_shift; }
int32_t orc_bandwidth(const orc_plan *p) { return p->kl + p->ku + 1; }

void orc_destroy(orc_plan *p) {
    if (!p) return;
    free(p->indptr); free(p->indices); free(p->a); free(p->b);
    free(p->shifts); free(p->weights); free(p->ab); free(p->ipiv);
    free(p->umin); free(p->umax); free(p->uinfo); free(p);
}

/* rhs = 1j * (B @ u) */
static void rhs_ib_u(const orc_plan *p, const c128 *u, c128 *rhs) {
    for (int64_t r = 0; r < p->n; ++r) {
        double sr = 0.0, si = 0.0;
        for (int32_t q = p->indptr[r]; q < p->indptr[r + 1]; ++q) {
            c128 x = u[p->indices[q]];
            sr += p->b[q] * x.re;
            si += p->b[q] * x.im;
        }
        rhs[r] = cmk(-si, sr);
    }
}

/* residual r = rhs - S_j (x_hi + x_lo), evaluated in double-double */
static void residual_dd(const orc_plan *p, int j, const c128 *rhs, const c128 *xh,
                        const c128 *xl, c128 *res) {
    const c128 s = p->shifts[j];
    for (int64_t r = 0; r < p->n; ++r) {
        dd acc_re = {rhs[r].re, 0.0}, acc_im = {rhs[r].im, 0.0};
        for (int32_t q = p->indptr[r]; q < p->indptr[r + 1]; ++q) {
            int64_t c = p->indices[q];
            c128 e = form_entry(p->tau, p->a[q], p->b[q], s);
            dd xr = two_sum(xh[c].re, xl[c].re), xi = two_sum(xh[c].im, xl[c].im);
            /* (e.re + i e.im)(xr + i xi) */
            dd pr = dd_add(dd_mul_d(xr, e.re), dd_neg(dd_mul_d(xi, e.im)));
            dd pi = dd_add(dd_mul_d(xi, e.re), dd_mul_d(xr, e.im));
            acc_re = dd_add(acc_re, dd_neg(pr));
            acc_im = dd_add(acc_im, dd_neg(pi));
        }
        res[r] = cmk(acc_re.hi + acc_re.lo, acc_im.hi + acc_im.lo);
    }
}

/*
 * One step.  mode 0 = reference restatement (fl(beta*x), Kahan ascending j);
 * mode 1 = truth (dd-refined x, exact products, dd sum).
 * xs_out (optional, k*n) receives the per-shift solutions (hi part).
 * max_rel_corr (optional) receives the last refinement correction size.
 */
int orc_step(orc_plan *p, const c128 *u_in, c128 *u_out, int32_t mode, c128 *xs_out,
             double *max_rel_corr) {
    const int64_t n = p->n;
    const int k = p->k;
    c128 *rhs = malloc(sizeof(c128) * (n ? n : 1));
    c128 *work = malloc(sizeof(c128) * (size_t)k * (n ? n : 1));
    c128 *work_lo = mode ? calloc((size_t)k * (n ? n : 1), sizeof(c128)) : NULL;
    rhs_ib_u(p, u_in, rhs);
    double worst = 0.0;
    #pragma omp parallel for schedule(dynamic) num_threads(p->nthreads) reduction(max:worst)
    for (int j = 0; j < k; ++j) {
        c128 *x = work + (size_t)j * n;
        memcpy(x, rhs, sizeof(c128) * n);
        gbtrs(p, j, x);
        if (mode == 1) {
            c128 *xl = work_lo + (size_t)j * n;
            c128 *res = malloc(sizeof(c128) * (n ? n : 1));
            double rel = 0.0;
            for (int it = 0; it < 6; ++it) {
                residual_dd(p, j, rhs, x, xl, res);
                gbtrs(p, j, res);
                double nd = 0.0, nx = 0.0;
                for (int64_t i = 0; i < n; ++i) {
                    dd sr = dd_add_d(two_sum(x[i].re, xl[i].re), res[i].re);
                    dd si = dd_add_d(two_sum(x[i].im, xl[i].im), res[i].im);
                    x[i] = cmk(sr.hi, si.hi);
                    xl[i] = cmk(sr.lo, si.lo);
                    nd += res[i].re * res[i].re + res[i].im * res[i].im;
                    nx += x[i].re * x[i].re + x[i].im * x[i].im;
                }
                rel = nx > 0 ? sqrt(nd / nx) : 0.0;
                if (rel < 1e-22) break;
            }
            if (rel > worst) worst = rel;
            free(res);
        }
    }
    if (xs_out) memcpy(xs_out, work, sizeof(c128) * (size_t)k * n);
    if (mode == 0) {
        /* work[j] = weights[j] * x_j ; _kahan_rows ascending j */
        for (int64_t i = 0; i < n; ++i) {
            c128 acc = {0.0, 0.0}, comp = {0.0, 0.0};
            for (int j = 0; j < k; ++j) {
                c128 row = cmul(p->weights[j], work[(size_t)j * n + i]);
                c128 y = csub(row, comp);
                c128 t = cadd(acc, y);
                comp = csub(csub(t, acc), y);
                acc = t;
            }
            u_out[i] = acc;
        }
    } else {
        for (int64_t i = 0; i < n; ++i) {
            dd sre = {0.0, 0.0}, sim = {0.0, 0.0};
            for (int j = 0; j < k; ++j) {
                c128 bw = p->weights[j];
                dd xr = two_sum(work[(size_t)j * n + i].re, work_lo[(size_t)j * n + i].re);
                dd xi = two_sum(work[(size_t)j * n + i].im, work_lo[(size_t)j * n + i].im);
                sre = dd_add(sre, dd_add(dd_mul_d(xr, bw.re), dd_neg(dd_mul_d(xi, bw.im))));
                sim = dd_add(sim, dd_add(dd_mul_d(xi, bw.re), dd_mul_d(xr, bw.im)));
            }
            u_out[i] = cmk(sre.hi + sre.lo, sim.hi + sim.lo);
        }
    }
    if (max_rel_corr) *max_rel_corr = worst;
    free(rhs); free(work); free(work_lo);
    return 0;
}

/* Per-shift solve of an arbitrary rhs (reference-mode gbtrs), x = S_j^{-1} b. */
int orc_solve(const orc_plan *p, int32_t j, const c128 *b, c128 *x) {
    memcpy(x, b, sizeof(c128) * p->n);
    gbtrs(p, j, x);
    return 0;
}

/* ||rhs - S_j x|| / ||rhs|| evaluated in double-double. */
double orc_rel_residual(const orc_plan *p, int32_t j, const c128 *rhs, const c128 *x) {
    c128 *res = malloc(sizeof(c128) * (p->n ? p->n : 1));
    c128 *zero = calloc(p->n ? p->n : 1, sizeof(c128));
    residual_dd(p, j, rhs, x, zero, res);
    double nr = 0.0, nb = 0.0;
    for (int64_t i = 0; i < p->n; ++i) {
        nr += res[i].re * res[i].re + res[i].im * res[i].im;
        nb += rhs[i].re * rhs[i].re + rhs[i].im * rhs[i].im;
    }
    free(res); free(zero);
    return nb > 0 ? sqrt(nr / nb) : sqrt(nr);
}

/* per-shift singularity screen data of the band LU (tests): extremes of |U_ii|
 * and zgbtf2's info, as the reference's BandedFactorization sees them */
void orc_screen(const orc_plan *p, double *umin, double *umax, int32_t *info) {
    for (int j = 0; j < p->k; ++j) {
        umin[j] = p->umin[j];
        umax[j] = p->umax[j];
        info[j] = p->uinfo[j];
    }
}

/* rhs helper exported for tests */
void orc_rhs(const orc_plan *p, const c128 *u, c128 *rhs) { rhs_ib_u(p, u, rhs); }

const char *orc_message(const orc_plan *p) { return p->msg; }
