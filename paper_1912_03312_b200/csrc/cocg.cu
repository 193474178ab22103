// cocg.cu -- lockstep-over-shifts Jacobi-COCG for general CSR pencils (2D/3D,
// P2 1D, dense test pencils).  Replaces, for non-tridiagonal patterns, the
// reference's factorize() (which falls back to a dense LU there,
// solvers.py:108-115) and the K back-substitutions of rexi_step
// (integrate.py:208-222).
//
// Layout: every per-shift vector is [row][kp] complex128 (shift index fastest)
// so one warp = 32 shifts of one row: the shared CSR pattern and the A/B
// values are read once per row for all shifts (broadcast) and every gather of
// a neighbour's vector entries is a contiguous 512-B segment.  The shifted
// entries tau*a - (1j*sigma)*b are formed on the fly with the reference's
// rounding.
//
// Per iteration two kernels (two reductions -- the COCG recurrences need them):
//   A: p = z + beta*p_old (own row, double-buffered), q = S p (neighbour p
//      recomputed from the gathered z, p_old), mu = p^T q
//   B: x += alpha p, r -= alpha q, z = D^{-1} r, rho' = r^T z, |r|^2
// Per-shift dots are reduced per CTA in fixed order and finished by the last
// CTA to arrive (deterministic, independent of how shifts are sharded), which
// also computes alpha / beta, freezes converged shifts and flags breakdown.
// Converged shifts are frozen (their lanes do no memory traffic).
// Refinement: r = b - S x with error-free products (double-double), a
// correction solve, x += dx.  The final step output is the beta-weighted
// double-double sum over shifts.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "cocg.cuh"

namespace rexi {

constexpr int CG_NT = 256;           // threads per CTA (8 warps)
constexpr int CG_WARPS = CG_NT / 32;

struct CgMat {
    int64_t n;
    const int32_t *indptr, *indices;
    const double *ta, *ta_im, *b;          // per nnz: fl(tau a), fl(tau a_im), b
    const double *dta, *dta_im, *db;       // per row: the diagonal entry's values
};

struct CgVec {
    c128 *x, *r, *z, *p0, *p1, *q;         // [n][kp]
    const c128 *bvec;                      // per-shift rhs [n][kp] or nullptr
    const c128 *bshared;                   // shared rhs [n] or nullptr
};

struct CgScal {
    double2 *rho, *mu, *alpha, *beta;      // [kp]
    double *rnorm2, *bnorm2;               // [kp]
    int *active;                           // [kp] 1 = iterating
    int *iters;                            // [kp]
    int *status;                           // [kp] 0 ok, 1 breakdown, 2 non-finite
    int *nactive;                          // [1]
    double2 *part_a;                       // [grid][kp] partials
    double2 *part_b;                       // [grid][kp]
    double *part_c;                        // [grid][kp]
    unsigned int *counter;                 // [2]
    double tol;
};

struct CgGeom {
    int kp, kw, G, rpw;                    // lanes per group, groups per row, rows per warp
    int k;                                 // real shifts (lanes >= k are padding)
};

__device__ __forceinline__ c128 cdiv_c(c128 a, c128 b) { return cmul(a, crcp(b)); }

__device__ __forceinline__ void lane_geom(const CgGeom &g, int &j, int &roff, int64_t &item0,
                                          int64_t &stride) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * CG_WARPS + (threadIdx.x >> 5);
    const int64_t W = (int64_t)gridDim.x * CG_WARPS;
    const int grp = (int)(w % g.G);
    j = grp * g.kw + (lane % g.kw);
    roff = lane / g.kw;
    item0 = w / g.G;
    stride = W / g.G;
}

// shift index of thread u inside a CTA (same for every CTA)
__device__ __forceinline__ int thread_shift(const CgGeom &g, int u) {
    const int w = blockIdx.x * CG_WARPS + (u >> 5);   // global warp of thread u in this CTA
    const int grp = w % g.G;
    return grp * g.kw + ((u & 31) % g.kw);
}

// last-CTA-done: returns true in the single CTA that finishes last
__device__ __forceinline__ bool last_block(unsigned int *counter) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int prev = atomicAdd(counter, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

// ---------------------------------------------------------------------------
// reduce helpers: each thread holds one complex / real partial for shift j;
// write per-CTA partials part[cta][kp] summed in fixed thread order
// ---------------------------------------------------------------------------
__device__ void block_reduce_c(c128 v, const CgGeom &g, double2 *part, int kp) {
    __shared__ double2 sm[CG_NT];
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int t = threadIdx.x; t < kp; t += CG_NT) {
        double2 s = make_double2(0.0, 0.0);
        for (int u = 0; u < CG_NT; ++u)
            if (thread_shift(g, u) == t) s = cadd(s, sm[u]);
        part[(size_t)blockIdx.x * kp + t] = s;
    }
    __syncthreads();
}

__device__ void block_reduce_r(double v, const CgGeom &g, double *part, int kp) {
    __shared__ double sm[CG_NT];
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int t = threadIdx.x; t < kp; t += CG_NT) {
        double s = 0.0;
        for (int u = 0; u < CG_NT; ++u)
            if (thread_shift(g, u) == t) s += sm[u];
        part[(size_t)blockIdx.x * kp + t] = s;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// init: x = 0, r = b, z = D^-1 r, p_old = 0; rho = r^T z, |b|^2
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CG_NT) k_cg_init(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    int j, roff;
    int64_t item, stride;
    lane_geom(g, j, roff, item, stride);
    const int kp = g.kp;
    const c128 sg = S.sigma[j];
    c128 rho = cmk(0.0, 0.0);
    double bn = 0.0;
    for (int64_t it = item; it * g.rpw < M.n; it += stride) {
        const int64_t i = it * g.rpw + roff;
        if (i >= M.n) continue;
        const c128 b = V.bshared ? V.bshared[i] : V.bvec[i * kp + j];
        const c128 d = form_entry(M.dta[i], M.dta_im[i], M.db[i], sg);
        const c128 z = cdiv_c(b, d);
        V.x[i * kp + j] = cmk(0.0, 0.0);
        V.r[i * kp + j] = b;
        V.z[i * kp + j] = z;
        V.p0[i * kp + j] = cmk(0.0, 0.0);
        rho = cadd(rho, cmul(b, z));
        bn += cabs2(b);
    }
    block_reduce_c(rho, g, Sc.part_a, kp);
    block_reduce_r(bn, g, Sc.part_c, kp);
    if (last_block(Sc.counter)) {
        for (int t = threadIdx.x; t < kp; t += CG_NT) {
            double2 s = make_double2(0.0, 0.0);
            double sb = 0.0;
            for (unsigned c = 0; c < gridDim.x; ++c) {
                s = cadd(s, Sc.part_a[(size_t)c * kp + t]);
                sb += Sc.part_c[(size_t)c * kp + t];
            }
            Sc.rho[t] = s;
            Sc.bnorm2[t] = sb;
            Sc.rnorm2[t] = sb;
            Sc.beta[t] = make_double2(0.0, 0.0);
            Sc.iters[t] = 0;
            Sc.status[t] = 0;
            Sc.active[t] = (t < g.k && sb > 0.0) ? 1 : 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int na = 0;
            for (int t = 0; t < kp; ++t) na += Sc.active[t];
            *Sc.nactive = na;
            Sc.counter[0] = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// A: p_new = z + beta p_old (own row); q = S p_new; mu = p^T q
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CG_NT) k_cg_spmv(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g,
                                                    int parity) {
    if (*Sc.nactive == 0) return;
    int j, roff;
    int64_t item, stride;
    lane_geom(g, j, roff, item, stride);
    const int kp = g.kp;
    const bool act = Sc.active[j] != 0;
    const c128 sg = S.sigma[j];
    const c128 beta = Sc.beta[j];
    const c128 *pold = parity ? V.p1 : V.p0;
    c128 *pnew = parity ? V.p0 : V.p1;
    c128 mu = cmk(0.0, 0.0);
    for (int64_t it = item; it * g.rpw < M.n; it += stride) {
        const int64_t i = it * g.rpw + roff;
        if (i >= M.n || !act) continue;
        c128 acc = cmk(0.0, 0.0);
        c128 pi = cmk(0.0, 0.0);
        const int32_t q0 = M.indptr[i], q1 = M.indptr[i + 1];
        for (int32_t q = q0; q < q1; ++q) {
            const int64_t c = M.indices[q];
            const c128 pc = cadd(V.z[c * kp + j], cmul(beta, pold[c * kp + j]));
            const c128 e = form_entry(M.ta[q], M.ta_im[q], M.b[q], sg);
            acc = cadd(acc, cmul(e, pc));
            if (c == i) pi = pc;
        }
        pnew[i * kp + j] = pi;
        V.q[i * kp + j] = acc;
        mu = cadd(mu, cmul(pi, acc));
    }
    block_reduce_c(mu, g, Sc.part_a, kp);
    if (last_block(Sc.counter)) {
        for (int t = threadIdx.x; t < kp; t += CG_NT) {
            if (!Sc.active[t]) continue;
            double2 s = make_double2(0.0, 0.0);
            for (unsigned c = 0; c < gridDim.x; ++c) s = cadd(s, Sc.part_a[(size_t)c * kp + t]);
            Sc.mu[t] = s;
            const double2 rho = Sc.rho[t];
            const double ms = cabs2(s);
            if (!(ms > 0.0) || !isfinite(ms)) {
                Sc.status[t] = isfinite(ms) ? 1 : 2;
                Sc.active[t] = 0;
                Sc.alpha[t] = make_double2(0.0, 0.0);
            } else {
                Sc.alpha[t] = cdiv_c(rho, s);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) Sc.counter[0] = 0;
    }
}

// ---------------------------------------------------------------------------
// B: x += alpha p; r -= alpha q; z = D^-1 r; rho' = r^T z; |r|^2; freeze
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CG_NT) k_cg_update(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g,
                                                      int parity, int max_iters) {
    if (*Sc.nactive == 0) return;
    int j, roff;
    int64_t item, stride;
    lane_geom(g, j, roff, item, stride);
    const int kp = g.kp;
    const bool act = Sc.active[j] != 0;
    const c128 sg = S.sigma[j];
    const c128 alpha = Sc.alpha[j];
    const c128 *pnew = parity ? V.p0 : V.p1;
    c128 rho = cmk(0.0, 0.0);
    double rn = 0.0;
    for (int64_t it = item; it * g.rpw < M.n; it += stride) {
        const int64_t i = it * g.rpw + roff;
        if (i >= M.n || !act) continue;
        const size_t o = (size_t)i * kp + j;
        const c128 p = pnew[o], q = V.q[o];
        V.x[o] = cadd(V.x[o], cmul(alpha, p));
        const c128 r = csub(V.r[o], cmul(alpha, q));
        V.r[o] = r;
        const c128 d = form_entry(M.dta[i], M.dta_im[i], M.db[i], sg);
        const c128 z = cdiv_c(r, d);
        V.z[o] = z;
        rho = cadd(rho, cmul(r, z));
        rn += cabs2(r);
    }
    block_reduce_c(rho, g, Sc.part_b, kp);
    block_reduce_r(rn, g, Sc.part_c, kp);
    if (last_block(Sc.counter + 1)) {
        for (int t = threadIdx.x; t < kp; t += CG_NT) {
            if (!Sc.active[t]) continue;
            double2 s = make_double2(0.0, 0.0);
            double sr = 0.0;
            for (unsigned c = 0; c < gridDim.x; ++c) {
                s = cadd(s, Sc.part_b[(size_t)c * kp + t]);
                sr += Sc.part_c[(size_t)c * kp + t];
            }
            Sc.rnorm2[t] = sr;
            Sc.iters[t] += 1;
            const double2 rho_old = Sc.rho[t];
            const double ro = cabs2(rho_old);
            if (!isfinite(sr)) {
                Sc.status[t] = 2;
                Sc.active[t] = 0;
            } else if (sr <= Sc.tol * Sc.tol * Sc.bnorm2[t]) {
                Sc.active[t] = 0;                              // converged: freeze
            } else if (!(ro > 0.0)) {
                Sc.status[t] = 1;
                Sc.active[t] = 0;
            } else if (Sc.iters[t] >= max_iters) {
                Sc.status[t] = 3;
                Sc.active[t] = 0;
            } else {
                Sc.beta[t] = cdiv_c(s, rho_old);
                Sc.rho[t] = s;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int na = 0;
            for (int t = 0; t < kp; ++t) na += Sc.active[t];
            *Sc.nactive = na;
            Sc.counter[1] = 0;
        }
    }
}

// r_j = b - S_j x_j with error-free products, double-double sum, rounded once
__global__ void __launch_bounds__(CG_NT) k_cg_residual(CgMat M, CgVec V, ShiftDev S, CgGeom g,
                                                        c128 *out) {
    int j, roff;
    int64_t item, stride;
    lane_geom(g, j, roff, item, stride);
    const int kp = g.kp;
    const c128 sg = S.sigma[j];
    for (int64_t it = item; it * g.rpw < M.n; it += stride) {
        const int64_t i = it * g.rpw + roff;
        if (i >= M.n) continue;
        const c128 b = V.bshared ? V.bshared[i] : V.bvec[i * kp + j];
        ddacc re = {b.x, 0.0}, im = {b.y, 0.0};
        for (int32_t q = M.indptr[i]; q < M.indptr[i + 1]; ++q) {
            const c128 e = form_entry(M.ta[q], M.ta_im[q], M.b[q], sg);
            const c128 x = V.x[(int64_t)M.indices[q] * kp + j];
            dd p;
            p = two_prod(e.x, x.x); ddacc_add(re, -p.hi); re.lo = __dsub_rn(re.lo, p.lo);
            p = two_prod(e.y, x.y); ddacc_add(re, p.hi); re.lo = __dadd_rn(re.lo, p.lo);
            p = two_prod(e.x, x.y); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
            p = two_prod(e.y, x.x); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
        }
        out[i * kp + j] = cmk(__dadd_rn(re.hi, re.lo), __dadd_rn(im.hi, im.lo));
    }
}

// rhs = 1j * (B @ u), CSR row order, no FMA (reference integrate.py:204)
__global__ void k_cg_rhs(CgMat M, const c128 *__restrict__ u, c128 *__restrict__ rhs) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M.n) return;
    double sr = 0.0, si = 0.0;
    for (int32_t q = M.indptr[i]; q < M.indptr[i + 1]; ++q) {
        const double b = M.b[q];
        const c128 x = u[M.indices[q]];
        sr = __dadd_rn(sr, __dmul_rn(b, x.x));
        si = __dadd_rn(si, __dmul_rn(b, x.y));
    }
    rhs[i] = cmk(-si, sr);
}

// acc (dd, SoA 4n) (+)= sum_j beta_j (x1_j [+ x2_j]), fixed shift order
__global__ void k_cg_accum(int64_t n, int kp, int k, const c128 *__restrict__ beta,
                           const c128 *__restrict__ x1, const c128 *__restrict__ x2, double *acc,
                           c128 *uout) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    ddacc re = {0.0, 0.0}, im = {0.0, 0.0};
    for (int jj = 0; jj < k; ++jj) {
        const c128 b = beta[jj];
        c128 x = x1[i * kp + jj];
        ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
        ddacc_add(im, fma(b.x, x.y, b.y * x.x));
        if (x2) {
            x = x2[i * kp + jj];
            ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
            ddacc_add(im, fma(b.x, x.y, b.y * x.x));
        }
    }
    dd sre = fast_two_sum(re.hi, re.lo), sim = fast_two_sum(im.hi, im.lo);
    if (uout) {
        uout[i] = cmk(__dadd_rn(sre.hi, sre.lo), __dadd_rn(sim.hi, sim.lo));
    } else {
        acc[i] = sre.hi;
        acc[n + i] = sre.lo;
        acc[2 * n + i] = sim.hi;
        acc[3 * n + i] = sim.lo;
    }
}

__global__ void k_cg_transpose(const c128 *__restrict__ X, const c128 *__restrict__ X2, int64_t n,
                               int kp, int k, c128 *__restrict__ out) {
    int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gt >= n * (int64_t)k) return;
    int j = (int)(gt / n);
    int64_t i = gt % n;
    c128 v = X[i * kp + j];
    if (X2) v = cadd(v, X2[i * kp + j]);
    out[gt] = v;
}

__global__ void k_axpy_inplace(c128 *x, const c128 *y, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = cadd(x[i], y[i]);
}

cudaError_t cocg_axpy_inplace(c128 *x, const c128 *y, int64_t n, cudaStream_t st) {
    k_axpy_inplace<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, y, n);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct CocgImpl {
    CgMat M{};
    CgVec V{};
    CgScal Sc{};
    CgGeom g{};
    int grid = 0;
    c128 *rhs = nullptr;       // shared rhs [n]
    c128 *xsave = nullptr;     // first-solve x [n][kp] (refinement)
    c128 *res = nullptr;       // per-shift residual rhs [n][kp]
    int *h_nactive = nullptr;  // pinned
};

static int alloc_(CocgState &cg, void **p, size_t bytes, std::string &err) {
    cudaError_t e = cudaMalloc(p, bytes < 16 ? 16 : bytes);
    if (e != cudaSuccess) {
        err = std::string("cudaMalloc failed: ") + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? REXI_ERR_NOMEM : REXI_ERR_CUDA;
    }
    cg.allocs.push_back(*p);
    cg.bytes += (int64_t)bytes;
    return REXI_OK;
}

#define CGA(ptr, bytes)                                                   \
    do {                                                                  \
        int _rc = alloc_(cg, (void **)&(ptr), (size_t)(bytes), err);      \
        if (_rc) return _rc;                                              \
    } while (0)
#define CGK(expr)                                                         \
    do {                                                                  \
        cudaError_t _e = (expr);                                          \
        if (_e != cudaSuccess) {                                          \
            err = std::string(#expr) + ": " + cudaGetErrorString(_e);     \
            return REXI_ERR_CUDA;                                         \
        }                                                                 \
    } while (0)

int cocg_create(CocgState &cg, const rexi_desc *d, const ShiftDev &S, int refine, cudaStream_t st,
                std::string &err) {
    CocgImpl *im = new CocgImpl();
    cg.impl = im;
    cg.n = d->n;
    cg.nnz = d->nnz;
    cg.k = d->k;
    cg.refine = refine;
    cg.tol = d->tol > 0 ? d->tol : 1e-12;
    cg.max_iters = d->max_iters > 0 ? d->max_iters : 20000;
    cg.shift_offset = d->shift_offset;
    const int64_t n = d->n, nnz = d->nnz;
    const int kp = S.kp;
    // host: fl(tau*a) per nnz, diagonal positions
    std::vector<double> ta(nnz), tai(nnz), bb(nnz), dta(n, 0.0), dtai(n, 0.0), db(n, 0.0);
    std::vector<char> hasdiag(n, 0);
    for (int64_t r = 0; r < n; ++r)
        for (int32_t q = d->indptr[r]; q < d->indptr[r + 1]; ++q) {
            ta[q] = d->tau * d->a_vals[q];
            tai[q] = d->a_imag ? d->tau * d->a_imag[q] : 0.0;
            bb[q] = d->b_vals[q];
            if (d->indices[q] == r) {
                dta[r] = ta[q];
                dtai[r] = tai[q];
                db[r] = bb[q];
                hasdiag[r] = 1;
            }
        }
    for (int64_t r = 0; r < n; ++r)
        if (!hasdiag[r]) {
            err = "COCG needs a structurally present diagonal (row " + std::to_string(r) + ")";
            return REXI_ERR_UNSUPPORTED;
        }
    int32_t *ip, *ix;
    double *dta_, *dtai_, *db_, *ta_, *tai_, *bb_;
    CGA(ip, sizeof(int32_t) * (n + 1));
    CGA(ix, sizeof(int32_t) * nnz);
    CGA(ta_, sizeof(double) * nnz);
    CGA(tai_, sizeof(double) * nnz);
    CGA(bb_, sizeof(double) * nnz);
    CGA(dta_, sizeof(double) * n);
    CGA(dtai_, sizeof(double) * n);
    CGA(db_, sizeof(double) * n);
    CGK(cudaMemcpyAsync(ip, d->indptr, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(ix, d->indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(ta_, ta.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(tai_, tai.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(bb_, bb.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(dta_, dta.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(dtai_, dtai.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(db_, db.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    im->M = CgMat{n, ip, ix, ta_, tai_, bb_, dta_, dtai_, db_};
    // geometry
    CgGeom &g = im->g;
    g.kp = kp;
    g.kw = kp < 32 ? kp : 32;
    g.G = kp / g.kw;
    g.rpw = 32 / g.kw;
    g.k = d->k;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = ((n + g.rpw - 1) / g.rpw) * g.G;          // warp work items
    int64_t want = (items + CG_WARPS - 1) / CG_WARPS;
    int64_t cap = (int64_t)sms * 8;
    im->grid = (int)std::max<int64_t>(1, std::min(want, cap));
    // grid * CG_WARPS must be a multiple of G so every warp keeps one shift group
    while ((im->grid * CG_WARPS) % g.G) ++im->grid;
    // vectors
    const size_t vb = sizeof(c128) * (size_t)n * kp;
    CGA(im->V.x, vb);
    CGA(im->V.r, vb);
    CGA(im->V.z, vb);
    CGA(im->V.p0, vb);
    CGA(im->V.p1, vb);
    CGA(im->V.q, vb);
    CGA(im->rhs, sizeof(c128) * n);
    if (refine > 0) {
        CGA(im->xsave, vb);
        CGA(im->res, vb);
    }
    CgScal &Sc = im->Sc;
    CGA(Sc.rho, sizeof(double2) * kp);
    CGA(Sc.mu, sizeof(double2) * kp);
    CGA(Sc.alpha, sizeof(double2) * kp);
    CGA(Sc.beta, sizeof(double2) * kp);
    CGA(Sc.rnorm2, sizeof(double) * kp);
    CGA(Sc.bnorm2, sizeof(double) * kp);
    CGA(Sc.active, sizeof(int) * kp);
    CGA(Sc.iters, sizeof(int) * kp);
    CGA(Sc.status, sizeof(int) * kp);
    CGA(Sc.nactive, sizeof(int));
    CGA(Sc.part_a, sizeof(double2) * kp * im->grid);
    CGA(Sc.part_b, sizeof(double2) * kp * im->grid);
    CGA(Sc.part_c, sizeof(double) * kp * im->grid);
    CGA(Sc.counter, sizeof(unsigned int) * 2);
    CGK(cudaMemsetAsync(Sc.counter, 0, sizeof(unsigned int) * 2, st));
    Sc.tol = cg.tol;
    CGK(cudaMallocHost((void **)&im->h_nactive, sizeof(int)));
    CGK(cudaStreamSynchronize(st));
    return REXI_OK;
}

// solve S_j x_j = b for all shifts (b shared or per shift); x in V.x
static int cg_solve(CocgState &cg, CocgImpl *im, const ShiftDev &S, cudaStream_t st, int64_t *launches,
                    std::string &err, int *iters_out) {
    CgVec &V = im->V;
    k_cg_init<<<im->grid, CG_NT, 0, st>>>(im->M, V, im->Sc, S, im->g);
    CGK(cudaGetLastError());
    ++*launches;
    int it = 0, parity = 0;
    const int check_every = 8;
    for (;;) {
        for (int s = 0; s < check_every; ++s) {
            k_cg_spmv<<<im->grid, CG_NT, 0, st>>>(im->M, V, im->Sc, S, im->g, parity);
            k_cg_update<<<im->grid, CG_NT, 0, st>>>(im->M, V, im->Sc, S, im->g, parity, cg.max_iters);
            parity ^= 1;
            *launches += 2;
            ++it;
        }
        CGK(cudaGetLastError());
        CGK(cudaMemcpyAsync(im->h_nactive, im->Sc.nactive, sizeof(int), cudaMemcpyDeviceToHost, st));
        CGK(cudaStreamSynchronize(st));
        if (*im->h_nactive == 0 || it > cg.max_iters + check_every) break;
    }
    // status / iteration statistics
    const int kp = S.kp;
    std::vector<int> status(kp), iters(kp);
    CGK(cudaMemcpyAsync(status.data(), im->Sc.status, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
    CGK(cudaMemcpyAsync(iters.data(), im->Sc.iters, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
    CGK(cudaStreamSynchronize(st));
    int mx = 0;
    double mean = 0.0;
    for (int j = 0; j < cg.k; ++j) {
        mx = std::max(mx, iters[j]);
        mean += iters[j];
        if (iters_out) iters_out[j] += iters[j];
        if (status[j]) {
            char buf[256];
            const char *why = status[j] == 1 ? "COCG breakdown (rho or p^T S p vanished)"
                            : status[j] == 2 ? "non-finite values in COCG"
                                             : "COCG did not converge within max_iters";
            snprintf(buf, sizeof buf, "%s for shift j = %d after %d iterations", why,
                     cg.shift_offset + j, iters[j]);
            err = buf;
            return status[j] == 3 ? REXI_ERR_NOCONV : REXI_ERR_BREAKDOWN;
        }
    }
    cg.last_iters_max = std::max(cg.last_iters_max, mx);
    cg.last_iters_mean += mean / std::max(1, cg.k);
    return REXI_OK;
}

// all shifts, x_j = S_j^{-1} rhs (refined); leaves x in V.x (+ xsave if refined)
static int cg_solve_refined(CocgState &cg, CocgImpl *im, const ShiftDev &S, cudaStream_t st,
                            int64_t *launches, std::string &err) {
    cg.last_iters_max = 0;
    cg.last_iters_mean = 0.0;
    im->V.bshared = im->rhs;
    im->V.bvec = nullptr;
    im->Sc.tol = cg.tol;
    int rc = cg_solve(cg, im, S, st, launches, err, nullptr);
    if (rc) return rc;
    const int64_t n = cg.n;
    const int kp = S.kp;
    for (int r = 0; r < cg.refine; ++r) {
        // true residual in double-double against the accumulated solution
        if (r == 0) CGK(cudaMemcpyAsync(im->xsave, im->V.x, sizeof(c128) * n * kp, cudaMemcpyDeviceToDevice, st));
        else CGK(cocg_axpy_inplace(im->xsave, im->V.x, n * kp, st));
        CgVec Vr = im->V;
        Vr.x = im->xsave;
        k_cg_residual<<<im->grid, CG_NT, 0, st>>>(im->M, Vr, S, im->g, im->res);
        CGK(cudaGetLastError());
        ++*launches;
        im->V.bshared = nullptr;
        im->V.bvec = im->res;
        im->Sc.tol = std::max(1e-8, cg.tol);
        rc = cg_solve(cg, im, S, st, launches, err, nullptr);
        im->V.bshared = im->rhs;
        im->V.bvec = nullptr;
        im->Sc.tol = cg.tol;
        if (rc) return rc;
    }
    return REXI_OK;
}

int cocg_step(CocgState &cg, const ShiftDev &S, cudaStream_t st, const c128 *u, c128 *uout, double *acc,
              int64_t *launches, std::string &err) {
    CocgImpl *im = (CocgImpl *)cg.impl;
    const int64_t n = cg.n;
    k_cg_rhs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(im->M, u, im->rhs);
    CGK(cudaGetLastError());
    ++*launches;
    int rc = cg_solve_refined(cg, im, S, st, launches, err);
    if (rc) return rc;
    // u1 = sum_j beta_j (x_j [+ dx_j])
    const c128 *x1 = cg.refine > 0 ? im->xsave : im->V.x;
    const c128 *x2 = cg.refine > 0 ? im->V.x : nullptr;
    k_cg_accum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, S.kp, cg.k, S.beta, x1, x2, acc, uout);
    CGK(cudaGetLastError());
    ++*launches;
    return REXI_OK;
}

int cocg_solve_all(CocgState &cg, const ShiftDev &S, cudaStream_t st, const c128 *rhs, bool rhs_host,
                   c128 *x, std::string &err) {
    CocgImpl *im = (CocgImpl *)cg.impl;
    const int64_t n = cg.n;
    CGK(cudaMemcpyAsync(im->rhs, rhs, sizeof(c128) * n,
                        rhs_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    int64_t launches = 0;
    int rc = cg_solve_refined(cg, im, S, st, &launches, err);
    if (rc) return rc;
    const c128 *x1 = cg.refine > 0 ? im->xsave : im->V.x;
    const c128 *x2 = cg.refine > 0 ? im->V.x : nullptr;
    const int64_t t = n * (int64_t)cg.k;
    k_cg_transpose<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(x1, x2, n, S.kp, cg.k, x);
    CGK(cudaGetLastError());
    return REXI_OK;
}

void cocg_destroy(CocgState &cg) {
    for (void *p : cg.allocs) cudaFree(p);
    cg.allocs.clear();
    if (cg.impl) {
        CocgImpl *im = (CocgImpl *)cg.impl;
        if (im->h_nactive) cudaFreeHost(im->h_nactive);
        delete im;
        cg.impl = nullptr;
    }
}

}  // namespace rexi
