// pencil.cu -- the pencil (A, B) of one system on one GPU, for the two
// prepare/comparison paths next to the REXI step:
//
//   * rexi_pencil_spectral_radius  <- spectral_radius_estimate
//       (reference spatial.py:314-344): power iteration on B^-1 A with
//       B-pencil Rayleigh quotients |v^H A v / v^H B v|;
//   * rexi_pencil_cheb_step        <- chebyshev_step / chebyshev_run
//       (reference integrate.py:333-377): Clenshaw backward recurrence for
//       p(tau*M) u, one A-multiply and one B-solve per stage;
//   * rexi_pencil_solve_b          <- factorize(sys.B).solve
//       (reference solvers.py:76-80,108-115).
//
// The reference factors B once (banded or dense LU).  B is the real SPD mass
// matrix, so here every B-solve is a Jacobi-preconditioned CG on the shared
// CSR pattern (condition number of D^-1 B is O(1) for P1/P2 mass matrices,
// independent of h).  Per CG iteration two bandwidth-bound kernels:
//
//   dir: p = z + beta p;  q = B z + beta q   (gather z only, q recursively)
//        + partial p^H q
//   upd: x += alpha p;  r -= alpha q;  z = D^-1 r  + partials r^H z, r^H r
//
// Every reduction is a fixed tree (CTA tree over a grid fixed by n, then the
// last CTA folds the CTA partials in index order), so results are bitwise
// repeatable.  The scalar recurrences (alpha, beta, convergence) are
// finished on the device by that last CTA; kernels after convergence exit at
// their first instruction, and the host polls the done flag once per batch
// of iterations.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rexi_b200.h"
#include "common.cuh"

namespace rexi {
void set_global_error(const std::string &msg);
}

using namespace rexi;

namespace {

constexpr int PN_NT = 256;
constexpr int PN_BATCH = 8;   // CG iterations between host polls

struct PnMat {
    int64_t n;
    const int32_t *indptr, *indices;
    const double *a, *ai, *b, *dinv;   // ai may be null (real A)
};

struct PnScal {
    double rz, pq, alpha, beta, rr, bb, tolsq;
    double nrm2, rq;
    c128 num, den;
    int iters, maxit, done, status;
    unsigned ctr;
};

// ---------------------------------------------------------------------------
// deterministic reductions: CTA tree, then the last CTA folds the partials
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void cta_sum(double (&v)[NV], double *sh) {
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], off);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[w * NV + i] = v[i];
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            v[i] = l < PN_NT / 32 ? sh[l * NV + i] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], off);
        }
    }
}

// returns true in thread 0 of the last CTA, with the grid totals in tot
template <int NV>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], double *part, unsigned *ctr, double (&tot)[NV]) {
    __shared__ double sh[(PN_NT / 32) * NV];
    __shared__ bool last;
    cta_sum<NV>(v, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) part[(size_t)blockIdx.x * NV + i] = v[i];
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double u[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) u[i] = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += PN_NT)
#pragma unroll
        for (int i = 0; i < NV; ++i) u[i] += __ldcg(part + (size_t)b * NV + i);
    cta_sum<NV>(u, sh);
    if (threadIdx.x == 0) {
        *ctr = 0;
#pragma unroll
        for (int i = 0; i < NV; ++i) tot[i] = u[i];
        return true;
    }
    return false;
}

__device__ __forceinline__ c128 spmv_row(const int32_t *indptr, const int32_t *indices, const double *v_re,
                                         const double *v_im, const c128 *x, int64_t i) {
    double sr = 0.0, si = 0.0, tr = 0.0, ti = 0.0;
    const int32_t e0 = indptr[i], e1 = indptr[i + 1];
    for (int32_t e = e0; e < e1; ++e) {
        const c128 xc = x[indices[e]];
        const double vr = v_re[e];
        sr = fma(vr, xc.x, sr);
        si = fma(vr, xc.y, si);
        if (v_im) {
            const double vi = v_im[e];
            tr = fma(-vi, xc.y, tr);
            ti = fma(vi, xc.x, ti);
        }
    }
    return cmk(sr + tr, si + ti);
}

// ---------------------------------------------------------------------------
// CG on B x = rhs;  rhs = the vector y (mode 0) or A y (mode 1)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PN_NT) k_cg_init(PnMat M, const c128 *y, int mode, c128 *x, c128 *r, c128 *z,
                                                  c128 *p, c128 *q, PnScal *S, double *part) {
    double v[2] = {0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < M.n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 b = mode ? spmv_row(M.indptr, M.indices, M.a, M.ai, y, i) : y[i];
        const double d = M.dinv[i];
        r[i] = b;
        z[i] = cmk(d * b.x, d * b.y);
        x[i] = cmk(0.0, 0.0);
        p[i] = cmk(0.0, 0.0);
        q[i] = cmk(0.0, 0.0);
        const double b2 = b.x * b.x + b.y * b.y;
        v[0] += d * b2;
        v[1] += b2;
    }
    double t[2];
    if (grid_sum<2>(v, part, &S->ctr, t)) {
        S->rz = t[0];
        S->bb = t[1];
        S->rr = t[1];
        S->beta = 0.0;
        S->iters = 0;
        S->status = 0;
        S->done = t[1] == 0.0 ? 1 : 0;   // zero rhs: x = 0 exactly
        if (!isfinite(t[1])) { S->status = REXI_ERR_BREAKDOWN; S->done = 1; }
    }
}

__global__ void __launch_bounds__(PN_NT) k_cg_dir(PnMat M, const c128 *z, c128 *p, c128 *q, PnScal *S,
                                                 double *part) {
    if (*(volatile int *)&S->done) return;
    const double beta = S->beta;
    double v[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < M.n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 bz = spmv_row(M.indptr, M.indices, M.b, nullptr, z, i);
        const c128 pz = z[i], po = p[i], qo = q[i];
        const c128 pn = cmk(fma(beta, po.x, pz.x), fma(beta, po.y, pz.y));
        const c128 qn = cmk(fma(beta, qo.x, bz.x), fma(beta, qo.y, bz.y));
        p[i] = pn;
        q[i] = qn;
        v[0] += pn.x * qn.x + pn.y * qn.y;
    }
    double t[1];
    if (grid_sum<1>(v, part, &S->ctr, t)) {
        S->pq = t[0];
        if (!(t[0] > 0.0) || !isfinite(t[0])) {
            S->status = REXI_ERR_BREAKDOWN;
            S->done = 1;
        } else {
            S->alpha = S->rz / t[0];
        }
    }
}

__global__ void __launch_bounds__(PN_NT) k_cg_upd(PnMat M, c128 *x, c128 *r, c128 *z, const c128 *p,
                                                 const c128 *q, PnScal *S, double *part) {
    if (*(volatile int *)&S->done) return;
    const double alpha = S->alpha;
    double v[2] = {0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < M.n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 pi = p[i], qi = q[i];
        c128 xi = x[i], ri = r[i];
        xi = cmk(fma(alpha, pi.x, xi.x), fma(alpha, pi.y, xi.y));
        ri = cmk(fma(-alpha, qi.x, ri.x), fma(-alpha, qi.y, ri.y));
        const double d = M.dinv[i];
        x[i] = xi;
        r[i] = ri;
        z[i] = cmk(d * ri.x, d * ri.y);
        const double r2 = ri.x * ri.x + ri.y * ri.y;
        v[0] += d * r2;
        v[1] += r2;
    }
    double t[2];
    if (grid_sum<2>(v, part, &S->ctr, t)) {
        const int it = S->iters + 1;
        S->iters = it;
        S->rr = t[1];
        S->beta = t[0] / S->rz;
        S->rz = t[0];
        if (!isfinite(t[1])) {
            S->status = REXI_ERR_BREAKDOWN;
            S->done = 1;
        } else if (t[1] <= S->tolsq * S->bb) {
            S->done = 1;
        } else if (it >= S->maxit) {
            S->status = REXI_ERR_NOCONV;
            S->done = 1;
        }
    }
}

// ---------------------------------------------------------------------------
// power iteration pieces
// ---------------------------------------------------------------------------
// av = A v; num = v^H A v, den = v^H B v; rq = |num / den|
__global__ void __launch_bounds__(PN_NT) k_rq(PnMat M, const c128 *v, c128 *av, PnScal *S, double *part) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < M.n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 a = spmv_row(M.indptr, M.indices, M.a, M.ai, v, i);
        const c128 b = spmv_row(M.indptr, M.indices, M.b, nullptr, v, i);
        const c128 vi = v[i];
        av[i] = a;
        acc[0] += vi.x * a.x + vi.y * a.y;   // conj(v) a
        acc[1] += vi.x * a.y - vi.y * a.x;
        acc[2] += vi.x * b.x + vi.y * b.y;
        acc[3] += vi.x * b.y - vi.y * b.x;
    }
    double t[4];
    if (grid_sum<4>(acc, part, &S->ctr, t)) {
        S->num = cmk(t[0], t[1]);
        S->den = cmk(t[2], t[3]);
        S->rq = hypot(t[0], t[1]) / hypot(t[2], t[3]);
    }
}

__global__ void __launch_bounds__(PN_NT) k_norm2(int64_t n, const c128 *v, PnScal *S, double *part) {
    double acc[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 vi = v[i];
        acc[0] += vi.x * vi.x + vi.y * vi.y;
    }
    double t[1];
    if (grid_sum<1>(acc, part, &S->ctr, t)) S->nrm2 = t[0];
}

__global__ void __launch_bounds__(PN_NT) k_unit(int64_t n, const c128 *w, c128 *v, const PnScal *S) {
    const double nr = sqrt(S->nrm2);
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 wi = w[i];
        v[i] = cmk(wi.x / nr, wi.y / nr);
    }
}

// ---------------------------------------------------------------------------
// Clenshaw stage: out = a_k u + s2 x - b2   (s2 = 2*scale, or scale at k = 0)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PN_NT) k_clenshaw(int64_t n, c128 ak, double s2, const c128 *u, const c128 *x,
                                                   const c128 *b2, c128 *out) {
    for (int64_t i = (int64_t)blockIdx.x * PN_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * PN_NT) {
        const c128 ui = u[i], xi = x[i], bi = b2[i];
        const double tr = __dsub_rn(__dmul_rn(ak.x, ui.x), __dmul_rn(ak.y, ui.y));
        const double ti = __dadd_rn(__dmul_rn(ak.x, ui.y), __dmul_rn(ak.y, ui.x));
        out[i] = cmk(__dsub_rn(__dadd_rn(tr, __dmul_rn(s2, xi.x)), bi.x),
                     __dsub_rn(__dadd_rn(ti, __dmul_rn(s2, xi.y)), bi.y));
    }
}

__global__ void k_dinv(int64_t n, const int32_t *indptr, const int32_t *indices, const double *b, double *dinv,
                       int *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int32_t e = indptr[i]; e < indptr[i + 1]; ++e)
            if (indices[e] == i) d = b[e];
        if (!(d > 0.0)) atomicExch(bad, 1);
        dinv[i] = d > 0.0 ? 1.0 / d : 0.0;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct rexi_pencil {
    int device = 0;
    int64_t n = 0, nnz = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double tol = 1e-14;
    int max_iters = 1000;
    std::vector<void *> allocs;
    PnMat M{};
    c128 *v = nullptr, *w = nullptr, *av = nullptr;          // power iteration
    c128 *u = nullptr, *b1 = nullptr, *b2 = nullptr, *bn = nullptr;   // Clenshaw
    c128 *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;   // CG
    PnScal *S = nullptr;
    PnScal *h_S = nullptr;   // pinned
    double *part = nullptr;
    unsigned grid = 1;
    int64_t cg_iters_total = 0;
    int cg_iters_max = 0;
    int64_t launches = 0;
    std::string err;
};

namespace {

int pn_err(rexi_pencil *p, int code, const std::string &msg) {
    set_global_error(msg);
    if (p) p->err = msg;
    return code;
}

int pn_cuda(rexi_pencil *p, cudaError_t e, const char *what) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error in %s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    return pn_err(p, e == cudaErrorMemoryAllocation ? REXI_ERR_NOMEM : REXI_ERR_CUDA, buf);
}

#define PK(expr)                                                  \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return pn_cuda(pn, _e, #expr);     \
    } while (0)

template <typename T>
int pn_alloc(rexi_pencil *pn, T **ptr, size_t count) {
    void *d = nullptr;
    cudaError_t e = cudaMalloc(&d, count * sizeof(T) + 16);
    if (e == cudaSuccess) e = rexi_poison(d, count * sizeof(T) + 16);
    if (e != cudaSuccess) return pn_cuda(pn, e, "cudaMalloc");
    pn->allocs.push_back(d);
    *ptr = reinterpret_cast<T *>(d);
    return REXI_OK;
}

// B x = rhs (rhs = y, or A y when mode = 1); leaves x in pn->x
int pn_cg(rexi_pencil *pn, const c128 *y, int mode) {
    const unsigned g = pn->grid;
    k_cg_init<<<g, PN_NT, 0, pn->stream>>>(pn->M, y, mode, pn->x, pn->r, pn->z, pn->p, pn->q, pn->S, pn->part);
    pn->launches++;
    PK(cudaGetLastError());
    int done_iters = 0;
    for (;;) {
        for (int b = 0; b < PN_BATCH; ++b) {
            k_cg_dir<<<g, PN_NT, 0, pn->stream>>>(pn->M, pn->z, pn->p, pn->q, pn->S, pn->part);
            k_cg_upd<<<g, PN_NT, 0, pn->stream>>>(pn->M, pn->x, pn->r, pn->z, pn->p, pn->q, pn->S, pn->part);
            pn->launches += 2;
        }
        PK(cudaGetLastError());
        PK(cudaMemcpyAsync(pn->h_S, pn->S, sizeof(PnScal), cudaMemcpyDeviceToHost, pn->stream));
        PK(cudaStreamSynchronize(pn->stream));
        done_iters = pn->h_S->iters;
        if (pn->h_S->done) break;
    }
    pn->cg_iters_total += done_iters;
    if (done_iters > pn->cg_iters_max) pn->cg_iters_max = done_iters;
    if (pn->h_S->status == REXI_ERR_BREAKDOWN)
        return pn_err(pn, REXI_ERR_BREAKDOWN, "B-solve (CG) broke down: B is not symmetric positive definite");
    if (pn->h_S->status == REXI_ERR_NOCONV) {
        char buf[200];
        snprintf(buf, sizeof buf, "B-solve (CG) did not reach rel. residual %.1e in %d iterations", pn->tol,
                 pn->max_iters);
        return pn_err(pn, REXI_ERR_NOCONV, buf);
    }
    return REXI_OK;
}

int pn_copy_in(rexi_pencil *pn, c128 *dst, const rexi_c128 *src, int mem) {
    PK(cudaMemcpyAsync(dst, src, pn->n * sizeof(c128),
                       mem == REXI_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, pn->stream));
    return REXI_OK;
}

}  // namespace

extern "C" {

int rexi_pencil_create(const rexi_desc *d, rexi_pencil **out) {
    if (!out) return pn_err(nullptr, REXI_ERR_INVALID, "null output pointer");
    *out = nullptr;
    if (!d) return pn_err(nullptr, REXI_ERR_INVALID, "null descriptor");
    if (d->abi_version != REXI_ABI_VERSION) return pn_err(nullptr, REXI_ERR_INVALID, "ABI version mismatch");
    if (d->n < 1) return pn_err(nullptr, REXI_ERR_INVALID, "n must be >= 1");
    if (!d->indptr || !d->indices || !d->a_vals || !d->b_vals)
        return pn_err(nullptr, REXI_ERR_INVALID, "null input array");
    if (d->nnz != d->indptr[d->n]) return pn_err(nullptr, REXI_ERR_INVALID, "nnz does not match indptr[n]");
    for (int64_t q = 0; q < d->nnz; ++q)
        if (d->indices[q] < 0 || d->indices[q] >= d->n)
            return pn_err(nullptr, REXI_ERR_INVALID, "column index out of range");
    rexi_pencil *pn = new rexi_pencil();
    pn->device = d->device;
    pn->n = d->n;
    pn->nnz = d->nnz;
    if (d->tol > 0.0) pn->tol = d->tol;
    if (d->max_iters > 0) pn->max_iters = d->max_iters;
    auto fail = [&](int rc) {
        rexi_pencil_destroy(pn);
        return rc;
    };
    cudaError_t e = cudaSetDevice(d->device);
    if (e != cudaSuccess) return fail(pn_cuda(pn, e, "cudaSetDevice"));
    if (d->stream) {
        pn->stream = (cudaStream_t)d->stream;
    } else {
        e = cudaStreamCreateWithFlags(&pn->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return fail(pn_cuda(pn, e, "cudaStreamCreate"));
        pn->own_stream = true;
    }
    const int64_t n = d->n, nnz = d->nnz;
    int32_t *indptr, *indices;
    double *a, *ai = nullptr, *b, *dinv;
    int rc = REXI_OK;
    if ((rc = pn_alloc(pn, &indptr, n + 1)) || (rc = pn_alloc(pn, &indices, nnz ? nnz : 1)) ||
        (rc = pn_alloc(pn, &a, nnz ? nnz : 1)) || (rc = pn_alloc(pn, &b, nnz ? nnz : 1)) ||
        (rc = pn_alloc(pn, &dinv, n)))
        return fail(rc);
    if (d->a_imag && (rc = pn_alloc(pn, &ai, nnz ? nnz : 1))) return fail(rc);
    c128 **vecs[] = {&pn->v, &pn->w, &pn->av, &pn->u, &pn->b1, &pn->b2, &pn->bn,
                     &pn->x, &pn->r, &pn->z, &pn->p, &pn->q};
    for (c128 **vp : vecs)
        if ((rc = pn_alloc(pn, vp, n))) return fail(rc);
    // fixed grid (depends on n only -> the reduction trees do not depend on the device)
    const int64_t rows_per_cta = (int64_t)PN_NT * 4;
    pn->grid = (unsigned)std::min<int64_t>((n + rows_per_cta - 1) / rows_per_cta, 65535);
    if ((rc = pn_alloc(pn, &pn->part, (size_t)pn->grid * 4)) || (rc = pn_alloc(pn, &pn->S, 1))) return fail(rc);
    e = cudaMallocHost(&pn->h_S, sizeof(PnScal));
    if (e != cudaSuccess) return fail(pn_cuda(pn, e, "cudaMallocHost"));
    int *bad;
    if ((rc = pn_alloc(pn, &bad, 1))) return fail(rc);
#define PC(expr)                                                   \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return fail(pn_cuda(pn, _e, #expr)); \
    } while (0)
    PC(cudaMemcpyAsync(indptr, d->indptr, (n + 1) * 4, cudaMemcpyHostToDevice, pn->stream));
    if (nnz) {
        PC(cudaMemcpyAsync(indices, d->indices, nnz * 4, cudaMemcpyHostToDevice, pn->stream));
        PC(cudaMemcpyAsync(a, d->a_vals, nnz * 8, cudaMemcpyHostToDevice, pn->stream));
        PC(cudaMemcpyAsync(b, d->b_vals, nnz * 8, cudaMemcpyHostToDevice, pn->stream));
        if (ai) PC(cudaMemcpyAsync(ai, d->a_imag, nnz * 8, cudaMemcpyHostToDevice, pn->stream));
    }
    PnScal s0{};
    s0.tolsq = pn->tol * pn->tol;
    s0.maxit = pn->max_iters;
    PC(cudaMemcpyAsync(pn->S, &s0, sizeof s0, cudaMemcpyHostToDevice, pn->stream));
    PC(cudaMemsetAsync(bad, 0, sizeof(int), pn->stream));
    k_dinv<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, pn->stream>>>(n, indptr, indices, b, dinv,
                                                                                       bad);
    PC(cudaGetLastError());
    int hbad = 0;
    PC(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, pn->stream));
    PC(cudaStreamSynchronize(pn->stream));
#undef PC
    if (hbad) return fail(pn_err(pn, REXI_ERR_SINGULAR, "B has a non-positive diagonal entry (not SPD)"));
    pn->M = PnMat{n, indptr, indices, a, ai, b, dinv};
    *out = pn;
    return REXI_OK;
}

int rexi_pencil_solve_b(rexi_pencil *pn, const rexi_c128 *rhs, rexi_c128 *x, int32_t mem, int32_t *iterations) {
    if (!pn || !rhs || !x) return pn_err(pn, REXI_ERR_INVALID, "null argument");
    PK(cudaSetDevice(pn->device));
    int rc;
    if ((rc = pn_copy_in(pn, pn->u, rhs, mem))) return rc;
    if ((rc = pn_cg(pn, pn->u, 0))) return rc;
    PK(cudaMemcpyAsync(x, pn->x, pn->n * sizeof(c128),
                       mem == REXI_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, pn->stream));
    PK(cudaStreamSynchronize(pn->stream));
    if (iterations) *iterations = pn->h_S->iters;
    return REXI_OK;
}

int rexi_pencil_spectral_radius(rexi_pencil *pn, const rexi_c128 *v0, double tol, int32_t max_iters,
                                double *value, int32_t *iterations, int32_t *converged) {
    if (!pn || !v0 || !value) return pn_err(pn, REXI_ERR_INVALID, "null argument");
    if (max_iters < 1) return pn_err(pn, REXI_ERR_INVALID, "max_iters must be >= 1");
    PK(cudaSetDevice(pn->device));
    const unsigned g = pn->grid;
    int rc;
    // v = v0 / ||v0||
    if ((rc = pn_copy_in(pn, pn->w, v0, REXI_MEM_HOST))) return rc;
    k_norm2<<<g, PN_NT, 0, pn->stream>>>(pn->n, pn->w, pn->S, pn->part);
    k_unit<<<g, PN_NT, 0, pn->stream>>>(pn->n, pn->w, pn->v, pn->S);
    pn->launches += 2;
    PK(cudaGetLastError());
    double rq = 0.0, rq_prev = 0.0;
    bool have_prev = false, conv = false;
    int it = 0;
    for (it = 1; it <= max_iters; ++it) {
        k_rq<<<g, PN_NT, 0, pn->stream>>>(pn->M, pn->v, pn->av, pn->S, pn->part);
        pn->launches++;
        PK(cudaGetLastError());
        PK(cudaMemcpyAsync(pn->h_S, pn->S, sizeof(PnScal), cudaMemcpyDeviceToHost, pn->stream));
        PK(cudaStreamSynchronize(pn->stream));
        rq = pn->h_S->rq;
        if (have_prev && std::fabs(rq - rq_prev) <= tol * std::max(rq, 1e-300)) {
            conv = true;
            break;
        }
        rq_prev = rq;
        have_prev = true;
        if ((rc = pn_cg(pn, pn->av, 0))) return rc;
        k_norm2<<<g, PN_NT, 0, pn->stream>>>(pn->n, pn->x, pn->S, pn->part);
        k_unit<<<g, PN_NT, 0, pn->stream>>>(pn->n, pn->x, pn->v, pn->S);
        pn->launches += 2;
        PK(cudaGetLastError());
    }
    if (it > max_iters) it = max_iters;
    *value = rq;
    if (iterations) *iterations = it;
    if (converged) *converged = conv ? 1 : 0;
    return REXI_OK;
}

int rexi_pencil_cheb_step(rexi_pencil *pn, const rexi_c128 *coeffs, int32_t degree, double scale,
                          const rexi_c128 *u_in, rexi_c128 *u_out, int32_t n_steps, int32_t mem,
                          rexi_stats *stats) {
    if (!pn || !coeffs || !u_in || !u_out) return pn_err(pn, REXI_ERR_INVALID, "null argument");
    if (degree < 1) return pn_err(pn, REXI_ERR_INVALID, "degree must be >= 1");
    if (n_steps < 0) return pn_err(pn, REXI_ERR_INVALID, "n_steps must be >= 0");
    PK(cudaSetDevice(pn->device));
    const unsigned g = pn->grid;
    const int64_t n = pn->n;
    pn->cg_iters_total = 0;
    pn->cg_iters_max = 0;
    pn->launches = 0;
    cudaEvent_t e0, e1;
    PK(cudaEventCreate(&e0));
    PK(cudaEventCreate(&e1));
    PK(cudaEventRecord(e0, pn->stream));
    int rc;
    if ((rc = pn_copy_in(pn, pn->u, u_in, mem))) return rc;
    for (int s = 0; s < n_steps; ++s) {
        c128 *b1 = pn->b1, *b2 = pn->b2, *bn = pn->bn;
        PK(cudaMemsetAsync(b1, 0, n * sizeof(c128), pn->stream));
        PK(cudaMemsetAsync(b2, 0, n * sizeof(c128), pn->stream));
        for (int k = degree; k >= 0; --k) {
            if ((rc = pn_cg(pn, b1, 1))) return rc;   // x = B^-1 (A b1)
            const c128 ak = make_double2(coeffs[k].re, coeffs[k].im);
            const double s2 = k > 0 ? 2.0 * scale : scale;
            c128 *dst = k > 0 ? bn : pn->u;
            k_clenshaw<<<g, PN_NT, 0, pn->stream>>>(n, ak, s2, pn->u, pn->x, b2, dst);
            pn->launches++;
            PK(cudaGetLastError());
            if (k > 0) {   // (b1, b2) <- (b_new, b1)
                c128 *t = b2;
                b2 = b1;
                b1 = bn;
                bn = t;
            }
        }
    }
    PK(cudaMemcpyAsync(u_out, pn->u, n * sizeof(c128),
                       mem == REXI_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, pn->stream));
    PK(cudaEventRecord(e1, pn->stream));
    PK(cudaStreamSynchronize(pn->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->t_local_ms = ms;
        stats->steps = n_steps;
        stats->launches = pn->launches;
        stats->iters_max = pn->cg_iters_max;
        const int64_t solves = (int64_t)n_steps * (degree + 1);
        stats->iters_mean = solves ? (double)pn->cg_iters_total / (double)solves : 0.0;
        stats->bad_shift = -1;
    }
    return REXI_OK;
}

const char *rexi_pencil_last_error(const rexi_pencil *pn) { return pn ? pn->err.c_str() : rexi_last_error(); }

int rexi_pencil_wait_stream(rexi_pencil *pn, void *stream) {
    if (!pn) return pn_err(nullptr, REXI_ERR_INVALID, "null pencil");
    if ((cudaStream_t)stream == pn->stream) return REXI_OK;
    cudaSetDevice(pn->device);
    cudaEvent_t e = nullptr;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r == cudaSuccess) r = cudaEventRecord(e, (cudaStream_t)stream);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(pn->stream, e, 0);
    if (e) cudaEventDestroy(e);
    if (r != cudaSuccess) return pn_err(pn, REXI_ERR_CUDA, cudaGetErrorString(r));
    return REXI_OK;
}

int rexi_pencil_destroy(rexi_pencil *pn) {
    if (!pn) return REXI_OK;
    cudaSetDevice(pn->device);
    if (pn->stream) cudaStreamSynchronize(pn->stream);
    for (void *p : pn->allocs) cudaFree(p);
    if (pn->h_S) cudaFreeHost(pn->h_S);
    if (pn->own_stream && pn->stream) cudaStreamDestroy(pn->stream);
    delete pn;
    return REXI_OK;
}

}  // extern "C"
