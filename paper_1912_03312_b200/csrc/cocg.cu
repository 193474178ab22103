// cocg.cu -- lockstep-over-shifts Jacobi-COCG for general CSR pencils (2D/3D,
// P2 1D, dense test pencils).  Replaces, for non-tridiagonal patterns, the
// reference's factorize() (which falls back to a dense LU there,
// solvers.py:108-115) and the K back-substitutions of rexi_step
// (integrate.py:208-222).
//
// Layout: every per-shift vector is [row][kp_cur] complex128 with the shift
// lane fastest: one warp = up to 32 shift lanes of one row (or 32/kp_cur rows
// when fewer lanes are live), so the shared CSR pattern and A/B values are
// read once per row for all shifts and every neighbour gather is one
// contiguous segment.  Shifted entries tau*a - (1j*sigma)*b are formed on the
// fly with the reference's rounding.
//
// Iteration = two kernels (COCG needs two reductions per iteration), 160 B per
// live row-shift:
//   spmv  : x += alpha_prev p (the previous iteration's deferred update, see
//           CG_DEFER_X), p = z + beta p, q = S z + beta q (= S p by linearity:
//           only z is gathered), mu = p^T q.  Chunks are claimed from an
//           atomic counter, so all SMs work on one narrow wavefront and the
//           +-n neighbour rows of a 2D/3D stencil are L2 hits; the per-chunk
//           partials are indexed by chunk, so the reduction order is fixed.
//   update: z -= alpha D^-1 q (the preconditioned residual; r = D z is formed
//           for rho' = r^T z and |r|^2 only).
// Kernel families, all with the same rows per sub-block, per-lane operation
// order and partial tree (bitwise identical results):
//   k_cg_spmv_win / k_cg_update_tma : persistent producer/consumer pipelines,
//           every operand by cp.async.bulk into shared-memory stages (the
//           default wherever the plan has window tables / the layout has
//           >= 2 lanes);
//   k_cg_spmv_tma : tiles by bulk copy, z gathered (2D patterns without tables);
//   k_cg_spmv_st, k_cg_spmv, k_cg_spmv1, k_cg_update, k_cg_update1 : gather
//           kernels (complex A, patterns that fit no window budget, one lane).
// The last CTA of each kernel finishes the per-shift scalars (alpha, beta),
// freezes converged shifts and flags breakdown / non-finite values.
// Compaction: when at most half of the lanes are live, the live shifts are
// repacked (ascending shift order) into a layout half as wide; frozen shifts'
// x are written to the full-width solution first.  The work per iteration then
// follows the number of live shifts instead of K.
// Refinement: r = b - S x with error-free products (double-double), one
// correction solve, and the step output sum_j beta_j (x_j + dx_j) in
// double-double.
#include <cuda_runtime.h>

#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "cocg.cuh"

namespace rexi {

constexpr int CG_NT = 256;            // threads per CTA (8 warps)
constexpr int CG_WARPS = CG_NT / 32;

// Stencil classes (narrow layouts): rows whose column offsets (col - row) and
// B values equal those of a class share one table entry, so the narrow
// spmv streams only fl(tau a) (and fl(tau a_im)) per entry plus a 1-byte
// class id per row instead of index + a + b -- the matrix dominates the
// bytes of an iteration once few shifts are live.  The entries are formed
// from the same doubles in the same order: results are bitwise identical.
constexpr int CG_CLS_MAX = 64;        // classes (id 255: a row without one)
constexpr int CG_CLS_MAXNNZ = 32;     // entries per class row
struct CgClass {
    int nnz;
    int off[CG_CLS_MAXNNZ];
    double b[CG_CLS_MAXNNZ];
};

struct CgMat {
    int64_t n;
    const int32_t *indptr, *indices;
    const double *ta, *ta_im, *b;          // per nnz: fl(tau a), fl(tau a_im), b
    const double *dta, *dta_im, *db;       // per row: the diagonal entry's values
    const uint8_t *cls;                    // per row: stencil class or 255 (nullptr: none)
    const CgClass *classes;
};

struct CgVec {
    c128 *x, *z, *p, *q;                   // [n][kp] current (compacted) layout; the residual
                                           // is kept preconditioned only (r = D z, see k_cg_update)
    const c128 *bvec;                      // per-shift rhs [n][kp_full] or nullptr
    const c128 *bshared;                   // shared rhs [n] or nullptr
};

struct CgScal {                            // per lane of the current layout
    double2 *rho, *alpha, *beta;
    double *rnorm2, *bnorm2;
    int *active, *iters, *status;
    int *flush;                            // lane froze with its last x += alpha p still pending (CG_DEFER_X)
    int *nactive;                          // [1]
    double2 *part_a;                       // spmv partials [nchunks][kp]
    double2 *part_b;                       // update partials [grid][kp]
    double *part_c;                        // update partials [grid][kp]
    double2 *part_f, *part_f2;             // finish level partials [nranges][kp] (ping-pong)
    double *part_g, *part_g2;
    unsigned int *ctr;                     // [8] claim / done counters (parity)
    unsigned int *gctr;                    // [CG_GCTR] finish-tree group counters
    double *tolsq;                         // [kp] squared relative residual target per lane
};

struct CgGeom {
    int kp, kw, G, rpw;                    // lanes, lanes per warp group, groups, rows per warp
    int ld;                                // lanes stored per row (row stride of x, z, p, q): the live
                                           // prefix rounded up, <= kp; lanes >= ld are padding (never live)
    int slots, P, subs, cpc;               // row slots per pass, passes/claim, sub-blocks/claim, chunks/claim
    int64_t nchunks, nclaims;              // 64-row chunks, claims
    const int *lane_shift;                 // [kp] shift index of each lane
};

__device__ __forceinline__ c128 cdiv_c(c128 a, c128 b) { return cmul(a, crcp(b)); }

// Deferred x update (SURVEY 8(d)'s 160 B per live row-shift and iteration):
// x += alpha_k p_k is applied by the NEXT iteration's spmv, which holds p_k in
// registers anyway, so the update kernel touches only z and q (48 B) and the
// spmv 112 B, instead of 96 + 80.  A lane that freezes after update k keeps a
// `flush` flag: the next spmv (or the scatter that takes it out of the layout)
// applies the pending term.  Same operations in the same order per lane:
// bitwise identical to the undeferred form (CG_DEFER_X=0).
#ifndef CG_DEFER_X
#define CG_DEFER_X 1
#endif

#ifndef CG_GB
#define CG_GB 8   // z gathers in flight per thread (global-CSR spmv)
#endif

// (S z)_i for one lane, ascending CSR order, z gathers batched CG_GB at a
// time; a classed row takes its columns and B values from the class table
#ifndef CG_SPMV_UNROLL
#define CG_SPMV_UNROLL 4
#endif
constexpr int kSpmvUnroll = CG_SPMV_UNROLL;
template <bool CPLX, bool BATCH>
__device__ __forceinline__ c128 row_sz(const CgMat &M, int64_t i, const c128 *__restrict__ zv, uint32_t kp,
                                       int lane, c128 sg) {
    c128 acc = cmk(0.0, 0.0);
    const int32_t q0 = __ldg(M.indptr + i);
    const int cl = M.cls ? (int)__ldg(M.cls + i) : 255;
    if (cl != 255) {
        const CgClass &C = M.classes[cl];
        const int nz = C.nnz;
        if (!BATCH) {
#pragma unroll kSpmvUnroll
            for (int k = 0; k < nz; ++k) {
                const c128 e = form_entry(__ldg(M.ta + q0 + k), CPLX ? __ldg(M.ta_im + q0 + k) : 0.0, C.b[k], sg);
                acc = cadd(acc, cmul(e, zv[(uint32_t)(i + C.off[k]) * kp + lane]));
            }
            return acc;
        }
        for (int kb = 0; kb < nz; kb += CG_GB) {
            c128 zz[CG_GB];
#pragma unroll
            for (int k = 0; k < CG_GB; ++k)
                zz[k] = kb + k < nz ? zv[(uint32_t)(i + C.off[kb + k]) * kp + lane] : cmk(0.0, 0.0);
#pragma unroll
            for (int k = 0; k < CG_GB; ++k) {
                if (kb + k < nz) {
                    const int32_t q = q0 + kb + k;
                    const c128 e = form_entry(__ldg(M.ta + q), CPLX ? __ldg(M.ta_im + q) : 0.0, C.b[kb + k], sg);
                    acc = cadd(acc, cmul(e, zz[k]));
                }
            }
        }
        return acc;
    }
    const int32_t q1 = __ldg(M.indptr + i + 1);
    if (!BATCH) {
#pragma unroll kSpmvUnroll
        for (int32_t q = q0; q < q1; ++q) {
            const uint32_t c = (uint32_t)__ldg(M.indices + q);
            const c128 e = form_entry(__ldg(M.ta + q), CPLX ? __ldg(M.ta_im + q) : 0.0, __ldg(M.b + q), sg);
            acc = cadd(acc, cmul(e, zv[c * kp + lane]));
        }
        return acc;
    }
    for (int32_t qb = q0; qb < q1; qb += CG_GB) {
        uint32_t cc[CG_GB];
        c128 zz[CG_GB];
#pragma unroll
        for (int k = 0; k < CG_GB; ++k) cc[k] = qb + k < q1 ? (uint32_t)__ldg(M.indices + qb + k) : 0u;
#pragma unroll
        for (int k = 0; k < CG_GB; ++k) zz[k] = qb + k < q1 ? zv[cc[k] * kp + lane] : cmk(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < CG_GB; ++k) {
            if (qb + k < q1) {
                const int32_t q = qb + k;
                const c128 e = form_entry(__ldg(M.ta + q), CPLX ? __ldg(M.ta_im + q) : 0.0, __ldg(M.b + q), sg);
                acc = cadd(acc, cmul(e, zz[k]));
            }
        }
    }
    return acc;
}

// lane and row slot of this thread for one CTA pass
__device__ __forceinline__ void cta_geom(const CgGeom &g, int &lane, int &slot, int &slots) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int grp = w % g.G;
    lane = grp * g.kw + (l % g.kw);
    slot = (w / g.G) * g.rpw + l / g.kw;
    slots = (CG_WARPS / g.G) * g.rpw;
}

// faster fixed-order CTA reduction: lanes sharing a shift inside a warp
// (rows-per-warp > 1) combine by a butterfly, then thread t < kp sums the
// warps of its shift group in warp order
__device__ __forceinline__ double warp_same_shift(double v, int kw) {
    for (int off = kw; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}
__device__ __forceinline__ void cta_sum2(double2 v, double r, const CgGeom &g, double2 *smc, double *smr,
                                         double2 *outc, double *outr) {
    v.x = warp_same_shift(v.x, g.kw);
    v.y = warp_same_shift(v.y, g.kw);
    r = warp_same_shift(r, g.kw);
    smc[threadIdx.x] = v;
    smr[threadIdx.x] = r;
    __syncthreads();
    if (threadIdx.x < g.kp) {
        const int grp = threadIdx.x / g.kw, sl = threadIdx.x % g.kw;
        double2 s = make_double2(0.0, 0.0);
        double sr = 0.0;
        for (int w = grp; w < CG_WARPS; w += g.G) {
            s = cadd(s, smc[w * 32 + sl]);
            sr += smr[w * 32 + sl];
        }
        outc[threadIdx.x] = s;
        outr[threadIdx.x] = sr;
    }
    __syncthreads();
}

__device__ __forceinline__ bool arrive_last(unsigned int *done, unsigned int total) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == total - 1;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// ---------------------------------------------------------------------------
// Fixed reduction tree (independent of the lane layout, hence of K per GPU,
// sharding and compaction): a thread owns one 4-row sub-block of one shift
// (rows b, b+8, b+16, b+24 of a 32-row chunk, so a warp's row slots touch
// consecutive rows at every step) and sums its rows in order; a 32-row chunk sums its 8 sub-blocks in
// order; the finish kernels sum ranges of CG_RANGE chunks in chunk order,
// then the ranges in order.  Every per-shift scalar is therefore computed by
// the same operation sequence wherever the shift runs.
// ---------------------------------------------------------------------------
constexpr int CG_RANGE = 64;      // chunks per level-1 range, fan-in of the upper levels
constexpr int CG_SB = 4;          // rows per sub-block
constexpr int CG_CH = 8;          // sub-blocks per chunk
constexpr int CG_SBP = 1024;      // shared sub-block partial slots (subs_per_claim * kp)

// sub-block partials of a claim -> chunk partials part[chunk][lane]
template <typename T, typename Add>
__device__ __forceinline__ void chunk_partials(const T *sbp, const CgGeom &g, int64_t claim, T *part, Add add,
                                               T zero) {
    const int kp = g.kp;
    for (int w = threadIdx.x; w < g.cpc * kp; w += CG_NT) {
        const int cc = w / kp, l = w % kp;
        const int64_t chunk = claim * g.cpc + cc;
        if (chunk >= g.nchunks) continue;
        T s = zero;
        for (int b = 0; b < CG_CH; ++b) s = add(s, sbp[(cc * CG_CH + b) * kp + l]);
        part[(size_t)chunk * kp + l] = s;
    }
}

__device__ __forceinline__ double2 add_c(double2 a, double2 b) { return cadd(a, b); }
__device__ __forceinline__ double add_r(double a, double b) { return a + b; }

// ---------------------------------------------------------------------------
// init (full width, lane = shift): x = 0, z = D^-1 b, p_old = 0;
// partials of rho = r^T z and |b|^2
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CG_NT) k_cg_init(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    __shared__ double2 sbc[CG_SBP];
    __shared__ double sbr[CG_SBP];
    int lane, slot, slots;
    cta_geom(g, lane, slot, slots);
    const int kp = g.kp;
    const c128 sg = S.sigma[lane];
    for (int64_t claim = blockIdx.x; claim < g.nclaims; claim += gridDim.x) {
        for (int ps = 0; ps < g.P; ++ps) {
            const int sbl = ps * slots + slot;
            const int64_t gsb = claim * g.subs + sbl;   // sub-block b of chunk c: rows c*32 + b + 8k
            const int64_t r0 = (gsb / CG_CH) * (CG_SB * CG_CH) + gsb % CG_CH;
            c128 rho = cmk(0.0, 0.0);
            double bn = 0.0;
            for (int64_t i = r0; i < min(r0 + CG_SB * CG_CH, M.n); i += CG_CH) {
                const size_t o = (size_t)i * kp + lane;
                const c128 b = V.bshared ? V.bshared[i] : V.bvec[o];
                const c128 z = cdiv_c(b, form_entry(M.dta[i], M.dta_im[i], M.db[i], sg));
                V.x[o] = cmk(0.0, 0.0);
                V.z[o] = z;
                V.p[o] = cmk(0.0, 0.0);
                V.q[o] = cmk(0.0, 0.0);
                rho = cadd(rho, cmul(b, z));
                bn += cabs2(b);
            }
            sbc[sbl * kp + lane] = rho;
            sbr[sbl * kp + lane] = bn;
        }
        __syncthreads();
        chunk_partials<double2>(sbc, g, claim, Sc.part_b, add_c, make_double2(0.0, 0.0));
        chunk_partials<double>(sbr, g, claim, Sc.part_c, add_r, 0.0);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// spmv: w = S z (only z is gathered), then pointwise p <- z + beta p and
// q <- w + beta q (q = S p by linearity: S(z + beta p_old) = S z + beta q_old),
// mu = p^T q.  Gathering one vector instead of two halves the neighbour
// traffic through L2 (the bottleneck of the two-vector form).
// Claims (one or more 32-row chunks) are taken per CTA from an atomic counter:
// all SMs work on one coherent wavefront, so the +-n neighbour rows of a 2D/3D
// stencil are L2 hits.  The next claim is prefetched and the shared partials
// are double-buffered: one barrier per claim.  Element offsets fit in 32 bits
// (n * kp < 2^31 is checked at plan creation).
// ---------------------------------------------------------------------------
#ifndef CG_SPMV_MINB
#define CG_SPMV_MINB 3   // <= 85 registers: 3 CTAs/SM (the stencil-class path adds registers)
#endif
template <bool CPLX, bool BATCH>
__global__ void __launch_bounds__(CG_NT, CG_SPMV_MINB) k_cg_spmv(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    __shared__ double2 sbp[2][CG_SBP];
    __shared__ int64_t claim_q[2];
    if (*Sc.nactive == 0) return;
    int lane, slot, slots;
    cta_geom(g, lane, slot, slots);
    const uint32_t kp = (uint32_t)g.kp, ld = (uint32_t)g.ld;
    const bool act = Sc.active[lane] != 0;
    const bool fl = CG_DEFER_X && !act && Sc.flush[lane] != 0;
    const c128 sg = S.sigma[g.lane_shift[lane]];
    const c128 beta = Sc.beta[lane];
    const c128 alpha = Sc.alpha[lane];
    c128 *__restrict__ pv = V.p;
    c128 *__restrict__ qv = V.q;
    c128 *__restrict__ xv = V.x;
    const c128 *__restrict__ zv = V.z;
    if (threadIdx.x == 0) claim_q[0] = (int64_t)atomicAdd(Sc.ctr, 1u);
    __syncthreads();
    int buf = 0;
    for (;;) {
        const int64_t claim = claim_q[buf];
        if (claim >= g.nclaims) break;
        if (threadIdx.x == 0) claim_q[buf ^ 1] = (int64_t)atomicAdd(Sc.ctr, 1u);
        for (int ps = 0; ps < g.P; ++ps) {
            const int sbl = ps * slots + slot;
            const int64_t gsb = claim * g.subs + sbl;   // sub-block b of chunk c: rows c*32 + b + 8k
            const int64_t r0 = (gsb / CG_CH) * (CG_SB * CG_CH) + gsb % CG_CH;
            c128 mu = cmk(0.0, 0.0);
            if (act) {
                const int64_t r1 = min(r0 + CG_SB * CG_CH, M.n);
                for (int64_t i = r0; i < r1; i += CG_CH) {
                    const c128 acc = row_sz<CPLX, BATCH>(M, i, zv, ld, lane, sg);
                    const uint32_t o = (uint32_t)i * ld + lane;
                    const c128 po = pv[o];
                    if (CG_DEFER_X) xv[o] = cadd(xv[o], cmul(alpha, po));
                    const c128 pi = cadd(zv[o], cmul(beta, po));
                    const c128 qi = cadd(acc, cmul(beta, qv[o]));
                    pv[o] = pi;
                    qv[o] = qi;
                    mu = cadd(mu, cmul(pi, qi));
                }
            } else if (fl) {
                const int64_t r1 = min(r0 + CG_SB * CG_CH, M.n);
                for (int64_t i = r0; i < r1; i += CG_CH) {
                    const uint32_t o = (uint32_t)i * ld + lane;
                    xv[o] = cadd(xv[o], cmul(alpha, pv[o]));
                }
            }
            sbp[buf][sbl * kp + lane] = mu;
        }
        __syncthreads();   // sub-block partials complete, claim_q[buf^1] visible
        chunk_partials<double2>(sbp[buf], g, claim, Sc.part_a, add_c, make_double2(0.0, 0.0));
        buf ^= 1;
    }
}

// ---------------------------------------------------------------------------
// spmv with the claim's CSR slice staged in shared memory (wide layouts).
// Thread 0 bulk-copies (cp.async.bulk, one mbarrier per buffer) the indptr,
// indices and value slices of the NEXT claim while the CTA computes the
// current one, so the per-entry index/value reads are shared-memory
// broadcasts and only the z gathers go to L2/HBM.  Same rows, same order of
// operations as k_cg_spmv -> bitwise identical results.
// ---------------------------------------------------------------------------
constexpr int CG_ST_ROWS = 2 * CG_SB * CG_CH + 8;   // indptr slots per buffer (claims of <= 2 chunks)
constexpr int CG_ST_NNZ = 512;                      // entries per buffer
#ifndef CG_STB
#define CG_STB 8                                    // z gathers in flight per thread
#endif

struct StLayout {
    uint64_t *bar;      // [2]
    int *meta;          // [2][4]: indptr base, index base, value base
    int *ip, *ix;       // [2][CG_ST_ROWS], [2][CG_ST_NNZ + 8]
    double *ta, *tb, *ti;   // [2][CG_ST_NNZ + 8] each (ti only for complex A)
};

__host__ __device__ inline size_t st_smem_bytes(bool cplx) {
    return 128 + 2 * CG_ST_ROWS * 4 + 2 * (CG_ST_NNZ + 8) * 4 + (cplx ? 3 : 2) * 2 * (CG_ST_NNZ + 8) * 8;
}

__device__ __forceinline__ StLayout st_carve(unsigned char *smem, bool cplx) {
    StLayout L;
    L.bar = reinterpret_cast<uint64_t *>(smem);
    L.meta = reinterpret_cast<int *>(smem + 16);
    unsigned char *p = smem + 128;
    L.ip = reinterpret_cast<int *>(p);
    p += 2 * CG_ST_ROWS * 4;
    L.ix = reinterpret_cast<int *>(p);
    p += 2 * (CG_ST_NNZ + 8) * 4;
    L.ta = reinterpret_cast<double *>(p);
    p += 2 * (CG_ST_NNZ + 8) * 8;
    L.tb = reinterpret_cast<double *>(p);
    p += 2 * (CG_ST_NNZ + 8) * 8;
    L.ti = cplx ? reinterpret_cast<double *>(p) : nullptr;
    return L;
}

// thread 0: stage claim `claim` into buffer `b` (arrays padded by >= 32 B)
template <bool CPLX>
__device__ __forceinline__ void st_issue(const StLayout &L, int b, int64_t claim, const CgMat &M, const CgGeom &g,
                                         uint32_t extra_tx = 0) {
    const int64_t rows = (int64_t)g.cpc * CG_SB * CG_CH;
    const int64_t R0 = claim * rows, R1 = min(R0 + rows, M.n);
    const int64_t ipb = R0 & ~3ll, ipe = (R1 + 1 + 3) & ~3ll;
    const int32_t Q0 = __ldg(M.indptr + R0), Q1 = __ldg(M.indptr + R1);
    const int64_t xb = Q0 & ~3, xe = (Q1 + 3) & ~3;
    const int64_t vb = Q0 & ~1, ve = (Q1 + 1) & ~1;
    L.meta[b * 4 + 0] = (int)ipb;
    L.meta[b * 4 + 1] = (int)xb;
    L.meta[b * 4 + 2] = (int)vb;
    const uint32_t bip = (uint32_t)((ipe - ipb) * 4), bix = (uint32_t)((xe - xb) * 4), bv = (uint32_t)((ve - vb) * 8);
    mbar_expect_tx(L.bar + b, bip + bix + bv * (CPLX ? 3 : 2) + extra_tx);
    bulk_g2s(L.ip + b * CG_ST_ROWS, M.indptr + ipb, bip, L.bar + b);
    if (bix) bulk_g2s(L.ix + b * (CG_ST_NNZ + 8), M.indices + xb, bix, L.bar + b);
    if (bv) {
        bulk_g2s(L.ta + b * (CG_ST_NNZ + 8), M.ta + vb, bv, L.bar + b);
        bulk_g2s(L.tb + b * (CG_ST_NNZ + 8), M.b + vb, bv, L.bar + b);
        if (CPLX) bulk_g2s(L.ti + b * (CG_ST_NNZ + 8), M.ta_im + vb, bv, L.bar + b);
    }
}

#ifndef CG_STATIC
#define CG_STATIC 0   // A/B: static claim striding instead of the atomic claim counter
#endif
template <bool CPLX>
#ifndef CG_ST_MINB
#define CG_ST_MINB 3   // 80 registers: 3 CTAs/SM (swept: scripts/tune_spmv_minb.sh)
#endif
__global__ void __launch_bounds__(CG_NT, CG_ST_MINB) k_cg_spmv_st(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    __shared__ double2 sbp[2][CG_SBP];
    __shared__ int64_t claim_q[2];
    extern __shared__ __align__(128) unsigned char smem[];
    if (*Sc.nactive == 0) return;
    const StLayout L = st_carve(smem, CPLX);
    int lane, slot, slots;
    cta_geom(g, lane, slot, slots);
    const uint32_t kp = (uint32_t)g.kp, ld = (uint32_t)g.ld;
    const bool act = Sc.active[lane] != 0;
    const bool fl = CG_DEFER_X && !act && Sc.flush[lane] != 0;
    const c128 sg = S.sigma[g.lane_shift[lane]];
    const c128 beta = Sc.beta[lane];
    const c128 alpha = Sc.alpha[lane];
    c128 *__restrict__ pv = V.p;
    c128 *__restrict__ qv = V.q;
    c128 *__restrict__ xv = V.x;
    const c128 *__restrict__ zv = V.z;
    if (threadIdx.x == 0) {
        mbar_init(L.bar, 1);
        mbar_init(L.bar + 1, 1);
        fence_mbar_init();
        const int64_t c0 = CG_STATIC ? (int64_t)blockIdx.x : (int64_t)atomicAdd(Sc.ctr, 1u);
        claim_q[0] = c0;
        if (c0 < g.nclaims) st_issue<CPLX>(L, 0, c0, M, g);
    }
    __syncthreads();
    int buf = 0;
    uint32_t ph0 = 0, ph1 = 0;
    for (;;) {
        const int64_t claim = claim_q[buf];
        if (claim >= g.nclaims) break;
        if (threadIdx.x == 0) {
            const int64_t cn = CG_STATIC ? claim + gridDim.x : (int64_t)atomicAdd(Sc.ctr, 1u);
            claim_q[buf ^ 1] = cn;
            if (cn < g.nclaims) st_issue<CPLX>(L, buf ^ 1, cn, M, g);
        }
        mbar_wait(L.bar + buf, buf ? ph1 : ph0);
        if (buf) ph1 ^= 1u; else ph0 ^= 1u;
        const int *ip = L.ip + buf * CG_ST_ROWS;
        const int *ix = L.ix + buf * (CG_ST_NNZ + 8);
        const double *sta = L.ta + buf * (CG_ST_NNZ + 8);
        const double *stb = L.tb + buf * (CG_ST_NNZ + 8);
        const double *sti = CPLX ? L.ti + buf * (CG_ST_NNZ + 8) : nullptr;
        const int ipb = L.meta[buf * 4 + 0], xb = L.meta[buf * 4 + 1], vb = L.meta[buf * 4 + 2];
        for (int ps = 0; ps < g.P; ++ps) {
            const int sbl = ps * slots + slot;
            const int64_t gsb = claim * g.subs + sbl;   // sub-block b of chunk c: rows c*32 + b + 8k
            const int64_t r0 = (gsb / CG_CH) * (CG_SB * CG_CH) + gsb % CG_CH;
            c128 mu = cmk(0.0, 0.0);
            if (act) {
                const int64_t r1 = min(r0 + CG_SB * CG_CH, M.n);
                for (int64_t i = r0; i < r1; i += CG_CH) {
                    c128 acc = cmk(0.0, 0.0);
                    const int li = (int)(i - ipb);
                    const int32_t q0 = ip[li], q1 = ip[li + 1];
                    // batches of CG_STB entries: all gathers of a batch in flight
                    // before the (ascending-q) accumulation
                    for (int32_t qb = q0; qb < q1; qb += CG_STB) {
                        c128 zz[CG_STB];
                        uint32_t cc[CG_STB];
#pragma unroll
                        for (int k = 0; k < CG_STB; ++k) cc[k] = qb + k < q1 ? (uint32_t)ix[qb + k - xb] : 0u;
#pragma unroll
                        for (int k = 0; k < CG_STB; ++k)
                            zz[k] = qb + k < q1 ? zv[cc[k] * ld + lane] : cmk(0.0, 0.0);
#pragma unroll
                        for (int k = 0; k < CG_STB; ++k) {
                            if (qb + k < q1) {
                                const int qv = qb + k;
                                const c128 e = form_entry(sta[qv - vb], CPLX ? sti[qv - vb] : 0.0, stb[qv - vb], sg);
                                acc = cadd(acc, cmul(e, zz[k]));
                            }
                        }
                    }
                    const uint32_t o = (uint32_t)i * ld + lane;
                    const c128 po = pv[o];
                    if (CG_DEFER_X) xv[o] = cadd(xv[o], cmul(alpha, po));
                    const c128 pi = cadd(zv[o], cmul(beta, po));
                    const c128 qi = cadd(acc, cmul(beta, qv[o]));
                    pv[o] = pi;
                    qv[o] = qi;
                    mu = cadd(mu, cmul(pi, qi));
                }
            } else if (fl) {
                const int64_t r1 = min(r0 + CG_SB * CG_CH, M.n);
                for (int64_t i = r0; i < r1; i += CG_CH) {
                    const uint32_t o = (uint32_t)i * ld + lane;
                    xv[o] = cadd(xv[o], cmul(alpha, pv[o]));
                }
            }
            sbp[buf][sbl * kp + lane] = mu;
        }
        __syncthreads();   // sub-block partials complete, claim_q[buf^1] visible, buffer buf free
        chunk_partials<double2>(sbp[buf], g, claim, Sc.part_a, add_c, make_double2(0.0, 0.0));
        buf ^= 1;
    }
}

// ---------------------------------------------------------------------------
// spmv, widest layouts (kp = 32 or 64, real A): a persistent CTA per SM whose
// streaming operands never pass through registers.  A producer warp claims
// row chunks from the same atomic counter and bulk-copies (cp.async.bulk) the
// claim's p, q and x tiles -- each one contiguous range of 32 KB -- plus its
// CSR slice into one of two shared-memory stages; 16 consumer warps gather z
// (two rows' gathers in flight per thread), update the tiles in place and hand
// the stage back; the producer bulk-stores the three tiles and refills the
// stage.  The k_cg_spmv_st form keeps ~24 warps x (gathers | own loads) in
// flight per SM and is latency-bound at ~57 % of HBM; here 96 KB of loads and
// 96 KB of stores are in flight per SM independent of the gather latency.
// Same rows per sub-block, same operation order per lane, same partial tree:
// bitwise identical to the other spmv kernels.
// ---------------------------------------------------------------------------
constexpr int CGT_CW = 16;                      // consumer warps
constexpr int CGT_CT = CGT_CW * 32;             // consumer threads
constexpr int CGT_NT = CGT_CT + 32;             // + the producer warp
constexpr int CGT_TILE = CGT_CT * CG_SB;        // row-lanes per claim: 32 KB per vector
#ifndef CGT_ROWS_PAR
#define CGT_ROWS_PAR 1                          // swept with CGT_STB: scripts/tune_tma.sh (1 x 8 fastest)
#endif
constexpr int CGT_RP = CGT_ROWS_PAR;            // rows whose gathers are in flight together
#ifndef CGT_STB
#define CGT_STB 8                               // gathers in flight per row (96 registers, no spills)
#endif

__host__ __device__ inline size_t tma_smem_bytes() {
    return 128 + 2 * 3 * (size_t)CGT_TILE * sizeof(c128) + st_smem_bytes(false) + (size_t)(CGT_CT) * sizeof(double2);
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
// L2 eviction-priority hints (createpolicy): the streamed tiles go first, the z
// windows -- re-read by the stages of the neighbouring grid lines / planes -- last
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void *dst, const void *src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(CGT_CT) : "memory"); }

#if CG_DEFER_X
__global__ void __launch_bounds__(CGT_NT, 1) k_cg_spmv_tma(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (*Sc.nactive == 0) return;
    // header: full[2] (the CSR staging layout's barriers), done[2], claim[2]
    uint64_t *done = reinterpret_cast<uint64_t *>(smem + 64);
    int64_t *claim_q = reinterpret_cast<int64_t *>(smem + 96);
    c128 *tiles = reinterpret_cast<c128 *>(smem + 128);
    unsigned char *stp = smem + 128 + 2 * 3 * (size_t)CGT_TILE * sizeof(c128);
    const StLayout L = st_carve(stp, false);           // L.bar[2] = full[2]
    double2 *sbp = reinterpret_cast<double2 *>(stp + st_smem_bytes(false));
    const uint32_t kp = (uint32_t)g.kp, ld = (uint32_t)g.ld;
    const int64_t rows_pc = (int64_t)g.cpc * CG_SB * CG_CH;
    if (threadIdx.x == 0) {
        mbar_init(L.bar, 1);
        mbar_init(L.bar + 1, 1);
        mbar_init(done, 1);
        mbar_init(done + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x >= CGT_CT) {
        // ---- producer ----
        if (threadIdx.x != CGT_CT) return;
        int64_t prev[2] = {0, 0};
        uint32_t dph[2] = {0u, 0u};
        auto tile = [&](int s, int v) { return tiles + ((size_t)s * 3 + v) * CGT_TILE; };
        auto store = [&](int s, int64_t c) {
            const int64_t R0 = c * rows_pc, R1 = min(R0 + rows_pc, M.n);
            const uint32_t tb = (uint32_t)((R1 - R0) * ld * sizeof(c128));
            const size_t o = (size_t)R0 * ld;
            bulk_s2g(V.p + o, tile(s, 0), tb);
            bulk_s2g(V.q + o, tile(s, 1), tb);
            bulk_s2g(V.x + o, tile(s, 2), tb);
            bulk_commit();
        };
        int i = 0;
        for (;; ++i) {
            const int s = i & 1;
            if (i >= 2) {
                mbar_wait(done + s, dph[s]);
                dph[s] ^= 1u;
                store(s, prev[s]);
                bulk_wait_read0();   // the stage's tiles have been read out: refill
            }
            const int64_t c = (int64_t)atomicAdd(Sc.ctr, 1u);
            claim_q[s] = c;
            if (c >= g.nclaims) {
                mbar_arrive(L.bar + s);
                break;
            }
            prev[s] = c;
            const int64_t R0 = c * rows_pc, R1 = min(R0 + rows_pc, M.n);
            const uint32_t tb = (uint32_t)((R1 - R0) * ld * sizeof(c128));
            const size_t o = (size_t)R0 * ld;
            st_issue<false>(L, s, c, M, g, 3 * tb);
            bulk_g2s(tile(s, 0), V.p + o, tb, L.bar + s);
            bulk_g2s(tile(s, 1), V.q + o, tb, L.bar + s);
            bulk_g2s(tile(s, 2), V.x + o, tb, L.bar + s);
        }
        if (i >= 1) {   // the claim computed last sits in the other stage
            const int s = (i - 1) & 1;
            mbar_wait(done + s, dph[s]);
            store(s, prev[s]);
        }
        bulk_wait0();
        return;
    }
    // ---- consumers ----
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int lane = (w % g.G) * g.kw + (l % g.kw);
    const int sbl = (w / g.G) * g.rpw + l / g.kw;       // sub-block of the claim (one pass)
    const bool act = Sc.active[lane] != 0;
    const bool fl = !act && Sc.flush[lane] != 0;
    const c128 sg = S.sigma[g.lane_shift[lane]];
    const c128 beta = Sc.beta[lane];
    const c128 alpha = Sc.alpha[lane];
    const c128 *__restrict__ zv = V.z;
    uint32_t fph[2] = {0u, 0u};
    for (int it = 0;; ++it) {
        const int s = it & 1;
        mbar_wait(L.bar + s, fph[s]);
        fph[s] ^= 1u;
        const int64_t claim = claim_q[s];
        if (claim >= g.nclaims) break;
        c128 *tp = tiles + ((size_t)s * 3 + 0) * CGT_TILE;
        c128 *tq = tiles + ((size_t)s * 3 + 1) * CGT_TILE;
        c128 *tx = tiles + ((size_t)s * 3 + 2) * CGT_TILE;
        const int *ip = L.ip + s * CG_ST_ROWS;
        const int *ix = L.ix + s * (CG_ST_NNZ + 8);
        const double *sta = L.ta + s * (CG_ST_NNZ + 8);
        const double *stb = L.tb + s * (CG_ST_NNZ + 8);
        const int ipb = L.meta[s * 4 + 0], xb = L.meta[s * 4 + 1], vb = L.meta[s * 4 + 2];
        const int64_t R0 = claim * rows_pc;
        const int64_t gsb = claim * g.subs + sbl;   // sub-block b of chunk c: rows c*32 + b + 8k
        const int64_t r0 = (gsb / CG_CH) * (CG_SB * CG_CH) + gsb % CG_CH;
        c128 mu = cmk(0.0, 0.0);
        if (act) {
#pragma unroll
            for (int h = 0; h < CG_SB / CGT_RP; ++h) {
                int32_t q0[CGT_RP], q1[CGT_RP];
                c128 acc[CGT_RP];
                int nb = 0;
#pragma unroll
                for (int r = 0; r < CGT_RP; ++r) {
                    const int64_t i = r0 + (int64_t)(h * CGT_RP + r) * CG_CH;
                    const bool ok = i < M.n;
                    const int li = ok ? (int)(i - ipb) : 0;
                    q0[r] = ok ? ip[li] : 0;
                    q1[r] = ok ? ip[li + 1] : 0;
                    acc[r] = cmk(0.0, 0.0);
                    nb = max(nb, q1[r] - q0[r]);
                }
                for (int off = 0; off < nb; off += CGT_STB) {
                    c128 zz[CGT_RP][CGT_STB];
#pragma unroll
                    for (int r = 0; r < CGT_RP; ++r)
#pragma unroll
                        for (int k = 0; k < CGT_STB; ++k) {
                            const int32_t q = q0[r] + off + k;
                            const uint32_t cc = q < q1[r] ? (uint32_t)ix[q - xb] : 0u;
                            zz[r][k] = q < q1[r] ? zv[cc * ld + lane] : cmk(0.0, 0.0);
                        }
#pragma unroll
                    for (int r = 0; r < CGT_RP; ++r)
#pragma unroll
                        for (int k = 0; k < CGT_STB; ++k) {
                            const int32_t q = q0[r] + off + k;
                            if (q < q1[r]) {
                                const c128 e = form_entry(sta[q - vb], 0.0, stb[q - vb], sg);
                                acc[r] = cadd(acc[r], cmul(e, zz[r][k]));
                            }
                        }
                }
#pragma unroll
                for (int r = 0; r < CGT_RP; ++r) {
                    const int64_t i = r0 + (int64_t)(h * CGT_RP + r) * CG_CH;
                    if (i < M.n) {
                        const uint32_t o = (uint32_t)i * ld + lane;
                        const uint32_t t = (uint32_t)(i - R0) * ld + lane;
                        const c128 po = tp[t];
                        tx[t] = cadd(tx[t], cmul(alpha, po));
                        const c128 pi = cadd(zv[o], cmul(beta, po));
                        const c128 qi = cadd(acc[r], cmul(beta, tq[t]));
                        tp[t] = pi;
                        tq[t] = qi;
                        mu = cadd(mu, cmul(pi, qi));
                    }
                }
            }
        } else if (fl) {
            const int64_t r1 = min(r0 + CG_SB * CG_CH, M.n);
            for (int64_t i = r0; i < r1; i += CG_CH) {
                const uint32_t t = (uint32_t)(i - R0) * ld + lane;
                tx[t] = cadd(tx[t], cmul(alpha, tp[t]));
            }
        }
        bar_consumers();             // the previous claim's chunk partials have been read
        sbp[sbl * kp + lane] = mu;
        fence_proxy_async();         // tile writes -> visible to the bulk stores
        bar_consumers();
        if (threadIdx.x == 0) mbar_arrive(done + s);
        if (threadIdx.x < g.cpc * (int)kp) {
            const int cc = threadIdx.x / (int)kp, ll = threadIdx.x % (int)kp;
            const int64_t chunk = claim * g.cpc + cc;
            if (chunk < g.nchunks) {
                double2 sum = make_double2(0.0, 0.0);
                for (int b = 0; b < CG_CH; ++b) sum = cadd(sum, sbp[(cc * CG_CH + b) * kp + ll]);
                Sc.part_a[(size_t)chunk * kp + ll] = sum;
            }
        }
    }
}
#endif

// ---------------------------------------------------------------------------
// spmv, widest layouts of 2D-like patterns (kp = 64 or 128, real A): every
// operand arrives by bulk copy.  Rows are processed in stages of R = 1024 / kp
// rows.  At plan creation the columns of every stage are grouped into at most
// three runs of consecutive rows ("z windows": for a structured 2D mesh the
// lines above, around and below the stage's rows), and the stage's matrix
// slice is packed into one blob (local indptr, the window slot of every
// entry's column as uint16, fl(tau a), b).  The producer warp claims 32-row
// chunks from the atomic counter and, per stage, bulk-copies the p, q, x
// tiles, the z windows and the blob into one of two shared-memory stages; the
// consumers read every operand from shared memory -- no load latency in the
// row loop at all -- update the tiles in place, and the producer bulk-stores
// them.  L2 -> SM traffic equals the gather form's (each z row is fetched by
// the ~3 stages whose windows hold it); what changes is that ~100 KB of loads
// per SM are in flight whatever the consumers do.  Same rows per sub-block,
// same operation order per lane, same partial tree: bitwise identical to the
// other spmv kernels.
// ---------------------------------------------------------------------------
constexpr int CG_NWIN = 8;        // z windows per stage (2D stencils use 3, 3D ones 7)
struct WinStage {                 // 128 B per stage
    int64_t blob_off;             // byte offset of the stage's blob (16-B aligned)
    int32_t blob_bytes;           // multiple of 16
    int32_t off_zs, off_ta, off_b;   // byte offsets inside the blob (local indptr at 0)
    int32_t wstart[CG_NWIN], wrows[CG_NWIN];   // z windows: first row, rows (0: unused)
    int32_t own0;                 // window slot of the stage's first row
    int32_t pad[9];
};
static_assert(sizeof(WinStage) == 128, "WinStage is one 128-B directory entry");

struct CgWin {
    const WinStage *dir = nullptr;
    const unsigned char *blob = nullptr;
    int blob_max = 0;             // largest blob, rounded up to 128 B
    int zrows = 0;                // z-window rows of the largest stage (rounded up to 8)
    int64_t nstages = 0;
    int rl = 2;                   // row-lanes per consumer thread and stage (2: 2D tables, 1: 3D)
};

// RL row-lanes per consumer thread and stage: 2 for 2D-like patterns (three
// windows of R + 1..2 rows), 1 for 3D-like ones (seven windows: half the rows
// per stage keep them inside the shared-memory budget)
template <int KP, int RL> struct WinGeom {
    static constexpr int R = (CGT_CT * RL) / KP;         // rows per stage
    static constexpr int NST = R >= 32 ? 1 : (CG_SB * CG_CH) / R;   // stages per claim (a 32-row chunk)
    static constexpr int CPS = R >= 32 ? R / 32 : 1;     // chunks per stage (kp <= 32)
    static constexpr size_t tile_bytes = (size_t)R * KP * sizeof(c128);
};
// two stages of: three tiles, the z windows (zrows rows: the largest stage's, found at
// plan creation), the matrix blob
template <int KP, int RL>
__host__ __device__ inline size_t win_smem_bytes(int blob_max, int zrows) {
    return 128 + 2 * (3 * WinGeom<KP, RL>::tile_bytes + (size_t)zrows * KP * sizeof(c128) + (size_t)blob_max);
}
constexpr size_t CG_SMEM_MAX = 227 * 1024;

#if CG_DEFER_X
template <int KP, int RL>
__global__ void __launch_bounds__(CGT_NT, 1) k_cg_spmv_win(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g, CgWin W) {
    using G = WinGeom<KP, RL>;
    constexpr int R = G::R, NST = G::NST;
    extern __shared__ __align__(128) unsigned char smem[];
    if (*Sc.nactive == 0) return;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *done = reinterpret_cast<uint64_t *>(smem + 16);
    int64_t *slot_q = reinterpret_cast<int64_t *>(smem + 32);
    int4 *dirq = reinterpret_cast<int4 *>(smem + 64);   // per slot: blob offsets of zs / ta / b, own0
    const size_t zwin_bytes = (size_t)W.zrows * KP * sizeof(c128);
    const size_t stage_bytes = 3 * G::tile_bytes + zwin_bytes + (size_t)W.blob_max;
    const uint32_t ld = (uint32_t)g.ld;
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        mbar_init(done, 1);
        mbar_init(done + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x >= CGT_CT) {
        // ---- producer ----
        if (threadIdx.x != CGT_CT) return;
        int64_t prev[2] = {0, 0};
        uint32_t dph[2] = {0u, 0u};
#ifndef CGW_L2HINT
#define CGW_L2HINT 1   // A/B: eviction-priority hints on the bulk copies
#endif
        const uint64_t pol_s = l2_policy_evict_first(), pol_z = l2_policy_evict_last();
        auto ld_s = [&](void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
            if (CGW_L2HINT) bulk_g2s_hint(dst, src, bytes, bar, pol_s);
            else bulk_g2s(dst, src, bytes, bar);
        };
        auto ld_z = [&](void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
            if (CGW_L2HINT) bulk_g2s_hint(dst, src, bytes, bar, pol_z);
            else bulk_g2s(dst, src, bytes, bar);
        };
        auto st_s = [&](void *dst, const void *src, uint32_t bytes) {
            if (CGW_L2HINT) bulk_s2g_hint(dst, src, bytes, pol_s);
            else bulk_s2g(dst, src, bytes);
        };
        auto store = [&](int s, int64_t gs) {
            unsigned char *base = smem + 128 + (size_t)s * stage_bytes;
            const int64_t R0 = gs * R;
            const int64_t rows = min((int64_t)R, M.n - R0);
            if (rows > 0) {
                const uint32_t tb = (uint32_t)(rows * ld * sizeof(c128));
                const size_t o = (size_t)R0 * ld;
                st_s(V.p + o, base, tb);
                st_s(V.q + o, base + G::tile_bytes, tb);
                st_s(V.x + o, base + 2 * G::tile_bytes, tb);
            }
            bulk_commit();
        };
        int it = 0;
        bool ended = false;
        const int64_t nunits = (g.nchunks + G::CPS - 1) / G::CPS;   // claim unit: a chunk (kp >= 64) or a stage
        // The refill of a stage sits on the consumers' critical path, so nothing
        // with a global round trip stays in it: the next unit is claimed one unit
        // ahead and the next stage's directory entry is loaded one stage ahead
        // (CGW_LOOKAHEAD=0: both inside the refill, the first form of this kernel).
#ifndef CGW_LOOKAHEAD
#define CGW_LOOKAHEAD 1
#endif
        auto has_rows = [&](int64_t ch, int hh) { return ch < nunits && (ch * NST + hh) * R < M.n; };
        int64_t chunk = (int64_t)atomicAdd(Sc.ctr, 1u), chunk_nx = 0;
        bool nx_claimed = false;
        int h = 0;
        WinStage d{};
        if (CGW_LOOKAHEAD && has_rows(chunk, 0)) d = W.dir[chunk * NST];
        for (;; ++it) {
            const int s = it & 1;
            if (it >= 2) {
                mbar_wait(done + s, dph[s]);
                dph[s] ^= 1u;
                store(s, prev[s]);
                bulk_wait_read0();
            }
            if (chunk >= nunits) {
                slot_q[s] = -1;
                mbar_arrive(full + s);
                ended = true;
                break;
            }
            const int64_t gs = chunk * NST + h;
            slot_q[s] = gs;
            prev[s] = gs;
            const int64_t R0 = gs * R;
            const int64_t rows = min((int64_t)R, M.n - R0);
            if (rows <= 0) {            // stage past the last row of the last chunk
                mbar_arrive(full + s);
            } else {
                unsigned char *base = smem + 128 + (size_t)s * stage_bytes;
                if (!CGW_LOOKAHEAD) d = W.dir[gs];
                dirq[s] = make_int4(d.off_zs, d.off_ta, d.off_b, d.own0);
                const uint32_t tb = (uint32_t)(rows * ld * sizeof(c128));
                const uint32_t rb = ld * (uint32_t)sizeof(c128);
                uint32_t zr = 0;
#pragma unroll
                for (int k = 0; k < CG_NWIN; ++k) zr += (uint32_t)d.wrows[k];
                const uint32_t zb = zr * rb;
                mbar_expect_tx(full + s, 3 * tb + zb + (uint32_t)d.blob_bytes);
                const size_t o = (size_t)R0 * ld;
                unsigned char *zw = base + 3 * G::tile_bytes;
                uint32_t zo = 0;
#pragma unroll
                for (int k = 0; k < CG_NWIN; ++k)
                    if (d.wrows[k] > 0) {
                        ld_z(zw + zo, V.z + (size_t)d.wstart[k] * ld, (uint32_t)d.wrows[k] * rb, full + s);
                        zo += (uint32_t)d.wrows[k] * rb;
                    }
                ld_s(zw + zwin_bytes, W.blob + d.blob_off, (uint32_t)d.blob_bytes, full + s);
                ld_s(base, V.p + o, tb, full + s);
                ld_s(base + G::tile_bytes, V.q + o, tb, full + s);
                ld_s(base + 2 * G::tile_bytes, V.x + o, tb, full + s);
            }
            // the stage after this one
            if (CGW_LOOKAHEAD && !nx_claimed) {
                chunk_nx = (int64_t)atomicAdd(Sc.ctr, 1u);
                nx_claimed = true;
            }
            if (++h == NST) {
                h = 0;
                chunk = CGW_LOOKAHEAD ? chunk_nx : (int64_t)atomicAdd(Sc.ctr, 1u);
                nx_claimed = false;
            }
            if (CGW_LOOKAHEAD && has_rows(chunk, h)) d = W.dir[chunk * NST + h];
        }
        (void)ended;
        if (it >= 1) {   // the stage computed last sits in the other slot
            const int s = (it - 1) & 1;
            mbar_wait(done + s, dph[s]);
            store(s, prev[s]);
        }
        bulk_wait0();
        return;
    }
    // ---- consumers: RL row-lanes per thread and stage ----
    static_assert(RL == 2 || KP >= 32 || G::R >= 32, "one row-lane per thread: whole chunks per stage, or kp >= 32");
    static_assert(KP > 32 || NST <= 2, "terms over at most two stages per chunk");
    const int lane = threadIdx.x % KP;
    const int lr0 = threadIdx.x / KP;
    constexpr int LRS = CGT_CT / KP;                   // local-row distance of a thread's two rows
    constexpr bool SAME = LRS == CG_CH;                // a thread's rows all belong to sub-block lr0 (kp = 64);
                                                       // kp = 128: to sub-blocks lr0 and lr0 + 4
    constexpr bool TERMS = KP <= 32;                   // per-row terms, summed in tree order: a stage holds whole
                                                       // chunks (or, kp = 32 with one row-lane, half a chunk: NST = 2)
    const bool act = Sc.active[lane] != 0;
    const bool fl = !act && Sc.flush[lane] != 0;
    const c128 sg = S.sigma[g.lane_shift[lane]];
    const c128 beta = Sc.beta[lane];
    const c128 alpha = Sc.alpha[lane];
    uint32_t fph[2] = {0u, 0u};
    c128 mu[2] = {cmk(0.0, 0.0), cmk(0.0, 0.0)};
    for (int it = 0;; ++it) {
        const int s = it & 1;
        mbar_wait(full + s, fph[s]);
        fph[s] ^= 1u;
        const int64_t gs = slot_q[s];
        if (gs < 0) break;
        const int h = (int)(gs % NST);
        const int64_t chunk = gs / NST;
        unsigned char *base = smem + 128 + (size_t)s * stage_bytes;
        c128 *tp = reinterpret_cast<c128 *>(base);
        c128 *tq = reinterpret_cast<c128 *>(base + G::tile_bytes);
        c128 *tx = reinterpret_cast<c128 *>(base + 2 * G::tile_bytes);
        c128 *zw = reinterpret_cast<c128 *>(base + 3 * G::tile_bytes);
        const int64_t R0 = gs * R;
        const int rows = (int)min((int64_t)R, M.n - R0);
        if (h == 0 || (TERMS && NST == 1)) mu[0] = mu[1] = cmk(0.0, 0.0);
        if (rows > 0 && (act || fl)) {
            const unsigned char *blob = base + 3 * G::tile_bytes + zwin_bytes;
            const int4 dq = dirq[s];
            const int off_zs = dq.x, off_ta = dq.y, off_b = dq.z, own0 = dq.w;
            const int *ip = reinterpret_cast<const int *>(blob);
            const unsigned short *zs = reinterpret_cast<const unsigned short *>(blob + off_zs);
            const double *sta = reinterpret_cast<const double *>(blob + off_ta);
            const double *stb = reinterpret_cast<const double *>(blob + off_b);
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int lr = lr0 + r * LRS;
                if (lr < rows) {
                    const uint32_t t = (uint32_t)lr * ld + lane;
                    if (act) {
                        // accumulator of this row's sub-block (row h*R + lr of the chunk)
                        const int a = SAME ? 0 : (((h * R + lr) % CG_CH) != lr0);
                        const int q0 = ip[lr], q1 = ip[lr + 1];
                        c128 acc = cmk(0.0, 0.0);
#pragma unroll 4
                        for (int q = q0; q < q1; ++q) {
                            const c128 e = form_entry(sta[q], 0.0, stb[q], sg);
                            acc = cadd(acc, cmul(e, zw[(uint32_t)zs[q] * ld + lane]));
                        }
                        const c128 po = tp[t];
                        tx[t] = cadd(tx[t], cmul(alpha, po));
                        const c128 pi = cadd(zw[(uint32_t)(own0 + lr) * ld + lane], cmul(beta, po));
                        const c128 qi = cadd(acc, cmul(beta, tq[t]));
                        tp[t] = pi;
                        tq[t] = qi;
                        const c128 term = cmul(pi, qi);
                        if (TERMS && NST == 1) mu[r] = term;
                        else if (TERMS) { if (h == 0) mu[0] = term; else mu[1] = term; }
                        else if (a == 0) mu[0] = cadd(mu[0], term);
                        else mu[1] = cadd(mu[1], term);
                    } else {
                        tx[t] = cadd(tx[t], cmul(alpha, tp[t]));
                    }
                }
            }
        }
        fence_proxy_async();         // tile writes -> visible to the bulk stores
        bar_consumers();             // every consumer is done with the stage's z windows and tiles
        if (TERMS && (NST == 1 || h == NST - 1)) {
            // the stage holds G::CPS whole chunks (NST = 2: the chunk's second half, the
            // first half's terms are in mu[0]): per-row terms through the (now dead)
            // z-window area, then each chunk's tree (sub-block b = rows b, b+8, b+16,
            // b+24 in order from 0; the 8 sub-blocks in order from 0)
            double2 *trm = reinterpret_cast<double2 *>(zw);
            trm[lr0 * KP + lane] = mu[0];
            if (RL == 2 || NST == 2) trm[(lr0 + (NST == 2 ? R : LRS)) * KP + lane] = mu[1];
            bar_consumers();
            if (threadIdx.x < G::CPS * KP) {
                const int cc = threadIdx.x / KP, ll = threadIdx.x % KP;
                const int64_t chunk = NST == 2 ? gs / NST : gs * G::CPS + cc;
                if (chunk < g.nchunks) {
                    const double2 *tc = trm + (size_t)cc * (CG_SB * CG_CH) * KP + ll;
                    double2 sum = make_double2(0.0, 0.0);
#pragma unroll
                    for (int b = 0; b < CG_CH; ++b) {
                        double2 sb = make_double2(0.0, 0.0);
#pragma unroll
                        for (int k = 0; k < CG_SB; ++k) sb = cadd(sb, tc[(b + k * CG_CH) * KP]);
                        sum = cadd(sum, sb);
                    }
                    Sc.part_a[(size_t)chunk * KP + ll] = sum;
                }
            }
            fence_proxy_async();
            bar_consumers();
        } else if (h == NST - 1) {
            // chunk partial: the sub-block partials go through the (now dead) z-window area
            double2 *sbp = reinterpret_cast<double2 *>(zw);
            if (SAME) {
                sbp[lr0 * KP + lane] = mu[0];
            } else {
                sbp[lr0 * KP + lane] = mu[0];
                sbp[(lr0 + LRS) * KP + lane] = mu[1];
            }
            bar_consumers();
            if (threadIdx.x < KP) {
                double2 sum = make_double2(0.0, 0.0);
#pragma unroll
                for (int b = 0; b < CG_CH; ++b) sum = cadd(sum, sbp[b * KP + threadIdx.x]);
                Sc.part_a[(size_t)chunk * KP + threadIdx.x] = sum;
            }
            fence_proxy_async();     // the partial slots will be overwritten by the next bulk load
            bar_consumers();
        }
        if (threadIdx.x == 0) mbar_arrive(done + s);
    }
}
#endif

// ---------------------------------------------------------------------------
// update, widest layouts (kp = 64 or 128, real A): the same producer /
// consumer pipeline for the pointwise half of the iteration.  Stages of
// 2048 / kp rows (the z and q tiles, 32 KB each, plus the rows' diagonal data),
// three in flight per SM, claims strided over the CTAs; four row-lanes per
// consumer thread; only the z tile is stored.  Same per-lane arithmetic and
// partial tree as k_cg_update: bitwise identical.
// ---------------------------------------------------------------------------
template <int KP> struct UpdGeom {
    static constexpr int R = (CGT_CT * 4) / KP;          // rows per stage (four row-lanes per consumer thread)
    static constexpr int UNIT = R >= 32 ? R : 32;        // rows per claim unit: a stage of whole chunks, or a chunk
    static constexpr int NST = UNIT / R;                 // stages per unit (kp = 128: 2)
    static constexpr int CPS = R >= 32 ? R / 32 : 1;     // chunks per stage
    static constexpr bool TERMS = KP <= 32;              // per-row terms summed in tree order (a thread's rows
                                                         // belong to several sub-blocks' interleaved rows)
    static constexpr int NSTG = KP >= 8 ? 3 : 2;         // pipeline stages
    static constexpr size_t tile_bytes = (size_t)CGT_CT * 4 * sizeof(c128);   // 32 KB
    static constexpr size_t diag_bytes = ((size_t)R * 8 + 255) & ~(size_t)255;
    static constexpr size_t stage_bytes = 2 * tile_bytes + 2 * diag_bytes;    // z, q, dta[R], db[R]
    static constexpr size_t rterm_bytes = TERMS ? (size_t)CGT_CT * 4 * sizeof(double) : 0;
};
template <int KP>
__host__ __device__ inline size_t upd_smem_bytes() {
    return 128 + UpdGeom<KP>::NSTG * UpdGeom<KP>::stage_bytes + UpdGeom<KP>::rterm_bytes;
}

#if CG_DEFER_X
template <int KP>
__global__ void __launch_bounds__(CGT_NT, 1) k_cg_update_tma(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    using G = UpdGeom<KP>;
    constexpr int R = G::R, NST = G::NST, NSTG = G::NSTG;
    extern __shared__ __align__(128) unsigned char smem[];
    if (*Sc.nactive == 0) return;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);          // [3]
    uint64_t *done = reinterpret_cast<uint64_t *>(smem + 32);     // [3]
    const uint32_t ld = (uint32_t)g.ld;
    if (threadIdx.x == 0) {
        for (int k = 0; k < NSTG; ++k) {
            mbar_init(full + k, 1);
            mbar_init(done + k, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // this CTA's stages: units blockIdx.x, blockIdx.x + gridDim.x, ... (NST stages each)
    const int64_t nunits = (M.n + G::UNIT - 1) / G::UNIT;
    const int64_t my_units = nunits > blockIdx.x ? (nunits - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int64_t my_stages = my_units * NST;
    auto stage_of = [&](int64_t it) { return ((int64_t)blockIdx.x + (it / NST) * gridDim.x) * NST + it % NST; };
    if (threadIdx.x >= CGT_CT) {
        // ---- producer ----
        if (threadIdx.x != CGT_CT) return;
        uint32_t dph[NSTG] = {};
        for (int64_t it = 0; it < my_stages + NSTG; ++it) {
            const int s = (int)(it % NSTG);
            if (it >= NSTG) {
                // stage it - NSTG has been computed: store its z tile, free the slot
                const int64_t gp = stage_of(it - NSTG);
                mbar_wait(done + s, dph[s]);
                dph[s] ^= 1u;
                const int64_t R0 = gp * R;
                const int64_t rows = min((int64_t)R, M.n - R0);
                if (rows > 0) bulk_s2g(V.z + (size_t)R0 * ld, smem + 128 + (size_t)s * G::stage_bytes, (uint32_t)(rows * ld * sizeof(c128)));
                bulk_commit();
                if (it < my_stages) bulk_wait_read0();
            }
            if (it >= my_stages) continue;
            const int64_t gs = stage_of(it);
            const int64_t R0 = gs * R;
            const int64_t rows = min((int64_t)R, M.n - R0);
            if (rows <= 0) {
                mbar_arrive(full + s);
                continue;
            }
            unsigned char *base = smem + 128 + (size_t)s * G::stage_bytes;
            const uint32_t tb = (uint32_t)(rows * ld * sizeof(c128));
            const uint32_t db = (uint32_t)(((rows + 1) & ~(int64_t)1) * sizeof(double));
            mbar_expect_tx(full + s, 2 * tb + 2 * db);
            bulk_g2s(base, V.z + (size_t)R0 * ld, tb, full + s);
            bulk_g2s(base + G::tile_bytes, V.q + (size_t)R0 * ld, tb, full + s);
            bulk_g2s(base + 2 * G::tile_bytes, M.dta + R0, db, full + s);
            bulk_g2s(base + 2 * G::tile_bytes + G::diag_bytes, M.db + R0, db, full + s);
        }
        bulk_wait0();
        return;
    }
    // ---- consumers: four row-lanes per thread and stage ----
    const int lane = threadIdx.x % KP;
    const int lr0 = threadIdx.x / KP;
    constexpr int LRS = CGT_CT / KP;                   // kp = 64: 8, one sub-block per thread; kp = 128: 4
    const bool act = Sc.active[lane] != 0;
    const c128 sg = S.sigma[g.lane_shift[lane]];
    const c128 alpha = Sc.alpha[lane];
    uint32_t fph[NSTG] = {};
    c128 rho[G::TERMS ? 4 : 2];
    double rn[G::TERMS ? 4 : 2];
    double *rterm = reinterpret_cast<double *>(smem + 128 + NSTG * G::stage_bytes);
    for (int64_t it = 0; it < my_stages; ++it) {
        const int s = (int)(it % NSTG);
        mbar_wait(full + s, fph[s]);
        fph[s] ^= 1u;
        const int64_t gs = stage_of(it);
        const int h = (int)(it % NST);
        unsigned char *base = smem + 128 + (size_t)s * G::stage_bytes;
        c128 *tz = reinterpret_cast<c128 *>(base);
        c128 *tq = reinterpret_cast<c128 *>(base + G::tile_bytes);
        const double *sdta = reinterpret_cast<const double *>(base + 2 * G::tile_bytes);
        const double *sdb = reinterpret_cast<const double *>(base + 2 * G::tile_bytes + G::diag_bytes);
        const int rows = (int)min((int64_t)R, M.n - gs * R);
        if (h == 0 || G::TERMS) {
#pragma unroll
            for (int k = 0; k < (G::TERMS ? 4 : 2); ++k) {
                rho[k] = cmk(0.0, 0.0);
                rn[k] = 0.0;
            }
        }
        if (act) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int lr = lr0 + k * LRS;
                if (lr < rows) {
                    const uint32_t t = (uint32_t)lr * ld + lane;
                    const c128 q = tq[t];
                    const c128 d = form_entry(sdta[lr], 0.0, sdb[lr], sg);
                    const c128 z = csub(tz[t], cmul(alpha, cdiv_c(q, d)));
                    tz[t] = z;
                    const c128 r = cmul(d, z);
                    if (G::TERMS) {
                        rho[k] = cmul(r, z);
                        rn[k] = cabs2(r);
                    } else {
                        const int a = LRS == CG_CH ? 0 : (k & 1);
                        rho[a] = cadd(rho[a], cmul(r, z));
                        rn[a] += cabs2(r);
                    }
                }
            }
        }
        fence_proxy_async();         // z tile writes -> visible to the bulk store
        bar_consumers();
        if (G::TERMS) {
            // whole chunks per stage: per-row terms through the (now dead) q tile and the
            // real-term buffer, then each chunk's tree in order
            double2 *trm = reinterpret_cast<double2 *>(tq);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                trm[(lr0 + k * LRS) * KP + lane] = rho[k];
                rterm[(lr0 + k * LRS) * KP + lane] = rn[k];
            }
            bar_consumers();
            if (threadIdx.x < G::CPS * KP) {
                const int cc = threadIdx.x / KP, ll = threadIdx.x % KP;
                const int64_t chunk = gs * G::CPS + cc;
                if (chunk < g.nchunks) {
                    const double2 *tc = trm + (size_t)cc * (CG_SB * CG_CH) * KP + ll;
                    const double *tr = rterm + (size_t)cc * (CG_SB * CG_CH) * KP + ll;
                    double2 sum = make_double2(0.0, 0.0);
                    double sr = 0.0;
#pragma unroll
                    for (int b = 0; b < CG_CH; ++b) {
                        double2 sb = make_double2(0.0, 0.0);
                        double sbr = 0.0;
#pragma unroll
                        for (int k = 0; k < CG_SB; ++k) {
                            sb = cadd(sb, tc[(b + k * CG_CH) * KP]);
                            sbr += tr[(b + k * CG_CH) * KP];
                        }
                        sum = cadd(sum, sb);
                        sr += sbr;
                    }
                    Sc.part_b[(size_t)chunk * KP + ll] = sum;
                    Sc.part_c[(size_t)chunk * KP + ll] = sr;
                }
            }
            fence_proxy_async();     // the term slots will be overwritten by the next bulk load
            bar_consumers();
        } else if (h == NST - 1) {
            // chunk partials: the sub-block partials go through the (now dead) q tile
            double2 *sbc = reinterpret_cast<double2 *>(tq);
            double *sbr = reinterpret_cast<double *>(sbc + CG_CH * KP);
            sbc[lr0 * KP + lane] = rho[0];
            sbr[lr0 * KP + lane] = rn[0];
            if (LRS != CG_CH) {
                sbc[(lr0 + LRS) * KP + lane] = rho[1];
                sbr[(lr0 + LRS) * KP + lane] = rn[1];
            }
            bar_consumers();
            if (threadIdx.x < KP) {
                const int64_t chunk = gs / NST;
                double2 sum = make_double2(0.0, 0.0);
                double sr = 0.0;
#pragma unroll
                for (int b = 0; b < CG_CH; ++b) {
                    sum = cadd(sum, sbc[b * KP + threadIdx.x]);
                    sr += sbr[b * KP + threadIdx.x];
                }
                Sc.part_b[(size_t)chunk * KP + threadIdx.x] = sum;
                Sc.part_c[(size_t)chunk * KP + threadIdx.x] = sr;
            }
            fence_proxy_async();     // the partial slots will be overwritten by the next bulk load
            bar_consumers();
        }
        if (threadIdx.x == 0) mbar_arrive(done + s);
    }
}
#endif

// ---------------------------------------------------------------------------
// Width 1 (one live shift, the tail of a solve): one thread per row, a warp
// per 32-row chunk.  The sub-block partial (rows b, b+8, b+16, b+24 summed
// in that order from 0) and the chunk partial (sub-blocks 0..7 in order) are
// formed with shuffles in the same order as the general kernels, so the
// results are bitwise identical to them -- with 4x the threads in flight.
// ---------------------------------------------------------------------------
constexpr int CG1_NT = 256;

__device__ __forceinline__ double2 shfl_c(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// chunk partial of a warp's 32 per-row terms (lane = row in chunk)
__device__ __forceinline__ double2 chunk_sum_c(double2 t) {
    const int l = threadIdx.x & 31;
    const double2 t1 = shfl_c(t, (l + 8) & 31), t2 = shfl_c(t, (l + 16) & 31), t3 = shfl_c(t, (l + 24) & 31);
    const double2 mu = cadd(cadd(cadd(cadd(make_double2(0.0, 0.0), t), t1), t2), t3);   // lanes 0..7
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int b = 0; b < CG_CH; ++b) s = cadd(s, shfl_c(mu, b));
    return s;
}
__device__ __forceinline__ double chunk_sum_r(double t) {
    const int l = threadIdx.x & 31;
    const double t1 = __shfl_sync(0xffffffffu, t, (l + 8) & 31), t2 = __shfl_sync(0xffffffffu, t, (l + 16) & 31),
                 t3 = __shfl_sync(0xffffffffu, t, (l + 24) & 31);
    const double mu = (((0.0 + t) + t1) + t2) + t3;
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < CG_CH; ++b) s = s + __shfl_sync(0xffffffffu, mu, b);
    return s;
}

template <bool CPLX>
__global__ void __launch_bounds__(CG1_NT) k_cg_spmv1(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    if (*Sc.nactive == 0) return;
    const bool act = Sc.active[0] != 0;
    const bool fl = CG_DEFER_X && !act && Sc.flush[0] != 0;
    const c128 sg = S.sigma[g.lane_shift[0]];
    const c128 beta = Sc.beta[0];
    const c128 alpha = Sc.alpha[0];
    c128 *__restrict__ pv = V.p;
    c128 *__restrict__ qv = V.q;
    c128 *__restrict__ xv = V.x;
    const c128 *__restrict__ zv = V.z;
    const int l = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (CG1_NT / 32);
    for (int64_t c = (int64_t)blockIdx.x * (CG1_NT / 32) + (threadIdx.x >> 5); c < g.nchunks; c += wstride) {
        const int64_t i = c * (CG_SB * CG_CH) + l;
        c128 term = cmk(0.0, 0.0);
        if (act && i < M.n) {
            const c128 acc = row_sz<CPLX, true>(M, i, zv, 1u, 0, sg);
            const c128 po = pv[i];
            if (CG_DEFER_X) xv[i] = cadd(xv[i], cmul(alpha, po));
            const c128 pi = cadd(zv[i], cmul(beta, po));
            const c128 qi = cadd(acc, cmul(beta, qv[i]));
            pv[i] = pi;
            qv[i] = qi;
            term = cmul(pi, qi);
        } else if (fl && i < M.n) {
            xv[i] = cadd(xv[i], cmul(alpha, pv[i]));
        }
        const double2 s = chunk_sum_c(term);
        if (l == 0) Sc.part_a[c] = s;
    }
}

__global__ void __launch_bounds__(CG1_NT) k_cg_update1(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    if (*Sc.nactive == 0) return;
    const bool act = Sc.active[0] != 0;
    const c128 sg = S.sigma[g.lane_shift[0]];
    const c128 alpha = Sc.alpha[0];
    const int l = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (CG1_NT / 32);
    for (int64_t c = (int64_t)blockIdx.x * (CG1_NT / 32) + (threadIdx.x >> 5); c < g.nchunks; c += wstride) {
        const int64_t i = c * (CG_SB * CG_CH) + l;
        c128 trho = cmk(0.0, 0.0);
        double trn = 0.0;
        if (act && i < M.n) {
            const c128 q = V.q[i];
            if (!CG_DEFER_X) V.x[i] = cadd(V.x[i], cmul(alpha, V.p[i]));
            const c128 d = form_entry(M.dta[i], M.dta_im[i], M.db[i], sg);
            const c128 z = csub(V.z[i], cmul(alpha, cdiv_c(q, d)));
            V.z[i] = z;
            const c128 r = cmul(d, z);
            trho = cmul(r, z);
            trn = cabs2(r);
        }
        const double2 s = chunk_sum_c(trho);
        const double sr = chunk_sum_r(trn);
        if (l == 0) {
            Sc.part_b[c] = s;
            Sc.part_c[c] = sr;
        }
    }
}

// ---------------------------------------------------------------------------
// update: z -= alpha D^-1 q; partials of rho' = r^T z, |r|^2 with r = D z
// (48 B per live row-shift: z read + written, q read; x += alpha p is deferred
// to the next spmv, see CG_DEFER_X)
// (claims statically strided over CTAs: pointwise, no locality to exploit)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CG_NT) k_cg_update(CgMat M, CgVec V, CgScal Sc, ShiftDev S, CgGeom g) {
    __shared__ double2 sbc[CG_SBP];
    __shared__ double sbr[CG_SBP];
    if (*Sc.nactive == 0) return;
    int lane, slot, slots;
    cta_geom(g, lane, slot, slots);
    const int kp = g.kp;
    const bool act = Sc.active[lane] != 0;
    const c128 sg = S.sigma[g.lane_shift[lane]];
    const c128 alpha = Sc.alpha[lane];
    const c128 *__restrict__ pnew = V.p;
    for (int64_t claim = blockIdx.x; claim < g.nclaims; claim += gridDim.x) {
        for (int ps = 0; ps < g.P; ++ps) {
            const int sbl = ps * slots + slot;
            const int64_t gsb = claim * g.subs + sbl;   // sub-block b of chunk c: rows c*32 + b + 8k
            const int64_t r0 = (gsb / CG_CH) * (CG_SB * CG_CH) + gsb % CG_CH;
            c128 rho = cmk(0.0, 0.0);
            double rn = 0.0;
            if (act) {
                const int64_t r1 = min(r0 + CG_SB * CG_CH, M.n);
#pragma unroll 2
                for (int64_t i = r0; i < r1; i += CG_CH) {
                    const size_t o = (size_t)i * g.ld + lane;
                    const c128 q = V.q[o];
                    if (!CG_DEFER_X) V.x[o] = cadd(V.x[o], cmul(alpha, pnew[o]));
                    // preconditioned residual recurrence z <- z - alpha D^-1 q;
                    // r = D z is formed for the dots only (16 B per row-shift
                    // less than storing r and z)
                    const c128 d = form_entry(M.dta[i], M.dta_im[i], M.db[i], sg);
                    const c128 z = csub(V.z[o], cmul(alpha, cdiv_c(q, d)));
                    V.z[o] = z;
                    const c128 r = cmul(d, z);
                    rho = cadd(rho, cmul(r, z));
                    rn += cabs2(r);
                }
            }
            sbc[sbl * kp + lane] = rho;
            sbr[sbl * kp + lane] = rn;
        }
        __syncthreads();
        chunk_partials<double2>(sbc, g, claim, Sc.part_b, add_c, make_double2(0.0, 0.0));
        chunk_partials<double>(sbr, g, claim, Sc.part_c, add_r, 0.0);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// finish kernels: one thread per (range of CG_RANGE chunks, lane) sums its
// range in chunk order (loads batched, adds in order); the last CTA to arrive
// sums the ranges in order per lane and updates the per-shift scalars.
//   MODE 0 (after init):   rho, |b|^2 -> rho, bnorm2, active
//   MODE 1 (after spmv):   mu -> alpha (breakdown / non-finite -> status)
//   MODE 2 (after update): rho', |r|^2 -> freeze / beta / rho, nactive
// ---------------------------------------------------------------------------

template <bool REAL>
__device__ __forceinline__ void sum_range(const double2 *pa, const double *pc, int64_t c0, int64_t c1, int kp,
                                          int l, double2 &s, double &sr) {
    int64_t c = c0;
    for (; c + 8 <= c1; c += 8) {
        double2 v[8];
        double w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = pa[(size_t)(c + u) * kp + l];
            if (REAL) w[u] = pc[(size_t)(c + u) * kp + l];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = cadd(s, v[u]);
            if (REAL) sr += w[u];
        }
    }
    for (; c < c1; ++c) {
        s = cadd(s, pa[(size_t)c * kp + l]);
        if (REAL) sr += pc[(size_t)c * kp + l];
    }
}

// The tree: level-1 value r = ordered sum of chunk partials [64r, 64r+64),
// level-(k+1) value g = ordered sum of level-k values [64g, 64g+64), until
// one value per lane remains.  Every CTA stages the partials it sums into
// shared memory with coalesced loads and one thread per (value, lane) adds
// them in order (sum_range's order); the last CTA to finish the 64 inputs of
// a group (atomic counter per group and lane group) computes that group's
// value, so the levels run on many CTAs; the CTA holding a lane group's
// final value applies the per-shift scalar updates.
constexpr int CG_GCTR = 4096;
constexpr int CG_FL_NT = 256;
constexpr int CG_FL_MAXV = 2048;   // staged values per CTA

__device__ __forceinline__ bool arrive_count(unsigned int *ctr, unsigned int add, unsigned int total) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ctr, add) + add == total;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// ordered sums of nv groups (of up to CG_RANGE consecutive values each, starting
// at value index v0 of src) for LG lanes starting at l0: dst[(g0+v)*kp + l0 + l]
template <bool REAL>
__device__ __forceinline__ void fl_sum_groups(const double2 *src, const double *srcr, int64_t v0, int64_t nsrc,
                                             int nv, int kp, int l0, int LG, double2 *dst, double *dstr,
                                             int64_t g0, double2 *smv, double *smr) {
    const int64_t vend = min(v0 + (int64_t)nv * CG_RANGE, nsrc);
    const int cnt = (int)(vend - v0);
    for (int e = threadIdx.x; e < cnt * LG; e += CG_FL_NT) {
        const int64_t v = v0 + e / LG;
        const int l = l0 + e % LG;
        smv[e] = __ldcg(src + v * kp + l);
        if (REAL) smr[e] = __ldcg(srcr + v * kp + l);
    }
    __syncthreads();
    if (threadIdx.x < nv * LG) {
        const int gi = threadIdx.x / LG, l = threadIdx.x % LG;
        const int c0 = gi * CG_RANGE, c1 = min(c0 + CG_RANGE, cnt);
        if (c0 < cnt) {
            double2 acc = make_double2(0.0, 0.0);
            double accr = 0.0;
            for (int c = c0; c < c1; ++c) {
                acc = cadd(acc, smv[c * LG + l]);
                if (REAL) accr += smr[c * LG + l];
            }
            dst[(g0 + gi) * kp + l0 + l] = acc;
            if (REAL) dstr[(g0 + gi) * kp + l0 + l] = accr;
        }
    }
    __syncthreads();
}

// per-shift scalar update of lane l from its final reduced value(s)
template <int MODE>
__device__ __forceinline__ void finish_lane(CgScal &Sc, const CgGeom &g, int l, double2 s, double sr, int kreal,
                                            int max_iters) {
    if (MODE == 0) {
        Sc.rho[l] = s;
        Sc.bnorm2[l] = sr;
        Sc.rnorm2[l] = sr;
        Sc.beta[l] = make_double2(0.0, 0.0);
        Sc.alpha[l] = make_double2(0.0, 0.0);
        Sc.flush[l] = 0;
        Sc.iters[l] = 0;
        Sc.status[l] = 0;
        Sc.active[l] = (g.lane_shift[l] < kreal && sr > 0.0) ? 1 : 0;
    } else if (MODE == 1) {
        Sc.flush[l] = 0;   // the spmv just run applied a frozen lane's pending x term
        if (Sc.active[l]) {
            const double ms = cabs2(s);
            if (!(ms > 0.0) || !isfinite(ms)) {
                Sc.status[l] = isfinite(ms) ? 1 : 2;
                Sc.active[l] = 0;
                Sc.alpha[l] = make_double2(0.0, 0.0);
            } else {
                Sc.alpha[l] = cdiv_c(Sc.rho[l], s);
            }
        }
    } else if (Sc.active[l]) {
        Sc.rnorm2[l] = sr;
        Sc.iters[l] += 1;
        const double2 rho_old = Sc.rho[l];
        if (!isfinite(sr) || !isfinite(s.x) || !isfinite(s.y)) {
            Sc.status[l] = 2;
            Sc.active[l] = 0;
        } else if (sr <= Sc.tolsq[l] * Sc.bnorm2[l]) {
            Sc.active[l] = 0;                               // converged: freeze
        } else if (!(cabs2(rho_old) > 0.0)) {
            Sc.status[l] = 1;
            Sc.active[l] = 0;
        } else if (Sc.iters[l] >= max_iters) {
            Sc.status[l] = 3;
            Sc.active[l] = 0;
        } else {
            Sc.beta[l] = cdiv_c(s, rho_old);
            Sc.rho[l] = s;
        }
        if (CG_DEFER_X && !Sc.active[l]) Sc.flush[l] = 1;   // x += alpha p of this iteration is still pending
    }
}

template <int MODE>
__global__ void __launch_bounds__(CG_FL_NT) k_cg_finish(CgScal Sc, CgGeom g, int kreal, int max_iters) {
    extern __shared__ __align__(16) unsigned char fl_smem[];
    if (MODE != 0 && *Sc.nactive == 0) return;
    constexpr bool REAL = MODE != 1;
    double2 *smv = reinterpret_cast<double2 *>(fl_smem);
    double *smr = reinterpret_cast<double *>(smv + CG_FL_MAXV);
    const int kp = g.kp;
    const int LG = kp < 32 ? kp : 32;            // lanes per CTA
    const int nlg = kp / LG;
    const int TR = max(1, CG_FL_NT / (LG * CG_RANGE));   // level-1 values per CTA (divides 64)
    const int lg = blockIdx.x % nlg, rt = blockIdx.x / nlg;
    const int l0 = lg * LG;
    const double2 *pa = MODE == 1 ? Sc.part_a : Sc.part_b;
    const int64_t n1 = (g.nchunks + CG_RANGE - 1) / CG_RANGE;
    // level 1: TR ranges of chunk partials
    const int64_t r0 = (int64_t)rt * TR;
    const int nv = (int)min((int64_t)TR, n1 - r0);
    fl_sum_groups<REAL>(pa, Sc.part_c, r0 * CG_RANGE, g.nchunks, nv, kp, l0, LG, Sc.part_f, Sc.part_g, r0, smv, smr);
    // upper levels: the last arriver of each group of 64 computes its value
    const double2 *src = Sc.part_f;
    const double *srcr = Sc.part_g;
    double2 *dst = Sc.part_f2;
    double *dstr = Sc.part_g2;
    int64_t ncur = n1, grp = r0 / CG_RANGE, coff = 0;
    unsigned int add = (unsigned int)nv;
    while (ncur > 1) {
        const int64_t nnext = (ncur + CG_RANGE - 1) / CG_RANGE;
        const unsigned int total = (unsigned int)min((int64_t)CG_RANGE, ncur - grp * CG_RANGE);
        unsigned int *ctr = Sc.gctr + coff + grp * nlg + lg;
        if (!arrive_count(ctr, add, total)) return;
        if (threadIdx.x == 0) *ctr = 0;
        fl_sum_groups<REAL>(src, srcr, grp * CG_RANGE, ncur, 1, kp, l0, LG, dst, dstr, grp, smv, smr);
        coff += nnext * nlg;
        src = dst;
        srcr = dstr;
        dst += nnext * kp;
        dstr += nnext * kp;
        ncur = nnext;
        grp /= CG_RANGE;
        add = 1;
    }
    // this CTA holds its lane group's final values (src[l]); scalar updates
    for (int ll = threadIdx.x; ll < LG; ll += CG_FL_NT) {
        const int l = l0 + ll;
        finish_lane<MODE>(Sc, g, l, __ldcg(src + l), MODE != 1 ? __ldcg(srcr + l) : 0.0, kreal, max_iters);
    }
    // the last lane group to finish counts the live lanes and resets the claim counter
    if (!arrive_count(Sc.gctr + CG_GCTR - 1, 1u, (unsigned int)nlg)) return;
    if (threadIdx.x < 32) {
        if (MODE != 1) {
            int na = 0;
            for (int l = threadIdx.x; l < kp; l += 32) na += __ldcg(Sc.active + l);
            for (int off = 16; off > 0; off >>= 1) na += __shfl_xor_sync(0xffffffffu, na, off);
            if (threadIdx.x == 0) *Sc.nactive = na;
        }
        if (threadIdx.x == 0) {
            Sc.gctr[CG_GCTR - 1] = 0;
            if (MODE == 1) Sc.ctr[0] = 0;   // spmv claim counter
        }
    }
}

static inline int finish_grid(const CgGeom &g) {
    const int64_t n1 = (g.nchunks + CG_RANGE - 1) / CG_RANGE;
    const int LG = g.kp < 32 ? g.kp : 32;
    const int TR = std::max(1, CG_FL_NT / (LG * CG_RANGE));
    return (int)(((n1 + TR - 1) / TR) * (g.kp / LG));
}

static inline size_t finish_smem(int mode) { return (size_t)CG_FL_MAXV * (sizeof(double2) + (mode != 1 ? 8 : 0)); }

// ---------------------------------------------------------------------------
// compaction: dst[i][l'] = src[i][map[l']] (new width kp_new)
// ---------------------------------------------------------------------------
// (ld_old, ld_new: lanes stored per row before / after)
__global__ void k_cg_repack(const c128 *__restrict__ src, c128 *__restrict__ dst, int64_t n, int ld_old,
                            int ld_new, const int *__restrict__ map) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * ld_new) return;
    const int64_t i = t / ld_new;
    const int l = (int)(t % ld_new);
    dst[t] = src[i * ld_old + map[l]];
}

// x_out[i][lane_shift[l]] = x[i][l] for the lanes in mask
// (a lane with its last x += alpha p pending gets it here, see CG_DEFER_X)
__global__ void k_cg_scatter_x(const c128 *__restrict__ x, const c128 *__restrict__ p,
                               const double2 *__restrict__ alpha, const int *__restrict__ flush,
                               c128 *__restrict__ xout, int64_t n, int ld,
                               int kp_full, const int *__restrict__ lane_shift,
                               const int *__restrict__ mask) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * ld) return;
    const int64_t i = t / ld;
    const int l = (int)(t % ld);
    if (mask[l]) {
        c128 v = x[t];
        if (CG_DEFER_X && flush[l]) v = cadd(v, cmul(alpha[l], p[t]));
        xout[i * kp_full + lane_shift[l]] = v;
    }
}

// scalars of the kept lanes, in place safe (map[l'] >= l')
__global__ void k_cg_repack_scalars(CgScal Sc, int kp_new, const int *__restrict__ map) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int l = 0; l < kp_new; ++l) {
        const int s = map[l];
        Sc.rho[l] = Sc.rho[s];
        Sc.alpha[l] = Sc.alpha[s];
        Sc.beta[l] = Sc.beta[s];
        Sc.rnorm2[l] = Sc.rnorm2[s];
        Sc.bnorm2[l] = Sc.bnorm2[s];
        Sc.active[l] = Sc.active[s];
        Sc.flush[l] = Sc.flush[s];
        Sc.iters[l] = Sc.iters[s];
        Sc.status[l] = Sc.status[s];
        Sc.tolsq[l] = Sc.tolsq[s];
    }
}

// r_j = b - S_j x_j with error-free products, double-double sum, rounded once
// (full width: lane = shift)
__global__ void __launch_bounds__(CG_NT) k_cg_residual(CgMat M, const c128 *__restrict__ bshared,
                                                        const c128 *__restrict__ x, ShiftDev S, int kp,
                                                        c128 *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= M.n * kp) return;
    const int64_t i = t / kp;
    const int j = (int)(t % kp);
    const c128 sg = S.sigma[j];
    const c128 b = bshared[i];
    ddacc re = {b.x, 0.0}, im = {b.y, 0.0};
    for (int32_t q = M.indptr[i]; q < M.indptr[i + 1]; ++q) {
        const c128 e = form_entry(M.ta[q], M.ta_im[q], M.b[q], sg);
        const c128 v = x[(int64_t)M.indices[q] * kp + j];
        dd p;
        p = two_prod(e.x, v.x); ddacc_add(re, -p.hi); re.lo = __dsub_rn(re.lo, p.lo);
        p = two_prod(e.y, v.y); ddacc_add(re, p.hi); re.lo = __dadd_rn(re.lo, p.lo);
        p = two_prod(e.x, v.y); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
        p = two_prod(e.y, v.x); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
    }
    out[t] = cmk(__dadd_rn(re.hi, re.lo), __dadd_rn(im.hi, im.lo));
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

// acc (dd, SoA 4n) = sum_j beta_j (x1_j [+ x2_j]), fixed shift order
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
static inline void hook_begin(CocgState &cg, const char *name, double bytes) {
    if (cg.hook) cg.hook->begin(name, bytes);
}
// REXI_COCG_TRACE: profile names carry the layout width ("cg_spmv@16")
static const char *width_name(const char *base, int kp) {
    static const bool trace = getenv("REXI_COCG_TRACE") != nullptr;
    if (!trace) return base;
    static std::map<std::string, std::string> names;
    std::string key = std::string(base) + "@" + std::to_string(kp);
    auto it = names.find(key);
    if (it == names.end()) it = names.emplace(key, key).first;
    return it->second.c_str();
}
static inline void hook_end(CocgState &cg) {
    if (cg.hook) cg.hook->end();
}

struct CocgImpl {
    bool cplx = false;         // A has an imaginary part
    std::vector<double> wts;   // per shift: mean|beta| / |beta_j| (tolerance weights)
    CgMat M{};
    CgVec V{};
    CgScal Sc{};
    int kp_full = 0;
    int sms = 148;
    c128 *scratch = nullptr;   // repack staging [n][kp_full]
    c128 *xout = nullptr;      // full-width solution [n][kp_full]
    c128 *rhs = nullptr;       // shared rhs [n]
    c128 *xsave = nullptr;     // first-solve x [n][kp_full] (refinement)
    c128 *res = nullptr;       // residual rhs [n][kp_full]
    int *lane_shift = nullptr; // device [kp_full]
    int *map = nullptr;        // device [kp_full]
    int *mask = nullptr;       // device [kp_full]
    int *h_buf = nullptr;      // pinned [2 + 2*kp_full]
    bool stage_ok[3] = {false, false, false};   // [cpc]: every claim's CSR slice fits the staging buffers
    CgWin win[8];              // windowed spmv tables, [log2 kp] for kp = 4 .. 128 (dir == nullptr: not available)
};

static int alloc_(CocgState &cg, void **p, size_t bytes, std::string &err) {
    cudaError_t e = cudaMalloc(p, bytes < 16 ? 16 : bytes);
    if (e == cudaSuccess) e = rexi_poison(*p, bytes < 16 ? 16 : bytes);
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

static CgGeom make_geom(const CocgImpl *im, int kp, int64_t n, int warps = CG_WARPS, int ld = 0) {
    CgGeom g{};
    g.kp = kp;
    g.ld = ld > 0 ? ld : kp;
    g.kw = kp < 32 ? kp : 32;
    g.G = kp / g.kw;
    g.rpw = 32 / g.kw;
    g.slots = (warps / g.G) * g.rpw;                    // sub-blocks per CTA pass
    g.P = g.slots >= CG_CH ? 1 : CG_CH / g.slots;       // passes per claim
    g.subs = g.slots * g.P;                             // sub-blocks per claim (multiple of CG_CH)
    g.cpc = g.subs / CG_CH;                             // chunks per claim
    g.nchunks = (n + CG_SB * CG_CH - 1) / (CG_SB * CG_CH);
    g.nclaims = (g.nchunks + g.cpc - 1) / g.cpc;
    g.lane_shift = im->lane_shift;
    return g;
}

static int grid_for(const CocgImpl *im, const CgGeom &g, int64_t) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(g.nclaims, (int64_t)im->sms * 8));
}

// stage tables of the windowed spmv for layout width KP (see k_cg_spmv_win);
// leaves w.dir == nullptr when some stage's columns do not fit three windows
struct WinHost {                  // host image of one width's tables (built on a worker thread)
    bool ok = false;
    int rl = 0, blob_max = 0, zrows = 0;
    int64_t nstages = 0;
    std::vector<WinStage> dir;
    std::vector<unsigned char> blob;
};

template <int KP, int RL>
static void win_host(const rexi_desc *d, const std::vector<double> &ta, const std::vector<double> &bb, WinHost &out) {
    using G = WinGeom<KP, RL>;
    constexpr int R = G::R;
    out.ok = false;
    const int64_t n = d->n;
    const int64_t nchunks = (n + CG_SB * CG_CH - 1) / (CG_SB * CG_CH);
    const int64_t nstages = G::R >= 32 ? (nchunks + G::CPS - 1) / G::CPS : nchunks * G::NST;
    std::vector<WinStage> &dir = out.dir;
    std::vector<unsigned char> &blob = out.blob;
    dir.assign((size_t)nstages, WinStage{});
    blob.clear();
    blob.reserve((size_t)d->nnz * 19 + (size_t)nstages * 64);
    int blob_max = 0, zrows = 0;
    std::vector<int32_t> cols;
    auto al16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
    for (int64_t gs = 0; gs < nstages; ++gs) {
        WinStage e{};
        const int64_t R0 = gs * R, R1 = std::min<int64_t>(n, R0 + R);
        if (R0 >= n) {
            dir[(size_t)gs] = e;
            continue;
        }
        const int32_t Q0 = d->indptr[R0], Q1 = d->indptr[R1];
        cols.assign(d->indices + Q0, d->indices + Q1);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        std::vector<std::pair<int32_t, int32_t>> runs;   // [first, last]
        for (int32_t c : cols) {
            if (!runs.empty() && c == runs.back().second + 1) runs.back().second = c;
            else runs.push_back({c, c});
        }
        while (runs.size() > (size_t)CG_NWIN) {   // merge the closest pair
            size_t best = 0;
            for (size_t k = 1; k + 1 < runs.size(); ++k)
                if (runs[k + 1].first - runs[k].second < runs[best + 1].first - runs[best].second) best = k;
            runs[best].second = runs[best + 1].second;
            runs.erase(runs.begin() + (long)best + 1);
        }
        int total = 0, own0 = -1;
        for (size_t k = 0; k < runs.size(); ++k) {
            e.wstart[k] = runs[k].first;
            e.wrows[k] = runs[k].second - runs[k].first + 1;
            if (runs[k].first <= R0 && R1 - 1 <= runs[k].second) own0 = total + (int)(R0 - runs[k].first);
            total += e.wrows[k];
        }
        // not window-shaped (the windows alone would overflow the two stages): keep the gather kernels
        if (own0 < 0 || Q1 - Q0 > 65535 || win_smem_bytes<KP, RL>(0, total) > CG_SMEM_MAX) return;
        zrows = std::max(zrows, total);
        e.own0 = own0;
        const int rows = (int)(R1 - R0), nz = Q1 - Q0;
        const size_t b_ip = al16(4 * (size_t)(rows + 1)), b_zs = al16(2 * (size_t)nz), b_v = al16(8 * (size_t)nz);
        e.blob_off = (int64_t)blob.size();
        e.off_zs = (int32_t)b_ip;
        e.off_ta = (int32_t)(b_ip + b_zs);
        e.off_b = (int32_t)(b_ip + b_zs + b_v);
        e.blob_bytes = (int32_t)(b_ip + b_zs + 2 * b_v);
        blob.resize(blob.size() + (size_t)e.blob_bytes, 0);
        unsigned char *bp = blob.data() + e.blob_off;
        int32_t *ipl = reinterpret_cast<int32_t *>(bp);
        for (int r = 0; r <= rows; ++r) ipl[r] = d->indptr[R0 + r] - Q0;
        unsigned short *zs = reinterpret_cast<unsigned short *>(bp + e.off_zs);
        double *pa = reinterpret_cast<double *>(bp + e.off_ta), *pb = reinterpret_cast<double *>(bp + e.off_b);
        for (int32_t q = Q0; q < Q1; ++q) {
            const int32_t c = d->indices[q];
            int base = 0, slot = -1;
            for (size_t k = 0; k < runs.size(); ++k) {
                if (c >= runs[k].first && c <= runs[k].second) {
                    slot = base + (c - runs[k].first);
                    break;
                }
                base += e.wrows[k];
            }
            zs[q - Q0] = (unsigned short)slot;
            pa[q - Q0] = ta[(size_t)q];
            pb[q - Q0] = bb[(size_t)q];
        }
        blob_max = std::max(blob_max, (int)e.blob_bytes);
        dir[(size_t)gs] = e;
    }
    blob_max = (blob_max + 127) & ~127;
    zrows = std::max((zrows + 7) & ~7, CG_SB * CG_CH);   // the dead window area also stages a chunk's terms
    if (win_smem_bytes<KP, RL>(blob_max, zrows) > CG_SMEM_MAX) return;
    out.ok = true;
    out.rl = RL;
    out.blob_max = blob_max;
    out.zrows = zrows;
    out.nstages = nstages;
}

// two row-lanes per thread where the stages' windows and blob fit the shared-memory
// budget, else one (3D-like patterns, and the narrow layouts whose stages are mostly
// matrix)
template <int KP>
static void win_host_any(const rexi_desc *d, const std::vector<double> &ta, const std::vector<double> &bb, WinHost &out) {
    if (KP >= 8) win_host<KP, 2>(d, ta, bb, out);
    if (!out.ok) win_host<KP, 1>(d, ta, bb, out);
}

static int win_upload(CocgState &cg, const WinHost &h, CgWin &w, cudaStream_t st, std::string &err) {
    if (!h.ok) return REXI_OK;
    WinStage *ddir;
    unsigned char *dblob;
    CGA(ddir, sizeof(WinStage) * h.dir.size());
    CGA(dblob, h.blob.size() + 16);
    CGK(cudaMemcpyAsync(ddir, h.dir.data(), sizeof(WinStage) * h.dir.size(), cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(dblob, h.blob.data(), h.blob.size(), cudaMemcpyHostToDevice, st));
    CGK(cudaStreamSynchronize(st));   // the host vectors go out of scope
    w.rl = h.rl;
    w.dir = ddir;
    w.blob = dblob;
    w.blob_max = h.blob_max;
    w.zrows = h.zrows;
    w.nstages = h.nstages;
    return REXI_OK;
}

// Dynamic shared-memory limits of the big-shared-memory kernels.  Function
// attributes are per device, so this runs at every plan creation on the plan's
// device (a process-wide "done" flag would leave the other GPUs of an
// in-process multi-GPU stepper without them).
static cudaError_t cocg_set_smem_attrs() {
    cudaError_t e = cudaSuccess;
#define REXI_ATTR(fn, bytes)                                                                          \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes))
    REXI_ATTR(k_cg_spmv_st<true>, st_smem_bytes(true));
    REXI_ATTR(k_cg_spmv_st<false>, st_smem_bytes(false));
#if CG_DEFER_X
    REXI_ATTR(k_cg_spmv_tma, tma_smem_bytes());
    REXI_ATTR(k_cg_update_tma<1>, upd_smem_bytes<1>());
    REXI_ATTR(k_cg_update_tma<2>, upd_smem_bytes<2>());
    REXI_ATTR(k_cg_update_tma<4>, upd_smem_bytes<4>());
    REXI_ATTR(k_cg_update_tma<8>, upd_smem_bytes<8>());
    REXI_ATTR(k_cg_update_tma<16>, upd_smem_bytes<16>());
    REXI_ATTR(k_cg_update_tma<32>, upd_smem_bytes<32>());
    REXI_ATTR(k_cg_update_tma<64>, upd_smem_bytes<64>());
    REXI_ATTR(k_cg_update_tma<128>, upd_smem_bytes<128>());
    // the windowed spmv's need depends on the plan's tables: allow the per-block maximum
    auto w1 = k_cg_spmv_win<1, 1>;   auto w2 = k_cg_spmv_win<2, 1>;   auto w4 = k_cg_spmv_win<4, 1>;
    auto w8a = k_cg_spmv_win<8, 2>;  auto w8b = k_cg_spmv_win<8, 1>;  auto w16a = k_cg_spmv_win<16, 2>;
    auto w16b = k_cg_spmv_win<16, 1>; auto w32a = k_cg_spmv_win<32, 2>; auto w32b = k_cg_spmv_win<32, 1>;
    auto w64a = k_cg_spmv_win<64, 2>; auto w64b = k_cg_spmv_win<64, 1>; auto w128a = k_cg_spmv_win<128, 2>;
    auto w128b = k_cg_spmv_win<128, 1>;
    REXI_ATTR(w1, CG_SMEM_MAX);   REXI_ATTR(w2, CG_SMEM_MAX);   REXI_ATTR(w4, CG_SMEM_MAX);
    REXI_ATTR(w8a, CG_SMEM_MAX);  REXI_ATTR(w8b, CG_SMEM_MAX);  REXI_ATTR(w16a, CG_SMEM_MAX);
    REXI_ATTR(w16b, CG_SMEM_MAX); REXI_ATTR(w32a, CG_SMEM_MAX); REXI_ATTR(w32b, CG_SMEM_MAX);
    REXI_ATTR(w64a, CG_SMEM_MAX); REXI_ATTR(w64b, CG_SMEM_MAX); REXI_ATTR(w128a, CG_SMEM_MAX);
    REXI_ATTR(w128b, CG_SMEM_MAX);
#endif
#undef REXI_ATTR
    return e;
}

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
    cg.gid.resize(d->k);
    for (int j = 0; j < d->k; ++j) cg.gid[j] = d->shift_ids ? d->shift_ids[j] : d->shift_offset + j;
    cg.shift_iters.assign(d->k, 0);
    for (auto &e : cg.ev) CGK(cudaEventCreate(&e));
    const int64_t n = d->n, nnz = d->nnz;
    const int kp = S.kp;
    im->kp_full = kp;
    {
        double mean = 0.0;
        for (int j = 0; j < d->k; ++j) mean += std::hypot(d->weights[j].re, d->weights[j].im);
        mean /= std::max(1, d->k);
        if (d->weight_ref > 0.0) mean = d->weight_ref;   // global reference (sharded runs)
        im->wts.assign(kp, 1.0);
        for (int j = 0; j < d->k; ++j) {
            const double b = std::hypot(d->weights[j].re, d->weights[j].im);
            im->wts[j] = b > 0.0 ? mean / b : 1e30;
        }
        if (const char *e = getenv("REXI_COCG_WEIGHTED"))
            if (atoi(e) == 0) std::fill(im->wts.begin(), im->wts.end(), 1.0);
    }
    std::vector<double> ta(nnz), tai(nnz), bb(nnz), dta(n, 0.0), dtai(n, 0.0), db(n, 0.0);
    std::vector<char> hasdiag(n, 0);
    for (int64_t r = 0; r < n; ++r)
        for (int32_t q = d->indptr[r]; q < d->indptr[r + 1]; ++q) {
            ta[q] = d->tau * d->a_vals[q];
            tai[q] = d->a_imag ? d->tau * d->a_imag[q] : 0.0;
            if (tai[q] != 0.0) im->cplx = true;
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
    // +32 B of zeroed padding: the staged spmv bulk-copies 16-B aligned supersets
    CGA(ip, sizeof(int32_t) * (n + 1) + 32);
    CGA(ix, sizeof(int32_t) * nnz + 32);
    CGA(ta_, sizeof(double) * nnz + 32);
    CGA(tai_, sizeof(double) * nnz + 32);
    CGA(bb_, sizeof(double) * nnz + 32);
    CGK(cudaMemsetAsync(ip, 0, sizeof(int32_t) * (n + 1) + 32, st));
    CGK(cudaMemsetAsync(ix, 0, sizeof(int32_t) * nnz + 32, st));
    CGK(cudaMemsetAsync(ta_, 0, sizeof(double) * nnz + 32, st));
    CGK(cudaMemsetAsync(tai_, 0, sizeof(double) * nnz + 32, st));
    CGK(cudaMemsetAsync(bb_, 0, sizeof(double) * nnz + 32, st));
    for (int cpc = 1; cpc <= 2; ++cpc) {
        const int64_t rows = (int64_t)cpc * CG_SB * CG_CH;
        bool ok = !getenv("REXI_COCG_NOSTAGE");
        for (int64_t r0 = 0; ok && r0 < n; r0 += rows) {
            const int64_t r1 = std::min<int64_t>(r0 + rows, n);
            const int64_t q0 = d->indptr[r0], q1 = d->indptr[r1];
            if (((q1 + 3) & ~3ll) - (q0 & ~3ll) > CG_ST_NNZ) ok = false;
        }
        im->stage_ok[cpc] = ok;
    }
    CGA(dta_, sizeof(double) * n + 16);   // + padding: the TMA update rounds odd row counts up
    CGA(dtai_, sizeof(double) * n + 16);
    CGA(db_, sizeof(double) * n + 16);
    CGK(cudaMemsetAsync(dta_, 0, sizeof(double) * n + 16, st));
    CGK(cudaMemsetAsync(db_, 0, sizeof(double) * n + 16, st));
    CGK(cudaMemcpyAsync(ip, d->indptr, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(ix, d->indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(ta_, ta.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(tai_, tai.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(bb_, bb.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(dta_, dta.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(dtai_, dtai.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CGK(cudaMemcpyAsync(db_, db.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    im->M = CgMat{n, ip, ix, ta_, tai_, bb_, dta_, dtai_, db_, nullptr, nullptr};
    {
        // stencil classes for the narrow-layout spmv (see CgClass)
        std::vector<uint8_t> cls((size_t)n, 255);
        std::vector<CgClass> classes;
        int64_t classed = 0;
        if (!getenv("REXI_COCG_NOCLS")) {
            std::unordered_map<std::string, int> ids;
            int prev = -1;
            std::string key;
            auto matches = [&](int id, int64_t r, int32_t q0, int nz) {
                const CgClass &C = classes[id];
                if (C.nnz != nz) return false;
                for (int k = 0; k < nz; ++k)
                    if ((int64_t)d->indices[q0 + k] - r != C.off[k] || memcmp(&bb[q0 + k], &C.b[k], sizeof(double)))
                        return false;
                return true;
            };
            for (int64_t r = 0; r < n; ++r) {
                const int32_t q0 = d->indptr[r], q1 = d->indptr[r + 1];
                const int nz = q1 - q0;
                if (nz <= 0 || nz > CG_CLS_MAXNNZ) continue;
                if (prev >= 0 && matches(prev, r, q0, nz)) {
                    cls[r] = (uint8_t)prev;
                    ++classed;
                    continue;
                }
                key.assign(reinterpret_cast<const char *>(&nz), sizeof nz);
                for (int k = 0; k < nz; ++k) {
                    const int32_t off = (int32_t)((int64_t)d->indices[q0 + k] - r);
                    key.append(reinterpret_cast<const char *>(&off), sizeof off);
                    key.append(reinterpret_cast<const char *>(&bb[q0 + k]), sizeof(double));
                }
                auto it = ids.find(key);
                int id;
                if (it != ids.end()) {
                    id = it->second;
                } else if ((int)classes.size() < CG_CLS_MAX) {
                    CgClass C{};
                    C.nnz = nz;
                    for (int k = 0; k < nz; ++k) {
                        C.off[k] = (int32_t)((int64_t)d->indices[q0 + k] - r);
                        C.b[k] = bb[q0 + k];
                    }
                    id = (int)classes.size();
                    classes.push_back(C);
                    ids.emplace(key, id);
                } else {
                    prev = -1;
                    continue;
                }
                cls[r] = (uint8_t)id;
                prev = id;
                ++classed;
            }
        }
        if (classed * 2 >= n) {   // worth a table: most rows share few stencils
            uint8_t *cls_;
            CgClass *cl_;
            CGA(cls_, (size_t)n);
            CGA(cl_, sizeof(CgClass) * classes.size());
            CGK(cudaMemcpyAsync(cls_, cls.data(), (size_t)n, cudaMemcpyHostToDevice, st));
            CGK(cudaMemcpyAsync(cl_, classes.data(), sizeof(CgClass) * classes.size(), cudaMemcpyHostToDevice, st));
            im->M.cls = cls_;
            im->M.classes = cl_;
        }
    }
#if CG_DEFER_X
    if (!im->cplx && !getenv("REXI_COCG_NOWIN")) {
        // windowed all-TMA spmv for the wide layouts: two row-lanes per thread where the
        // stages' columns fit the window budget (2D-like patterns), else one (3D-like,
        // kp >= 64 only), else the gather kernels stay
        // one host thread per width (the builds are independent passes over the pattern).
        // One lane: the thread-per-row kernel over stencil classes streams 8 B per entry
        // against the blob's 18 and measured faster (54 vs 59 us at 1M rows): table on request.
        WinHost wh[8];
        std::vector<std::thread> th;
        const bool want1 = getenv("REXI_COCG_WINMIN") && atoi(getenv("REXI_COCG_WINMIN")) <= 1;
        if (want1) th.emplace_back([&] { win_host_any<1>(d, ta, bb, wh[0]); });
        if (kp >= 2) th.emplace_back([&] { win_host_any<2>(d, ta, bb, wh[1]); });
        if (kp >= 4) th.emplace_back([&] { win_host_any<4>(d, ta, bb, wh[2]); });
        if (kp >= 8) th.emplace_back([&] { win_host_any<8>(d, ta, bb, wh[3]); });
        if (kp >= 16) th.emplace_back([&] { win_host_any<16>(d, ta, bb, wh[4]); });
        if (kp >= 32) th.emplace_back([&] { win_host_any<32>(d, ta, bb, wh[5]); });
        if (kp >= 64) th.emplace_back([&] { win_host_any<64>(d, ta, bb, wh[6]); });
        if (kp >= 128) th.emplace_back([&] { win_host_any<128>(d, ta, bb, wh[7]); });
        for (auto &t : th) t.join();
        int rc = REXI_OK;
        for (int w = 0; w < 8 && !rc; ++w) rc = win_upload(cg, wh[w], im->win[w], st, err);
        if (rc) return rc;
        if (getenv("REXI_COCG_REQUIRE_WIN")) {   // tests: fail instead of silently keeping the gather kernels
            int lg = 0;
            while ((1 << lg) < kp) ++lg;
            if (kp > 128 || !im->win[lg].dir) {
                err = "REXI_COCG_REQUIRE_WIN: no window tables for the " + std::to_string(kp) + "-lane layout";
                return REXI_ERR_UNSUPPORTED;
            }
        }
    }
#endif
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&im->sms, cudaDevAttrMultiProcessorCount, dev);
    CGK(cocg_set_smem_attrs());
    if ((double)n * kp >= 2147483647.0) {
        err = "COCG plan too large for 32-bit element offsets (n * k_pad >= 2^31); split the shifts";
        return REXI_ERR_UNSUPPORTED;
    }
    const size_t vb = sizeof(c128) * (size_t)n * kp;
    CGA(im->V.x, vb);
    CGA(im->V.z, vb);
    CGA(im->V.p, vb);
    CGA(im->V.q, vb);
    CGA(im->scratch, vb);
    CGA(im->xout, vb);
    CGA(im->rhs, sizeof(c128) * n);
    if (refine > 0) {
        CGA(im->xsave, vb);
        CGA(im->res, vb);
    }
    CGA(im->lane_shift, sizeof(int) * kp);
    CGA(im->map, sizeof(int) * kp);
    CGA(im->mask, sizeof(int) * kp);
    CgScal &Sc = im->Sc;
    CGA(Sc.rho, sizeof(double2) * kp);
    CGA(Sc.alpha, sizeof(double2) * kp);
    CGA(Sc.beta, sizeof(double2) * kp);
    CGA(Sc.rnorm2, sizeof(double) * kp);
    CGA(Sc.bnorm2, sizeof(double) * kp);
    CGA(Sc.active, sizeof(int) * kp);
    CGA(Sc.iters, sizeof(int) * kp);
    CGA(Sc.status, sizeof(int) * kp);
    CGA(Sc.flush, sizeof(int) * kp);
    CGA(Sc.nactive, sizeof(int));
    int64_t part_max = 1;                     // largest nchunks*kp over the layouts compaction can reach
    for (int w = 1; w <= kp; w *= 2) part_max = std::max<int64_t>(part_max, make_geom(im, w, n).nchunks * w);
    CGA(Sc.part_a, sizeof(double2) * (size_t)part_max);
    CGA(Sc.part_b, sizeof(double2) * (size_t)part_max);
    CGA(Sc.part_c, sizeof(double) * (size_t)part_max);
    const int64_t nranges_max = (make_geom(im, kp, n).nchunks + CG_RANGE - 1) / CG_RANGE;
    CGA(Sc.part_f, sizeof(double2) * (size_t)kp * nranges_max);
    CGA(Sc.part_g, sizeof(double) * (size_t)kp * nranges_max);
    CGA(Sc.part_f2, sizeof(double2) * (size_t)kp * nranges_max);
    CGA(Sc.part_g2, sizeof(double) * (size_t)kp * nranges_max);
    CGA(Sc.ctr, sizeof(unsigned int) * 8);
    CGK(cudaMemsetAsync(Sc.ctr, 0, sizeof(unsigned int) * 8, st));
    CGA(Sc.gctr, sizeof(unsigned int) * CG_GCTR);
    CGK(cudaMemsetAsync(Sc.gctr, 0, sizeof(unsigned int) * CG_GCTR, st));
    for (int mode = 0; mode < 3; ++mode) {
        cudaError_t fe = mode == 0 ? cudaFuncSetAttribute(k_cg_finish<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)finish_smem(0))
                       : mode == 1 ? cudaFuncSetAttribute(k_cg_finish<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)finish_smem(1))
                                   : cudaFuncSetAttribute(k_cg_finish<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)finish_smem(2));
        CGK(fe);
    }
    CGA(Sc.tolsq, sizeof(double) * kp);
    CGK(cudaMallocHost((void **)&im->h_buf, sizeof(int) * (2 + 2 * kp)));
    CGK(cudaStreamSynchronize(st));
    return REXI_OK;
}

// repack the live lanes into a layout of width kp_new (host decides the map)
static int cg_repack(CocgImpl *im, int kp_old, int ld_old, int kp_new, int ld_new, const std::vector<int> &map,
                     const std::vector<int> &drop_mask, std::vector<int> &lane_shift,
                     cudaStream_t st, std::string &err) {
    const int64_t n = im->M.n;
    // 1) frozen lanes being dropped: x -> full-width solution
    CGK(cudaMemcpyAsync(im->mask, drop_mask.data(), sizeof(int) * kp_old, cudaMemcpyHostToDevice, st));
    const int64_t t_old = n * ld_old;
    k_cg_scatter_x<<<(unsigned)((t_old + 255) / 256), 256, 0, st>>>(im->V.x, im->V.p, im->Sc.alpha, im->Sc.flush,
                                                                   im->xout, n, ld_old, im->kp_full,
                                                                   im->lane_shift, im->mask);
    // 2) live vectors x, r, z, p(current) -> new width, through the scratch array
    CGK(cudaMemcpyAsync(im->map, map.data(), sizeof(int) * kp_new, cudaMemcpyHostToDevice, st));
    const int64_t t_new = n * ld_new;
    c128 **vecs[4] = {&im->V.x, &im->V.z, &im->V.p, &im->V.q};
    for (c128 **v : vecs) {
        k_cg_repack<<<(unsigned)((t_new + 255) / 256), 256, 0, st>>>(*v, im->scratch, n, ld_old, ld_new, im->map);
        std::swap(*v, im->scratch);
    }
    k_cg_repack_scalars<<<1, 32, 0, st>>>(im->Sc, kp_new, im->map);
    std::vector<int> ls(kp_new);
    for (int l = 0; l < kp_new; ++l) ls[l] = lane_shift[map[l]];
    lane_shift = ls;
    CGK(cudaMemcpyAsync(im->lane_shift, lane_shift.data(), sizeof(int) * kp_new, cudaMemcpyHostToDevice, st));
    CGK(cudaGetLastError());
    return REXI_OK;
}

// solve S_j x_j = b for all shifts (b shared or per shift); result in im->xout
static int cg_solve(CocgState &cg, CocgImpl *im, const ShiftDev &S, cudaStream_t st, int64_t *launches,
                    std::string &err, double tol, double cap) {
    const int64_t n = cg.n;
    int kp = im->kp_full;
    std::vector<int> lane_shift(kp), valid(kp);
    for (int l = 0; l < kp; ++l) {
        lane_shift[l] = l;
        valid[l] = l < cg.k;
    }
    CGK(cudaMemcpyAsync(im->lane_shift, lane_shift.data(), sizeof(int) * kp, cudaMemcpyHostToDevice, st));
    {
        // weighted per-shift targets: shift j's error enters u1 scaled by |beta_j|,
        // so tol_j = min(cap, tol * mean|beta| / |beta_j|) keeps sum_j |beta_j| e_j
        // at the uniform-tol budget while small-weight shifts stop early
        std::vector<double> tsq(kp);
        for (int l = 0; l < kp; ++l) {
            const double t = std::min(cap, tol * im->wts[l]);
            tsq[l] = t * t;
        }
        CGK(cudaMemcpyAsync(im->Sc.tolsq, tsq.data(), sizeof(double) * kp, cudaMemcpyHostToDevice, st));
    }
    int ld = kp;   // lanes stored per row
    CgGeom g = make_geom(im, kp, n);
    int grid = grid_for(im, g, n);
    const double nnzb = 28.0 * (double)cg.nnz + 4.0 * (double)(n + 1);   // CSR pattern + 3 value arrays
    hook_begin(cg, "cg_init", 80.0 * n * kp);
    k_cg_init<<<grid, CG_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
    k_cg_finish<0><<<finish_grid(g), CG_FL_NT, finish_smem(0), st>>>(im->Sc, g, cg.k, cg.max_iters);
    hook_end(cg);
    CGK(cudaGetLastError());
    *launches += 2;
    int live = cg.k;
    int packed_live = std::min(cg.k, kp);   // live lanes at the last (re)pack
    std::vector<int> h_it(kp);
    int it = 0;
    const int check_every = 8;
    // failed lane l (current layout) -> error naming its shift
    auto lane_failure = [&](int l, int status) -> int {
        int iters = 0;
        cudaMemcpy(&iters, im->Sc.iters + l, sizeof(int), cudaMemcpyDeviceToHost);
        char buf[256];
        const char *why = status == 1 ? "COCG breakdown (rho or p^T S p vanished)"
                        : status == 2 ? "non-finite values in COCG"
                                      : "COCG did not converge within max_iters";
        const int ls = lane_shift[l];
        snprintf(buf, sizeof buf, "%s for shift j = %d after %d iterations", why,
                 ls < cg.k ? cg.gid[ls] : cg.shift_offset + ls, iters);
        err = buf;
        return status == 3 ? REXI_ERR_NOCONV : REXI_ERR_BREAKDOWN;
    };
    // REXI_COCG_TRACE=1: iterations and host time spent at each layout width
    static const bool trace = getenv("REXI_COCG_TRACE") != nullptr;
    auto tr_t0 = std::chrono::steady_clock::now();
    int tr_it0 = 0;
    auto trace_phase = [&](int width, int live_now) {
        if (!trace) return;
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[cocg] width %3d  iters %5d..%5d  live at end %3d  %.3f ms\n", width, tr_it0, it,
                live_now, std::chrono::duration<double, std::milli>(t1 - tr_t0).count());
        tr_t0 = t1;
        tr_it0 = it;
    };
    static const bool batch_all = getenv("REXI_COCG_BATCH") != nullptr;   // A/B switch
    for (;;) {
        for (int s = 0; s < check_every; ++s) {
            hook_begin(cg, width_name("cg_spmv", kp), (CG_DEFER_X ? 112.0 : 80.0) * n * live + nnzb);
#if CG_DEFER_X
            static const bool no_tma = getenv("REXI_COCG_NOTMA") != nullptr;   // A/B switch
            static const int win_min = getenv("REXI_COCG_WINMIN") ? atoi(getenv("REXI_COCG_WINMIN")) : 2;
            int lg = 0;
            while ((1 << lg) < kp) ++lg;
            const CgWin *wn = kp >= win_min && kp <= 128 ? &im->win[lg] : nullptr;
            if (!no_tma && wn && wn->dir) {
                // layouts whose stages fit the z-window budget: every operand by bulk copy
                const CgGeom gw = make_geom(im, kp, n, CG_WARPS, ld);
                const int gg = (int)std::max<int64_t>(1, std::min<int64_t>(wn->nstages, (int64_t)im->sms));
#define REXI_WIN_LAUNCH(KPV, RLV)                                                                          \
    {                                                                                                      \
        const int sm_ = (int)win_smem_bytes<KPV, RLV>(wn->blob_max, wn->zrows);                            \
        k_cg_spmv_win<KPV, RLV><<<gg, CGT_NT, sm_, st>>>(im->M, im->V, im->Sc, S, gw, *wn);                \
    }
                if (kp == 1) REXI_WIN_LAUNCH(1, 1)
                else if (kp == 2) REXI_WIN_LAUNCH(2, 1)
                else if (kp == 4) REXI_WIN_LAUNCH(4, 1)
                else if (kp == 8 && wn->rl == 2) REXI_WIN_LAUNCH(8, 2)
                else if (kp == 8) REXI_WIN_LAUNCH(8, 1)
                else if (kp == 16 && wn->rl == 2) REXI_WIN_LAUNCH(16, 2)
                else if (kp == 16) REXI_WIN_LAUNCH(16, 1)
                else if (kp == 32 && wn->rl == 2) REXI_WIN_LAUNCH(32, 2)
                else if (kp == 32) REXI_WIN_LAUNCH(32, 1)
                else if (kp == 64 && wn->rl == 2) REXI_WIN_LAUNCH(64, 2)
                else if (kp == 64) REXI_WIN_LAUNCH(64, 1)
                else if (wn->rl == 2) REXI_WIN_LAUNCH(128, 2)
                else REXI_WIN_LAUNCH(128, 1)
#undef REXI_WIN_LAUNCH
            } else if (!no_tma && !im->cplx && (kp == 32 || kp == 64) && im->stage_ok[kp / 32 == 2 ? 1 : 2] &&
                cg.nnz <= (int64_t)CG_GB * n) {
                // widest layouts, short rows (2D stencils): persistent TMA-pipelined spmv,
                // one CTA per SM (cfg 3 steps 2-4 -3.6 % with the live-prefix row stride;
                // 15-entry 3D rows keep the staged kernel, whose larger L1 serves their
                // gathers: cfg 5 +5 % with this one; scripts/tune_tma.sh, tune_ld.sh)
                const CgGeom gt = make_geom(im, kp, n, CGT_CW, ld);
                const int gg = (int)std::max<int64_t>(1, std::min<int64_t>(gt.nclaims, (int64_t)im->sms));
                k_cg_spmv_tma<<<gg, CGT_NT, tma_smem_bytes(), st>>>(im->M, im->V, im->Sc, S, gt);
            } else
#endif
            if (g.cpc <= 2 && im->stage_ok[g.cpc]) {
                const size_t sm = st_smem_bytes(im->cplx);
                if (im->cplx) k_cg_spmv_st<true><<<grid, CG_NT, sm, st>>>(im->M, im->V, im->Sc, S, g);
                else k_cg_spmv_st<false><<<grid, CG_NT, sm, st>>>(im->M, im->V, im->Sc, S, g);
            } else if (g.kp == 1 && cg.nnz <= (int64_t)CG_GB * n) {
                // one lane, rows within one gather batch (2D stencils): a thread per row
                // (78 -> 71 us at 1M rows).  Longer rows (3D) keep the 4-rows-per-thread
                // batched kernel, measured faster there (209 vs 224 us at 2M rows).
                const int g1 = (int)std::min<int64_t>((g.nchunks + 7) / 8, (int64_t)im->sms * 16);
                if (im->cplx) k_cg_spmv1<true><<<g1, CG1_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
                else k_cg_spmv1<false><<<g1, CG1_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
            } else if (g.kp == 1 || batch_all) {   // batched gathers (measured faster only at one lane)
                if (im->cplx) k_cg_spmv<true, true><<<grid, CG_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
                else k_cg_spmv<false, true><<<grid, CG_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
            } else {
                if (im->cplx) k_cg_spmv<true, false><<<grid, CG_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
                else k_cg_spmv<false, false><<<grid, CG_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
            }
            k_cg_finish<1><<<finish_grid(g), CG_FL_NT, finish_smem(1), st>>>(im->Sc, g, cg.k, cg.max_iters);
            hook_end(cg);
            hook_begin(cg, width_name("cg_update", kp), (CG_DEFER_X ? 48.0 : 96.0) * n * live + 24.0 * n);
#if CG_DEFER_X
            static const bool no_utma = getenv("REXI_COCG_NOUTMA") != nullptr;   // A/B switch
            static const int utma_min = getenv("REXI_COCG_UTMAMIN") ? atoi(getenv("REXI_COCG_UTMAMIN")) : 2;   // one lane: k_cg_update1 measured faster (33.6 vs 36.2 us)
            if (!no_utma && !no_tma && !im->cplx && kp >= utma_min && kp <= 128) {
#define REXI_UPD_LAUNCH(KPV)                                                                              \
    {                                                                                                     \
        const int64_t nu = (n + UpdGeom<KPV>::UNIT - 1) / UpdGeom<KPV>::UNIT;                             \
        const int gg = (int)std::max<int64_t>(1, std::min<int64_t>(nu, (int64_t)im->sms));                \
        k_cg_update_tma<KPV><<<gg, CGT_NT, upd_smem_bytes<KPV>(), st>>>(im->M, im->V, im->Sc, S, g);       \
    }
                switch (kp) {
                    case 1: REXI_UPD_LAUNCH(1) break;
                    case 2: REXI_UPD_LAUNCH(2) break;
                    case 4: REXI_UPD_LAUNCH(4) break;
                    case 8: REXI_UPD_LAUNCH(8) break;
                    case 16: REXI_UPD_LAUNCH(16) break;
                    case 32: REXI_UPD_LAUNCH(32) break;
                    case 64: REXI_UPD_LAUNCH(64) break;
                    default: REXI_UPD_LAUNCH(128) break;
                }
#undef REXI_UPD_LAUNCH
            } else
#endif
            if (g.kp == 1) {
                const int g1 = (int)std::min<int64_t>((g.nchunks + 7) / 8, (int64_t)im->sms * 16);
                k_cg_update1<<<g1, CG1_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
            } else {
                k_cg_update<<<grid, CG_NT, 0, st>>>(im->M, im->V, im->Sc, S, g);
            }
            k_cg_finish<2><<<finish_grid(g), CG_FL_NT, finish_smem(2), st>>>(im->Sc, g, cg.k, cg.max_iters);
            hook_end(cg);
            *launches += 4;
            ++it;
        }
        CGK(cudaGetLastError());
        int *h_na = im->h_buf, *h_act = im->h_buf + 2, *h_st = im->h_buf + 2 + im->kp_full;
        CGK(cudaMemcpyAsync(h_na, im->Sc.nactive, sizeof(int), cudaMemcpyDeviceToHost, st));
        CGK(cudaMemcpyAsync(h_act, im->Sc.active, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
        CGK(cudaStreamSynchronize(st));
        const int na = *h_na;
        live = na;
        if (trace && getenv("REXI_COCG_TRACE_LIVE")) fprintf(stderr, "[cocg]   it %5d  width %3d  live %3d\n", it, kp, na);
        if (na == 0 || it > cg.max_iters + check_every) {
            trace_phase(kp, na);
            break;
        }
        // compaction: halve the layout while the live lanes fit; otherwise, once
        // kp/8 more lanes have frozen inside the layout, repack the live lanes
        // into a prefix of the same width.  A frozen lane costs bandwidth while
        // it sits between live ones (2 lanes per 32-B sector, 32 per warp
        // segment) and none as trailing padding: the wide phases run at ~80 %
        // live lanes.  Repacking moves 128 B per live row-shift, about 0.7 of an
        // iteration.  Per-lane results are unchanged (layout-independent
        // reduction tree).
        int kp_new = kp;
        while (kp_new > 1 && na <= kp_new / 2) kp_new /= 2;
        bool prefix = false;
        static const bool no_prefix = getenv("REXI_COCG_NOPREFIX") != nullptr;   // A/B switch
        static const int repack_div = getenv("REXI_COCG_REPACK_DIV") ? std::max(1, atoi(getenv("REXI_COCG_REPACK_DIV"))) : 8;
        static const int repack_min = getenv("REXI_COCG_REPACK_MINKP") ? atoi(getenv("REXI_COCG_REPACK_MINKP")) : 16;
        if (!no_prefix && kp_new == kp && kp >= repack_min && packed_live - na >= std::max(1, kp / repack_div))
            for (int l = na; l < kp && !prefix; ++l) prefix = h_act[l] != 0;
        if (kp_new < kp || prefix) {
            if (kp_new < kp) trace_phase(kp, na);
            // a frozen lane leaving the layout takes its status with it: report
            // a failed one now
            CGK(cudaMemcpyAsync(h_st, im->Sc.status, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
            CGK(cudaMemcpyAsync(h_it.data(), im->Sc.iters, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
            CGK(cudaStreamSynchronize(st));
            for (int l = 0; l < kp; ++l)
                if (valid[l] && !h_act[l] && h_st[l]) return lane_failure(l, h_st[l]);
            for (int l = 0; l < kp; ++l)
                if (valid[l] && !h_act[l] && lane_shift[l] < cg.k) cg.shift_iters[lane_shift[l]] += h_it[l];
            packed_live = na;
            // live lanes keep ascending shift order; frozen valid lanes hand their
            // x to the full-width solution; padding lanes (a copy of lane map[0],
            // inactive, invalid) fill the new width
            std::vector<int> map, drop(kp, 0);
            for (int l = 0; l < kp; ++l) {
                if (h_act[l]) map.push_back(l);
                else if (valid[l]) drop[l] = 1;
            }
            const int live = (int)map.size();
            for (int l = live; l < kp_new; ++l) map.push_back(map[0]);
            // rows keep only the live prefix (rounded up to 32-B sectors): what the
            // kernels stream -- the TMA kernels move whole rows -- follows the live
            // lanes.  scripts/tune_repack.sh: 2 lanes against 8 (whole 128-B lines)
            // cfg 3 -1.2 %, cfg 5 -2 %; repacking twice as often no further gain
            static const bool no_ld = getenv("REXI_COCG_NOLD") != nullptr;   // A/B switch
            static const int ld_gran = getenv("REXI_COCG_LDGRAN") ? std::max(1, atoi(getenv("REXI_COCG_LDGRAN"))) : 2;
            const int gran = kp_new >= 16 ? ld_gran : std::min(2, ld_gran);
            const int ld_new = no_ld ? kp_new : std::min(kp_new, (live + gran - 1) / gran * gran);
            int rc = cg_repack(im, kp, ld, kp_new, ld_new, map, drop, lane_shift, st, err);
            if (rc) return rc;
            std::vector<int> act(kp_new, 1);
            valid.assign(kp_new, 1);
            for (int l = live; l < kp_new; ++l) act[l] = valid[l] = 0;
            CGK(cudaMemcpyAsync(im->Sc.active, act.data(), sizeof(int) * kp_new, cudaMemcpyHostToDevice, st));
            kp = kp_new;
            ld = ld_new;
            g = make_geom(im, kp, n, CG_WARPS, ld);
            grid = grid_for(im, g, n);
        }
    }
    // statistics / failures (per current lane -> shift)
    std::vector<int> status(kp);
    CGK(cudaMemcpyAsync(status.data(), im->Sc.status, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
    CGK(cudaMemcpyAsync(h_it.data(), im->Sc.iters, sizeof(int) * kp, cudaMemcpyDeviceToHost, st));
    // remaining valid lanes' x -> full-width solution
    CGK(cudaMemcpyAsync(im->mask, valid.data(), sizeof(int) * kp, cudaMemcpyHostToDevice, st));
    k_cg_scatter_x<<<(unsigned)((n * ld + 255) / 256), 256, 0, st>>>(im->V.x, im->V.p, im->Sc.alpha, im->Sc.flush,
                                                                    im->xout, n, ld, im->kp_full,
                                                                    im->lane_shift, im->mask);
    CGK(cudaGetLastError());
    CGK(cudaStreamSynchronize(st));
    for (int l = 0; l < kp; ++l)
        if (valid[l] && lane_shift[l] < cg.k && status[l]) return lane_failure(l, status[l]);
    for (int l = 0; l < kp; ++l)
        if (valid[l] && lane_shift[l] < cg.k) cg.shift_iters[lane_shift[l]] += h_it[l];
    return REXI_OK;
}

// all shifts, x_j = S_j^{-1} rhs (refined): result x1 (+ x2)
static int cg_solve_refined(CocgState &cg, CocgImpl *im, const ShiftDev &S, cudaStream_t st,
                            int64_t *launches, std::string &err, const c128 **x1, const c128 **x2) {
    std::fill(cg.shift_iters.begin(), cg.shift_iters.end(), 0);
    im->V.bshared = im->rhs;
    im->V.bvec = nullptr;
    // with refinement the first solve stops at tol*100 (the dd-residual
    // correction supplies the remaining digits)
    // targets: first solve min(1e-9, 1e-10 w_j), correction min(5e-4, 1e-5 w_j):
    // every shift ends at a true relative residual <= cap1 * cap2 = 5e-13
    // (north_star: <= 1e-12), u1 ~2e-10 from truth at BASELINE conditioning
    // (north_star: <= 1e-8).  Sweep: scripts/tune_tol3.sh -- the former
    // correction targets (1e-4, 1e-6 w_j) bought residuals of 1e-13 at +10 %
    // step time.
    double tol1 = cg.refine > 0 ? std::min(1e-8, cg.tol * 100.0) : cg.tol;
    double tol2 = 1e-5;
    double cap1 = cg.refine > 0 ? 1e-9 : cg.tol, cap2 = 5e-4;
    if (const char *e = getenv("REXI_COCG_TOL1")) tol1 = atof(e);   // tuning knobs
    if (const char *e = getenv("REXI_COCG_TOL2")) tol2 = atof(e);
    if (const char *e = getenv("REXI_COCG_CAP1")) cap1 = atof(e);
    if (const char *e = getenv("REXI_COCG_CAP2")) cap2 = atof(e);
    int rc = cg_solve(cg, im, S, st, launches, err, tol1, std::max(tol1, cap1));
    if (rc) return rc;
    *x1 = im->xout;
    *x2 = nullptr;
    if (cg.refine <= 0) return REXI_OK;
    const int64_t n = cg.n;
    const int kp = im->kp_full;
    CGK(cudaMemcpyAsync(im->xsave, im->xout, sizeof(c128) * n * kp, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < cg.refine; ++r) {
        if (r > 0) CGK(cocg_axpy_inplace(im->xsave, im->xout, n * kp, st));
        hook_begin(cg, "cg_residual", 32.0 * n * cg.k + 28.0 * cg.nnz);
        k_cg_residual<<<(unsigned)((n * kp + CG_NT - 1) / CG_NT), CG_NT, 0, st>>>(im->M, im->rhs, im->xsave, S, kp,
                                                                               im->res);
        hook_end(cg);
        CGK(cudaGetLastError());
        ++*launches;
        im->V.bshared = nullptr;
        im->V.bvec = im->res;
        rc = cg_solve(cg, im, S, st, launches, err, tol2, std::max(tol2, cap2));
        im->V.bshared = im->rhs;
        im->V.bvec = nullptr;
        if (rc) return rc;
    }
    *x1 = im->xsave;
    *x2 = im->xout;
    return REXI_OK;
}

static void iter_summary(CocgState &cg) {
    int mx = 0;
    double sum = 0.0;
    for (int v : cg.shift_iters) {
        mx = std::max(mx, v);
        sum += v;
    }
    cg.last_iters_max = mx;
    cg.last_iters_mean = cg.k ? sum / cg.k : 0.0;
}

void cocg_collect_phase(CocgState &cg) {
    if (!cg.ev_pending) return;
    cg.ev_pending = false;
    float a = 0.f, b = 0.f;
    if (cudaEventSynchronize(cg.ev[3]) != cudaSuccess) return;
    cudaEventElapsedTime(&a, cg.ev[0], cg.ev[1]);
    cudaEventElapsedTime(&b, cg.ev[2], cg.ev[3]);
    cg.t_rhs_ms += a;
    cg.t_acc_ms += b;
}

int cocg_step(CocgState &cg, const ShiftDev &S, cudaStream_t st, const c128 *u, c128 *uout, double *acc,
              int64_t *launches, std::string &err) {
    CocgImpl *im = (CocgImpl *)cg.impl;
    const int64_t n = cg.n;
    cocg_collect_phase(cg);
    CGK(cudaEventRecord(cg.ev[0], st));
    k_cg_rhs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(im->M, u, im->rhs);
    CGK(cudaGetLastError());
    CGK(cudaEventRecord(cg.ev[1], st));
    ++*launches;
    const c128 *x1 = nullptr, *x2 = nullptr;
    int rc = cg_solve_refined(cg, im, S, st, launches, err, &x1, &x2);
    iter_summary(cg);
    if (rc) return rc;
    CGK(cudaEventRecord(cg.ev[2], st));
    hook_begin(cg, "cg_accum", (x2 ? 32.0 : 16.0) * n * cg.k + 32.0 * n);
    k_cg_accum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, im->kp_full, cg.k, S.beta, x1, x2, acc, uout);
    hook_end(cg);
    CGK(cudaGetLastError());
    CGK(cudaEventRecord(cg.ev[3], st));
    cg.ev_pending = true;
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
    const c128 *x1 = nullptr, *x2 = nullptr;
    int rc = cg_solve_refined(cg, im, S, st, &launches, err, &x1, &x2);
    iter_summary(cg);
    if (rc) return rc;
    const int64_t t = n * (int64_t)cg.k;
    k_cg_transpose<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(x1, x2, n, im->kp_full, cg.k, x);
    CGK(cudaGetLastError());
    return REXI_OK;
}

void cocg_destroy(CocgState &cg) {
    for (auto &e : cg.ev)
        if (e) {
            cudaEventDestroy(e);
            e = nullptr;
        }
    for (void *p : cg.allocs) cudaFree(p);
    cg.allocs.clear();
    if (cg.impl) {
        CocgImpl *im = (CocgImpl *)cg.impl;
        if (im->h_buf) cudaFreeHost(im->h_buf);
        delete im;
        cg.impl = nullptr;
    }
}

}  // namespace rexi
