// tridiag_kernels.cu -- sm_100a kernels of the 1D (tridiagonal) REXI path.
// Algorithm and layout: see tridiag.cuh and DESIGN.md ("1D path").
#include "tridiag.cuh"
#include "tridiag_launch.h"

namespace rexi {

enum { RHS_L0 = 0, RHS_LV = 1, RHS_ST = 2, RHS_LVDD = 3 };

struct BlkArgs {
    L0Dev z;
    LevelDev L;
    ShiftDev S;
    const c128 *rhs0;                 // RHS_L0: shared rhs [n]
    const c128 *rin_a, *rin_b;        // RHS_LV: previous level ypart / lc [n][kp]
    const c128 *rst;                  // RHS_ST: stored per-shift rhs [n][kp]
    const cdh *rdd_a, *rdd_b;         // RHS_LVDD: previous level dd ypart / lc
    const c128 *Xnext;                // S3: next-level solution [P][kp]
    double *acc;                      // dd partial, SoA 4*n
    c128 *uout;                       // rounded output (final_out)
    int acc_add;                      // 1: add to acc instead of overwrite
    int final_out;                    // 1: write uout instead of acc
};

template <int RHS>
__device__ __forceinline__ c128 rhs_at(const BlkArgs &a, int64_t i, int j) {
    const int kp = a.S.kp;
    if constexpr (RHS == RHS_L0) return a.rhs0[i];
    else if constexpr (RHS == RHS_LV) return cadd(a.rin_a[i * kp + j], a.rin_b[i * kp + j]);
    else if constexpr (RHS == RHS_LVDD) return cdd_round(cdd_add(cdh_unpack(a.rdd_a[i * kp + j]), cdh_unpack(a.rdd_b[i * kp + j])));
    else return a.rst[i * kp + j];
}

// ---------------------------------------------------------------------------
// Block kernel: PHASE 1 = interior solve with zero halos -> reduced rhs;
//               PHASE 3 = interior solve with known interface values.
// ---------------------------------------------------------------------------
template <int M, bool L0, int RHS, int PHASE, bool WRITE_X, bool ACCUM>
__global__ void __launch_bounds__(TRI_THREADS) k_block(BlkArgs a) {
    extern __shared__ c128 tile[];
    const int kp = a.S.kp;
    const int tid = threadIdx.x;
    const int64_t gt = (int64_t)blockIdx.x * TRI_THREADS + tid;
    const int j = (int)(gt & (kp - 1));
    const int64_t p = gt / kp;
    const int64_t P = a.L.P;
    const int64_t n = a.L.n;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    const c128 sg = a.S.sigma[j];

    c128 y[M];
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (PHASE == 3 && active) {
        xs = a.Xnext[p * kp + j];
        if (p + 1 < P) xn = a.Xnext[(p + 1) * kp + j];
    }
    y[0] = xs;
#pragma unroll
    for (int q = 1; q < M; ++q) y[q] = cmk(0.0, 0.0);

    // forward: y_q = invd_q (d_q - a_q y_{q-1})
#pragma unroll
    for (int q = 1; q < M; ++q) {
        if (q <= cnt) {
            const int64_t i = base + q;
            c128 d = rhs_at<RHS>(a, i, j);
            c128 ai = co_sub<L0>(a.z, a.L, a.S, i, j, sg);
            c128 iv = a.L.invd[i * kp + j];
            y[q] = cmul(iv, cfnma(d, ai, y[q - 1]));
        }
    }
    c128 ylast = y[0];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q == cnt) ylast = y[q];
    // backward: x_q = y_q - invd_q (c_q x_{q+1})
    c128 xnext = xn;
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        if (q <= cnt) {
            const int64_t i = base + q;
            c128 ci = co_sup<L0>(a.z, a.L, a.S, i, j, sg);
            c128 iv = a.L.invd[i * kp + j];
            c128 xi = cfnma(y[q], iv, cmul(ci, xnext));
            y[q] = xi;
            xnext = xi;
        }
    }

    if constexpr (PHASE == 1) {
        if (active) {
            c128 yfirst = cnt >= 1 ? y[1] : cmk(0.0, 0.0);
            c128 ds = rhs_at<RHS>(a, base, j);
            c128 cs = co_sup<L0>(a.z, a.L, a.S, base, j, sg);
            a.L.ypart[p * kp + j] = cfnma(ds, cs, yfirst);
            if (p + 1 < P) {
                c128 an = co_sub<L0>(a.z, a.L, a.S, base + M, j, sg);
                a.L.lc[(p + 1) * kp + j] = cneg(cmul(an, ylast));
            }
            if (p == 0) a.L.lc[j] = cmk(0.0, 0.0);
        }
    } else {
        if constexpr (WRITE_X) {
            if (active) {
                a.L.X[base * kp + j] = xs;
#pragma unroll
                for (int q = 1; q < M; ++q)
                    if (q <= cnt) a.L.X[(base + q) * kp + j] = y[q];
            }
        }
        if constexpr (ACCUM) {
            // beta-weighted accumulation over shifts through a smem tile
            const int bpc = TRI_THREADS / kp;             // blocks per CTA
            const int rows = bpc * M;                      // rows per CTA
            const int ld = kp + 1;                         // padded row stride
            const int b = tid / kp;
#pragma unroll
            for (int q = 0; q < M; ++q) {
                c128 v = (q == 0) ? xs : y[q];
                if (q > cnt) v = cmk(0.0, 0.0);
                tile[(b * M + q) * ld + j] = v;
            }
            __syncthreads();
            const int tpr = kp >= M ? kp / M : 1;          // threads per row
            const int stride_rows = TRI_THREADS / tpr;
            const int sub = tid % tpr;
            const int64_t row0 = (int64_t)blockIdx.x * bpc * M;
            for (int r = tid / tpr; r < rows; r += stride_rows) {
                cdd s = cdd_zero();
                for (int jj = sub; jj < kp; jj += tpr)
                    s = cdd_fma(s, a.S.beta[jj], tile[r * ld + jj]);
                for (int off = tpr >> 1; off > 0; off >>= 1) {
                    cdd o;
                    o.re.hi = __shfl_down_sync(0xffffffffu, s.re.hi, off, tpr);
                    o.re.lo = __shfl_down_sync(0xffffffffu, s.re.lo, off, tpr);
                    o.im.hi = __shfl_down_sync(0xffffffffu, s.im.hi, off, tpr);
                    o.im.lo = __shfl_down_sync(0xffffffffu, s.im.lo, off, tpr);
                    s = cdd_add(s, o);
                }
                const int64_t row = row0 + r;
                if (sub == 0 && row < n) {
                    if (a.acc_add) {
                        cdd prev = {{a.acc[row], a.acc[n + row]}, {a.acc[2 * n + row], a.acc[3 * n + row]}};
                        s = cdd_add(prev, s);
                    }
                    if (a.final_out) {
                        a.uout[row] = cdd_round(s);
                    } else {
                        a.acc[row] = s.re.hi;
                        a.acc[n + row] = s.re.lo;
                        a.acc[2 * n + row] = s.im.hi;
                        a.acc[3 * n + row] = s.im.lo;
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// rhs = 1j * (B @ u)  (reference integrate.py:204; CSR row order, no FMA)
// ---------------------------------------------------------------------------
__global__ void k_rhs(L0Dev z, int64_t n, const c128 *__restrict__ u, c128 *__restrict__ rhs) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sr = 0.0, si = 0.0;
    if (i > 0) {
        double b = __ldg(z.b_sub + i);
        c128 x = u[i - 1];
        sr = __dadd_rn(sr, __dmul_rn(b, x.x));
        si = __dadd_rn(si, __dmul_rn(b, x.y));
    }
    {
        double b = __ldg(z.b_dia + i);
        c128 x = u[i];
        sr = __dadd_rn(sr, __dmul_rn(b, x.x));
        si = __dadd_rn(si, __dmul_rn(b, x.y));
    }
    if (i + 1 < n) {
        double b = __ldg(z.b_sup + i);
        c128 x = u[i + 1];
        sr = __dadd_rn(sr, __dmul_rn(b, x.x));
        si = __dadd_rn(si, __dmul_rn(b, x.y));
    }
    rhs[i] = cmk(-si, sr);
}

// ---------------------------------------------------------------------------
// residual r_j = rhs - S_j x_j, evaluated with error-free products and a
// double-double sum, rounded once (level 0, refinement)
// ---------------------------------------------------------------------------
__global__ void k_residual(L0Dev z, LevelDev L, ShiftDev S, const c128 *__restrict__ rhs0,
                           c128 *__restrict__ res) {
    const int kp = S.kp;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = L.n;
    if (gt >= n * kp) return;
    const int j = (int)(gt & (kp - 1));
    const int64_t i = gt / kp;
    const c128 sg = S.sigma[j];
    const c128 d = rhs0[i];
    cdd acc = {{d.x, 0.0}, {d.y, 0.0}};
    if (i > 0) acc = cdd_sub_prod(acc, co_sub<true>(z, L, S, i, j, sg), L.X[(i - 1) * kp + j]);
    acc = cdd_sub_prod(acc, co_dia<true>(z, L, S, i, j, sg), L.X[i * kp + j]);
    if (i + 1 < n) acc = cdd_sub_prod(acc, co_sup<true>(z, L, S, i, j, sg), L.X[(i + 1) * kp + j]);
    res[i * kp + j] = cdd_round(acc);
}

// ---------------------------------------------------------------------------
// Top level: direct solve, one thread per shift
// ---------------------------------------------------------------------------
__global__ void k_top_solve(LevelDev L, ShiftDev S, const c128 *__restrict__ rin_a,
                            const c128 *__restrict__ rin_b, const cdh *__restrict__ rdd_a,
                            const cdh *__restrict__ rdd_b) {
    const int kp = S.kp;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= kp) return;
    const int64_t n = L.n;
    c128 yp = cmk(0.0, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        c128 d = rdd_a ? cdd_round(cdd_add(cdh_unpack(rdd_a[i * kp + j]), cdh_unpack(rdd_b[i * kp + j])))
                       : cadd(rin_a[i * kp + j], rin_b[i * kp + j]);
        c128 ai = L.sym ? (i > 0 ? L.sup[(i - 1) * kp + j] : cmk(0.0, 0.0)) : L.sub[i * kp + j];
        yp = cmul(L.invd[i * kp + j], cfnma(d, ai, yp));
        L.X[i * kp + j] = yp;
    }
    c128 xnext = cmk(0.0, 0.0);
    for (int64_t i = n - 1; i >= 0; --i) {
        c128 ci = L.sup[i * kp + j];
        c128 xi = cfnma(L.X[i * kp + j], L.invd[i * kp + j], cmul(ci, xnext));
        L.X[i * kp + j] = xi;
        xnext = xi;
    }
}

// ---------------------------------------------------------------------------
// Prepare-time kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pivot_stats(c128 d, double &mn, double &mx) {
    double v = sqrt(cabs2(d));
    if (!(v == v) || isinf(v)) v = 0.0;   // non-finite counts as singular
    mn = fmin(mn, v);
    mx = fmax(mx, v);
}
__device__ __forceinline__ void pivot_commit(unsigned long long *pmin, unsigned long long *pmax,
                                             int j, double mn, double mx) {
    // non-negative doubles order like their bit patterns
    atomicMin(pmin + j, (unsigned long long)__double_as_longlong(mn));
    atomicMax(pmax + j, (unsigned long long)__double_as_longlong(mx));
}

template <int M, bool L0>
__global__ void k_factor(L0Dev z, LevelDev L, ShiftDev S, unsigned long long *pmin,
                         unsigned long long *pmax) {
    const int kp = S.kp;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = (int)(gt & (kp - 1));
    const int64_t p = gt / kp;
    if (p >= L.P) return;
    const int64_t base = p * M;
    const int cnt = (int)min((int64_t)M, L.n - base) - 1;
    const c128 sg = S.sigma[j];
    double mn = INFINITY, mx = 0.0;
    c128 ivp = cmk(0.0, 0.0), g = cmk(0.0, 0.0);
    c128 phiF = cmk(0.0, 0.0), phiL = cmk(0.0, 0.0), psiF = cmk(0.0, 0.0), psiL = cmk(0.0, 0.0);
    if (cnt >= 1) {
        for (int q = 1; q <= cnt; ++q) {
            const int64_t i = base + q;
            c128 bq = co_dia<L0>(z, L, S, i, j, sg);
            c128 delta = bq;
            c128 ai = cmk(0.0, 0.0);
            if (q > 1) {
                ai = co_sub<L0>(z, L, S, i, j, sg);
                c128 cm = co_sup<L0>(z, L, S, i - 1, j, sg);
                delta = csub(bq, cmul(ai, cmul(cm, ivp)));
            }
            pivot_stats(delta, mn, mx);
            c128 iv = crcp(delta);
            L.invd[i * kp + j] = iv;
            g = (q == 1) ? iv : cneg(cmul(iv, cmul(ai, g)));
            ivp = iv;
        }
        const int64_t r0 = base + 1, r1 = base + cnt;
        const c128 t = ivp;                                   // (T^-1)_{r1,r1}
        // bottom-up pivot at r0 -> (T^-1)_{r0,r0}
        c128 dh = co_dia<L0>(z, L, S, r1, j, sg);
        for (int64_t i = r1 - 1; i >= r0; --i) {
            c128 ci = co_sup<L0>(z, L, S, i, j, sg);
            c128 an = co_sub<L0>(z, L, S, i + 1, j, sg);
            dh = csub(co_dia<L0>(z, L, S, i, j, sg), cmul(cmul(ci, an), crcp(dh)));
        }
        const c128 h = crcp(dh);
        // (T^-1)_{r0,r1} by the backward product
        c128 zq = t;
        for (int64_t i = r1 - 1; i >= r0; --i)
            zq = cneg(cmul(L.invd[i * kp + j], cmul(co_sup<L0>(z, L, S, i, j, sg), zq)));
        const c128 a0 = co_sub<L0>(z, L, S, r0, j, sg);
        const c128 c1 = co_sup<L0>(z, L, S, r1, j, sg);
        phiF = cmul(a0, h);
        phiL = cmul(a0, g);
        psiF = cmul(c1, zq);
        psiL = cmul(c1, t);
    }
    L.phiF[p * kp + j] = phiF;
    L.phiL[p * kp + j] = phiL;
    L.psiF[p * kp + j] = psiF;
    L.psiL[p * kp + j] = psiL;
    if (cnt >= 1) pivot_commit(pmin, pmax, j, mn, mx);
}

// next level row p: L_p = -a_s phiL_{p-1}, D_p = b_s - a_s psiL_{p-1} - c_s phiF_p, U_p = -c_s psiF_p
template <int M, bool L0>
__global__ void k_assemble(L0Dev z, LevelDev L, LevelDev N, ShiftDev S) {
    const int kp = S.kp;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = (int)(gt & (kp - 1));
    const int64_t p = gt / kp;
    if (p >= L.P) return;
    const c128 sg = S.sigma[j];
    const int64_t s = p * M;
    c128 as = co_sub<L0>(z, L, S, s, j, sg);
    c128 bs = co_dia<L0>(z, L, S, s, j, sg);
    c128 cs = co_sup<L0>(z, L, S, s, j, sg);
    c128 lv = cmk(0.0, 0.0), dv = bs, uv = cmk(0.0, 0.0);
    if (p > 0) {
        lv = cneg(cmul(as, L.phiL[(p - 1) * kp + j]));
        dv = csub(dv, cmul(as, L.psiL[(p - 1) * kp + j]));
    }
    dv = csub(dv, cmul(cs, L.phiF[p * kp + j]));
    if (p + 1 < L.P) uv = cneg(cmul(cs, L.psiF[p * kp + j]));
    if (!N.sym) N.sub[p * kp + j] = lv;
    N.dia[p * kp + j] = dv;
    N.sup[p * kp + j] = uv;
}

__global__ void k_top_factor(LevelDev L, ShiftDev S, unsigned long long *pmin,
                             unsigned long long *pmax) {
    const int kp = S.kp;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= kp) return;
    double mn = INFINITY, mx = 0.0;
    c128 ivp = cmk(0.0, 0.0);
    for (int64_t i = 0; i < L.n; ++i) {
        c128 delta = L.dia[i * kp + j];
        if (i > 0) {
            const c128 ai = L.sym ? L.sup[(i - 1) * kp + j] : L.sub[i * kp + j];
            delta = csub(delta, cmul(ai, cmul(L.sup[(i - 1) * kp + j], ivp)));
        }
        pivot_stats(delta, mn, mx);
        ivp = crcp(delta);
        L.invd[i * kp + j] = ivp;
    }
    pivot_commit(pmin, pmax, j, mn, mx);
}

// [n][kp] -> [k][n] (shift-major) for rexi_plan_solve
__global__ void k_transpose_out(const c128 *__restrict__ X, int64_t n, int kp, int k,
                                c128 *__restrict__ out) {
    int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gt >= n * (int64_t)k) return;
    int j = (int)(gt / n);
    int64_t i = gt % n;
    out[gt] = X[i * kp + j];
}

// combine G double-double partials (SoA 4*n each) in fixed order
__global__ void k_combine(const double *__restrict__ parts, int g, int64_t n, c128 *__restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    cdd s = cdd_zero();
    for (int q = 0; q < g; ++q) {
        const double *pp = parts + (size_t)q * 4 * n;
        cdd v = {{pp[i], pp[n + i]}, {pp[2 * n + i], pp[3 * n + i]}};
        s = cdd_add(s, v);
    }
    out[i] = cdd_round(s);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static size_t accum_smem(int kp) { return (size_t)(TRI_THREADS / kp) * TRI_M * (kp + 1) * sizeof(c128); }

template <bool L0, int RHS, int PHASE, bool WRITE_X, bool ACCUM>
static cudaError_t launch_block(const BlkArgs &a, cudaStream_t st) {
    auto kern = k_block<TRI_M, L0, RHS, PHASE, WRITE_X, ACCUM>;
    const int64_t threads = a.L.P * a.S.kp;
    const int64_t grid = (threads + TRI_THREADS - 1) / TRI_THREADS;
    size_t smem = ACCUM ? accum_smem(a.S.kp) : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)grid, TRI_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t tri_launch_rhs(const L0Dev &z, int64_t n, const c128 *u, c128 *rhs, cudaStream_t st) {
    k_rhs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(z, n, u, rhs);
    return cudaGetLastError();
}

cudaError_t tri_launch_residual(const L0Dev &z, const LevelDev &L, const ShiftDev &S,
                                const c128 *rhs0, c128 *res, cudaStream_t st) {
    int64_t t = L.n * S.kp;
    k_residual<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(z, L, S, rhs0, res);
    return cudaGetLastError();
}

cudaError_t tri_launch_s1(const L0Dev &z, const LevelDev &L, const ShiftDev &S, int level,
                          const c128 *rhs0, const c128 *rst, const c128 *rin_a,
                          const c128 *rin_b, cudaStream_t st) {
    BlkArgs a{};
    a.z = z; a.L = L; a.S = S;
    a.rhs0 = rhs0; a.rst = rst; a.rin_a = rin_a; a.rin_b = rin_b;
    if (level == 0) {
        if (rst) return launch_block<true, RHS_ST, 1, false, false>(a, st);
        return launch_block<true, RHS_L0, 1, false, false>(a, st);
    }
    return launch_block<false, RHS_LV, 1, false, false>(a, st);
}

cudaError_t tri_launch_s3(const L0Dev &z, const LevelDev &L, const ShiftDev &S, int level,
                          const c128 *rhs0, const c128 *rst, const c128 *rin_a,
                          const c128 *rin_b, const c128 *Xnext, int out_mode, double *acc,
                          int acc_add, c128 *uout, cudaStream_t st) {
    BlkArgs a{};
    a.z = z; a.L = L; a.S = S;
    a.rhs0 = rhs0; a.rst = rst; a.rin_a = rin_a; a.rin_b = rin_b; a.Xnext = Xnext;
    a.acc = acc; a.acc_add = acc_add; a.uout = uout; a.final_out = uout != nullptr;
    if (level > 0) return launch_block<false, RHS_LV, 3, true, false>(a, st);
    // level 0
    if (rst) {
        if (out_mode == TRI_OUT_ACC) return launch_block<true, RHS_ST, 3, false, true>(a, st);
        return launch_block<true, RHS_ST, 3, true, false>(a, st);
    }
    if (out_mode == TRI_OUT_ACC) return launch_block<true, RHS_L0, 3, false, true>(a, st);
    if (out_mode == TRI_OUT_X_ACC) return launch_block<true, RHS_L0, 3, true, true>(a, st);
    return launch_block<true, RHS_L0, 3, true, false>(a, st);
}

cudaError_t tri_launch_top_solve(const LevelDev &L, const ShiftDev &S, const c128 *rin_a,
                                 const c128 *rin_b, cudaStream_t st) {
    k_top_solve<<<(S.kp + 63) / 64, 64, 0, st>>>(L, S, rin_a, rin_b, nullptr, nullptr);
    return cudaGetLastError();
}

cudaError_t tri_launch_top_solve_dd(const LevelDev &L, const ShiftDev &S, const cdh *rdd_a,
                                    const cdh *rdd_b, cudaStream_t st) {
    k_top_solve<<<(S.kp + 63) / 64, 64, 0, st>>>(L, S, nullptr, nullptr, rdd_a, rdd_b);
    return cudaGetLastError();
}

cudaError_t tri_launch_lv_dd(const LevelDev &L, const ShiftDev &S, int phase, const cdh *rdd_a,
                             const cdh *rdd_b, const c128 *Xnext, cudaStream_t st) {
    BlkArgs a{};
    a.L = L; a.S = S; a.rdd_a = rdd_a; a.rdd_b = rdd_b; a.Xnext = Xnext;
    if (phase == 1) return launch_block<false, RHS_LVDD, 1, false, false>(a, st);
    return launch_block<false, RHS_LVDD, 3, true, false>(a, st);
}

cudaError_t tri_launch_factor(const L0Dev &z, const LevelDev &L, const LevelDev *next,
                              const ShiftDev &S, int level, unsigned long long *pmin,
                              unsigned long long *pmax, cudaStream_t st) {
    if (L.top) {
        k_top_factor<<<(S.kp + 63) / 64, 64, 0, st>>>(L, S, pmin, pmax);
        return cudaGetLastError();
    }
    int64_t t = L.P * S.kp;
    unsigned grid = (unsigned)((t + 127) / 128);
    if (level == 0) {
        k_factor<TRI_M, true><<<grid, 128, 0, st>>>(z, L, S, pmin, pmax);
        k_assemble<TRI_M, true><<<grid, 128, 0, st>>>(z, L, *next, S);
    } else {
        k_factor<TRI_M, false><<<grid, 128, 0, st>>>(z, L, S, pmin, pmax);
        k_assemble<TRI_M, false><<<grid, 128, 0, st>>>(z, L, *next, S);
    }
    return cudaGetLastError();
}

cudaError_t tri_launch_transpose(const c128 *X, int64_t n, int kp, int k, c128 *out, cudaStream_t st) {
    int64_t t = n * (int64_t)k;
    k_transpose_out<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(X, n, kp, k, out);
    return cudaGetLastError();
}

cudaError_t launch_combine(const double *parts, int g, int64_t n, c128 *out, cudaStream_t st) {
    k_combine<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(parts, g, n, out);
    return cudaGetLastError();
}

}  // namespace rexi
