// tridiag_l0.cu -- level-0 kernels of the 1D path, TMA-fed (v2).
//
// Every CTA owns a tile of T_r = (L0_NT / kp) * M consecutive rows for all kp
// shift lanes.  Per-shift arrays are [row][kp], so the tile of the inverse
// pivots (and of the stored residual) is ONE contiguous range of
// T_r*kp*16 = L0_NT*M*16 = 32 KB: a single cp.async.bulk (TMA bulk copy)
// stages it into shared memory, completion on an mbarrier.  Each thread then
// runs the forward/backward sweeps of one block (M rows) for one shift out of
// shared memory, so the long dependent row chain no longer serialises HBM
// loads.  Shared per-row inputs (rhs, the A/B off-diagonals) are broadcast
// __ldg loads.
//
// Kernels (refine = 0):  S1 (reduce) ... levels >= 1 ... S3ACC (solve + sum)
// Kernels (refine = 1):  S1 ... K2 (solve + sum + dd residual + correction
//                        reduce) ... levels >= 1 ... K3 (correction solve + sum)
#include "tridiag.cuh"
#include "tridiag_launch.h"

namespace rexi {

constexpr int L0_NT = 128;    // threads per CTA

struct L0Args {
    L0Dev z;
    LevelDev L;
    ShiftDev S;
    const c128 *rhs0;     // [n]
    const c128 *X1;       // next-level solution [P][kp]
    const c128 *rres_in;  // K3
    c128 *rres_out;       // K2
    double *acc;          // dd partial SoA 4*n
    c128 *uout;
    int acc_add;
    int final_out;
};

struct L0Smem {
    uint64_t bar;
    uint64_t pad;
};

template <int M>
__device__ __forceinline__ int rows_per_cta(int kp) { return (L0_NT / kp) * M; }

// stage nt tiles of per-shift data (rows [row0, row1)) into shared memory
__device__ __forceinline__ void stage_tiles(uint64_t *bar, c128 *t0, const c128 *g0, c128 *t1,
                                            const c128 *g1, int64_t row0, int64_t row1, int kp) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t bytes = (uint32_t)((row1 - row0) * kp * sizeof(c128));
        mbar_expect_tx(bar, g1 ? 2 * bytes : bytes);
        bulk_g2s(t0, g0 + row0 * kp, bytes, bar);
        if (g1) bulk_g2s(t1, g1 + row0 * kp, bytes, bar);
    }
}

// beta-weighted sum over the kp shift lanes of every tile row, fixed order,
// fp64 products accumulated with error-free TwoSum; writes acc or uout
template <int M>
__device__ __forceinline__ void reduce_rows(const c128 *tile, const L0Args &a, int64_t row0) {
    const int kp = a.S.kp;
    const int rows = rows_per_cta<M>(kp);
    const int tpr = L0_NT / rows > 0 ? L0_NT / rows : 1;
    const int sub = threadIdx.x % tpr;
    const int64_t n = a.L.n;
    for (int r = threadIdx.x / tpr; r < rows; r += L0_NT / tpr) {
        ddacc re = {0.0, 0.0}, im = {0.0, 0.0};
        for (int jj = sub; jj < kp; jj += tpr) {
            const c128 b = a.S.beta[jj];
            const c128 x = tile[r * kp + jj];
            ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
            ddacc_add(im, fma(b.x, x.y, b.y * x.x));
        }
        dd sre = fast_two_sum(re.hi, re.lo), sim = fast_two_sum(im.hi, im.lo);
        for (int off = tpr >> 1; off > 0; off >>= 1) {
            dd ore, oim;
            ore.hi = __shfl_down_sync(0xffffffffu, sre.hi, off, tpr);
            ore.lo = __shfl_down_sync(0xffffffffu, sre.lo, off, tpr);
            oim.hi = __shfl_down_sync(0xffffffffu, sim.hi, off, tpr);
            oim.lo = __shfl_down_sync(0xffffffffu, sim.lo, off, tpr);
            sre = dd_add(sre, ore);
            sim = dd_add(sim, oim);
        }
        const int64_t row = row0 + r;
        if (sub == 0 && row < n) {
            if (a.acc_add) {
                sre = dd_add(sre, dd{a.acc[row], a.acc[n + row]});
                sim = dd_add(sim, dd{a.acc[2 * n + row], a.acc[3 * n + row]});
            }
            if (a.final_out) {
                a.uout[row] = cmk(__dadd_rn(sre.hi, sre.lo), __dadd_rn(sim.hi, sim.lo));
            } else {
                a.acc[row] = sre.hi;
                a.acc[n + row] = sre.lo;
                a.acc[2 * n + row] = sim.hi;
                a.acc[3 * n + row] = sim.lo;
            }
        }
    }
}

// error-free accumulation of -e*x into a complex double-double (Dot2 style)
__device__ __forceinline__ void dot2_sub(ddacc &re, ddacc &im, c128 e, c128 x) {
    dd p;
    p = two_prod(e.x, x.x); ddacc_add(re, -p.hi); re.lo = __dsub_rn(re.lo, p.lo);
    p = two_prod(e.y, x.y); ddacc_add(re, p.hi); re.lo = __dadd_rn(re.lo, p.lo);
    p = two_prod(e.x, x.y); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
    p = two_prod(e.y, x.x); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
}

// ---------------------------------------------------------------------------
// S1: interior solves with zero halos -> reduced rhs (ypart, lc)
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(L0_NT) k_l0_s1(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    L0Smem *sm = reinterpret_cast<L0Smem *>(smem_raw);
    c128 *tinv = reinterpret_cast<c128 *>(smem_raw + 128);
    const int kp = a.S.kp;
    const int bpc = L0_NT / kp;
    const int b = threadIdx.x / kp, j = threadIdx.x % kp;
    const int64_t n = a.L.n, P = a.L.P;
    const int64_t row0 = (int64_t)blockIdx.x * bpc * M;
    const int64_t row1 = min(row0 + (int64_t)bpc * M, n);
    stage_tiles(&sm->bar, tinv, a.L.invd, nullptr, nullptr, row0, row1, kp);
    const int64_t p = (int64_t)blockIdx.x * bpc + b;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    const c128 sg = a.S.sigma[j];
    const c128 *ti = tinv + (size_t)b * M * kp + j;
    mbar_wait(&sm->bar, 0);
    if (!active) return;

    c128 y[M];
    y[0] = cmk(0.0, 0.0);
#pragma unroll
    for (int q = 1; q < M; ++q) {
        y[q] = cmk(0.0, 0.0);
        if (q <= cnt) {
            const int64_t i = base + q;
            const c128 ai = form_entry(__ldg(a.z.ta_sub + i), __ldg(a.z.ta_sub_im + i), __ldg(a.z.b_sub + i), sg);
            y[q] = cmul(ti[q * kp], cfnma(a.rhs0[i], ai, y[q - 1]));
        }
    }
    c128 ylast = y[0];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q == cnt) ylast = y[q];
    c128 xnext = cmk(0.0, 0.0);
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        if (q <= cnt) {
            const int64_t i = base + q;
            const c128 ci = form_entry(__ldg(a.z.ta_sup + i), __ldg(a.z.ta_sup_im + i), __ldg(a.z.b_sup + i), sg);
            xnext = cfnma(y[q], ti[q * kp], cmul(ci, xnext));
            y[q] = xnext;
        }
    }
    const c128 yfirst = cnt >= 1 ? y[1] : cmk(0.0, 0.0);
    const c128 cs = form_entry(__ldg(a.z.ta_sup + base), __ldg(a.z.ta_sup_im + base), __ldg(a.z.b_sup + base), sg);
    a.L.ypart[p * kp + j] = cfnma(a.rhs0[base], cs, yfirst);
    if (p + 1 < P) {
        const int64_t s1 = base + M;
        const c128 an = form_entry(__ldg(a.z.ta_sub + s1), __ldg(a.z.ta_sub_im + s1), __ldg(a.z.b_sub + s1), sg);
        a.L.lc[(p + 1) * kp + j] = cneg(cmul(an, ylast));
    }
    if (p == 0) a.L.lc[j] = cmk(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// S3ACC: solve with the interface values known, beta-weighted sum -> out
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(L0_NT) k_l0_s3acc(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    L0Smem *sm = reinterpret_cast<L0Smem *>(smem_raw);
    c128 *tinv = reinterpret_cast<c128 *>(smem_raw + 128);
    const int kp = a.S.kp;
    const int bpc = L0_NT / kp;
    const int b = threadIdx.x / kp, j = threadIdx.x % kp;
    const int64_t n = a.L.n, P = a.L.P;
    const int64_t row0 = (int64_t)blockIdx.x * bpc * M;
    const int64_t row1 = min(row0 + (int64_t)bpc * M, n);
    stage_tiles(&sm->bar, tinv, a.L.invd, nullptr, nullptr, row0, row1, kp);
    const int64_t p = (int64_t)blockIdx.x * bpc + b;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    const c128 sg = a.S.sigma[j];
    c128 *ti = tinv + (size_t)b * M * kp + j;
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (active) {
        xs = a.X1[p * kp + j];
        if (p + 1 < P) xn = a.X1[(p + 1) * kp + j];
    }
    mbar_wait(&sm->bar, 0);
    if (active) {
        c128 y[M];
        y[0] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q) {
            y[q] = cmk(0.0, 0.0);
            if (q <= cnt) {
                const int64_t i = base + q;
                const c128 ai = form_entry(__ldg(a.z.ta_sub + i), __ldg(a.z.ta_sub_im + i), __ldg(a.z.b_sub + i), sg);
                y[q] = cmul(ti[q * kp], cfnma(a.rhs0[i], ai, y[q - 1]));
            }
        }
        c128 xnext = xn;
#pragma unroll
        for (int q = M - 1; q >= 1; --q) {
            c128 v = cmk(0.0, 0.0);
            if (q <= cnt) {
                const int64_t i = base + q;
                const c128 ci = form_entry(__ldg(a.z.ta_sup + i), __ldg(a.z.ta_sup_im + i), __ldg(a.z.b_sup + i), sg);
                xnext = cfnma(y[q], ti[q * kp], cmul(ci, xnext));
                v = xnext;
            }
            ti[q * kp] = v;                // x overwrites the consumed inverse pivot
        }
        ti[0] = xs;                        // interface row
    } else {
#pragma unroll
        for (int q = 0; q < M; ++q) ti[q * kp] = cmk(0.0, 0.0);
    }
    __syncthreads();
    reduce_rows<M>(tinv, a, row0);
}

// ---------------------------------------------------------------------------
// K2 (refine): S3 + sum(beta x) + dd residual of the interior rows + the
// correction's reduce (dd interface pieces, so the residual at interface rows
// is formed exactly from the two blocks that own its terms)
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(L0_NT) k_l0_k2(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    L0Smem *sm = reinterpret_cast<L0Smem *>(smem_raw);
    const int kp = a.S.kp;
    const int bpc = L0_NT / kp;
    c128 *tinv = reinterpret_cast<c128 *>(smem_raw + 128);
    c128 *tx = tinv + (size_t)bpc * M * kp;
    const int b = threadIdx.x / kp, j = threadIdx.x % kp;
    const int64_t n = a.L.n, P = a.L.P;
    const int64_t row0 = (int64_t)blockIdx.x * bpc * M;
    const int64_t row1 = min(row0 + (int64_t)bpc * M, n);
    stage_tiles(&sm->bar, tinv, a.L.invd, nullptr, nullptr, row0, row1, kp);
    const int64_t p = (int64_t)blockIdx.x * bpc + b;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    const c128 sg = a.S.sigma[j];
    const c128 *ti = tinv + (size_t)b * M * kp + j;
    c128 *tc = tx + (size_t)b * M * kp + j;
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (active) {
        xs = a.X1[p * kp + j];
        if (p + 1 < P) xn = a.X1[(p + 1) * kp + j];
    }
    mbar_wait(&sm->bar, 0);
    c128 y[M];
    if (active) {
        y[0] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q) {
            y[q] = cmk(0.0, 0.0);
            if (q <= cnt) {
                const int64_t i = base + q;
                const c128 ai = form_entry(__ldg(a.z.ta_sub + i), __ldg(a.z.ta_sub_im + i), __ldg(a.z.b_sub + i), sg);
                y[q] = cmul(ti[q * kp], cfnma(a.rhs0[i], ai, y[q - 1]));
            }
        }
        c128 xnext = xn;
#pragma unroll
        for (int q = M - 1; q >= 1; --q) {
            c128 v = cmk(0.0, 0.0);
            if (q <= cnt) {
                const int64_t i = base + q;
                const c128 ci = form_entry(__ldg(a.z.ta_sup + i), __ldg(a.z.ta_sup_im + i), __ldg(a.z.b_sup + i), sg);
                xnext = cfnma(y[q], ti[q * kp], cmul(ci, xnext));
                v = xnext;
            }
            tc[q * kp] = v;
        }
        tc[0] = xs;
    } else {
#pragma unroll
        for (int q = 0; q < M; ++q) tc[q * kp] = cmk(0.0, 0.0);
    }
    __syncthreads();
    reduce_rows<M>(tx, a, row0);
    if (!active) return;

    // residual r_q = d_q - a_q x_{q-1} - b_q x_q - c_q x_{q+1}, interior rows
#pragma unroll
    for (int q = 1; q < M; ++q) {
        if (q <= cnt) {
            const int64_t i = base + q;
            const c128 d = a.rhs0[i];
            const c128 xm = tc[(q - 1) * kp];
            const c128 x0 = tc[q * kp];
            const c128 xp = q < cnt ? tc[(q + 1) * kp] : xn;
            ddacc re = {d.x, 0.0}, im = {d.y, 0.0};
            dot2_sub(re, im, form_entry(__ldg(a.z.ta_sub + i), __ldg(a.z.ta_sub_im + i), __ldg(a.z.b_sub + i), sg), xm);
            dot2_sub(re, im, form_entry(__ldg(a.z.ta_dia + i), __ldg(a.z.ta_dia_im + i), __ldg(a.z.b_dia + i), sg), x0);
            dot2_sub(re, im, form_entry(__ldg(a.z.ta_sup + i), __ldg(a.z.ta_sup_im + i), __ldg(a.z.b_sup + i), sg), xp);
            const c128 r = cmk(__dadd_rn(re.hi, re.lo), __dadd_rn(im.hi, im.lo));
            a.rres_out[i * kp + j] = r;
            y[q] = r;
        }
    }
    // interface pieces (double-double, combined by the next level)
    ddacc p1re, p1im;
    {
        const c128 d = a.rhs0[base];
        p1re = {d.x, 0.0};
        p1im = {d.y, 0.0};
        dot2_sub(p1re, p1im, form_entry(__ldg(a.z.ta_dia + base), __ldg(a.z.ta_dia_im + base), __ldg(a.z.b_dia + base), sg), xs);
        const c128 x1 = cnt >= 1 ? tc[kp] : xn;
        dot2_sub(p1re, p1im, form_entry(__ldg(a.z.ta_sup + base), __ldg(a.z.ta_sup_im + base), __ldg(a.z.b_sup + base), sg), x1);
    }
    // correction reduce: S1 with rhs = r
    y[0] = cmk(0.0, 0.0);
#pragma unroll
    for (int q = 1; q < M; ++q) {
        if (q <= cnt) {
            const int64_t i = base + q;
            const c128 ai = form_entry(__ldg(a.z.ta_sub + i), __ldg(a.z.ta_sub_im + i), __ldg(a.z.b_sub + i), sg);
            y[q] = cmul(ti[q * kp], cfnma(y[q], ai, y[q - 1]));
        }
    }
    c128 ylast = y[0];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q == cnt) ylast = y[q];
    c128 xnext = cmk(0.0, 0.0);
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        if (q <= cnt) {
            const int64_t i = base + q;
            const c128 ci = form_entry(__ldg(a.z.ta_sup + i), __ldg(a.z.ta_sup_im + i), __ldg(a.z.b_sup + i), sg);
            xnext = cfnma(y[q], ti[q * kp], cmul(ci, xnext));
            y[q] = xnext;
        }
    }
    const c128 yfirst = cnt >= 1 ? y[1] : cmk(0.0, 0.0);
    const c128 cs = form_entry(__ldg(a.z.ta_sup + base), __ldg(a.z.ta_sup_im + base), __ldg(a.z.b_sup + base), sg);
    const c128 t1 = cneg(cmul(cs, yfirst));
    ddacc_add(p1re, t1.x);
    ddacc_add(p1im, t1.y);
    a.L.ypdd[p * kp + j] = cdd{{p1re.hi, p1re.lo}, {p1im.hi, p1im.lo}};
    if (p + 1 < P) {
        const int64_t s1 = base + M;
        const c128 an = form_entry(__ldg(a.z.ta_sub + s1), __ldg(a.z.ta_sub_im + s1), __ldg(a.z.b_sub + s1), sg);
        const c128 xl = cnt >= 1 ? tc[cnt * kp] : xs;
        ddacc p2re = {0.0, 0.0}, p2im = {0.0, 0.0};
        dot2_sub(p2re, p2im, an, xl);
        const c128 t2 = cneg(cmul(an, ylast));
        ddacc_add(p2re, t2.x);
        ddacc_add(p2im, t2.y);
        a.L.lcdd[(p + 1) * kp + j] = cdd{{p2re.hi, p2re.lo}, {p2im.hi, p2im.lo}};
    }
    if (p == 0) a.L.lcdd[j] = cdd_zero();
}

// ---------------------------------------------------------------------------
// K3 (refine): correction solve with the stored residual, sum(beta dx) += acc
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(L0_NT) k_l0_k3(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    L0Smem *sm = reinterpret_cast<L0Smem *>(smem_raw);
    const int kp = a.S.kp;
    const int bpc = L0_NT / kp;
    c128 *tinv = reinterpret_cast<c128 *>(smem_raw + 128);
    c128 *tr = tinv + (size_t)bpc * M * kp;
    const int b = threadIdx.x / kp, j = threadIdx.x % kp;
    const int64_t n = a.L.n, P = a.L.P;
    const int64_t row0 = (int64_t)blockIdx.x * bpc * M;
    const int64_t row1 = min(row0 + (int64_t)bpc * M, n);
    stage_tiles(&sm->bar, tinv, a.L.invd, tr, a.rres_in, row0, row1, kp);
    const int64_t p = (int64_t)blockIdx.x * bpc + b;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    const c128 sg = a.S.sigma[j];
    const c128 *ti = tinv + (size_t)b * M * kp + j;
    c128 *tc = tr + (size_t)b * M * kp + j;
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (active) {
        xs = a.X1[p * kp + j];
        if (p + 1 < P) xn = a.X1[(p + 1) * kp + j];
    }
    mbar_wait(&sm->bar, 0);
    if (active) {
        c128 y[M];
        y[0] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q) {
            y[q] = cmk(0.0, 0.0);
            if (q <= cnt) {
                const int64_t i = base + q;
                const c128 ai = form_entry(__ldg(a.z.ta_sub + i), __ldg(a.z.ta_sub_im + i), __ldg(a.z.b_sub + i), sg);
                y[q] = cmul(ti[q * kp], cfnma(tc[q * kp], ai, y[q - 1]));
            }
        }
        c128 xnext = xn;
#pragma unroll
        for (int q = M - 1; q >= 1; --q) {
            c128 v = cmk(0.0, 0.0);
            if (q <= cnt) {
                const int64_t i = base + q;
                const c128 ci = form_entry(__ldg(a.z.ta_sup + i), __ldg(a.z.ta_sup_im + i), __ldg(a.z.b_sup + i), sg);
                xnext = cfnma(y[q], ti[q * kp], cmul(ci, xnext));
                v = xnext;
            }
            tc[q * kp] = v;
        }
        tc[0] = xs;
    } else {
#pragma unroll
        for (int q = 0; q < M; ++q) tc[q * kp] = cmk(0.0, 0.0);
    }
    __syncthreads();
    reduce_rows<M>(tr, a, row0);
}

// ---------------------------------------------------------------------------
template <typename K>
static cudaError_t launch_l0(K kern, const L0Args &a, int tiles, cudaStream_t st) {
    const int kp = a.S.kp;
    const int64_t rows = (int64_t)(L0_NT / kp) * TRI_M;
    const int64_t grid = (a.L.n + rows - 1) / rows;
    const size_t smem = 128 + (size_t)tiles * rows * kp * sizeof(c128);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, L0_NT, smem, st>>>(a);
    return cudaGetLastError();
}

bool l0v2_supported(int kp) { return kp <= L0_NT; }

cudaError_t l0_launch_s1(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                         cudaStream_t st) {
    L0Args a{};
    a.z = z; a.L = L; a.S = S; a.rhs0 = rhs0;
    return launch_l0(k_l0_s1<TRI_M>, a, 1, st);
}

cudaError_t l0_launch_s3acc(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                            const c128 *X1, double *acc, c128 *uout, cudaStream_t st) {
    L0Args a{};
    a.z = z; a.L = L; a.S = S; a.rhs0 = rhs0; a.X1 = X1; a.acc = acc; a.uout = uout;
    a.acc_add = 0; a.final_out = uout != nullptr;
    return launch_l0(k_l0_s3acc<TRI_M>, a, 1, st);
}

cudaError_t l0_launch_k2(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                         const c128 *X1, double *acc, c128 *rres, cudaStream_t st) {
    L0Args a{};
    a.z = z; a.L = L; a.S = S; a.rhs0 = rhs0; a.X1 = X1; a.acc = acc; a.rres_out = rres;
    a.acc_add = 0; a.final_out = 0;
    return launch_l0(k_l0_k2<TRI_M>, a, 2, st);
}

cudaError_t l0_launch_k3(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *X1,
                         const c128 *rres, double *acc, c128 *uout, cudaStream_t st) {
    L0Args a{};
    a.z = z; a.L = L; a.S = S; a.X1 = X1; a.rres_in = rres; a.acc = acc; a.uout = uout;
    a.acc_add = 1; a.final_out = uout != nullptr;
    return launch_l0(k_l0_k3<TRI_M>, a, 2, st);
}

}  // namespace rexi
