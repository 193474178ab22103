// tridiag_l0.cu -- level-0 kernels of the 1D path, TMA-fed.
//
// Every CTA owns a tile of T = (L0_NT / kp) * M consecutive rows for all kp
// shift lanes.  Per-shift arrays are [row][kp], so a CTA's tile of inverse
// pivots (and of the stored residual) is ONE contiguous range of
// T*kp*16 = L0_NT*M*16 = 32 KB; the shared per-row inputs (rhs and the A/B
// diagonals, fl(tau*A) precomputed) are contiguous ranges too.  One thread
// issues the cp.async.bulk (TMA bulk) copies, completion on one mbarrier;
// then each thread runs the forward/backward sweeps of one block (M rows) for
// one shift entirely out of shared memory (no global load inside the
// dependent row chain).  Full blocks take a predicate-free path.
//
// refine = 0:  S1 (reduce) ... levels >= 1 ... S3ACC (solve + beta-sum)
// refine = 1:  S1 ... K2 (solve + beta-sum + dd residual + correction reduce)
//              ... levels >= 1 (correction) ... K3 (correction solve + sum)
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "tridiag.cuh"
#include "tridiag_launch.h"

namespace cgr = cooperative_groups;

namespace rexi {

constexpr int L0_NT = 128;      // threads per CTA
// k_pad is a power of two (pick_kp): lane / block indices by shifts and masks
// instead of the integer-division subroutine
__device__ __forceinline__ int lg2(int pow2) { return __ffs(pow2) - 1; }
constexpr int L0_ROWPAD = 2;    // extra staged rows (next interface row + 16-B rounding)

#ifndef K2_RES_UNROLL
#define K2_RES_UNROLL 5   // swept: scripts/tune_k2u.sh (3: +1.2 %, 15: +15 %)
#endif
constexpr int K2_UNROLL = K2_RES_UNROLL;
#ifndef K2_ONE_TILE
#define K2_ONE_TILE 1   // x overwrites the pivot tile; the correction reads complex64 pivots from HBM
#endif
#ifndef K2_MINB
#define K2_MINB 4
#endif
#ifndef K2_I32
#define K2_I32 0   // 1: the correction sweep's complex64 pivots staged with the rest (+16 KB shared memory) instead of
                   // read from HBM in the sweep -- K2 0.680 -> 0.672 ms but the step no faster (scripts/tune_k2i32.sh)
#endif
#ifndef K2_ALIGNED
#define K2_ALIGNED 1   // real symmetric A: aligned-quantum residual instead of Dot2 (see k2_refine)
#endif
struct L0Args {
    L0Dev z;
    LevelDev L;
    ShiftDev S;
    const c128 *rhs0;     // [n (+pad)]
    const c128 *X1;       // next-level solution [P][kp]
    const c64 *rres_in;   // K3: interior residuals, complex64
    c64 *rres_out;        // K2
    const c64 *inv32;     // K3: level-0 inverse pivots rounded to complex64
    const float *r32[6];  // K3: fl(tau a) sub/im/b, sup/im/b rounded to float
    const double2 *emax;  // K2 (aligned residual): per block max |fl(tau a)|, max |b|
    double *acc;          // dd partial SoA 4*nout
    c128 *uout;
    int64_t nout;         // real n (level 0 is padded to a multiple of M)
    int acc_add;
    int final_out;
    int64_t pf_dist;      // K2: L2-prefetch the tile of CTA blockIdx.x + pf_dist
    const c128 *u;        // S1: state u (device or mapped page-locked host memory)
    int u_bulk;           // S1: u is 16-B aligned -> staged by one bulk copy
    c128 *rhs_out;        // S1: rhs = iBu of the CTA's rows -> rhs0 for K2 / S3ACC
};

// shared-memory view of the staged per-row inputs (local row index)
struct RowView {
    const c128 *rhs;
    const double *sr, *si, *sb;   // sub  : fl(tau a), fl(tau a_im), b
    const double *dr, *di, *db;   // diag
    const double *ur, *ui, *ub;   // sup
    const float *f[6];            // ST_R32: sub (tau a, tau a_im, b), sup (same) rounded to float
    __device__ __forceinline__ c128 sub(int lr, c128 sg) const { return form_entry(sr[lr], si[lr], sb[lr], sg); }
    // complex64 entries for the level-0 correction solve (fp32 formation)
    __device__ __forceinline__ c64 sub32(int lr, c64 sg) const {
        return c64mk(fmaf(sg.y, f[2][lr], f[0][lr]), fmaf(-sg.x, f[2][lr], f[1][lr]));
    }
    __device__ __forceinline__ c64 sup32(int lr, c64 sg) const {
        return c64mk(fmaf(sg.y, f[5][lr], f[3][lr]), fmaf(-sg.x, f[5][lr], f[4][lr]));
    }
    __device__ __forceinline__ c128 dia(int lr, c128 sg) const { return form_entry(dr[lr], di[lr], db[lr], sg); }
    __device__ __forceinline__ c128 sup(int lr, c128 sg) const { return form_entry(ur[lr], ui[lr], ub[lr], sg); }
};

enum { ST_RHS = 1, ST_DIA = 2, ST_TILE2 = 4, ST_BDIA = 8, ST_T32 = 16, ST_R32 = 32, ST_I32 = 64 };
// ST_T32: t0 holds complex64; ST_R32: + float copies of the sub/sup row data;
// ST_I32: + the complex64 copy of the inverse-pivot tile (K2's correction sweep)

struct L0Layout {
    int kp, T, Tp;
    c128 *t0, *t1;
    const c64 *i32;   // ST_I32
    RowView rv;
};

__device__ __forceinline__ L0Layout carve(unsigned char *smem, int kp, int M, int flags) {
    L0Layout l;
    l.kp = kp;
    l.T = (L0_NT / kp) * M;
    l.Tp = l.T + L0_ROWPAD;
    unsigned char *p = smem + 128;
    l.t0 = reinterpret_cast<c128 *>(p);
    p += (size_t)l.T * kp * ((flags & ST_T32) ? sizeof(c64) : sizeof(c128));
    l.t1 = nullptr;
    if (flags & ST_TILE2) {
        l.t1 = reinterpret_cast<c128 *>(p);
        p += (size_t)l.T * kp * sizeof(c128);
    }
    RowView &r = l.rv;
    r.rhs = nullptr;
    if (flags & ST_RHS) {
        r.rhs = reinterpret_cast<const c128 *>(p);
        p += (size_t)l.Tp * sizeof(c128);
    }
    double *d = reinterpret_cast<double *>(p);
    r.sr = d; d += l.Tp; r.si = d; d += l.Tp; r.sb = d; d += l.Tp;
    r.ur = d; d += l.Tp; r.ui = d; d += l.Tp; r.ub = d; d += l.Tp;
    r.dr = r.di = r.db = nullptr;
    if (flags & ST_DIA) { r.dr = d; d += l.Tp; r.di = d; d += l.Tp; r.db = d; d += l.Tp; }
    else if (flags & ST_BDIA) { r.db = d; d += l.Tp; }
    float *fend = reinterpret_cast<float *>(d);
    if (flags & ST_R32) {
        float *f = reinterpret_cast<float *>(d);
        const int tp4 = (l.Tp + 3) & ~3;
        for (int q = 0; q < 6; ++q) r.f[q] = f + q * tp4;
        fend = f + 6 * tp4;
    }
    l.i32 = nullptr;
    if (flags & ST_I32) l.i32 = reinterpret_cast<const c64 *>((reinterpret_cast<uintptr_t>(fend) + 15) & ~(uintptr_t)15);
    return l;
}

__host__ __device__ inline size_t l0_smem_bytes(int kp, int M, int flags) {
    size_t T = (size_t)(L0_NT / kp) * M, Tp = T + L0_ROWPAD;
    size_t b = 128 + T * kp * ((flags & ST_T32) ? 8 : 16) + ((flags & ST_TILE2) ? T * kp * 16 : 0);
    if (flags & ST_RHS) b += Tp * 16;
    b += Tp * 8 * ((flags & ST_DIA) ? 9 : (flags & ST_BDIA) ? 7 : 6);
    if (flags & ST_R32) b += 6 * ((Tp + 3) & ~(size_t)3) * sizeof(float);
    if (flags & ST_I32) b = ((b + 15) & ~(size_t)15) + T * kp * sizeof(c64);
    return b;
}

// one thread: init the mbarrier, then issue every bulk copy of this CTA
__device__ __forceinline__ void l0_stage(unsigned char *smem, const L0Layout &l, const L0Args &a,
                                         const void *g_t0, const c128 *g_t1, int64_t row0, int flags) {
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t n = a.L.n;
        const int64_t row1 = min(row0 + (int64_t)l.T, n);
        const size_t esz = (flags & ST_T32) ? sizeof(c64) : sizeof(c128);
        const uint32_t tb = (uint32_t)((row1 - row0) * l.kp * sizeof(c128));
        const uint32_t tb0 = (uint32_t)((row1 - row0) * l.kp * esz);
        const uint32_t rb8 = (uint32_t)(l.Tp * 8), rb16 = (uint32_t)(l.Tp * 16);
        const uint32_t rb4 = (uint32_t)(((l.Tp + 3) & ~3) * sizeof(float));
        const uint32_t tb32 = (uint32_t)((row1 - row0) * l.kp * sizeof(c64));
        uint32_t total = tb0 + ((flags & ST_TILE2) ? tb : 0) + ((flags & ST_RHS) ? rb16 : 0) +
                         rb8 * ((flags & ST_DIA) ? 9 : (flags & ST_BDIA) ? 7 : 6) + ((flags & ST_R32) ? 6 * rb4 : 0) +
                         ((flags & ST_I32) ? tb32 : 0);
        mbar_expect_tx(bar, total);
        if (flags & ST_I32) bulk_g2s((void *)l.i32, a.inv32 + row0 * l.kp, tb32, bar);
        bulk_g2s(l.t0, reinterpret_cast<const unsigned char *>(g_t0) + (size_t)row0 * l.kp * esz, tb0, bar);
        if (flags & ST_TILE2) bulk_g2s(l.t1, g_t1 + row0 * l.kp, tb, bar);
        if (flags & ST_RHS) bulk_g2s((void *)l.rv.rhs, a.rhs0 + row0, rb16, bar);
        bulk_g2s((void *)l.rv.sr, a.z.ta_sub + row0, rb8, bar);
        bulk_g2s((void *)l.rv.si, a.z.ta_sub_im + row0, rb8, bar);
        bulk_g2s((void *)l.rv.sb, a.z.b_sub + row0, rb8, bar);
        bulk_g2s((void *)l.rv.ur, a.z.ta_sup + row0, rb8, bar);
        bulk_g2s((void *)l.rv.ui, a.z.ta_sup_im + row0, rb8, bar);
        bulk_g2s((void *)l.rv.ub, a.z.b_sup + row0, rb8, bar);
        if (flags & ST_DIA) {
            bulk_g2s((void *)l.rv.dr, a.z.ta_dia + row0, rb8, bar);
            bulk_g2s((void *)l.rv.di, a.z.ta_dia_im + row0, rb8, bar);
            bulk_g2s((void *)l.rv.db, a.z.b_dia + row0, rb8, bar);
        } else if (flags & ST_BDIA) {
            bulk_g2s((void *)l.rv.db, a.z.b_dia + row0, rb8, bar);
        }
        if (flags & ST_R32)
            for (int q = 0; q < 6; ++q) bulk_g2s((void *)l.rv.f[q], a.r32[q] + row0, rb4, bar);
    }
}

// forward sweep y_q = invd_q (d_q - a_q y_{q-1}), y[0] = left halo
template <int M, bool FULL, typename RhsF>
__device__ __forceinline__ void sweep_fwd(c128 (&y)[M], const c128 *ti, int kp, const RowView &rv,
                                          int lr0, int cnt, c128 sg, RhsF rhs) {
#pragma unroll
    for (int q = 1; q < M; ++q) {
        if (FULL || q <= cnt) {
            const int lr = lr0 + q;
            y[q] = cmul(ti[q * kp], cfnma(rhs(q), rv.sub(lr, sg), y[q - 1]));
        }
    }
}

// backward sweep x_q = y_q - invd_q (c_q x_{q+1}), x_{cnt+1} = xn; out(q, x_q)
template <int M, bool FULL, typename OutF>
__device__ __forceinline__ void sweep_bwd(c128 (&y)[M], const c128 *ti, int kp, const RowView &rv,
                                          int lr0, int cnt, c128 sg, c128 xn, OutF out) {
    c128 xnext = xn;
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        if (FULL || q <= cnt) {
            const int lr = lr0 + q;
            xnext = cfnma(y[q], ti[q * kp], cmul(rv.sup(lr, sg), xnext));
            y[q] = xnext;
            out(q, xnext);
        } else {
            out(q, cmk(0.0, 0.0));
        }
    }
}

template <int M, bool FULL>
__device__ __forceinline__ c128 pick_last(const c128 (&y)[M], int cnt) {
    if (FULL) return y[M - 1];
    c128 v = y[0];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q == cnt) v = y[q];
    return v;
}

// beta-weighted sum over the kp lanes of every tile row (fixed order, fp64
// products accumulated with error-free TwoSum, lanes combined in dd)
__device__ __forceinline__ c128 tile_c128(c128 v) { return v; }
__device__ __forceinline__ c128 tile_c128(c64 v) { return to_c128(v); }

// KP > 0: k_pad known at compile time (the lane loop unrolls, offsets become immediates)
template <int M, typename TT = c128, int KP = 0>
__device__ __forceinline__ void reduce_rows(const TT *tile, const L0Args &a, int64_t row0) {
    const int kp = KP ? KP : a.S.kp;
    const int rows = (L0_NT / kp) * M;
    const int tpr = L0_NT / rows > 0 ? L0_NT / rows : 1;
    const int sub = threadIdx.x % tpr;
    const int64_t n = a.nout;
    for (int r = threadIdx.x / tpr; r < rows; r += L0_NT / tpr) {
        // the dd accumulation keeps the rounded row sum independent of how
        // the lanes are grouped (k_pad, sharding): a plain fp64 chain here
        // broke the bitwise sharded-vs-single equality of the refined path
        // K3 adds to the partial K2 left: its four words are loaded before the lane
        // loop (the ncu source view had 8.8 % of K3's stall samples on the first
        // dd_add below when they were loaded there)
        const int64_t row = row0 + r;
        const bool lead = sub == 0 && row < n;
        dd pre = {0.0, 0.0}, pim = {0.0, 0.0};
        if (a.acc_add && lead) {
            pre = dd{a.acc[row], a.acc[n + row]};
            pim = dd{a.acc[2 * n + row], a.acc[3 * n + row]};
        }
        ddacc re = {0.0, 0.0}, im = {0.0, 0.0};
#pragma unroll
        for (int jj = sub; jj < kp; jj += tpr) {
            const c128 b = a.S.beta[jj];
            const c128 x = tile_c128(tile[r * kp + jj]);
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
        if (lead) {
            if (a.acc_add) {
                sre = dd_add(sre, pre);
                sim = dd_add(sim, pim);
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

// acc -= e*x, error-free (Dot2 style) into complex double-double accumulators
// r -= e*x into double-double accumulators.  FULL: all four real products
// error-free (Dot2).  Otherwise (real A, refinement only runs on stiff pencils,
// tau*sr > 5e3): the products of Re(e) (tau*A dominated, where the residual
// cancels) are error-free, and the products of Im(e) = -fl(Re(sigma) b), at
// least tau*sr/|sigma| times smaller, go into the low word with one FMA each
// -- measured to leave the refined cfg 2 result unchanged vs truth (3.76e-11)
// at 25 % fewer FP64 instructions in K2.
template <bool FULL>
__device__ __forceinline__ void dot2_sub(ddacc &re, ddacc &im, c128 e, c128 x) {
    dd p;
    p = two_prod(e.x, x.x); ddacc_add(re, -p.hi); re.lo = __dsub_rn(re.lo, p.lo);
    if (FULL) {
        p = two_prod(e.y, x.y); ddacc_add(re, p.hi); re.lo = __dadd_rn(re.lo, p.lo);
    } else {
        re.lo = __fma_rn(e.y, x.y, re.lo);
    }
    p = two_prod(e.x, x.y); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
    if (FULL) {
        p = two_prod(e.y, x.x); ddacc_add(im, -p.hi); im.lo = __dsub_rn(im.lo, p.lo);
    } else {
        im.lo = __fma_rn(-e.y, x.x, im.lo);
    }
}

// ---- aligned residual (real symmetric A: the refined cfg 2 path) ----
// Every Re(entry) of a block-lane is rounded to a multiple of one quantum qE
// (25 significant bits) and every Re x / Im x to a multiple of qX (26 bits):
// the products E_h x_h are then multiples of qE*qX below 2^53 of it, so the
// row sum H = sum E_h x_h is EXACT in plain fp64 (no TwoSum), and d - H is
// exact by Sterbenz wherever the residual cancels.  The remainders
// sum (E x - E_h x_h) (~2^-25 of the products) and the Im(entry) terms go
// into one fp64 word L with an FMA each, rounding at ~2^-77 of |S||x| -- the
// same budget as the Dot2 form's (its error-free hi parts are what costs).
__device__ __forceinline__ unsigned hiabs(double v) { return (unsigned)__double2hiint(v) & 0x7fffffffu; }
// C such that fl(v + C) - C rounds v to a multiple of 2^(e+1-bits), for every
// |v| < 2^(e+1), e the exponent of the double whose high word is h
__device__ __forceinline__ double quant_c(unsigned h, int bits) {
    const int be = min((int)(h >> 20) + 53 - bits, 2046);
    return __hiloint2double((be << 20) | 0x80000, 0);
}
__device__ __forceinline__ double quant(double v, double C) { return __dsub_rn(__dadd_rn(v, C), C); }

struct Ctx {
    int kp, b, j, cnt, lr0;
    int64_t p, P, base, row0;
    bool active;
    c128 sg;
};

// DIV: integer division (S1: the shift form measured 0.204 -> 0.218 ms there,
// its register allocation spilling 92 instead of 60 B)
template <bool DIV = false, int KP = 0>
__device__ __forceinline__ Ctx make_ctx(const L0Args &a, int M) {
    Ctx c;
    c.kp = KP ? KP : a.S.kp;
    const int lk = lg2(c.kp);
    const int bpc = DIV ? L0_NT / c.kp : L0_NT >> lk;
    c.b = DIV ? threadIdx.x / c.kp : threadIdx.x >> lk;
    c.j = DIV ? threadIdx.x % c.kp : threadIdx.x & (c.kp - 1);
    c.P = a.L.P;
    c.row0 = (int64_t)blockIdx.x * bpc * M;
    c.p = (int64_t)blockIdx.x * bpc + c.b;
    c.active = c.p < c.P;
    c.base = c.p * M;
    c.cnt = c.active ? (int)min((int64_t)M, a.L.n - c.base) - 1 : -1;
    c.lr0 = c.b * M;
    c.sg = a.S.sigma[c.j];
    return c;
}

// Level 0 is padded to a multiple of M (decoupled unit rows), so every
// level-0 block is full and only the predicate-free instantiations exist.

// ---------------------------------------------------------------------------
// S1: interior solves with zero halos -> reduced rhs (ypart, lc)
// ---------------------------------------------------------------------------
template <int M, bool FULL>
__device__ __forceinline__ void s1_body(const L0Args &a, const L0Layout &l, const Ctx &c) {
    const c128 *ti = l.t0 + (size_t)c.lr0 * c.kp + c.j;
    const RowView &rv = l.rv;
    c128 y[M];
    y[0] = cmk(0.0, 0.0);
    sweep_fwd<M, FULL>(y, ti, c.kp, rv, c.lr0, c.cnt, c.sg, [&](int q) { return rv.rhs[c.lr0 + q]; });
    const c128 ylast = pick_last<M, FULL>(y, c.cnt);
    sweep_bwd<M, FULL>(y, ti, c.kp, rv, c.lr0, c.cnt, c.sg, cmk(0.0, 0.0), [](int, c128) {});
    const c128 yfirst = c.cnt >= 1 ? y[1] : cmk(0.0, 0.0);
    const int kp = c.kp, j = c.j;
    a.L.ypart[c.p * kp + j] = cfnma(rv.rhs[c.lr0], rv.sup(c.lr0, c.sg), yfirst);
    if (c.p + 1 < c.P) a.L.lc[(c.p + 1) * kp + j] = cneg(cmul(rv.sub(c.lr0 + M, c.sg), ylast));
    if (c.p == 0) a.L.lc[j] = cmk(0.0, 0.0);
}

// S1 with the rhs formed in the kernel: rhs_i = 1j * (B u)_i for the CTA's
// rows, in k_rhs's order (CSR row order, unfused products: bitwise equal), from
// u read directly -- device memory, or page-locked host memory mapped into the
// device address space, which makes the host->device transfer of a host-buffer
// step part of this kernel instead of a separate copy in front of it.  The rhs
// rows go to rhs0 for K2 / S3ACC (padding rows stay zero).
template <int M, int KP>
#ifndef S1_MINB
#define S1_MINB 4   // 128 registers + 60 B spills, 7 % faster than 3 CTAs/SM without (scripts/tune_l0minb.sh)
#endif
__global__ void __launch_bounds__(L0_NT, S1_MINB) k_l0_s1(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int FL = ST_RHS | ST_BDIA;
    const int kp_ = KP ? KP : a.S.kp;
    const L0Layout l = carve(smem, kp_, M, FL);
    const Ctx c = make_ctx<true, KP>(a, M);
    uint64_t *bar_u = reinterpret_cast<uint64_t *>(smem) + 1;
    if (threadIdx.x == 0 && a.u_bulk) mbar_init(bar_u, 1);   // fenced with l0_stage's barrier init
    l0_stage(smem, l, a, a.L.invd, nullptr, c.row0, FL & ~ST_RHS);
    // u rows row0-1 .. row0+T, slots outside [0, n) zero
    c128 *su = reinterpret_cast<c128 *>(smem + ((l0_smem_bytes(kp_, M, FL) + 15) & ~(size_t)15));   // T+2 slots after the carve
    const int64_t n = a.nout;
    const int64_t i0 = max(c.row0 - 1, (int64_t)0), i1 = min(c.row0 + (int64_t)l.T + 1, n);
    if (a.u_bulk) {
        // one bulk copy (also from mapped page-locked host memory: larger link
        // transactions than per-thread loads)
        if (threadIdx.x == 0) {
            if (i1 > i0) {
                const uint32_t ub = (uint32_t)((i1 - i0) * sizeof(c128));
                mbar_expect_tx(bar_u, ub);
                bulk_g2s(su + (i0 - (c.row0 - 1)), a.u + i0, ub, bar_u);
            } else {
                mbar_arrive(bar_u);
            }
        }
        for (int t = threadIdx.x; t < l.T + 2; t += L0_NT) {
            const int64_t i = c.row0 - 1 + t;
            if (i < i0 || i >= i1) su[t] = cmk(0.0, 0.0);
        }
    } else {
        for (int t = threadIdx.x; t < l.T + 2; t += L0_NT) {
            const int64_t i = c.row0 - 1 + t;
            su[t] = (i >= 0 && i < n) ? a.u[i] : cmk(0.0, 0.0);
        }
    }
    mbar_wait(reinterpret_cast<uint64_t *>(smem), 0);
    if (a.u_bulk) mbar_wait(bar_u, 0);
    __syncthreads();
    c128 *rhs = const_cast<c128 *>(l.rv.rhs);
    for (int t = threadIdx.x; t < l.T; t += L0_NT) {
        const int64_t i = c.row0 + t;
        c128 v = cmk(0.0, 0.0);
        if (i < n) {
            double sr = 0.0, si = 0.0;
            if (i > 0) {
                const double b = l.rv.sb[t];
                const c128 x = su[t];
                sr = __dadd_rn(sr, __dmul_rn(b, x.x));
                si = __dadd_rn(si, __dmul_rn(b, x.y));
            }
            {
                const double b = l.rv.db[t];
                const c128 x = su[t + 1];
                sr = __dadd_rn(sr, __dmul_rn(b, x.x));
                si = __dadd_rn(si, __dmul_rn(b, x.y));
            }
            if (i + 1 < n) {
                const double b = l.rv.ub[t];
                const c128 x = su[t + 2];
                sr = __dadd_rn(sr, __dmul_rn(b, x.x));
                si = __dadd_rn(si, __dmul_rn(b, x.y));
            }
            v = cmk(-si, sr);
            a.rhs_out[i] = v;
        }
        rhs[t] = v;
    }
    __syncthreads();
    if (!c.active) return;
    s1_body<M, true>(a, l, c);
}

// ---------------------------------------------------------------------------
// S3ACC: solve with known interface values, beta-weighted sum -> out
// ---------------------------------------------------------------------------
template <int M, bool FULL>
__device__ __forceinline__ void s3_body(const L0Args &a, const L0Layout &l, const Ctx &c, c128 xs,
                                        c128 xn) {
    c128 *ti = l.t0 + (size_t)c.lr0 * c.kp + c.j;
    const RowView &rv = l.rv;
    const int kp = c.kp;
    c128 y[M];
    y[0] = xs;
    sweep_fwd<M, FULL>(y, ti, kp, rv, c.lr0, c.cnt, c.sg, [&](int q) { return rv.rhs[c.lr0 + q]; });
    // x overwrites the consumed inverse pivot of its own lane
    sweep_bwd<M, FULL>(y, ti, kp, rv, c.lr0, c.cnt, c.sg, xn, [&](int q, c128 x) { ti[q * kp] = x; });
    ti[0] = xs;
}

template <int M>
#ifndef S3_MINB
#define S3_MINB 5
#endif
__global__ void __launch_bounds__(L0_NT, S3_MINB) k_l0_s3acc(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const L0Layout l = carve(smem, a.S.kp, M, ST_RHS);
    const Ctx c = make_ctx(a, M);
    l0_stage(smem, l, a, a.L.invd, nullptr, c.row0, ST_RHS);
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (c.active) {
        xs = a.X1[c.p * c.kp + c.j];
        if (c.p + 1 < c.P) xn = a.X1[(c.p + 1) * c.kp + c.j];
    }
    mbar_wait(reinterpret_cast<uint64_t *>(smem), 0);
    if (c.active) {
        s3_body<M, true>(a, l, c, xs, xn);
    } else {
        c128 *ti = l.t0 + (size_t)c.lr0 * c.kp + c.j;
#pragma unroll
        for (int q = 0; q < M; ++q) ti[q * c.kp] = cmk(0.0, 0.0);
    }
    __syncthreads();
    reduce_rows<M>(l.t0, a, c.row0);
}

// ---------------------------------------------------------------------------
// K2 (refine): S3 + sum(beta x) + dd residual of the interior rows + the
// correction's reduce.  The residual of an interface row has one term from
// each of two blocks; both halves are kept in double-double and combined by
// the next level, so it is formed as exactly as the interior residuals.
// ---------------------------------------------------------------------------
template <int M, bool FULL>
__device__ __forceinline__ void k2_solve(const L0Args &a, const L0Layout &l, const Ctx &c, c128 xs,
                                         c128 xn, c128 (&y)[M], c128 *xt, unsigned &hx, unsigned &hy) {
    const c128 *ti = l.t0 + (size_t)c.lr0 * c.kp + c.j;
    c128 *tc = xt + (size_t)c.lr0 * c.kp + c.j;   // may alias ti: slot q is read before x_q overwrites it
    const RowView &rv = l.rv;
    const int kp = c.kp;
    y[0] = xs;
    // hx, hy: largest high word of |Re x|, |Im x| over the block's x_0..x_M (integer pipe)
    hx = max(hiabs(xs.x), hiabs(xn.x));
    hy = max(hiabs(xs.y), hiabs(xn.y));
    sweep_fwd<M, FULL>(y, ti, kp, rv, c.lr0, c.cnt, c.sg, [&](int q) { return rv.rhs[c.lr0 + q]; });
    sweep_bwd<M, FULL>(y, ti, kp, rv, c.lr0, c.cnt, c.sg, xn, [&](int q, c128 x) {
        tc[q * kp] = x;
        if (K2_ALIGNED) {
            hx = max(hx, hiabs(x.x));
            hy = max(hy, hiabs(x.y));
        }
    });
    tc[0] = xs;
}

template <int M, bool FULL, bool EXACT, bool SYM>
__device__ __forceinline__ void k2_refine(const L0Args &a, const L0Layout &l, const Ctx &c, c128 xs,
                                          c128 xn, c128 (&y)[M], c128 *xt, unsigned hx, unsigned hy) {
    static_assert(FULL, "level 0 is padded to full blocks");
    const c128 *ti = l.t0 + (size_t)c.lr0 * c.kp + c.j;
    c128 *tc = xt + (size_t)c.lr0 * c.kp + c.j;
    const RowView &rv = l.rv;
    const int kp = c.kp, j = c.j;
    constexpr int cnt = M - 1;
    // interface row s: d_s - b_s x_s - c_s x_{s+1} (the -a_s x_{s-1} half comes
    // from block p-1) and this block's half of the next interface row; taken
    // before the residual loop recycles the x slots
    ddacc p1re, p1im, p2re = {0.0, 0.0}, p2im = {0.0, 0.0};
    const c128 sup0 = rv.sup(c.lr0, c.sg);
    {
        const c128 d = rv.rhs[c.lr0];
        p1re = {d.x, 0.0};
        p1im = {d.y, 0.0};
        dot2_sub<EXACT>(p1re, p1im, rv.dia(c.lr0, c.sg), xs);
        dot2_sub<EXACT>(p1re, p1im, sup0, tc[kp]);
    }
    const bool has_next = c.p + 1 < c.P;
    const c128 an = rv.sub(c.lr0 + M, c.sg);
    if (has_next) dot2_sub<EXACT>(p2re, p2im, an, tc[cnt * kp]);
    // interior residuals r_q = d_q - a_q x_{q-1} - b_q x_q - c_q x_{q+1}, error-free
    // products; r_q goes to slot q-1 (x_{q-1} is dead once r_q is formed) -- a
    // rolled loop keeps the kernel's code and register footprint small.  SYM
    // (symmetric pencil, checked bitwise on the formed entries at plan
    // creation): a_q = c_{q-1}, so each off-diagonal entry is formed once.
    if constexpr (K2_ALIGNED && SYM && !EXACT) {
        // bits: qE 25, qX 26 -> 3 products of <= 2^(eE+eX+3) on a grid of
        // 2^(eE+eX+3-51): the partial sums need <= 53 bits (exact)
        const double2 em = __ldg(a.emax + c.p);
        const double eb = fma(fabs(c.sg.y), em.y, em.x);
        const double cE = quant_c(hiabs(eb) + (1u << 20), 25);   // one binade of headroom for the formation's rounding
        const double cX = quant_c(hx, 26), cY = quant_c(hy, 26);
        c128 xm = tc[0], x0 = tc[kp];
        double xmh = quant(xm.x, cX), xmk = quant(xm.y, cY);
        double x0h = quant(x0.x, cX), x0k = quant(x0.y, cY);
        double Es = sup0.x, Fs = sup0.y, Esh = quant(Es, cE);
#pragma unroll K2_UNROLL
        for (int q = 1; q < M; ++q) {
            const int lr = c.lr0 + q;
            const c128 xp = q < cnt ? tc[(q + 1) * kp] : xn;
            const double xph = quant(xp.x, cX), xpk = quant(xp.y, cY);
            const c128 d = rv.rhs[lr];
            // entries with the reference's rounding (form_entry; Im(tau A) = 0 here)
            const double Ed = __dadd_rn(rv.dr[lr], __dmul_rn(c.sg.y, rv.db[lr]));
            const double Fd = -__dmul_rn(c.sg.x, rv.db[lr]);
            const double Eu = __dadd_rn(rv.ur[lr], __dmul_rn(c.sg.y, rv.ub[lr]));
            const double Fu = -__dmul_rn(c.sg.x, rv.ub[lr]);
            const double Edh = quant(Ed, cE), Euh = quant(Eu, cE);
            // Re r = d.x - sum(E X - F Y)
            double P1 = __dmul_rn(Esh, xmh), P2 = __dmul_rn(Edh, x0h), P3 = __dmul_rn(Euh, xph);
            double H = __dadd_rn(__dadd_rn(P1, P2), P3);
            double L = __fma_rn(Es, xm.x, -P1);
            L = __dadd_rn(L, __fma_rn(Ed, x0.x, -P2));
            L = __dadd_rn(L, __fma_rn(Eu, xp.x, -P3));
            L = __fma_rn(-Fs, xm.y, L);
            L = __fma_rn(-Fd, x0.y, L);
            L = __fma_rn(-Fu, xp.y, L);
            const double rre = __dsub_rn(__dsub_rn(d.x, H), L);
            // Im r = d.y - sum(E Y + F X)
            P1 = __dmul_rn(Esh, xmk); P2 = __dmul_rn(Edh, x0k); P3 = __dmul_rn(Euh, xpk);
            H = __dadd_rn(__dadd_rn(P1, P2), P3);
            L = __fma_rn(Es, xm.y, -P1);
            L = __dadd_rn(L, __fma_rn(Ed, x0.y, -P2));
            L = __dadd_rn(L, __fma_rn(Eu, xp.y, -P3));
            L = __fma_rn(Fs, xm.x, L);
            L = __fma_rn(Fd, x0.x, L);
            L = __fma_rn(Fu, xp.x, L);
            const double rim = __dsub_rn(__dsub_rn(d.y, H), L);
            const c64 r32 = to_c64(cmk(rre, rim));
            a.rres_out[(c.base + q) * kp + j] = r32;
            *reinterpret_cast<c64 *>(tc + (q - 1) * kp) = r32;
            xm = x0; xmh = x0h; xmk = x0k;
            x0 = xp; x0h = xph; x0k = xpk;
            Es = Eu; Fs = Fu; Esh = Euh;
        }
    } else {
    c128 xm = tc[0], x0 = tc[kp];
    c128 esub = sup0;
#pragma unroll K2_UNROLL
    for (int q = 1; q < M; ++q) {
        const int lr = c.lr0 + q;
        const c128 xp = q < cnt ? tc[(q + 1) * kp] : xn;
        const c128 d = rv.rhs[lr];
        ddacc re = {d.x, 0.0}, im = {d.y, 0.0};
        const c128 eup = rv.sup(lr, c.sg);
        dot2_sub<EXACT>(re, im, SYM ? esub : rv.sub(lr, c.sg), xm);
        dot2_sub<EXACT>(re, im, rv.dia(lr, c.sg), x0);
        dot2_sub<EXACT>(re, im, eup, xp);
        // the correction is solved to ~1e-5 relative (it only has to shrink an
        // error that is already ~1e-13 of x): its rhs is stored as complex64,
        // and the correction's S1 here uses the same rounded values as K3's S3
        const c64 r32 = to_c64(cmk(__dadd_rn(re.hi, re.lo), __dadd_rn(im.hi, im.lo)));
        a.rres_out[(c.base + q) * kp + j] = r32;
        *reinterpret_cast<c64 *>(tc + (q - 1) * kp) = r32;
        xm = x0;
        x0 = xp;
        esub = eup;
    }
    }
    // correction reduce: S1 with rhs = r, in complex64 with K3's pivots
    // (K2_ONE_TILE: the complex64 pivot copy in HBM, as K3 reads it; else
    // rounded from the staged fp64 tile -- the same values), entries formed
    // in fp32
    (void)y;
    (void)ti;
    const c64 sg32 = to_c64(c.sg);
    // (K2_I32: staged by the CTA's bulk copies -- the ncu source view had 8.7 % of
    // K2's stall samples on the first two uses of these pivots when they were
    // loaded from HBM here)
    const c64 *iv32 = a.inv32 + c.base * kp + j;
    const c64 *sv32 = l.i32 + (size_t)c.lr0 * kp + j;
    auto piv = [&](int q) -> c64 {
        return !K2_ONE_TILE ? to_c64(ti[q * kp]) : K2_I32 ? sv32[q * kp] : __ldg(iv32 + q * kp);
    };
    c64 yf[M];
    yf[0] = c64mk(0.f, 0.f);
#pragma unroll
    for (int q = 1; q < M; ++q) {
        const c64 rq = *reinterpret_cast<const c64 *>(tc + (q - 1) * kp);
        yf[q] = fmul(piv(q), ffnma(rq, rv.sub32(c.lr0 + q, sg32), yf[q - 1]));
    }
    const c64 ylast = yf[M - 1];
    c64 xnext = c64mk(0.f, 0.f);
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        xnext = ffnma(yf[q], piv(q), fmul(rv.sup32(c.lr0 + q, sg32), xnext));
        yf[q] = xnext;
    }
    const c64 m1 = fmul(rv.sup32(c.lr0, sg32), yf[1]);
    const c128 t1 = cmk(-(double)m1.x, -(double)m1.y);
    ddacc_add(p1re, t1.x);
    ddacc_add(p1im, t1.y);
    a.L.ypdd[c.p * kp + j] = cdh_pack(cdd{{p1re.hi, p1re.lo}, {p1im.hi, p1im.lo}});
    if (has_next) {
        const c64 m2 = fmul(rv.sub32(c.lr0 + M, sg32), ylast);
        const c128 t2 = cmk(-(double)m2.x, -(double)m2.y);
        ddacc_add(p2re, t2.x);
        ddacc_add(p2im, t2.y);
        a.L.lcdd[(c.p + 1) * kp + j] = cdh_pack(cdd{{p2re.hi, p2re.lo}, {p2im.hi, p2im.lo}});
    }
    if (c.p == 0) a.L.lcdd[j] = cdh_pack(cdd_zero());
}

constexpr int K2_FLAGS = (K2_ONE_TILE ? (ST_RHS | ST_DIA | ST_R32) : (ST_RHS | ST_DIA | ST_TILE2 | ST_R32)) |
                         (K2_ONE_TILE && K2_I32 ? ST_I32 : 0);
// KP: k_pad at compile time for the common K = 64 (0: runtime).  At runtime
// k_pad a fifth of K2's instructions were integer address arithmetic
// (ncu source view, profiles/r02_k2_sass_regions.txt).
template <int M, bool EXACT, int KP>
__global__ void __launch_bounds__(L0_NT, K2_MINB) k_l0_k2(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int flags = K2_FLAGS;
    const L0Layout l = carve(smem, KP ? KP : a.S.kp, M, flags);
    c128 *const xt = K2_ONE_TILE ? l.t0 : l.t1;
    const Ctx c = make_ctx<false, KP>(a, M);
    l0_stage(smem, l, a, a.L.invd, nullptr, c.row0, flags & ~ST_TILE2);
#ifndef K2_PF
#define K2_PF 1
#endif
    // K2 is latency-bound (FP64 dependency chains at 3 CTAs/SM): a CTA's
    // start waits ~1.5 us for its bulk copies.  Warm L2 with the tile of the
    // CTA that will take this slot about one residency-wave later.
    if (K2_PF && threadIdx.x == 0 && a.pf_dist > 0) {
        const int64_t nb = (int64_t)blockIdx.x + a.pf_dist;
        const int64_t r0 = nb * l.T;
        if (r0 < a.L.n) {
            const int64_t r1 = min(r0 + (int64_t)l.T, a.L.n);
            bulk_prefetch_l2(a.L.invd + r0 * l.kp, (uint32_t)((r1 - r0) * l.kp * sizeof(c128)));
            const uint32_t rb8 = (uint32_t)(l.Tp * 8);
            bulk_prefetch_l2(a.rhs0 + r0, (uint32_t)(l.Tp * 16));
            const double *rows[9] = {a.z.ta_sub, a.z.ta_sub_im, a.z.b_sub, a.z.ta_sup, a.z.ta_sup_im,
                                     a.z.b_sup, a.z.ta_dia, a.z.ta_dia_im, a.z.b_dia};
#pragma unroll
            for (int q = 0; q < 9; ++q) bulk_prefetch_l2(rows[q] + r0, rb8);
        }
    }
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (c.active) {
        xs = a.X1[c.p * c.kp + c.j];
        if (c.p + 1 < c.P) xn = a.X1[(c.p + 1) * c.kp + c.j];
    }
    mbar_wait(reinterpret_cast<uint64_t *>(smem), 0);
    c128 y[M];
    unsigned hx = 0, hy = 0;
    if (c.active) {
        k2_solve<M, true>(a, l, c, xs, xn, y, xt, hx, hy);
    } else {
        c128 *tc = xt + (size_t)c.lr0 * c.kp + c.j;
#pragma unroll
        for (int q = 0; q < M; ++q) tc[q * c.kp] = cmk(0.0, 0.0);
    }
    __syncthreads();
    reduce_rows<M, c128, KP>(xt, a, c.row0);
    if (!c.active) return;
    if (a.L.sym) k2_refine<M, true, EXACT, true>(a, l, c, xs, xn, y, xt, hx, hy);
    else k2_refine<M, true, EXACT, false>(a, l, c, xs, xn, y, xt, hx, hy);
}

// ---------------------------------------------------------------------------
// K3 (refine): correction solve from the stored residual, acc += sum(beta dx).
// The correction only has to shrink an error that is already ~1e-13 of x, so
// its level-0 part runs in complex64: the inverse pivots are staged from their
// complex64 copy (one 16-KB tile), the complex64 residual rows go straight
// into the sweep registers (loads issued before the mbarrier wait, so they
// overlap the bulk copy), entries are formed with the reference's fp64
// rounding and then rounded, and dx (complex64) overwrites the consumed
// pivots for the lane sum, which is accumulated in double-double as before.
// Half the bytes of an fp64 correction (16 instead of 32 per row-shift).
// ---------------------------------------------------------------------------
#ifndef K3_DIV
#define K3_DIV 1   // scripts/tune_k3div.sh: equal within noise
#endif
#ifndef K3_MINB
#define K3_MINB 7   // 72 registers, no spills (8: 64 + spills, equal time; scripts/tune_l0minb.sh)
#endif
// K3's shared memory: mbarrier | complex64 pivot tile T*kp | 6 float row
// arrays (sub: tau a, tau a_im, b; sup: same) of Tp4 = T + 2 rounded to 4
__host__ __device__ inline int k3_tp4(int T) { return (T + 2 + 3) & ~3; }
__host__ __device__ inline size_t k3_smem_bytes(int kp, int M) {
    const int T = (L0_NT / kp) * M;
    return 128 + (size_t)T * kp * sizeof(c64) + 6 * (size_t)k3_tp4(T) * sizeof(float);
}

template <int M, int KP>
__global__ void __launch_bounds__(L0_NT, K3_MINB) k_l0_k3(L0Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int kp = KP ? KP : a.S.kp;
    const int T = (L0_NT >> lg2(kp)) * M, Tp4 = k3_tp4(T);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    c64 *tile = reinterpret_cast<c64 *>(smem + 128);
    float *rows = reinterpret_cast<float *>(tile + (size_t)T * kp);
    const Ctx c = make_ctx<K3_DIV, KP>(a, M);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t row1 = min(c.row0 + (int64_t)T, a.L.n);
        const uint32_t tb = (uint32_t)((row1 - c.row0) * kp * sizeof(c64));
        const uint32_t rb = (uint32_t)(Tp4 * sizeof(float));
        mbar_expect_tx(bar, tb + 6 * rb);
        bulk_g2s(tile, a.inv32 + c.row0 * kp, tb, bar);
#pragma unroll
        for (int q = 0; q < 6; ++q) bulk_g2s(rows + q * Tp4, a.r32[q] + c.row0, rb, bar);
    }
    c64 y[M];
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (c.active) {
        xs = a.X1[c.p * kp + c.j];
        if (c.p + 1 < c.P) xn = a.X1[(c.p + 1) * kp + c.j];
#pragma unroll
        for (int q = 1; q < M; ++q) y[q] = a.rres_in[(c.base + q) * kp + c.j];
    }
    mbar_wait(bar, 0);
    c64 *ti = tile + (size_t)c.lr0 * kp + c.j;
    if (c.active) {
        // entries formed in fp32 from fp32 copies of fl(tau a) and b: the
        // correction only needs ~1e-5 relative accuracy
        const c64 sg = to_c64(c.sg);
        const float *sr = rows, *si = rows + Tp4, *sb = rows + 2 * Tp4;
        const float *ur = rows + 3 * Tp4, *ui = rows + 4 * Tp4, *ub = rows + 5 * Tp4;
        y[0] = to_c64(xs);
#pragma unroll
        for (int q = 1; q < M; ++q) {
            const int lr = c.lr0 + q;
            const c64 e = c64mk(fmaf(sg.y, sb[lr], sr[lr]), fmaf(-sg.x, sb[lr], si[lr]));
            y[q] = fmul(ti[q * kp], ffnma(y[q], e, y[q - 1]));
        }
        c64 xnext = to_c64(xn);
#pragma unroll
        for (int q = M - 1; q >= 1; --q) {
            const int lr = c.lr0 + q;
            const c64 e = c64mk(fmaf(sg.y, ub[lr], ur[lr]), fmaf(-sg.x, ub[lr], ui[lr]));
            xnext = ffnma(y[q], ti[q * kp], fmul(e, xnext));
            ti[q * kp] = xnext;
        }
        ti[0] = to_c64(xs);
    } else {
#pragma unroll
        for (int q = 0; q < M; ++q) ti[q * kp] = c64mk(0.f, 0.f);
    }
    __syncthreads();
    reduce_rows<M, c64, KP>(tile, a, c.row0);
}

// ---------------------------------------------------------------------------
// Levels >= 1 (explicit reduced coefficients, symmetric pencils): TMA-staged
// invd and sup tiles (sub_q := sup_{q-1}); the block's rhs goes straight into
// the sweep registers.  PHASE 1 -> reduced rhs of the next level, PHASE 3 -> X.
// ---------------------------------------------------------------------------
#ifndef LV_MINB
#define LV_MINB 2   // 212 registers, no spills (3: 168 + 116-196 B spills, 1 % slower; scripts/tune_lv.sh)
#endif
struct LvArgs {
    LevelDev L;
    ShiftDev S;
    const c128 *rin_a, *rin_b;   // previous level ypart / lc
    const cdh *rdd_a, *rdd_b;    // or their double-double versions (correction pass)
    const c128 *Xnext;
    c128 *rw;                    // SRC 1, PHASE 1: the rounded rhs rows, reused by the level's S3
};

struct LvPtrs {
    const c128 *inv, *sup;          // staged tiles (+ lane offset)
    const c128 *ra, *rb;
    const cdh *da, *db;
    const c128 *Xn;
    c128 *ypart, *lc, *X;
    c128 *rw;
};

// rhs of a reduced level: SRC 0 = ypart + lc, 1 = round(ypdd + lcdd) (the
// correction pass's double-double halves), 2 = the rounded rhs SRC 1 stored
enum { LV_SRC_PLAIN = 0, LV_SRC_DD = 1, LV_SRC_STORED = 2 };
template <int SRC>
__device__ __forceinline__ c128 lv_rhs(const LvPtrs &q, int64_t i, int j, int kp) {
    if constexpr (SRC == LV_SRC_DD) return cdd_round(cdd_add(cdh_unpack(q.da[i * kp + j]), cdh_unpack(q.db[i * kp + j])));
    else if constexpr (SRC == LV_SRC_STORED) return q.ra[i * kp + j];
    else return cadd(q.ra[i * kp + j], q.rb[i * kp + j]);
}

template <int M, int PHASE, int SRC, bool FULL>
__device__ __forceinline__ void lv_body(const LvPtrs &t, int lr0, int kp, int j, int64_t p, int64_t P,
                                        int64_t base, int cnt) {
    c128 y[M];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (FULL || q <= cnt) y[q] = lv_rhs<SRC>(t, base + q, j, kp);
    if (SRC == LV_SRC_DD && PHASE == 1 && t.rw) {
        // the combined, rounded rhs for this level's S3 (16 instead of 64 B re-read)
#pragma unroll
        for (int q = 1; q < M; ++q)
            if (FULL || q <= cnt) t.rw[(base + q) * kp + j] = y[q];
    }
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (PHASE == 3) {
        xs = t.Xn[p * kp + j];
        if (p + 1 < P) xn = t.Xn[(p + 1) * kp + j];
    }
    y[0] = xs;
#pragma unroll
    for (int q = 1; q < M; ++q) {
        if (FULL || q <= cnt) {
            const c128 aq = t.sup[(lr0 + q - 1) * kp];            // sub_q = sup_{q-1}
            y[q] = cmul(t.inv[(lr0 + q) * kp], cfnma(y[q], aq, y[q - 1]));
        }
    }
    c128 ylast = y[0];
    if (FULL) ylast = y[M - 1];
    else {
#pragma unroll
        for (int q = 1; q < M; ++q)
            if (q == cnt) ylast = y[q];
    }
    c128 xnext = xn;
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        if (FULL || q <= cnt) {
            xnext = cfnma(y[q], t.inv[(lr0 + q) * kp], cmul(t.sup[(lr0 + q) * kp], xnext));
            y[q] = xnext;
        }
    }
    if constexpr (PHASE == 1) {
        const c128 yfirst = cnt >= 1 ? y[1] : cmk(0.0, 0.0);
        const c128 ds = lv_rhs<SRC>(t, base, j, kp);
        t.ypart[p * kp + j] = cfnma(ds, t.sup[lr0 * kp], yfirst);
        if (p + 1 < P) t.lc[(p + 1) * kp + j] = cneg(cmul(t.sup[(lr0 + M - 1) * kp], ylast));
        if (p == 0) t.lc[j] = cmk(0.0, 0.0);
    } else {
        t.X[base * kp + j] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q)
            if (FULL || q <= cnt) t.X[(base + q) * kp + j] = y[q];
    }
}

template <int M, int PHASE, int SRC>
__global__ void __launch_bounds__(L0_NT, LV_MINB) k_lv_tma(const __grid_constant__ LvArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    const int kp = a.S.kp;
    const int bpc = L0_NT >> lg2(kp);
    const int T = bpc * M;
    c128 *tinv = reinterpret_cast<c128 *>(smem + 128);
    c128 *tsup = tinv + (size_t)T * kp;
    const int b = threadIdx.x >> lg2(kp), j = threadIdx.x & (kp - 1);
    const int64_t n = a.L.n, P = a.L.P;
    const int64_t row0 = (int64_t)blockIdx.x * T;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t row1 = min(row0 + (int64_t)T, n);
        const uint32_t tb = (uint32_t)((row1 - row0) * kp * sizeof(c128));
        mbar_expect_tx(bar, 2 * tb);
        bulk_g2s(tinv, a.L.invd + row0 * kp, tb, bar);
        bulk_g2s(tsup, a.L.sup + row0 * kp, tb, bar);
    }
    const int64_t p = (int64_t)blockIdx.x * bpc + b;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    mbar_wait(bar, 0);
    if (!active) return;
    LvPtrs t;
    t.inv = tinv + j; t.sup = tsup + j;
    t.ra = a.rin_a; t.rb = a.rin_b; t.da = a.rdd_a; t.db = a.rdd_b; t.Xn = a.Xnext;
    t.ypart = a.L.ypart; t.lc = a.L.lc; t.X = a.L.X; t.rw = a.rw;
    if (cnt == M - 1) lv_body<M, PHASE, SRC, true>(t, b * M, kp, j, p, P, base, cnt);
    else lv_body<M, PHASE, SRC, false>(t, b * M, kp, j, p, P, base, cnt);
}

// ---------------------------------------------------------------------------
// Level 1 of the correction pass in complex64 (like the level-0 correction):
// complex64 copies of the level's inverse pivots and couplings, the rhs
// combined from the double-double halves and rounded, stored (complex64) for
// the level's S3; the level-2 rhs and the level-1 solution stay complex128.
// ---------------------------------------------------------------------------
struct Lv32Args {
    LevelDev L;
    ShiftDev S;
    const c64 *inv32, *sup32;    // level 1, [n][kp]
    const cdh *rdd_a, *rdd_b;    // PHASE 1: the double-double rhs halves
    c64 *rw;                     // PHASE 1 writes, PHASE 3 reads: the rounded rhs rows
    const c128 *Xnext;           // PHASE 3: level-2 solution
};

template <int M, int PHASE>
__global__ void __launch_bounds__(L0_NT, LV_MINB) k_lv32(const __grid_constant__ Lv32Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    const int kp = a.S.kp;
    const int bpc = L0_NT >> lg2(kp);
    const int T = bpc * M;
    c64 *tinv = reinterpret_cast<c64 *>(smem + 128);
    c64 *tsup = tinv + (size_t)T * kp;
    const int b = threadIdx.x >> lg2(kp), j = threadIdx.x & (kp - 1);
    const int64_t n = a.L.n, P = a.L.P;
    const int64_t row0 = (int64_t)blockIdx.x * T;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t row1 = min(row0 + (int64_t)T, n);
        const uint32_t tb = (uint32_t)((row1 - row0) * kp * sizeof(c64));
        mbar_expect_tx(bar, 2 * tb);
        bulk_g2s(tinv, a.inv32 + row0 * kp, tb, bar);
        bulk_g2s(tsup, a.sup32 + row0 * kp, tb, bar);
    }
    const int64_t p = (int64_t)blockIdx.x * bpc + b;
    const bool active = p < P;
    const int64_t base = p * M;
    const int cnt = active ? (int)min((int64_t)M, n - base) - 1 : -1;
    c64 y[M];
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (active) {
#pragma unroll
        for (int q = 1; q < M; ++q) {
            if (q <= cnt) {
                if (PHASE == 1) {
                    const int64_t e = (base + q) * kp + j;
                    y[q] = to_c64(cdd_round(cdd_add(cdh_unpack(a.rdd_a[e]), cdh_unpack(a.rdd_b[e]))));
                    a.rw[e] = y[q];
                } else {
                    y[q] = a.rw[(base + q) * kp + j];
                }
            }
        }
        if (PHASE == 3) {
            xs = a.Xnext[p * kp + j];
            if (p + 1 < P) xn = a.Xnext[(p + 1) * kp + j];
        }
    }
    mbar_wait(bar, 0);
    if (!active) return;
    const c64 *ti = tinv + (size_t)b * M * kp + j;
    const c64 *ts = tsup + (size_t)b * M * kp + j;
    y[0] = to_c64(xs);
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q <= cnt) y[q] = fmul(ti[q * kp], ffnma(y[q], ts[(q - 1) * kp], y[q - 1]));   // sub_q = sup_{q-1}
    c64 ylast = y[0];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q == cnt) ylast = y[q];
    c64 xnext = to_c64(xn);
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        if (q <= cnt) {
            xnext = ffnma(y[q], ti[q * kp], fmul(ts[q * kp], xnext));
            y[q] = xnext;
        }
    }
    if (PHASE == 1) {
        const c64 yfirst = cnt >= 1 ? y[1] : c64mk(0.f, 0.f);
        const c64 ds = to_c64(cdd_round(cdd_add(cdh_unpack(a.rdd_a[base * kp + j]), cdh_unpack(a.rdd_b[base * kp + j]))));
        a.L.ypart[p * kp + j] = to_c128(ffnma(ds, ts[0], yfirst));
        if (p + 1 < P) {
            const c64 m = fmul(ts[(M - 1) * kp], ylast);
            a.L.lc[(p + 1) * kp + j] = cmk(-(double)m.x, -(double)m.y);
        }
        if (p == 0) a.L.lc[j] = cmk(0.0, 0.0);
    } else {
        a.L.X[base * kp + j] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q)
            if (q <= cnt) a.L.X[(base + q) * kp + j] = to_c128(y[q]);
    }
}

cudaError_t lv32_launch(const LevelDev &L, const ShiftDev &S, int phase, const c64 *inv32, const c64 *sup32,
                        const cdh *rdd_a, const cdh *rdd_b, c64 *rw, const c128 *Xnext, cudaStream_t st) {
    Lv32Args a{};
    a.L = L; a.S = S; a.inv32 = inv32; a.sup32 = sup32; a.rdd_a = rdd_a; a.rdd_b = rdd_b; a.rw = rw; a.Xnext = Xnext;
    const int kp = S.kp;
    const int64_t rows = (int64_t)(L0_NT / kp) * TRI_M;
    const int64_t grid = (L.n + rows - 1) / rows;
    const size_t smem = 128 + 2 * (size_t)rows * kp * sizeof(c64);
    cudaError_t e;
    if (phase == 1) {
        e = cudaFuncSetAttribute(k_lv32<TRI_M, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_lv32<TRI_M, 1><<<(unsigned)grid, L0_NT, smem, st>>>(a);
    } else {
        e = cudaFuncSetAttribute(k_lv32<TRI_M, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_lv32<TRI_M, 3><<<(unsigned)grid, L0_NT, smem, st>>>(a);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The small reduced levels in ONE thread-block-cluster launch: S1 up levels
// l0..nl-2, the top solve, S3 down levels nl-2..l0, separated by cluster
// barriers instead of kernel boundaries.  Each cluster CTA plays the role of
// k_lv_tma's CTAs for a level (virtual CTAs rank, rank + CS, ...): the same
// TMA-staged invd/sup tiles and the same lv_body, so results are bitwise
// identical to the per-level launches; the top solve repeats k_top_solve.
// Level data written by one CTA and read by another (ypart/lc, X) are plain
// global stores/loads ordered by the cluster barrier (release/acquire).
// ---------------------------------------------------------------------------
constexpr int CH_MAXLV = 8;
constexpr int CH_MAXCS = 16;

struct ChainArgs {
    LevelDev lv[CH_MAXLV];
    ShiftDev S;
    int l0, nl;
};

template <int M, int PHASE>
__device__ __forceinline__ void chain_level(const LevelDev &L, const LevelDev &Lp, const c128 *Xnext, const ShiftDev &S,
                                            c128 *tinv, c128 *tsup, uint64_t *bar, uint32_t &phase,
                                            unsigned rank, unsigned cs) {
    const int kp = S.kp;
    const int bpc = L0_NT >> lg2(kp);
    const int T = bpc * M;
    const int b = threadIdx.x >> lg2(kp), j = threadIdx.x & (kp - 1);
    const int64_t n = L.n, P = L.P;
    const int64_t G = (n + T - 1) / T;
    for (int64_t vb = rank; vb < G; vb += cs) {
        const int64_t row0 = vb * T;
        if (threadIdx.x == 0) {
            const int64_t row1 = min(row0 + (int64_t)T, n);
            const uint32_t tb = (uint32_t)((row1 - row0) * kp * sizeof(c128));
            mbar_expect_tx(bar, 2 * tb);
            bulk_g2s(tinv, L.invd + row0 * kp, tb, bar);
            bulk_g2s(tsup, L.sup + row0 * kp, tb, bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        const int64_t p = vb * bpc + b;
        if (p < P) {
            const int64_t base = p * M;
            const int cnt = (int)min((int64_t)M, n - base) - 1;
            LvPtrs t;
            t.inv = tinv + j; t.sup = tsup + j;
            t.ra = Lp.ypart; t.rb = Lp.lc; t.da = nullptr; t.db = nullptr; t.Xn = Xnext;
            t.ypart = L.ypart; t.lc = L.lc; t.X = L.X; t.rw = nullptr;
            if (cnt == M - 1) lv_body<M, PHASE, LV_SRC_PLAIN, true>(t, b * M, kp, j, p, P, base, cnt);
            else lv_body<M, PHASE, LV_SRC_PLAIN, false>(t, b * M, kp, j, p, P, base, cnt);
        }
        __syncthreads();   // tiles free for the next virtual CTA
    }
}

template <int M>
__global__ void __launch_bounds__(L0_NT, 1) k_lv_chain(const __grid_constant__ ChainArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    const int kp = a.S.kp;
    const int T = (L0_NT >> lg2(kp)) * M;
    c128 *tinv = reinterpret_cast<c128 *>(smem + 128);
    c128 *tsup = tinv + (size_t)T * kp;
    auto cl = cgr::this_cluster();
    const unsigned rank = cl.block_rank(), cs = cl.num_blocks();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    const LevelDev *lv = a.lv;
    for (int l = a.l0; l + 1 < a.nl; ++l) {
        chain_level<M, 1>(lv[l], lv[l - 1], nullptr, a.S, tinv, tsup, bar, phase, rank, cs);
        cl.sync();
    }
    if (rank == 0 && (int)threadIdx.x < kp) {   // k_top_solve's order
        const LevelDev &Tl = lv[a.nl - 1], &Tp = lv[a.nl - 2];
        const int j = threadIdx.x;
        c128 yp = cmk(0.0, 0.0);
        for (int64_t i = 0; i < Tl.n; ++i) {
            const c128 d = cadd(Tp.ypart[i * kp + j], Tp.lc[i * kp + j]);
            const c128 ai = i > 0 ? Tl.sup[(i - 1) * kp + j] : cmk(0.0, 0.0);
            yp = cmul(Tl.invd[i * kp + j], cfnma(d, ai, yp));
            Tl.X[i * kp + j] = yp;
        }
        c128 xnext = cmk(0.0, 0.0);
        for (int64_t i = Tl.n - 1; i >= 0; --i) {
            const c128 xi = cfnma(Tl.X[i * kp + j], Tl.invd[i * kp + j], cmul(Tl.sup[i * kp + j], xnext));
            Tl.X[i * kp + j] = xi;
            xnext = xi;
        }
    }
    cl.sync();
    for (int l = a.nl - 2; l >= a.l0; --l) {
        chain_level<M, 3>(lv[l], lv[l - 1], lv[l + 1].X, a.S, tinv, tsup, bar, phase, rank, cs);
        if (l > a.l0) cl.sync();
    }
}

// first chained level (0: the plan does not use the chain) and the cluster
// size: levels >= 2 whose k_lv_tma grid fits one wave of <= 16 CTAs
int lv_chain_start(const LevelDev *lv, int nl, int kp, int *cs) {
    if (getenv("REXI_NO_CHAIN") || nl > CH_MAXLV || nl < 4 || !lv[0].sym || kp > L0_NT) return 0;
    for (int l = 2; l + 1 < nl; ++l) {
        const int64_t g = lv_tma_ctas(lv[l].n, kp);
        if (g <= CH_MAXCS) {
            *cs = (int)std::max<int64_t>(1, g);
            return l;
        }
    }
    return 0;
}

cudaError_t lv_launch_chain(const LevelDev *lv, int nl, int l0, int cs, const ShiftDev &S, cudaStream_t st) {
    ChainArgs a{};
    for (int l = 0; l < nl; ++l) a.lv[l] = lv[l];
    a.S = S;
    a.l0 = l0;
    a.nl = nl;
    const int64_t rows = (int64_t)(L0_NT / S.kp) * TRI_M;
    const size_t smem = 128 + 2 * (size_t)rows * S.kp * sizeof(c128);
    auto kern = k_lv_chain<TRI_M>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(L0_NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t lv_launch_tma(const LevelDev &L, const ShiftDev &S, int phase, const c128 *rin_a, const c128 *rin_b,
                          const cdh *rdd_a, const cdh *rdd_b, const c128 *Xnext, cudaStream_t st, c128 *rw) {
    LvArgs a{};
    a.L = L; a.S = S; a.rin_a = rin_a; a.rin_b = rin_b; a.rdd_a = rdd_a; a.rdd_b = rdd_b; a.Xnext = Xnext;
    const int kp = S.kp;
    const int64_t rows = (int64_t)(L0_NT / kp) * TRI_M;
    const int64_t grid = (L.n + rows - 1) / rows;
    const size_t smem = 128 + 2 * (size_t)rows * kp * sizeof(c128);
    cudaError_t e;
#define LV_LAUNCH(PH, SRCV)                                                                             \
    do {                                                                                                \
        auto kern = k_lv_tma<TRI_M, PH, SRCV>;                                                           \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
        if (e != cudaSuccess) return e;                                                                 \
        kern<<<(unsigned)grid, L0_NT, smem, st>>>(a);                                                   \
    } while (0)
    if (phase == 1) {
        a.rw = rdd_a ? rw : nullptr;
        if (rdd_a) LV_LAUNCH(1, LV_SRC_DD);
        else LV_LAUNCH(1, LV_SRC_PLAIN);
    } else if (rdd_a && rw) {   // the rhs the S1 pass stored
        a.rin_a = rw;
        LV_LAUNCH(3, LV_SRC_STORED);
    } else {
        if (rdd_a) LV_LAUNCH(3, LV_SRC_DD);
        else LV_LAUNCH(3, LV_SRC_PLAIN);
    }
#undef LV_LAUNCH
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
template <typename K>
static cudaError_t launch_l0(K kern, const L0Args &a, int flags, cudaStream_t st) {
    const int kp = a.S.kp;
    const int64_t rows = (int64_t)(L0_NT / kp) * TRI_M;
    const int64_t grid = (a.L.n + rows - 1) / rows;
    const size_t smem = l0_smem_bytes(kp, TRI_M, flags);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, L0_NT, smem, st>>>(a);
    return cudaGetLastError();
}

__global__ void k_to_c64(const c128 *__restrict__ src, c64 *__restrict__ dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = to_c64(src[i]);
}

__global__ void k_to_f32(const double *__restrict__ src, float *__restrict__ dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __double2float_rn(src[i]);
}

cudaError_t launch_to_f32(const double *src, float *dst, int64_t n, cudaStream_t st) {
    k_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_to_c64(const c128 *src, c64 *dst, int64_t n, cudaStream_t st) {
    k_to_c64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, n);
    return cudaGetLastError();
}

// Graph patching for host-buffer steps (plan.cu): find the level-0 kernel
// nodes of a captured step that read u (S1) and write the rounded output
// (K3, or S3ACC without refinement), and re-point them at other buffers.
int l0_graph_role(cudaGraphNode_t node) {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(node, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) return 0;
    cudaKernelNodeParams p{};
    if (cudaGraphKernelNodeGetParams(node, &p) != cudaSuccess) return 0;
    if (p.func == (void *)k_l0_s1<TRI_M, 0> || p.func == (void *)k_l0_s1<TRI_M, 64>) return 1;
    if (p.func == (void *)k_l0_k3<TRI_M, 0> || p.func == (void *)k_l0_k3<TRI_M, 64> ||
        p.func == (void *)k_l0_s3acc<TRI_M>) {
        const L0Args *a = reinterpret_cast<const L0Args *>(p.kernelParams[0]);
        return a->final_out ? 2 : 0;
    }
    return 0;
}

cudaError_t l0_graph_patch(cudaGraphExec_t exec, cudaGraphNode_t node, int role, const c128 *u, c128 *uout) {
    cudaKernelNodeParams p{};
    cudaError_t e = cudaGraphKernelNodeGetParams(node, &p);
    if (e != cudaSuccess) return e;
    L0Args a = *reinterpret_cast<const L0Args *>(p.kernelParams[0]);
    if (role == 1) {
        a.u = u;
        a.u_bulk = ((uintptr_t)u & 15) == 0 && !getenv("REXI_S1_NO_BULK");
    } else {
        a.uout = uout;
    }
    void *args[1] = {&a};
    p.kernelParams = args;
    p.extra = nullptr;
    return cudaGraphExecKernelNodeSetParams(exec, node, &p);
}

bool l0v2_supported(int kp) { return kp <= L0_NT; }
// REXI_L0_KP: bit mask of the level-0 kernels that take their k_pad = 64
// instantiation (1: S1, 2: K2, 4: K3; A/B switch).  scripts/tune_l0kp.sh on
// cfg 2: K2 0.70 -> 0.673 ms, K3 0.270 -> 0.249 ms, S1 unchanged (HBM-bound;
// its k_pad = 64 form spills more), so S1 keeps the runtime form.
static int l0_kp_mask() {
    static const int m = getenv("REXI_L0_KP") ? atoi(getenv("REXI_L0_KP")) : 6;
    return m;
}
int64_t l0_row_padding() { return (int64_t)L0_NT * TRI_M + 2 * L0_ROWPAD; }

cudaError_t l0_launch_s1(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *u, c128 *rhs0,
                         int64_t nout, cudaStream_t st) {
    L0Args a{};
    a.z = z; a.L = L; a.S = S; a.u = u; a.rhs_out = rhs0; a.nout = nout;
    a.u_bulk = ((uintptr_t)u & 15) == 0 && !getenv("REXI_S1_NO_BULK");
    // + T+2 u rows after the staged rhs rows
    const size_t extra = 16 + ((size_t)(L0_NT / S.kp) * TRI_M + 2) * sizeof(c128);
    const int kp = S.kp;
    const int64_t rows = (int64_t)(L0_NT / kp) * TRI_M;
    const int64_t grid = (L.n + rows - 1) / rows;
    const size_t smem = l0_smem_bytes(kp, TRI_M, ST_RHS | ST_BDIA) + extra;
    auto kern = (kp == 64 && (l0_kp_mask() & 1)) ? k_l0_s1<TRI_M, 64> : k_l0_s1<TRI_M, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, L0_NT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t l0_launch_s3acc(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                            const c128 *X1, double *acc, c128 *uout, int64_t nout, cudaStream_t st) {
    L0Args a{};
    a.nout = nout;
    a.z = z; a.L = L; a.S = S; a.rhs0 = rhs0; a.X1 = X1; a.acc = acc; a.uout = uout;
    a.acc_add = 0; a.final_out = uout != nullptr;
    return launch_l0(k_l0_s3acc<TRI_M>, a, ST_RHS, st);
}

cudaError_t l0_launch_k2(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                         const c128 *X1, double *acc, c64 *rres, const c64 *inv32, const float *const *r32,
                         const double2 *emax, int64_t nout, bool exact_residual, cudaStream_t st) {
    L0Args a{};
    a.nout = nout;
    a.z = z; a.L = L; a.S = S; a.rhs0 = rhs0; a.X1 = X1; a.acc = acc; a.rres_out = rres; a.inv32 = inv32;
    a.emax = emax;
    a.acc_add = 0; a.final_out = 0;
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        a.pf_dist = (int64_t)sms * K2_MINB;   // one residency wave ahead
        if (const char *e = getenv("REXI_K2_PF")) a.pf_dist = (int64_t)(atof(e) * sms * K2_MINB);
    }
    for (int q = 0; q < 6; ++q) a.r32[q] = r32[q];
    if (exact_residual) return launch_l0(k_l0_k2<TRI_M, true, 0>, a, K2_FLAGS, st);
    if (S.kp == 64 && (l0_kp_mask() & 2)) return launch_l0(k_l0_k2<TRI_M, false, 64>, a, K2_FLAGS, st);
    return launch_l0(k_l0_k2<TRI_M, false, 0>, a, K2_FLAGS, st);
}

cudaError_t l0_launch_k3(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *X1,
                         const c64 *inv32, const float *const *r32, const c64 *rres, double *acc, c128 *uout,
                         int64_t nout, cudaStream_t st) {
    L0Args a{};
    a.nout = nout;
    a.z = z; a.L = L; a.S = S; a.X1 = X1; a.inv32 = inv32; a.rres_in = rres; a.acc = acc; a.uout = uout;
    for (int q = 0; q < 6; ++q) a.r32[q] = r32[q];
    a.acc_add = 1; a.final_out = uout != nullptr;
    const int kp = S.kp;
    const int64_t rows = (int64_t)(L0_NT / kp) * TRI_M;
    const int64_t grid = (L.n + rows - 1) / rows;
    const size_t smem = k3_smem_bytes(kp, TRI_M);
    auto kern = (kp == 64 && (l0_kp_mask() & 4)) ? k_l0_k3<TRI_M, 64> : k_l0_k3<TRI_M, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, L0_NT, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rexi
