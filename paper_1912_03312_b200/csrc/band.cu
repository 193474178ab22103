// band.cu -- direct solver for narrow banded pencils: the reference's P2 1D
// systems (pentadiagonal, solvers.py:39-80 via zgbtrf/zgbtrs on bandwidth 5,
// spatial.py:202-216), and any pattern with half bandwidth 2..4.
//
// Partitioned band LU, all K shifts in lockstep (lane = shift, fastest in
// every per-shift array):
//   * the rows are cut into P blocks of M; the first B rows of every block
//     p >= 1 are its interface rows Gamma_p, the rest its interior I_p (block 0
//     is all interior).  Interiors of different blocks never couple (they are
//     separated by B interface rows), so S_II is block diagonal;
//   * prepare factors every interior block without pivoting (stable for
//     these pencils: the imaginary part -Re(sigma) B is definite, the same
//     argument as the tridiagonal path) and forms the Schur complement on the
//     interface rows, R = S_GG - S_GI S_II^-1 S_IG, which is block
//     tridiagonal with B x B blocks, factored by block LU (explicit inverses
//     of the B x B pivots, partial pivoting inside them);
//   * a step: rhs = iBu (k_band_rhs, CSR order), interior solves with zero
//     halos -> reduced rhs (k_band_s1), the block-tridiagonal interface solve
//     one thread per shift (k_band_red), interior solves with the interface
//     values known (k_band_s3), and the beta-weighted double-double lane sum
//     (k_band_accum, the fixed-order sum of the other paths).  With
//     refinement the residual b - S x is formed with error-free products and
//     a double-double sum (k_band_residual) and solved for once more.
// The interface solve is sequential over the P blocks, so M ~ sqrt(4n) keeps
// the interior sweeps and the interface chain balanced; this solver is aimed
// at the reference's P2 sizes (thousands to ~1e5 rows), where one step is a
// handful of microsecond-scale launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "band.cuh"
#include "tridiag_launch.h"

namespace rexi {

namespace {

struct BandDev {
    int64_t n, npad;
    int M, P, kp;
    const double *ta, *tai, *bb;   // [(2B+1)][npad]: fl(tau a), fl(tau a_im), b of entry (r, r+d)
    c128 *lo, *up, *dinv;          // interior factors: [npad][B][kp], [npad][B][kp], [npad][kp]
    c128 *spk;                     // spikes [P][4][B*B][kp]: Etop, Ebot, Ftop, Fbot
    c128 *rl, *rdi, *ru;           // interface system [P][B*B][kp]: A_j, D_j^-1, C_j at the level block j
                                   // is eliminated (block cyclic reduction; j = p - 1)
    c128 *ral, *rga;               // BCR multipliers of the survivors [sum_l ns_l][B*B][kp]
    c128 *gcon;                    // reduced-rhs pieces [P][2][B][kp]
    c128 *xg;                      // interface solution [P][B][kp]
    c128 *X;                       // sweep scratch [npad][kp]
};

struct BandImpl {
    BandDev D{};
    c128 *rhs = nullptr;           // shared rhs [npad]
    c128 *X1 = nullptr, *X2 = nullptr, *res = nullptr;   // [npad][kp]
    double *pstat = nullptr;       // [2*kp] pivot |.| min / max per lane (prepare)
    bool staged = false;           // shared-memory staged step kernels (M = 64, small P)
};

template <int B>
__device__ __forceinline__ c128 ent(const BandDev &D, int64_t r, int d, c128 sg) {
    const size_t o = (size_t)(d + B) * D.npad + r;
    return form_entry(__ldg(D.ta + o), __ldg(D.tai + o), __ldg(D.bb + o), sg);
}

__device__ __forceinline__ int64_t blk_i0(int p, int M, int B) { return p == 0 ? 0 : (int64_t)p * M + B; }

__device__ __forceinline__ c128 crecip_c(c128 b) {
    if (fabs(b.x) >= fabs(b.y)) {
        const double r = b.y / b.x, den = b.x + r * b.y;
        return cmk(1.0 / den, -r / den);
    }
    const double r = b.x / b.y, den = b.y + r * b.x;
    return cmk(r / den, -1.0 / den);
}

// factor access: the interior factors in HBM ([row][coef][kp], read-only
// path) or staged in shared memory ([row][2B+1][lg], lo | up | dinv)
template <int B>
struct GlobalF {
    const c128 *__restrict__ lo;
    const c128 *__restrict__ up;
    const c128 *__restrict__ dinv;
    int kp, lane;
    __device__ __forceinline__ c128 l(int64_t r, int q) const { return __ldg(lo + ((size_t)r * B + q) * kp + lane); }
    __device__ __forceinline__ c128 u(int64_t r, int q) const { return __ldg(up + ((size_t)r * B + q) * kp + lane); }
    __device__ __forceinline__ c128 d(int64_t r) const { return __ldg(dinv + (size_t)r * kp + lane); }
};
template <int B>
struct SmemF {
    const c128 *f;
    int64_t r0;
    int lg, ll;
    __device__ __forceinline__ c128 l(int64_t r, int q) const { return f[((r - r0) * (2 * B + 1) + q) * lg + ll]; }
    __device__ __forceinline__ c128 u(int64_t r, int q) const {
        return f[((r - r0) * (2 * B + 1) + B + q) * lg + ll];
    }
    __device__ __forceinline__ c128 d(int64_t r) const { return f[((r - r0) * (2 * B + 1) + 2 * B) * lg + ll]; }
};

// interior solve of rows [r0, r1) for one lane: forward with the unit lower
// factor (y' into the scratch Yt(r)), backward with the upper factor (y handed
// to out(r, y)).  The loads of the next rows are independent of the dependent
// chain and go out ahead of it.
template <int B, typename F, typename Yt, typename Rhs, typename Out>
__device__ __forceinline__ void interior_solve_f(const F &f, Yt yt, int64_t r0, int64_t r1, Rhs rhs, Out out) {
    c128 w[B];
#pragma unroll
    for (int q = 0; q < B; ++q) w[q] = cmk(0.0, 0.0);
#pragma unroll 4
    for (int64_t r = r0; r < r1; ++r) {
        c128 v = rhs(r);
#pragma unroll
        for (int q = 0; q < B; ++q) v = cfnma(v, f.l(r, q), w[q]);
#pragma unroll
        for (int q = B - 1; q > 0; --q) w[q] = w[q - 1];
        w[0] = v;
        yt(r) = v;
    }
#pragma unroll
    for (int q = 0; q < B; ++q) w[q] = cmk(0.0, 0.0);
#pragma unroll 4
    for (int64_t r = r1 - 1; r >= r0; --r) {
        c128 v = yt(r);
#pragma unroll
        for (int q = 0; q < B; ++q) v = cfnma(v, f.u(r, q), w[q]);
        v = cmul(f.d(r), v);
#pragma unroll
        for (int q = B - 1; q > 0; --q) w[q] = w[q - 1];
        w[0] = v;
        out(r, v);
    }
}

template <int B, typename Rhs, typename Out>
__device__ __forceinline__ void interior_solve(const BandDev &D, c128 *__restrict__ Yt, int64_t r0, int64_t r1,
                                               int lane, Rhs rhs, Out out) {
    const GlobalF<B> f{D.lo, D.up, D.dinv, D.kp, lane};
    const int kp = D.kp;
    interior_solve_f<B>(f, [&](int64_t r) -> c128 & { return Yt[(size_t)r * kp + lane]; }, r0, r1, rhs, out);
}

__device__ __forceinline__ bool thread_block_lane(const BandDev &D, int &p, int &lane) {
    const int per = blockDim.x / D.kp;
    lane = threadIdx.x % D.kp;
    p = blockIdx.x * per + threadIdx.x / D.kp;
    return p < D.P;
}

// ---- prepare: interior no-pivot band LU + spikes -------------------------
template <int B>
__global__ void k_band_factor(BandDev D, ShiftDev S, double *pstat) {
    int p, lane;
    if (!thread_block_lane(D, p, lane)) return;
    const int kp = D.kp, M = D.M;
    const c128 sg = S.sigma[lane];
    const int64_t r0 = blk_i0(p, M, B), r1 = (int64_t)(p + 1) * M;
    // window of the previous B rows of U: urow[i][e] = u_{t, t+e}, t = r-1-i
    c128 urow[B][B + 1], udi[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        udi[i] = cmk(0.0, 0.0);
#pragma unroll
        for (int e = 0; e <= B; ++e) urow[i][e] = cmk(0.0, 0.0);
    }
    double pmin = INFINITY, pmax = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
        c128 a[2 * B + 1];
#pragma unroll
        for (int e = 0; e <= 2 * B; ++e) {
            const int64_t c = r + e - B;
            a[e] = (c >= r0 && c < r1) ? ent<B>(D, r, e - B, sg) : cmk(0.0, 0.0);
        }
        // eliminate columns r-B .. r-1 in increasing order (Doolittle, no pivot)
#pragma unroll
        for (int e = 0; e < B; ++e) {            // column c = r - B + e, U row index i = B - 1 - e
            const int i = B - 1 - e;
            const c128 l = cmul(a[e], udi[i]);
            D.lo[((size_t)r * B + i) * kp + lane] = l;   // q = r - 1 - c = i
#pragma unroll
            for (int f = 1; f <= B; ++f)                  // columns c + f, f <= B  -> a index e + f
                if (e + f <= 2 * B) a[e + f] = cfnma(a[e + f], l, urow[i][f]);
        }
        const c128 dg = a[B];
        const double ad = hypot(dg.x, dg.y);
        pmin = fmin(pmin, ad);
        pmax = isfinite(ad) ? fmax(pmax, ad) : INFINITY;   // fmax would drop a NaN
        const c128 di = crecip_c(dg);
        D.dinv[(size_t)r * kp + lane] = di;
#pragma unroll
        for (int q = 0; q < B; ++q) D.up[((size_t)r * B + q) * kp + lane] = a[B + 1 + q];
#pragma unroll
        for (int i = B - 1; i > 0; --i) {
            udi[i] = udi[i - 1];
#pragma unroll
            for (int e = 0; e <= B; ++e) urow[i][e] = urow[i - 1][e];
        }
        udi[0] = di;
#pragma unroll
        for (int e = 0; e <= B; ++e) urow[0][e] = a[B + e];
    }
    // pivot extremes per lane (atomic min/max on the bit patterns of non-negative doubles)
    atomicMin(reinterpret_cast<unsigned long long *>(pstat) + lane, (unsigned long long)__double_as_longlong(pmin));
    atomicMax(reinterpret_cast<unsigned long long *>(pstat) + kp + lane,
              (unsigned long long)__double_as_longlong(isfinite(pmax) ? pmax : INFINITY));
    // spikes: S_Ip^-1 S_{Ip, Gamma_p} (E, p >= 1) and S_Ip^-1 S_{Ip, Gamma_p+1} (F, p <= P-2),
    // kept at the first B and the last B interior rows
    for (int which = 0; which < 2; ++which) {
        if (which == 0 && p == 0) continue;
        if (which == 1 && p == D.P - 1) continue;
        const int64_t cbase = which == 0 ? (int64_t)p * M : (int64_t)(p + 1) * M;
        for (int col = 0; col < B; ++col) {
            const int64_t c = cbase + col;
            c128 *const etop = D.spk + ((size_t)p * 4 + 2 * which) * B * B * kp;
            c128 *const ebot = D.spk + ((size_t)p * 4 + 2 * which + 1) * B * B * kp;
            interior_solve<B>(
                D, D.X, r0, r1, lane,
                [&](int64_t r) {
                    const int64_t dd = c - r;
                    return (dd >= -B && dd <= B) ? ent<B>(D, r, (int)dd, sg) : cmk(0.0, 0.0);
                },
                [&](int64_t r, c128 y) {
                    if (r < r0 + B) etop[(size_t)((r - r0) * B + col) * kp + lane] = y;
                    if (r >= r1 - B) ebot[(size_t)((r - (r1 - B)) * B + col) * kp + lane] = y;
                });
        }
    }
}

// B x B complex helpers (row-major [i][j])
template <int B>
__device__ __forceinline__ void mm_sub(c128 (&c)[B][B], const c128 (&a)[B][B], const c128 (&b)[B][B]) {
    // c -= a b
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) {
            c128 s = c[i][j];
#pragma unroll
            for (int t = 0; t < B; ++t) s = cfnma(s, a[i][t], b[t][j]);
            c[i][j] = s;
        }
}
template <int B>
__device__ __forceinline__ void mm(c128 (&c)[B][B], const c128 (&a)[B][B], const c128 (&b)[B][B]) {
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) {
            c128 s = cmk(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < B; ++t) s = cadd(s, cmul(a[i][t], b[t][j]));
            c[i][j] = s;
        }
}
// inverse by Gauss-Jordan with partial pivoting (|re| + |im|); returns min |pivot|
template <int B>
__device__ double inv_bb(const c128 (&a_in)[B][B], c128 (&inv)[B][B]) {
    c128 a[B][B];
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) {
            a[i][j] = a_in[i][j];
            inv[i][j] = cmk(i == j ? 1.0 : 0.0, 0.0);
        }
    double pmin = INFINITY;
    for (int c = 0; c < B; ++c) {
        int pr = c;
        double best = fabs(a[c][c].x) + fabs(a[c][c].y);
        for (int i = c + 1; i < B; ++i) {
            const double v = fabs(a[i][c].x) + fabs(a[i][c].y);
            if (v > best) {
                best = v;
                pr = i;
            }
        }
        if (pr != c)
            for (int j = 0; j < B; ++j) {
                c128 t = a[c][j]; a[c][j] = a[pr][j]; a[pr][j] = t;
                t = inv[c][j]; inv[c][j] = inv[pr][j]; inv[pr][j] = t;
            }
        pmin = fmin(pmin, hypot(a[c][c].x, a[c][c].y));
        const c128 r = crecip_c(a[c][c]);
        for (int j = 0; j < B; ++j) {
            a[c][j] = cmul(a[c][j], r);
            inv[c][j] = cmul(inv[c][j], r);
        }
        for (int i = 0; i < B; ++i) {
            if (i == c) continue;
            const c128 f = a[i][c];
            for (int j = 0; j < B; ++j) {
                a[i][j] = cfnma(a[i][j], f, a[c][j]);
                inv[i][j] = cfnma(inv[i][j], f, inv[c][j]);
            }
        }
    }
    return pmin;
}

template <int B>
__device__ __forceinline__ void load_bb(c128 (&m)[B][B], const c128 *base, int kp, int lane) {
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) m[i][j] = __ldg(base + (size_t)(i * B + j) * kp + lane);
}
template <int B>
__device__ __forceinline__ void store_bb(const c128 (&m)[B][B], c128 *base, int kp, int lane) {
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) base[(size_t)(i * B + j) * kp + lane] = m[i][j];
}

// couplings of interface block p: S_GG (Gamma_p x Gamma_p), S_GIprev (Gamma_p x
// last B rows of I_{p-1}), S_GIcur (Gamma_p x first B rows of I_p)
template <int B>
__device__ __forceinline__ void couplings(const BandDev &D, int p, c128 sg, c128 (&gg)[B][B], c128 (&gp)[B][B],
                                          c128 (&gc)[B][B]) {
    const int64_t g0 = (int64_t)p * D.M;
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) {
            gg[i][j] = ent<B>(D, g0 + i, j - i, sg);
            const int dp = j - i - B, dc = B + j - i;
            gp[i][j] = dp >= -B ? ent<B>(D, g0 + i, dp, sg) : cmk(0.0, 0.0);
            gc[i][j] = dc <= B ? ent<B>(D, g0 + i, dc, sg) : cmk(0.0, 0.0);
        }
}

// ---- prepare: the interface system's block cyclic reduction, one thread per shift
// The block-tridiagonal interface system  A_j x_{j-1} + D_j x_j + C_j x_{j+1} = g_j
// (j = p - 1 = 0 .. nb-1, nb = P - 1) is reduced odd-even: at level l (h = 2^l)
// the active blocks are the multiples of h, those with j/h odd are eliminated
// through their neighbours j +- h (multiples of 2h, the survivors), and a
// survivor s takes  alpha_s = -A_s D_{s-h}^-1,  gamma_s = -C_s D_{s+h}^-1,
//   A_s <- alpha_s A_{s-h},  C_s <- gamma_s C_{s+h},
//   D_s <- D_s + alpha_s C_{s-h} + gamma_s A_{s+h},  g_s <- g_s + alpha_s g_{s-h} + gamma_s g_{s+h}.
// Block 0 is left at the top; the back substitution runs the levels down:
//   x_e = D_e^-1 (g_e - A_e x_{e-h} - C_e x_{e+h}).
// A solve is 2 ceil(log2 nb) dependent levels instead of a chain over the
// blocks.  Stored: per block its (A, D^-1, C) at its elimination level (rl,
// rdi, ru); per (level, survivor) alpha and gamma (ral, rga, compact).
__host__ __device__ inline int bcr_levels(int nb) {
    int L = 0;
    while ((1 << L) < nb) ++L;
    return L;
}
// survivors of level l: multiples of 2^(l+1) in [0, nb)
__host__ __device__ inline int bcr_nsurv(int nb, int l) { return (nb - 1) / (2 << l) + 1; }
__host__ __device__ inline int bcr_off(int nb, int l) {
    int o = 0;
    for (int q = 0; q < l; ++q) o += bcr_nsurv(nb, q);
    return o;
}

template <int B>
__device__ __forceinline__ void band_blocks(const BandDev &D, int p, c128 sg, int lane, c128 (&Dp)[B][B],
                                            c128 (&Cp)[B][B], c128 (&Ap)[B][B]) {
    const int kp = D.kp;
    c128 gp[B][B], gc[B][B], sp[B][B];
    couplings<B>(D, p, sg, Dp, gp, gc);
    // D_p = S_GG - S_GIprev Fbot_{p-1} - S_GIcur Etop_p
    load_bb<B>(sp, D.spk + ((size_t)(p - 1) * 4 + 3) * B * B * kp, kp, lane);
    mm_sub<B>(Dp, gp, sp);
    load_bb<B>(sp, D.spk + ((size_t)p * 4 + 0) * B * B * kp, kp, lane);
    mm_sub<B>(Dp, gc, sp);
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) {
            Cp[i][j] = cmk(0.0, 0.0);
            Ap[i][j] = cmk(0.0, 0.0);
        }
    if (p + 1 < D.P) {   // C_p = -S_GIcur Ftop_p
        load_bb<B>(sp, D.spk + ((size_t)p * 4 + 2) * B * B * kp, kp, lane);
        mm_sub<B>(Cp, gc, sp);
    }
    if (p >= 2) {        // A_p = -S_GIprev Ebot_{p-1}
        load_bb<B>(sp, D.spk + ((size_t)(p - 1) * 4 + 1) * B * B * kp, kp, lane);
        mm_sub<B>(Ap, gp, sp);
    }
}

template <int B>
__device__ __forceinline__ void ldm(c128 (&m)[B][B], const c128 *base, int kp, int lane) {
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) m[i][j] = base[(size_t)(i * B + j) * kp + lane];
}

template <int B>
__global__ void k_band_rfactor(BandDev D, ShiftDev S, double *pstat) {
    const int lane = blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= D.kp) return;
    const int kp = D.kp, nb = D.P - 1;
    if (nb < 1) return;
    const c128 sg = S.sigma[lane];
    double pmin = INFINITY;
    auto note = [&](double pv) { pmin = isfinite(pv) ? fmin(pmin, pv) : 0.0; };
    auto at = [&](c128 *arr, int j) { return arr + (size_t)(j + 1) * B * B * kp; };
    // level-0 blocks: A in rl, D in rdi (inverted at elimination), C in ru
    for (int j = 0; j < nb; ++j) {
        c128 Dp[B][B], Cp[B][B], Ap[B][B];
        band_blocks<B>(D, j + 1, sg, lane, Dp, Cp, Ap);
        store_bb<B>(Ap, at(D.rl, j), kp, lane);
        store_bb<B>(Dp, at(D.rdi, j), kp, lane);
        store_bb<B>(Cp, at(D.ru, j), kp, lane);
    }
    const int L = bcr_levels(nb);
    for (int l = 0; l < L; ++l) {
        const int h = 1 << l;
        // the eliminated blocks of this level: D^-1 in place
        for (int e = h; e < nb; e += 2 * h) {
            c128 Dm[B][B], inv[B][B];
            ldm<B>(Dm, at(D.rdi, e), kp, lane);
            note(inv_bb<B>(Dm, inv));
            store_bb<B>(inv, at(D.rdi, e), kp, lane);
        }
        // the survivors: multipliers and updated blocks
        for (int s2 = 0; s2 < nb; s2 += 2 * h) {
            c128 As[B][B], Cs[B][B], Ds[B][B], al[B][B], ga[B][B], t[B][B], m[B][B], nA[B][B], nC[B][B];
            ldm<B>(As, at(D.rl, s2), kp, lane);
            ldm<B>(Ds, at(D.rdi, s2), kp, lane);
            ldm<B>(Cs, at(D.ru, s2), kp, lane);
#pragma unroll
            for (int i = 0; i < B; ++i)
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    al[i][j] = ga[i][j] = nA[i][j] = nC[i][j] = cmk(0.0, 0.0);
                }
            if (s2 - h >= 0) {
                ldm<B>(m, at(D.rdi, s2 - h), kp, lane);          // D_{s-h}^-1
                mm_sub<B>(al, As, m);                          // alpha = -A_s D_{s-h}^-1
                ldm<B>(t, at(D.ru, s2 - h), kp, lane);            // C_{s-h}
                mm<B>(m, al, t);
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) Ds[i][j] = cadd(Ds[i][j], m[i][j]);
                ldm<B>(t, at(D.rl, s2 - h), kp, lane);            // A_{s-h}
                mm<B>(nA, al, t);
            }
            if (s2 + h < nb) {
                ldm<B>(m, at(D.rdi, s2 + h), kp, lane);          // D_{s+h}^-1
                mm_sub<B>(ga, Cs, m);                          // gamma = -C_s D_{s+h}^-1
                ldm<B>(t, at(D.rl, s2 + h), kp, lane);            // A_{s+h}
                mm<B>(m, ga, t);
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) Ds[i][j] = cadd(Ds[i][j], m[i][j]);
                ldm<B>(t, at(D.ru, s2 + h), kp, lane);            // C_{s+h}
                mm<B>(nC, ga, t);
            }
            const int k = bcr_off(nb, l) + s2 / (2 * h);
            store_bb<B>(al, D.ral + (size_t)k * B * B * kp, kp, lane);
            store_bb<B>(ga, D.rga + (size_t)k * B * B * kp, kp, lane);
            store_bb<B>(nA, at(D.rl, s2), kp, lane);
            store_bb<B>(Ds, at(D.rdi, s2), kp, lane);
            store_bb<B>(nC, at(D.ru, s2), kp, lane);
        }
    }
    {   // the top block
        c128 Dm[B][B], inv[B][B];
        ldm<B>(Dm, at(D.rdi, 0), kp, lane);
        note(inv_bb<B>(Dm, inv));
        store_bb<B>(inv, at(D.rdi, 0), kp, lane);
    }
    atomicMin(reinterpret_cast<unsigned long long *>(pstat) + lane, (unsigned long long)__double_as_longlong(pmin));
}

// ---- step kernels ----------------------------------------------------------
// rhs = 1j * (B @ u): CSR column order (the band's d = -B..B), no FMA
// (integrate.py:204); absent entries hold b = 0 and add exactly nothing
template <int B>
__global__ void k_band_rhs(BandDev D, const c128 *__restrict__ u, c128 *__restrict__ rhs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.npad) return;
    double sr = 0.0, si = 0.0;
    if (i < D.n) {
#pragma unroll
        for (int d = -B; d <= B; ++d) {
            const int64_t c = i + d;
            if (c < 0 || c >= D.n) continue;
            const double b = D.bb[(size_t)(d + B) * D.npad + i];
            const c128 x = u[c];
            sr = __dadd_rn(sr, __dmul_rn(b, x.x));
            si = __dadd_rn(si, __dmul_rn(b, x.y));
        }
    }
    rhs[i] = cmk(-si, sr);
}

template <int B>
__device__ __forceinline__ c128 rhs_at(const BandDev &D, const c128 *sh, const c128 *ps, int64_t r, int lane) {
    return sh ? __ldg(sh + r) : __ldg(ps + (size_t)r * D.kp + lane);
}

// interior solves with zero halos -> the pieces of the reduced rhs
template <int B>
__global__ void k_band_s1(BandDev D, ShiftDev S, const c128 *__restrict__ rsh, const c128 *__restrict__ rps) {
    int p, lane;
    if (!thread_block_lane(D, p, lane)) return;
    const int kp = D.kp, M = D.M;
    const c128 sg = S.sigma[lane];
    const int64_t r0 = blk_i0(p, M, B), r1 = (int64_t)(p + 1) * M;
    // only the first and the last B rows of y feed the reduced rhs
    c128 yf[B], yl[B];
    interior_solve<B>(
        D, D.X, r0, r1, lane, [&](int64_t r) { return rhs_at<B>(D, rsh, rps, r, lane); },
        [&](int64_t r, c128 y) {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (r == r0 + i) yf[i] = y;
                if (r == r1 - B + i) yl[i] = y;
            }
        });
    c128 *gc = D.gcon + (size_t)p * 2 * B * kp;
    if (p >= 1) {        // t_p = S_{Gamma_p, I_p(first B)} y
        c128 gg[B][B], gp[B][B], gcur[B][B];
        couplings<B>(D, p, sg, gg, gp, gcur);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            c128 s = cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < B; ++j) s = cadd(s, cmul(gcur[i][j], yf[j]));
            gc[(size_t)i * kp + lane] = s;
        }
    }
    if (p + 1 < D.P) {   // s_p = S_{Gamma_p+1, I_p(last B)} y
        c128 gg[B][B], gp[B][B], gcur[B][B];
        couplings<B>(D, p + 1, sg, gg, gp, gcur);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            c128 s = cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < B; ++j) s = cadd(s, cmul(gp[i][j], yl[j]));
            gc[(size_t)(B + i) * kp + lane] = s;
        }
    }
}

// block-cyclic-reduction solve of the interface system for one shift.  The
// caller supplies accessors: A(j)/Di(j)/C(j) -> B x B blocks, al(k)/ga(k) ->
// the level multipliers (compact index), g(j)/x(j) -> B-vector slots (g is
// reduced in place); thread tid of nthr cooperating threads, sync() between
// levels
template <int B, typename MA, typename MDi, typename MC, typename MAl, typename MGa, typename VG, typename VX,
          typename Sync>
__device__ __forceinline__ void bcr_solve(int nb, int tid, int nthr, MA A, MDi Di, MC C, MAl al, MGa ga, VG g, VX x,
                                          Sync sync) {
    const int L = bcr_levels(nb);
    for (int l = 0; l < L; ++l) {
        const int h = 1 << l, off = bcr_off(nb, l);
        for (int s2 = 2 * h * tid; s2 < nb; s2 += 2 * h * nthr) {
            c128 v[B], M0[B][B];
#pragma unroll
            for (int i = 0; i < B; ++i) v[i] = g(s2)[i];
            if (s2 - h >= 0) {
                al(off + s2 / (2 * h), M0);
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) v[i] = cadd(v[i], cmul(M0[i][j], g(s2 - h)[j]));
            }
            if (s2 + h < nb) {
                ga(off + s2 / (2 * h), M0);
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) v[i] = cadd(v[i], cmul(M0[i][j], g(s2 + h)[j]));
            }
#pragma unroll
            for (int i = 0; i < B; ++i) g(s2)[i] = v[i];
        }
        sync();
    }
    if (tid == 0) {
        c128 M0[B][B];
        Di(0, M0);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            c128 t = cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < B; ++j) t = cadd(t, cmul(M0[i][j], g(0)[j]));
            x(0)[i] = t;
        }
    }
    sync();
    for (int l = L - 1; l >= 0; --l) {
        const int h = 1 << l;
        for (int e = h + 2 * h * tid; e < nb; e += 2 * h * nthr) {
            c128 v[B], M0[B][B];
#pragma unroll
            for (int i = 0; i < B; ++i) v[i] = g(e)[i];
            A(e, M0);
#pragma unroll
            for (int i = 0; i < B; ++i)
#pragma unroll
                for (int j = 0; j < B; ++j) v[i] = cfnma(v[i], M0[i][j], x(e - h)[j]);
            if (e + h < nb) {
                C(e, M0);
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) v[i] = cfnma(v[i], M0[i][j], x(e + h)[j]);
            }
            Di(e, M0);
#pragma unroll
            for (int i = 0; i < B; ++i) {
                c128 t = cmk(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < B; ++j) t = cadd(t, cmul(M0[i][j], v[j]));
                x(e)[i] = t;
            }
        }
        sync();
    }
}

// a proxy for a B-vector stored with a lane stride
struct StridedVec {
    c128 *base;
    int stride;
    __device__ __forceinline__ c128 &operator[](int i) const { return base[(size_t)i * stride]; }
};

// interface system from HBM, one thread per shift (larger problems)
template <int B>
__global__ void k_band_red(BandDev D, const c128 *__restrict__ rsh, const c128 *__restrict__ rps) {
    const int lane = blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= D.kp) return;
    const int kp = D.kp, M = D.M, nb = D.P - 1;
    if (nb < 1) return;
    // g_j in the sweep scratch (D.X), x_j in xg (block p = j + 1)
    for (int j = 0; j < nb; ++j) {
        const int p = j + 1;
        const c128 *gprev = D.gcon + ((size_t)(p - 1) * 2 * B + B) * kp;
        const c128 *gcur = D.gcon + (size_t)p * 2 * B * kp;
#pragma unroll
        for (int i = 0; i < B; ++i)
            D.X[((size_t)j * B + i) * kp + lane] =
                csub(csub(rhs_at<B>(D, rsh, rps, (int64_t)p * M + i, lane), __ldg(gprev + (size_t)i * kp + lane)),
                     __ldg(gcur + (size_t)i * kp + lane));
    }
    auto blk = [&](const c128 *arr, int j, c128 (&o)[B][B]) { load_bb<B>(o, arr + (size_t)(j + 1) * B * B * kp, kp, lane); };
    bcr_solve<B>(
        nb, 0, 1, [&](int j, c128 (&o)[B][B]) { blk(D.rl, j, o); }, [&](int j, c128 (&o)[B][B]) { blk(D.rdi, j, o); },
        [&](int j, c128 (&o)[B][B]) { blk(D.ru, j, o); },
        [&](int k, c128 (&o)[B][B]) { load_bb<B>(o, D.ral + (size_t)k * B * B * kp, kp, lane); },
        [&](int k, c128 (&o)[B][B]) { load_bb<B>(o, D.rga + (size_t)k * B * B * kp, kp, lane); },
        [&](int j) { return StridedVec{D.X + (size_t)j * B * kp + lane, kp}; },
        [&](int j) { return StridedVec{D.xg + (size_t)(j + 1) * B * kp + lane, kp}; }, [] {});
}

// interior solves with the interface values known -> x (all rows) in Xout
template <int B>
__global__ void k_band_s3(BandDev D, ShiftDev S, const c128 *__restrict__ rsh, const c128 *__restrict__ rps,
                          c128 *Xout) {
    int p, lane;
    if (!thread_block_lane(D, p, lane)) return;
    const int kp = D.kp, M = D.M;
    const c128 sg = S.sigma[lane];
    const int64_t r0 = blk_i0(p, M, B), r1 = (int64_t)(p + 1) * M;
    c128 xa[B], xb[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        xa[i] = p >= 1 ? D.xg[((size_t)p * B + i) * kp + lane] : cmk(0.0, 0.0);
        xb[i] = p + 1 < D.P ? D.xg[((size_t)(p + 1) * B + i) * kp + lane] : cmk(0.0, 0.0);
    }
    const int64_t ga = (int64_t)p * M, gb = (int64_t)(p + 1) * M;
    interior_solve<B>(D, D.X, r0, r1, lane, [&](int64_t r) {
        c128 v = rhs_at<B>(D, rsh, rps, r, lane);
        if (p >= 1 && r < r0 + B) {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                const int64_t dd = ga + i - r;
                if (dd >= -B) v = cfnma(v, ent<B>(D, r, (int)dd, sg), xa[i]);
            }
        }
        if (p + 1 < D.P && r >= r1 - B) {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                const int64_t dd = gb + i - r;
                if (dd <= B) v = cfnma(v, ent<B>(D, r, (int)dd, sg), xb[i]);
            }
        }
        return v;
    }, [&](int64_t r, c128 y) { Xout[(size_t)r * kp + lane] = y; });
    if (p >= 1)
#pragma unroll
        for (int i = 0; i < B; ++i) Xout[(size_t)(ga + i) * kp + lane] = xa[i];
}

// res = rhs - S x, error-free products, double-double sum, rounded once
template <int B>
__global__ void k_band_residual(BandDev D, ShiftDev S, const c128 *__restrict__ rsh, const c128 *__restrict__ X,
                                c128 *__restrict__ res) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= D.npad * D.kp) return;
    const int64_t i = t / D.kp;
    const int lane = (int)(t % D.kp);
    if (i >= D.n) {
        res[t] = cmk(0.0, 0.0);
        return;
    }
    const c128 sg = S.sigma[lane];
    const c128 b = rsh[i];
    ddacc re = {b.x, 0.0}, im = {b.y, 0.0};
#pragma unroll
    for (int d = -B; d <= B; ++d) {
        const int64_t c = i + d;
        if (c < 0 || c >= D.n) continue;
        const c128 e = ent<B>(D, i, d, sg);
        const c128 v = X[(size_t)c * D.kp + lane];
        dd pr;
        pr = two_prod(e.x, v.x); ddacc_add(re, -pr.hi); re.lo = __dsub_rn(re.lo, pr.lo);
        pr = two_prod(e.y, v.y); ddacc_add(re, pr.hi); re.lo = __dadd_rn(re.lo, pr.lo);
        pr = two_prod(e.x, v.y); ddacc_add(im, -pr.hi); im.lo = __dsub_rn(im.lo, pr.lo);
        pr = two_prod(e.y, v.x); ddacc_add(im, -pr.hi); im.lo = __dsub_rn(im.lo, pr.lo);
    }
    res[t] = cmk(__dadd_rn(re.hi, re.lo), __dadd_rn(im.hi, im.lo));
}

// acc (dd, SoA 4n) or uout = sum_j beta_j (x1_j [+ x2_j]), fixed shift order
// (the same per-row operations as the COCG accumulation)
__global__ void k_band_accum(int64_t n, int kp, int k, const c128 *__restrict__ beta, const c128 *__restrict__ x1,
                             const c128 *__restrict__ x2, double *acc, c128 *uout) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    ddacc re = {0.0, 0.0}, im = {0.0, 0.0};
    for (int jj = 0; jj < k; ++jj) {
        const c128 b = beta[jj];
        c128 x = x1[(size_t)i * kp + jj];
        ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
        ddacc_add(im, fma(b.x, x.y, b.y * x.x));
        if (x2) {
            x = x2[(size_t)i * kp + jj];
            ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
            ddacc_add(im, fma(b.x, x.y, b.y * x.x));
        }
    }
    const dd sre = fast_two_sum(re.hi, re.lo), sim = fast_two_sum(im.hi, im.lo);
    if (uout) {
        uout[i] = cmk(__dadd_rn(sre.hi, sre.lo), __dadd_rn(sim.hi, sim.lo));
    } else {
        acc[i] = sre.hi;
        acc[n + i] = sre.lo;
        acc[2 * n + i] = sim.hi;
        acc[3 * n + i] = sim.lo;
    }
}

// ---- shared-memory staged step kernels (P small: the reference's P2 sizes) --
// One CTA per (block, group of BLG lanes): all threads copy the block's factor
// rows and rhs into shared memory (independent coalesced loads, ~one memory
// latency), then one thread per lane runs the dependent sweeps out of shared
// memory instead of paying an HBM/L2 round trip every few rows.
#ifndef BAND_BLG
#define BAND_BLG 8   // swept (scripts/tune_blg.sh, P2 acceptance step): 16: 45.5 us, 8: 43.7, 4: 43.6
#endif
constexpr int BLG = BAND_BLG;
constexpr int BST_NT = 256;

template <int B>
__host__ __device__ inline size_t band_st_smem(int M, int lg) {
    return (size_t)M * lg * sizeof(c128) * (2 * B + 3);   // factors + rhs + sweep scratch
}

template <int B>
__device__ __forceinline__ void band_stage(const BandDev &D, const c128 *rsh, const c128 *rps, int64_t r0,
                                           int64_t r1, int lane0, int lg, c128 *f, c128 *rb) {
    const int m = (int)(r1 - r0);
    const int kp = D.kp;
    const int nf = m * (2 * B + 1) * lg;
    for (int idx = threadIdx.x; idx < nf; idx += blockDim.x) {
        const int l = idx % lg, cr = idx / lg;
        const int co = cr % (2 * B + 1), rr = cr / (2 * B + 1);
        const int64_t r = r0 + rr;
        const int lane = lane0 + l;
        const c128 *src = co < B       ? D.lo + ((size_t)r * B + co) * kp + lane
                          : co < 2 * B ? D.up + ((size_t)r * B + co - B) * kp + lane
                                       : D.dinv + (size_t)r * kp + lane;
        cp_async16(f + idx, src);
    }
    if (rsh) {
        for (int idx = threadIdx.x; idx < m; idx += blockDim.x) cp_async16(rb + idx, rsh + r0 + idx);
    } else {
        for (int idx = threadIdx.x; idx < m * lg; idx += blockDim.x)
            cp_async16(rb + idx, rps + (size_t)(r0 + idx / lg) * kp + lane0 + idx % lg);
    }
    cp_async_wait_all();
    __syncthreads();
}

template <int B>
__global__ void __launch_bounds__(BST_NT) k_band_s1_st(BandDev D, ShiftDev S, const c128 *__restrict__ rsh,
                                                       const c128 *__restrict__ rps) {
    extern __shared__ __align__(16) unsigned char bsm[];
    const int p = blockIdx.x, lane0 = blockIdx.y * BLG;
    const int kp = D.kp, M = D.M;
    const int lg = min(BLG, kp - lane0);
    const int64_t r0 = blk_i0(p, M, B), r1 = (int64_t)(p + 1) * M;
    const int m = (int)(r1 - r0);
    c128 *f = reinterpret_cast<c128 *>(bsm);
    c128 *rb = f + (size_t)M * (2 * B + 1) * lg;
    c128 *yt = rb + (size_t)M * lg;
    band_stage<B>(D, rsh, rps, r0, r1, lane0, lg, f, rb);
    const int ll = threadIdx.x;
    if (ll >= lg) return;
    const int lane = lane0 + ll;
    const c128 sg = S.sigma[lane];
    const SmemF<B> fa{f, r0, lg, ll};
    c128 yf[B], yl[B];
    interior_solve_f<B>(
        fa, [&](int64_t r) -> c128 & { return yt[(size_t)(r - r0) * lg + ll]; }, r0, r1,
        [&](int64_t r) { return rsh ? rb[r - r0] : rb[(size_t)(r - r0) * lg + ll]; },
        [&](int64_t r, c128 y) {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (r == r0 + i) yf[i] = y;
                if (r == r1 - B + i) yl[i] = y;
            }
        });
    (void)m;
    c128 *gc = D.gcon + (size_t)p * 2 * B * kp;
    if (p >= 1) {
        c128 gg[B][B], gp[B][B], gcur[B][B];
        couplings<B>(D, p, sg, gg, gp, gcur);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            c128 s = cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < B; ++j) s = cadd(s, cmul(gcur[i][j], yf[j]));
            gc[(size_t)i * kp + lane] = s;
        }
    }
    if (p + 1 < D.P) {
        c128 gg[B][B], gp[B][B], gcur[B][B];
        couplings<B>(D, p + 1, sg, gg, gp, gcur);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            c128 s = cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < B; ++j) s = cadd(s, cmul(gp[i][j], yl[j]));
            gc[(size_t)(B + i) * kp + lane] = s;
        }
    }
}

// the beta-weighted dd lane sum of the rows [i0, i1) (k_band_accum's
// operations, bit for bit), for the last interior pass fused into its kernel
__device__ __forceinline__ void band_lane_sum(int64_t i0, int64_t i1, int64_t n, int kp, int k,
                                              const c128 *__restrict__ beta, const c128 *x1, const c128 *x2,
                                              double *acc, c128 *uout) {
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        if (i >= n) break;
        ddacc re = {0.0, 0.0}, im = {0.0, 0.0};
        for (int jj = 0; jj < k; ++jj) {
            const c128 b = beta[jj];
            c128 x = x1[(size_t)i * kp + jj];
            ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
            ddacc_add(im, fma(b.x, x.y, b.y * x.x));
            if (x2) {
                x = x2[(size_t)i * kp + jj];
                ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
                ddacc_add(im, fma(b.x, x.y, b.y * x.x));
            }
        }
        const dd sre = fast_two_sum(re.hi, re.lo), sim = fast_two_sum(im.hi, im.lo);
        if (uout) {
            uout[i] = cmk(__dadd_rn(sre.hi, sre.lo), __dadd_rn(sim.hi, sim.lo));
        } else {
            acc[i] = sre.hi;
            acc[n + i] = sre.lo;
            acc[2 * n + i] = sim.hi;
            acc[3 * n + i] = sim.lo;
        }
    }
}

struct BandFuse {      // the last pass's lane sum, fused into k_band_s3_st (lpc == kp)
    int on, k;
    const c128 *beta, *x1;   // x1: the first pass's x when this is the correction pass, else null
    double *acc;
    c128 *uout;
};

template <int B>
__global__ void __launch_bounds__(BST_NT) k_band_s3_st(BandDev D, ShiftDev S, const c128 *__restrict__ rsh,
                                                       const c128 *__restrict__ rps, c128 *Xout, int lpc,
                                                       BandFuse fu) {
    extern __shared__ __align__(16) unsigned char bsm[];
    const int p = blockIdx.x, lane0 = blockIdx.y * lpc;
    const int kp = D.kp, M = D.M;
    const int lg = min(lpc, kp - lane0);
    const int64_t r0 = blk_i0(p, M, B), r1 = (int64_t)(p + 1) * M;
    c128 *f = reinterpret_cast<c128 *>(bsm);
    c128 *rb = f + (size_t)M * (2 * B + 1) * lg;
    c128 *yt = rb + (size_t)M * lg;
    band_stage<B>(D, rsh, rps, r0, r1, lane0, lg, f, rb);
    const int ll = threadIdx.x;
    if (ll < lg) {
    const int lane = lane0 + ll;
    const c128 sg = S.sigma[lane];
    c128 xa[B], xb[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        xa[i] = p >= 1 ? D.xg[((size_t)p * B + i) * kp + lane] : cmk(0.0, 0.0);
        xb[i] = p + 1 < D.P ? D.xg[((size_t)(p + 1) * B + i) * kp + lane] : cmk(0.0, 0.0);
    }
    const int64_t ga = (int64_t)p * M, gb = (int64_t)(p + 1) * M;
    const SmemF<B> fa{f, r0, lg, ll};
    interior_solve_f<B>(
        fa, [&](int64_t r) -> c128 & { return yt[(size_t)(r - r0) * lg + ll]; }, r0, r1,
        [&](int64_t r) {
            c128 v = rsh ? rb[r - r0] : rb[(size_t)(r - r0) * lg + ll];
            if (p >= 1 && r < r0 + B) {
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    const int64_t dd = ga + i - r;
                    if (dd >= -B) v = cfnma(v, ent<B>(D, r, (int)dd, sg), xa[i]);
                }
            }
            if (p + 1 < D.P && r >= r1 - B) {
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    const int64_t dd = gb + i - r;
                    if (dd <= B) v = cfnma(v, ent<B>(D, r, (int)dd, sg), xb[i]);
                }
            }
            return v;
        },
        [&](int64_t r, c128 y) { Xout[(size_t)r * kp + lane] = y; });
    if (p >= 1)
#pragma unroll
        for (int i = 0; i < B; ++i) Xout[(size_t)(ga + i) * kp + lane] = xa[i];
    }
    if (fu.on) {   // every lane of the block's rows is in this CTA: sum them here
        __syncthreads();
        band_lane_sum((int64_t)p * M, (int64_t)(p + 1) * M, D.n, kp, fu.k, fu.beta, fu.x1 ? fu.x1 : Xout,
                      fu.x1 ? Xout : nullptr, fu.acc, fu.uout);
    }
}

// interface system, a CTA per rlg(B) shifts: all threads stage the shifts'
// BCR blocks, multipliers and reduced rhs in shared memory (cp.async, every
// copy in flight), then the CTA's threads split each level's blocks among
// themselves (256 / rlg threads per shift, a barrier between levels)
template <int B>
__host__ __device__ constexpr int band_rlg() { return 1; }   // swept (P2 acceptance): 4 lanes per CTA 27.0 us, 1 lane 18.7 us
template <int B>
__host__ __device__ inline size_t band_red_lane_elems(int P) {
    const int nb = P > 1 ? P - 1 : 1;
    return (size_t)nb * (3 * B * B + 2 * B) + (size_t)bcr_off(nb, bcr_levels(nb)) * 2 * B * B;
}
template <int B>
__host__ __device__ inline size_t band_red_smem(int P) {
    return band_red_lane_elems<B>(P) * band_rlg<B>() * sizeof(c128);
}

template <int B>
__global__ void __launch_bounds__(256) k_band_red_st(BandDev D, const c128 *__restrict__ rsh,
                                                     const c128 *__restrict__ rps) {
    extern __shared__ __align__(16) unsigned char bsm[];
    constexpr int RL = band_rlg<B>();
    const int lane0 = blockIdx.x * RL;
    const int kp = D.kp, M = D.M, nb = D.P - 1;
    const int lg = min(RL, kp - lane0);
    const int ns = bcr_off(nb, bcr_levels(nb));
    const size_t per = band_red_lane_elems<B>(D.P);
    c128 *sm = reinterpret_cast<c128 *>(bsm);
    // per lane l: [A | Di | C] nb x 3B^2, [al | ga] ns x 2B^2, g nb x B, x nb x B
    auto base = [&](int l) { return sm + (size_t)l * per; };
    const int W3 = 3 * B * B;
    for (int idx = threadIdx.x; idx < nb * W3 * lg; idx += blockDim.x) {
        const int l = idx % lg, r = idx / lg;
        const int j = r / W3, e = r % W3;
        const c128 *arr = e < B * B ? D.rl : e < 2 * B * B ? D.rdi : D.ru;
        cp_async16(base(l) + (size_t)j * W3 + e, arr + ((size_t)(j + 1) * B * B + e % (B * B)) * kp + lane0 + l);
    }
    for (int idx = threadIdx.x; idx < ns * 2 * B * B * lg; idx += blockDim.x) {
        const int l = idx % lg, r = idx / lg;
        const int k = r / (2 * B * B), e = r % (2 * B * B);
        const c128 *arr = e < B * B ? D.ral : D.rga;
        cp_async16(base(l) + (size_t)nb * W3 + (size_t)k * 2 * B * B + e,
                   arr + ((size_t)k * B * B + e % (B * B)) * kp + lane0 + l);
    }
    for (int idx = threadIdx.x; idx < nb * B * lg; idx += blockDim.x) {
        const int l = idx % lg, r = idx / lg;
        const int j = r / B, i = r % B, p = j + 1, lane = lane0 + l;
        const c128 *gprev = D.gcon + ((size_t)(p - 1) * 2 * B + B) * kp;
        const c128 *gcur = D.gcon + (size_t)p * 2 * B * kp;
        base(l)[(size_t)nb * W3 + (size_t)ns * 2 * B * B + (size_t)j * B + i] =
            csub(csub(rhs_at<B>(D, rsh, rps, (int64_t)p * M + i, lane), __ldg(gprev + (size_t)i * kp + lane)),
                 __ldg(gcur + (size_t)i * kp + lane));
    }
    cp_async_wait_all();
    __syncthreads();
    constexpr int TPL = 256 / RL;
    const int l = threadIdx.x / TPL, tid = threadIdx.x % TPL;
    const int ll = l < lg ? l : 0;                  // idle lanes still join the barriers
    const int nthr = l < lg ? TPL : 0;
    c128 *b0 = base(ll);
    c128 *gv = b0 + (size_t)nb * W3 + (size_t)ns * 2 * B * B;
    c128 *xv = gv + (size_t)nb * B;
    auto mat = [&](const c128 *src, c128 (&o)[B][B]) {
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
            for (int j = 0; j < B; ++j) o[i][j] = src[i * B + j];
    };
    bcr_solve<B>(
        // an idle lane's threads get tid = nb: no work, but the same barriers
        nb, nthr ? tid : nb, nthr ? TPL : 1, [&](int j, c128 (&o)[B][B]) { mat(b0 + (size_t)j * W3, o); },
        [&](int j, c128 (&o)[B][B]) { mat(b0 + (size_t)j * W3 + B * B, o); },
        [&](int j, c128 (&o)[B][B]) { mat(b0 + (size_t)j * W3 + 2 * B * B, o); },
        [&](int k, c128 (&o)[B][B]) { mat(b0 + (size_t)nb * W3 + (size_t)k * 2 * B * B, o); },
        [&](int k, c128 (&o)[B][B]) { mat(b0 + (size_t)nb * W3 + (size_t)k * 2 * B * B + B * B, o); },
        [&](int j) { return StridedVec{gv + (size_t)j * B, 1}; }, [&](int j) { return StridedVec{xv + (size_t)j * B, 1}; },
        [] { __syncthreads(); });
    for (int idx = threadIdx.x; idx < nb * B * lg; idx += blockDim.x) {
        const int l2 = idx % lg, r = idx / lg;
        const int j = r / B, i = r % B;
        const c128 *xs = base(l2) + (size_t)nb * W3 + (size_t)ns * 2 * B * B + (size_t)nb * B;
        D.xg[((size_t)(j + 1) * B + i) * kp + lane0 + l2] = xs[(size_t)j * B + i];
    }
}

int launch_nt(int kp) { return std::max(128, kp); }
int launch_grid(const BandDev &D) {
    const int per = launch_nt(D.kp) / D.kp;
    return (D.P + per - 1) / per;
}

template <int B>
cudaError_t solve_chain(BandImpl *im, const ShiftDev &S, cudaStream_t st, const c128 *rsh, const c128 *rps,
                        c128 *Xout, int64_t *launches, ProfHook *hook, int kreal, BandFuse fu = BandFuse{}) {
    BandDev &D = im->D;
    const int nt = launch_nt(D.kp), grid = launch_grid(D);
    const double lane_rows = (double)D.npad * kreal;
    const dim3 sgrid(D.P, (D.kp + BLG - 1) / BLG);
    const size_t ssm = band_st_smem<B>(D.M, std::min(BLG, D.kp)), rsm = band_red_smem<B>(D.P);
    if (hook) hook->begin("band_s1", 16.0 * lane_rows * ((2 * B + 1) + 2) + (rps ? 16.0 * lane_rows : 16.0 * D.npad));
    if (im->staged) k_band_s1_st<B><<<sgrid, BST_NT, ssm, st>>>(D, S, rsh, rps);
    else k_band_s1<B><<<grid, nt, 0, st>>>(D, S, rsh, rps);
    if (hook) hook->end();
    if (hook) hook->begin("band_red", 0.0);
    if (im->staged && D.P > 1)
        k_band_red_st<B><<<(D.kp + band_rlg<B>() - 1) / band_rlg<B>(), 256, rsm, st>>>(D, rsh, rps);
    else k_band_red<B><<<(D.kp + 31) / 32, 32, 0, st>>>(D, rsh, rps);
    if (hook) hook->end();
    if (hook) hook->begin("band_s3", 16.0 * lane_rows * ((2 * B + 1) + 2) + (rps ? 16.0 * lane_rows : 16.0 * D.npad));
    if (im->staged) {
        // the last pass of a step sums the lanes in the same kernel: all of a
        // block's lanes in one CTA
        const int lpc = fu.on ? D.kp : BLG;
        const dim3 g3(D.P, (D.kp + lpc - 1) / lpc);
        k_band_s3_st<B><<<g3, BST_NT, band_st_smem<B>(D.M, std::min(lpc, D.kp)), st>>>(D, S, rsh, rps, Xout, lpc, fu);
    }
    else k_band_s3<B><<<grid, nt, 0, st>>>(D, S, rsh, rps, Xout);
    if (hook) hook->end();
    *launches += 3;
    return cudaGetLastError();
}

}  // namespace

#define BK(expr)                                                      \
    do {                                                              \
        cudaError_t _e = (expr);                                      \
        if (_e != cudaSuccess) {                                      \
            err = std::string(#expr) + ": " + cudaGetErrorString(_e); \
            return REXI_ERR_CUDA;                                     \
        }                                                             \
    } while (0)

static int balloc(BandState &bs, void **p, size_t bytes, std::string &err) {
    cudaError_t e = cudaMalloc(p, bytes < 16 ? 16 : bytes);
    if (e == cudaSuccess) e = rexi_poison(*p, bytes < 16 ? 16 : bytes);
    if (e != cudaSuccess) {
        err = std::string("cudaMalloc failed: ") + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? REXI_ERR_NOMEM : REXI_ERR_CUDA;
    }
    bs.allocs.push_back(*p);
    bs.bytes += (int64_t)bytes;
    return REXI_OK;
}
#define BA(ptr, bytes)                                                  \
    do {                                                                \
        int _rc = balloc(bs, (void **)&(ptr), (size_t)(bytes), err);    \
        if (_rc) return _rc;                                            \
    } while (0)

template <int B>
static int band_create_t(BandState &bs, BandImpl *im, const rexi_desc *d, const ShiftDev &S, cudaStream_t st,
                         std::string &err) {
    BandDev &D = im->D;
    const int kp = bs.kp;
    const int64_t n = d->n;
    // the interior sweeps (2M dependent rows) and the interface chain (2P
    // dependent blocks) balance at M ~ sqrt(n)
    int M = 16;
    while ((double)M * M < (double)n && M < 2048) M *= 2;
    M = std::max(M, 4 * B);
    // the reference's P2 sizes: blocks of 64 rows whose factors fit shared
    // memory, and an interface chain whose pieces fit one CTA's shared memory
#ifndef BAND_MST
#define BAND_MST 32   // swept (scripts/tune_mst.sh, P2 acceptance step): 64: 43.7 us, 32: 41.5, 16: 53.7
#endif
    constexpr int MST = BAND_MST;
    const int64_t pst = (n + MST - 1) / MST;
    if (!getenv("REXI_BAND_NOSTAGE") && band_red_smem<B>((int)std::min<int64_t>(pst, 1 << 20)) <= 200 * 1024 &&
        band_st_smem<B>(MST, std::min(BLG, kp)) <= 200 * 1024) {
        M = MST;
        im->staged = true;
    }
    const int P = (int)((n + M - 1) / M);
    const int64_t npad = (int64_t)P * M;
    bs.B = B;
    bs.n = n;
    bs.npad = npad;
    bs.M = M;
    bs.P = P;
    const int w = 2 * B + 1;
    std::vector<double> ta((size_t)w * npad, 0.0), tai((size_t)w * npad, 0.0), bb((size_t)w * npad, 0.0);
    for (int64_t r = 0; r < n; ++r)
        for (int32_t q = d->indptr[r]; q < d->indptr[r + 1]; ++q) {
            const int64_t dd = (int64_t)d->indices[q] - r;
            const size_t o = (size_t)(dd + B) * npad + r;
            ta[o] += d->tau * d->a_vals[q];
            tai[o] += d->a_imag ? d->tau * d->a_imag[q] : 0.0;
            bb[o] += d->b_vals[q];
        }
    for (int64_t r = n; r < npad; ++r) ta[(size_t)B * npad + r] = 1.0;   // decoupled unit rows
    double *dta, *dtai, *dbb;
    BA(dta, sizeof(double) * ta.size());
    BA(dtai, sizeof(double) * tai.size());
    BA(dbb, sizeof(double) * bb.size());
    BK(cudaMemcpyAsync(dta, ta.data(), sizeof(double) * ta.size(), cudaMemcpyHostToDevice, st));
    BK(cudaMemcpyAsync(dtai, tai.data(), sizeof(double) * tai.size(), cudaMemcpyHostToDevice, st));
    BK(cudaMemcpyAsync(dbb, bb.data(), sizeof(double) * bb.size(), cudaMemcpyHostToDevice, st));
    D.n = n;
    D.npad = npad;
    D.M = M;
    D.P = P;
    D.kp = kp;
    D.ta = dta;
    D.tai = dtai;
    D.bb = dbb;
    const size_t rows_kp = (size_t)npad * kp;
    BA(D.lo, sizeof(c128) * rows_kp * B);
    BA(D.up, sizeof(c128) * rows_kp * B);
    BA(D.dinv, sizeof(c128) * rows_kp);
    BA(D.spk, sizeof(c128) * (size_t)P * 4 * B * B * kp);
    BA(D.rl, sizeof(c128) * (size_t)P * B * B * kp);
    BA(D.rdi, sizeof(c128) * (size_t)P * B * B * kp);
    BA(D.ru, sizeof(c128) * (size_t)P * B * B * kp);
    {
        const int nb = std::max(1, P - 1);
        const size_t ns = (size_t)std::max(1, bcr_off(nb, bcr_levels(nb)));
        BA(D.ral, sizeof(c128) * ns * B * B * kp);
        BA(D.rga, sizeof(c128) * ns * B * B * kp);
    }
    BA(D.gcon, sizeof(c128) * (size_t)P * 2 * B * kp);
    BA(D.xg, sizeof(c128) * (size_t)P * B * kp);
    BA(D.X, sizeof(c128) * rows_kp);
    BK(cudaMemsetAsync(D.spk, 0, sizeof(c128) * (size_t)P * 4 * B * B * kp, st));
    BK(cudaMemsetAsync(D.gcon, 0, sizeof(c128) * (size_t)P * 2 * B * kp, st));
    BK(cudaMemsetAsync(D.xg, 0, sizeof(c128) * (size_t)P * B * kp, st));
    BA(im->rhs, sizeof(c128) * npad);
    BA(im->X1, sizeof(c128) * rows_kp);
    if (bs.refine > 0) {
        BA(im->X2, sizeof(c128) * rows_kp);
        BA(im->res, sizeof(c128) * rows_kp);
    }
    BA(im->pstat, sizeof(double) * 2 * kp);
    {
        std::vector<double> init(2 * kp, 0.0);
        for (int l = 0; l < kp; ++l) init[l] = INFINITY;
        BK(cudaMemcpyAsync(im->pstat, init.data(), sizeof(double) * 2 * kp, cudaMemcpyHostToDevice, st));
    }
    if (im->staged) {
        BK(cudaFuncSetAttribute(k_band_s1_st<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)band_st_smem<B>(M, std::min(BLG, kp))));
        BK(cudaFuncSetAttribute(k_band_s3_st<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::min<size_t>(band_st_smem<B>(M, std::max(BLG, kp)), 227 * 1024)));
        BK(cudaFuncSetAttribute(k_band_red_st<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)band_red_smem<B>(P)));
    }
    k_band_factor<B><<<launch_grid(D), launch_nt(kp), 0, st>>>(D, S, im->pstat);
    BK(cudaGetLastError());
    k_band_rfactor<B><<<(kp + 31) / 32, 32, 0, st>>>(D, S, im->pstat);
    BK(cudaGetLastError());
    std::vector<double> ps(2 * kp);
    BK(cudaMemcpyAsync(ps.data(), im->pstat, sizeof(double) * 2 * kp, cudaMemcpyDeviceToHost, st));
    BK(cudaStreamSynchronize(st));
    double worst = 1.0;
    for (int j = 0; j < bs.k; ++j) {
        const double mn = ps[j], mx = ps[kp + j];
        if (!(mn > 0.0) || !(mx < INFINITY)) {
            char buf[200];
            snprintf(buf, sizeof buf, "no-pivot band factorization broke down (pivot ratio = %.3e) [shift j = %d]",
                     mx > 0 ? mn / mx : 0.0, d->shift_ids ? d->shift_ids[j] : d->shift_offset + j);
            err = buf;
            return REXI_ERR_SINGULAR;
        }
        worst = std::min(worst, mn / mx);
    }
    bs.min_pivot_ratio = worst;
    return REXI_OK;
}

int band_create(BandState &bs, const rexi_desc *d, int B, const ShiftDev &S, int kp, int refine, cudaStream_t st,
                std::string &err) {
    BandImpl *im = new BandImpl();
    bs.impl = im;
    bs.k = d->k;
    bs.kp = kp;
    bs.refine = refine;
    switch (B) {
        case 2: return band_create_t<2>(bs, im, d, S, st, err);
        case 3: return band_create_t<3>(bs, im, d, S, st, err);
        case 4: return band_create_t<4>(bs, im, d, S, st, err);
        default:
            err = "BAND solver handles half bandwidths 2..4";
            return REXI_ERR_UNSUPPORTED;
    }
}

// the last pass sums the lanes in its own kernel when the staged sweeps hold
// every lane of a block in one CTA (k_band_s3_st, BandFuse)
template <int B>
static bool band_can_fuse(const BandImpl *im) {
    return im->staged && band_st_smem<B>(im->D.M, im->D.kp) <= 200 * 1024;
}

template <int B>
static int band_run(BandState &bs, const ShiftDev &S, cudaStream_t st, int64_t *launches, const c128 **x1,
                    const c128 **x2, std::string &err, bool *summed = nullptr, double *acc = nullptr,
                    c128 *uout = nullptr) {
    BandImpl *im = (BandImpl *)bs.impl;
    BandDev &D = im->D;
    const bool fuse = summed != nullptr && band_can_fuse<B>(im);
    if (summed) *summed = fuse;
    BandFuse fu{fuse ? 1 : 0, bs.k, S.beta, nullptr, acc, uout};
    BK(solve_chain<B>(im, S, st, im->rhs, nullptr, im->X1, launches, bs.hook, bs.k,
                      bs.refine > 0 ? BandFuse{} : fu));
    *x1 = im->X1;
    *x2 = nullptr;
    if (bs.refine > 0) {
        const int64_t t = D.npad * D.kp;
        if (bs.hook) bs.hook->begin("band_residual", 16.0 * t * 2 + 24.0 * (2 * B + 1) * D.npad);
        k_band_residual<B><<<(unsigned)((t + 255) / 256), 256, 0, st>>>(D, S, im->rhs, im->X1, im->res);
        if (bs.hook) bs.hook->end();
        BK(cudaGetLastError());
        ++*launches;
        fu.x1 = im->X1;
        BK(solve_chain<B>(im, S, st, nullptr, im->res, im->X2, launches, bs.hook, bs.k, fu));
        *x2 = im->X2;
    }
    return REXI_OK;
}

static int band_run_any(BandState &bs, const ShiftDev &S, cudaStream_t st, int64_t *launches, const c128 **x1,
                        const c128 **x2, std::string &err, bool *summed = nullptr, double *acc = nullptr,
                        c128 *uout = nullptr) {
    switch (bs.B) {
        case 2: return band_run<2>(bs, S, st, launches, x1, x2, err, summed, acc, uout);
        case 3: return band_run<3>(bs, S, st, launches, x1, x2, err, summed, acc, uout);
        default: return band_run<4>(bs, S, st, launches, x1, x2, err, summed, acc, uout);
    }
}

int band_step(BandState &bs, const ShiftDev &S, cudaStream_t st, const c128 *u, c128 *uout, double *acc,
              int64_t *launches, std::string &err) {
    BandImpl *im = (BandImpl *)bs.impl;
    BandDev &D = im->D;
    const unsigned g = (unsigned)((D.npad + 255) / 256);
    if (bs.hook) bs.hook->begin("band_rhs", 16.0 * 2 * D.n + 8.0 * (2 * bs.B + 1) * D.npad);
    switch (bs.B) {
        case 2: k_band_rhs<2><<<g, 256, 0, st>>>(D, u, im->rhs); break;
        case 3: k_band_rhs<3><<<g, 256, 0, st>>>(D, u, im->rhs); break;
        default: k_band_rhs<4><<<g, 256, 0, st>>>(D, u, im->rhs); break;
    }
    if (bs.hook) bs.hook->end();
    BK(cudaGetLastError());
    ++*launches;
    const c128 *x1 = nullptr, *x2 = nullptr;
    bool summed = false;
    int rc = band_run_any(bs, S, st, launches, &x1, &x2, err, &summed, acc, uout);
    if (rc) return rc;
    if (summed) return REXI_OK;
    if (bs.hook) bs.hook->begin("band_accum", (x2 ? 32.0 : 16.0) * D.n * bs.k + 32.0 * D.n);
    k_band_accum<<<(unsigned)((D.n + 255) / 256), 256, 0, st>>>(D.n, D.kp, bs.k, S.beta, x1, x2, acc, uout);
    if (bs.hook) bs.hook->end();
    BK(cudaGetLastError());
    ++*launches;
    return REXI_OK;
}

int band_solve_all(BandState &bs, const ShiftDev &S, cudaStream_t st, const c128 *rhs, c128 *x, std::string &err) {
    BandImpl *im = (BandImpl *)bs.impl;
    BandDev &D = im->D;
    BK(cudaMemsetAsync(im->rhs, 0, sizeof(c128) * D.npad, st));
    BK(cudaMemcpyAsync(im->rhs, rhs, sizeof(c128) * D.n, cudaMemcpyDeviceToDevice, st));
    int64_t launches = 0;
    const c128 *x1 = nullptr, *x2 = nullptr;
    int rc = band_run_any(bs, S, st, &launches, &x1, &x2, err);
    if (rc) return rc;
    if (x2) BK(cocg_axpy_inplace(im->X1, x2, D.npad * D.kp, st));
    BK(tri_launch_transpose(im->X1, D.n, D.kp, bs.k, x, st));
    return REXI_OK;
}

void band_destroy(BandState &bs) {
    for (void *p : bs.allocs) cudaFree(p);
    bs.allocs.clear();
    delete (BandImpl *)bs.impl;
    bs.impl = nullptr;
}

}  // namespace rexi
