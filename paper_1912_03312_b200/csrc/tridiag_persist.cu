// tridiag_persist.cu -- n REXI steps of a small 1D system in ONE launch
// (persistent multi-step loop for small configs, reference
// rexi_run integrate.py:229-245).
//
// For config-1-sized systems (10^3 rows) a step of the multi-kernel path is
// a chain of 8 dependent launches: launch latency, not work.  Here one
// thread-block cluster runs all n steps; the phases of a step are separated
// by hardware cluster barriers (~0.2 us) instead of kernel boundaries.
//
// Residency: CTA c of the cluster owns a fixed slice of level-0 blocks and
// keeps that slice's inverse pivots and A/B diagonals in shared memory for
// the whole launch (loaded once), so the level-0 phases read only shared
// memory plus the state u.  The small reduced levels stay in global memory
// (L2) and are read in batches.
//
// Every phase repeats the operation order of the multi-kernel path (k_rhs,
// tridiag_l0.cu S1 / S3ACC + reduce_rows, k_lv_tma / k_block, k_top_solve),
// so the result is bitwise identical to it (tests/test_gpu_persist.py).
//
// Phases of a step (levels 0..T, T = top with one row):
//   A  rhs = iBu of the slice's rows (shared), level-0 S1 of its blocks
//   B  levels 1..T-2 S1
//   C  level T-1 (one block): S1, top solve, S3 -- one thread per shift
//   D  levels T-2..1 S3
//   E  level-0 S3 of the slice into a shared tile + the beta-weighted
//      double-double row sums (lane order of reduce_rows) -> u_next
// Data written by another CTA is read after a cluster barrier
// (barrier.cluster.arrive.release / wait.acquire), which orders it for the
// plain loads used here (PTX memory model).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "tridiag.cuh"
#include "tridiag_launch.h"

namespace cgr = cooperative_groups;

namespace rexi {

constexpr int PS_NT = 256;

struct PersistArgs {
    L0Dev z;
    LevelDev lv[PS_MAXLV];
    int nl;                 // levels incl. top
    ShiftDev S;
    int64_t n;              // real rows (level 0 is padded to lv[0].n)
    int bc;                 // level-0 blocks per CTA
    const c128 *u_in;
    c128 *ua, *ub;          // state ping-pong [n]
    c128 *snaps;            // optional [n_steps][n]: state after every step
    c128 *final_out;        // optional: the last state also goes here (mapped page-locked host output)
    int n_steps;
    unsigned long long *tstamp;   // optional (REXI_PERSIST_TRACE): %globaltimer per phase, steps 0-2
};

// shared-memory slice of CTA c: rows [r0, r0 + R) of level 0 (R = bc * M)
struct Slice {
    c128 *inv;      // [R][kp] inverse pivots
    c128 *tile;     // [R][kp] x of the S3 pass (phase E)
    c128 *rhs;      // [R + 1] rhs = iBu (row r0 + R = next slice's first interface row)
    double *zd;     // 9 x [R + 1]: ta/ta_im/b of sub, dia, sup
};

__host__ __device__ inline size_t slice_bytes(int bc, int kp) {
    const size_t R = (size_t)bc * TRI_M;
    return 2 * R * kp * sizeof(c128) + (R + 1) * sizeof(c128) + 9 * (R + 1) * sizeof(double);
}

__device__ __forceinline__ Slice carve_slice(unsigned char *smem, int bc, int kp) {
    const int R = bc * TRI_M;
    Slice s;
    s.inv = reinterpret_cast<c128 *>(smem);
    s.tile = s.inv + (size_t)R * kp;
    s.rhs = s.tile + (size_t)R * kp;
    s.zd = reinterpret_cast<double *>(s.rhs + R + 1);
    return s;
}

__device__ __forceinline__ void stamp(const PersistArgs &a, int step, int &k) {
    if (a.tstamp && step < 3 && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.tstamp[step * 16 + k] = t;
    }
    ++k;
}

// entry of the level-0 shifted matrix from the slice's diagonals (form_entry,
// same rounding as co_sub<true> / co_sup<true>): d = 0 sub, 1 dia, 2 sup
__device__ __forceinline__ c128 zentry(const double *zd, int R1, int d, int r, c128 sg) {
    return form_entry(zd[(3 * d) * R1 + r], zd[(3 * d + 1) * R1 + r], zd[(3 * d + 2) * R1 + r], sg);
}

// k_rhs's rounding: rhs_i = 1j * (b_sub u_{i-1} + b_dia u_i + b_sup u_{i+1}), no FMA
__device__ __forceinline__ c128 rhs_row(double bs, double bd, double bu, const c128 *u, int64_t n, int64_t i) {
    if (i >= n) return cmk(0.0, 0.0);
    double sr = 0.0, si = 0.0;
    if (i > 0) {
        const c128 x = u[i - 1];
        sr = __dadd_rn(sr, __dmul_rn(bs, x.x));
        si = __dadd_rn(si, __dmul_rn(bs, x.y));
    }
    {
        const c128 x = u[i];
        sr = __dadd_rn(sr, __dmul_rn(bd, x.x));
        si = __dadd_rn(si, __dmul_rn(bd, x.y));
    }
    if (i + 1 < n) {
        const c128 x = u[i + 1];
        sr = __dadd_rn(sr, __dmul_rn(bu, x.x));
        si = __dadd_rn(si, __dmul_rn(bu, x.y));
    }
    return cmk(-si, sr);
}

// level-0 block b of the slice (tridiag_l0.cu sweeps on a full block), all
// operands from shared memory; PHASE 1 -> ypart/lc, PHASE 3 -> tile rows
template <int PHASE>
__device__ __forceinline__ void l0_block(const PersistArgs &a, const Slice &sl, int R, int64_t pb0, int b, int j,
                                         c128 *yp_out = nullptr, c128 *lc_out = nullptr) {
    constexpr int M = TRI_M;
    const LevelDev &L = a.lv[0];
    const int kp = a.S.kp;
    const int R1 = R + 1;
    const int64_t P = L.P, p = pb0 + b;
    const int lr0 = b * M;
    const c128 sg = a.S.sigma[j];
    c128 y[M];
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (PHASE == 3) {
        xs = a.lv[1].X[p * kp + j];
        if (p + 1 < P) xn = a.lv[1].X[(p + 1) * kp + j];
    }
    y[0] = xs;
#pragma unroll
    for (int q = 1; q < M; ++q) {
        const int r = lr0 + q;
        y[q] = cmul(sl.inv[r * kp + j], cfnma(sl.rhs[r], zentry(sl.zd, R1, 0, r, sg), y[q - 1]));
    }
    const c128 ylast = y[M - 1];
    c128 xnext = xn;
#pragma unroll
    for (int q = M - 1; q >= 1; --q) {
        const int r = lr0 + q;
        xnext = cfnma(y[q], sl.inv[r * kp + j], cmul(zentry(sl.zd, R1, 2, r, sg), xnext));
        y[q] = xnext;
    }
    if (PHASE == 1) {
        // straight into the level CTA's shared memory (distributed shared memory)
        yp_out[p * kp + j] = cfnma(sl.rhs[lr0], zentry(sl.zd, R1, 2, lr0, sg), y[1]);
        if (p + 1 < P) lc_out[(p + 1) * kp + j] = cneg(cmul(zentry(sl.zd, R1, 0, lr0 + M, sg), ylast));
        if (p == 0) lc_out[j] = cmk(0.0, 0.0);
    } else {
        c128 *tc = sl.tile + (size_t)lr0 * kp + j;
        tc[0] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q) tc[q * kp] = y[q];
    }
}

// dynamic shared memory of k_persist (offsets below are in c128 elements from here)
extern __shared__ __align__(16) unsigned char ps_smem[];

// one reduced level (l >= 1) as held by the level CTA: operands and the
// intermediate vectors in shared memory, addressed by element offsets from
// ps_smem so every access compiles to LDS/STS; level 1's solution goes to
// global memory (the level-0 S3 of the other CTAs reads it)
struct LvView {
    int invd, sup, sub;     // [n][kp] (sub unused for symmetric pencils)
    int rin_a, rin_b;       // previous level's ypart / lc  [n][kp]
    int yp, lc;             // this level's S1 outputs       [P][kp]
    int X;                  // this level's solution         [n][kp] (-1: global Xg)
    int Xn;                 // next level's solution         [P][kp]
    c128 *Xg;               // level 1: solution in global memory
    int n, P;
    int sym;
};

__device__ __forceinline__ c128 *psm() { return reinterpret_cast<c128 *>(ps_smem); }

__device__ __forceinline__ c128 lvv_sub(const LvView &V, int i, int j, int kp) {
    if (V.sym) return i > 0 ? psm()[V.sup + (i - 1) * kp + j] : cmk(0.0, 0.0);
    return psm()[V.sub + i * kp + j];
}

// reduced level block (k_lv_tma's lv_body / k_block with RHS_LV, same order)
template <int PHASE>
__device__ __forceinline__ void lv_block(const LvView V, int p, int j, int kp) {   // by value: offsets in registers
    constexpr int M = TRI_M;
    c128 *sm = psm();
    const int n = V.n, P = V.P, base = p * M;
    const int cnt = min(M, n - base) - 1;
    c128 y[M];
    c128 xs = cmk(0.0, 0.0), xn = cmk(0.0, 0.0);
    if (PHASE == 3) {
        xs = sm[V.Xn + p * kp + j];
        if (p + 1 < P) xn = sm[V.Xn + (p + 1) * kp + j];
    }
    y[0] = xs;
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q <= cnt) {
            const int i = base + q;
            const c128 d = cadd(sm[V.rin_a + i * kp + j], sm[V.rin_b + i * kp + j]);
            y[q] = cmul(sm[V.invd + i * kp + j], cfnma(d, lvv_sub(V, i, j, kp), y[q - 1]));
        }
    c128 ylast = y[0];
#pragma unroll
    for (int q = 1; q < M; ++q)
        if (q == cnt) ylast = y[q];
    c128 xnext = xn;
#pragma unroll
    for (int q = M - 1; q >= 1; --q)
        if (q <= cnt) {
            const int i = base + q;
            xnext = cfnma(y[q], sm[V.invd + i * kp + j], cmul(sm[V.sup + i * kp + j], xnext));
            y[q] = xnext;
        }
    if (PHASE == 1) {
        const c128 yfirst = cnt >= 1 ? y[1] : cmk(0.0, 0.0);
        const c128 ds = cadd(sm[V.rin_a + base * kp + j], sm[V.rin_b + base * kp + j]);
        sm[V.yp + p * kp + j] = cfnma(ds, sm[V.sup + base * kp + j], yfirst);
        if (p + 1 < P) sm[V.lc + (p + 1) * kp + j] = cneg(cmul(lvv_sub(V, base + M, j, kp), ylast));
        if (p == 0) sm[V.lc + j] = cmk(0.0, 0.0);
    } else if (V.X >= 0) {
        sm[V.X + base * kp + j] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q)
            if (q <= cnt) sm[V.X + (base + q) * kp + j] = y[q];
    } else {
        V.Xg[(int64_t)base * kp + j] = xs;
#pragma unroll
        for (int q = 1; q < M; ++q)
            if (q <= cnt) V.Xg[(int64_t)(base + q) * kp + j] = y[q];
    }
}

// k_top_solve for one lane (the top level's rows solved sequentially); the
// top's solution stays in shared memory (or global when the top is level 1)
__device__ __forceinline__ void top_solve(const LvView T, int j, int kp) {
    c128 *sm = psm();
    c128 *X = T.X >= 0 ? sm + T.X : T.Xg;
    c128 yp = cmk(0.0, 0.0);
    for (int i = 0; i < T.n; ++i) {
        const c128 d = cadd(sm[T.rin_a + i * kp + j], sm[T.rin_b + i * kp + j]);
        yp = cmul(sm[T.invd + i * kp + j], cfnma(d, lvv_sub(T, i, j, kp), yp));
        X[i * kp + j] = yp;
    }
    c128 xnext = cmk(0.0, 0.0);
    for (int i = T.n - 1; i >= 0; --i) {
        const c128 xi = cfnma(X[i * kp + j], sm[T.invd + i * kp + j], cmul(sm[T.sup + i * kp + j], xnext));
        X[i * kp + j] = xi;
        xnext = xi;
    }
}

// shared-memory footprint of the level CTA: staged level-0 outputs + every
// reduced level's operands and vectors (host and device use the same count)
__host__ __device__ inline size_t levels_bytes(const LevelDev *lv, int nl, int kp) {
    size_t e = 2 * (size_t)lv[0].P * kp;                           // staged ypart0 / lc0
    for (int l = 1; l < nl; ++l) {
        e += (size_t)lv[l].n * kp * (lv[l].sym ? 2 : 3);            // invd, sup (, sub)
        if (l <= nl - 2) e += 2 * (size_t)lv[l].P * kp;             // yp, lc
        if (l >= 2) e += (size_t)lv[l].n * kp;                       // X
    }
    return e * sizeof(c128);
}

// beta-weighted double-double sum of one row over the kp lanes, in the lane
// order and combine tree of tridiag_l0.cu reduce_rows (TPR lane groups)
template <int TPR>
__device__ __forceinline__ c128 row_sum_t(const c128 *trow, const ShiftDev &S) {
    dd gre[TPR], gim[TPR];
#pragma unroll
    for (int s = 0; s < TPR; ++s) {
        ddacc re = {0.0, 0.0}, im = {0.0, 0.0};
        for (int jj = s; jj < S.kp; jj += TPR) {
            const c128 b = S.beta[jj];
            const c128 x = trow[jj];
            ddacc_add(re, fma(b.x, x.x, -b.y * x.y));
            ddacc_add(im, fma(b.x, x.y, b.y * x.x));
        }
        gre[s] = fast_two_sum(re.hi, re.lo);
        gim[s] = fast_two_sum(im.hi, im.lo);
    }
#pragma unroll
    for (int off = TPR >> 1; off > 0; off >>= 1)
#pragma unroll
        for (int s = 0; s < off; ++s) {
            gre[s] = dd_add(gre[s], gre[s + off]);
            gim[s] = dd_add(gim[s], gim[s + off]);
        }
    return cmk(__dadd_rn(gre[0].hi, gre[0].lo), __dadd_rn(gim[0].hi, gim[0].lo));
}

__device__ __noinline__ c128 row_sum(const c128 *trow, const ShiftDev &S, int tpr) {
    switch (tpr) {
        case 1: return row_sum_t<1>(trow, S);
        case 2: return row_sum_t<2>(trow, S);
        case 4: return row_sum_t<4>(trow, S);
        default: return row_sum_t<8>(trow, S);
    }
}

__global__ void __launch_bounds__(PS_NT) k_persist(const __grid_constant__ PersistArgs pa) {
    unsigned char *smem = ps_smem;
    // one copy of the arguments in shared memory (read through references)
    __shared__ PersistArgs a_sh;
    __shared__ LvView views[PS_MAXLV];
    {
        const int words = (int)(sizeof(PersistArgs) / sizeof(int));
        const int *src = reinterpret_cast<const int *>(&pa);
        int *dst = reinterpret_cast<int *>(&a_sh);
        for (int w = threadIdx.x; w < words; w += PS_NT) dst[w] = src[w];
        __syncthreads();
    }
    const PersistArgs &a = a_sh;
    cgr::cluster_group cl = cgr::this_cluster();
    const int crank = (int)cl.block_rank();
    const int kp = a.S.kp;
    const int nl = a.nl;
    const int64_t P0 = a.lv[0].P, n0 = a.lv[0].n;
    const bool level_cta = crank == 0;
    // level-0 slice of CTA crank >= 1
    const int bc = a.bc;
    const int64_t pb0 = level_cta ? 0 : min((int64_t)(crank - 1) * bc, P0);
    const int64_t pb1 = level_cta ? 0 : min(pb0 + bc, P0);
    const int nb = (int)(pb1 - pb0);
    const int R = bc * TRI_M, R1 = R + 1;
    const int64_t r0 = pb0 * TRI_M;
    const Slice sl = carve_slice(smem, bc, kp);
    if (level_cta) {
        // resident: level 0's S1 outputs (written by the slices through
        // distributed shared memory) at offsets 0 and P0*kp, then every
        // reduced level's operands; views = offsets into ps_smem
        int off = 2 * (int)(P0 * kp);
        for (int l = 1; l < nl; ++l) {
            const LevelDev &L = a.lv[l];
            const int ne = (int)(L.n * kp);
            const int o_inv = off, o_sup = off + ne, o_sub = L.sym ? -1 : off + 2 * ne;
            off += ne * (L.sym ? 2 : 3);
            for (int e = threadIdx.x; e < ne; e += PS_NT) {
                psm()[o_inv + e] = L.invd[e];
                psm()[o_sup + e] = L.sup[e];
                if (o_sub >= 0) psm()[o_sub + e] = L.sub[e];
            }
            const int o_yp = off, o_lc = off + (int)(L.P * kp);
            if (l <= nl - 2) off += 2 * (int)(L.P * kp);
            const int o_x = l == 1 ? -1 : off;
            if (l >= 2) off += ne;
            if (threadIdx.x == 0) {
                LvView &V = views[l];
                V.invd = o_inv;
                V.sup = o_sup;
                V.sub = o_sub;
                V.n = (int)L.n;
                V.P = (int)L.P;
                V.sym = L.sym;
                V.rin_a = l == 1 ? 0 : views[l - 1].yp;
                V.rin_b = l == 1 ? (int)(P0 * kp) : views[l - 1].lc;
                V.yp = o_yp;
                V.lc = o_lc;
                V.X = o_x;
                V.Xg = a.lv[1].X;
                V.Xn = -1;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0)
            for (int l = 1; l < nl - 1; ++l) views[l].Xn = views[l + 1].X;
        __syncthreads();
    } else {
        // resident: the slice's inverse pivots and A/B diagonals
        const L0Dev &z = a.z;
        for (int64_t e = threadIdx.x; e < (int64_t)nb * TRI_M * kp; e += PS_NT)
            sl.inv[e] = a.lv[0].invd[r0 * kp + e];
        const double *src[9] = {z.ta_sub, z.ta_sub_im, z.b_sub, z.ta_dia, z.ta_dia_im, z.b_dia,
                                z.ta_sup, z.ta_sup_im, z.b_sup};
        for (int e = threadIdx.x; e < 9 * R1; e += PS_NT) {
            const int d = e / R1, r = e % R1;
            sl.zd[e] = (r <= nb * TRI_M && r0 + r < n0) ? src[d][r0 + r] : 0.0;
        }
        __syncthreads();
    }
    const int tpr = max(1, 128 / ((128 / kp) * TRI_M));   // reduce_rows' threads per row (L0_NT = 128)
    // the level CTA's staging arrays (offset 0 and P0*kp of its dynamic shared
    // memory), as seen from this CTA: the slices' S1 writes them directly
    c128 *rem_yp = cl.map_shared_rank(psm(), 0);
    c128 *rem_lc = rem_yp + P0 * kp;
    const c128 *u = a.u_in;
    for (int step = 0; step < a.n_steps; ++step) {
        int ts = 0;
        stamp(a, step, ts);
        c128 *un = (step & 1) ? a.ub : a.ua;   // the host copies the last one out
        // A (slice CTAs): rhs of the slice rows (+ next slice's first row), level-0 S1
        if (!level_cta) {
            for (int r = threadIdx.x; r <= nb * TRI_M; r += PS_NT)
                sl.rhs[r] = rhs_row(sl.zd[2 * R1 + r], sl.zd[5 * R1 + r], sl.zd[8 * R1 + r], u, a.n, r0 + r);
            __syncthreads();
            for (int it = threadIdx.x; it < nb * kp; it += PS_NT)
                l0_block<1>(a, sl, R, pb0, it / kp, it % kp, rem_yp, rem_lc);
        }
        cl.sync();
        stamp(a, step, ts);
        // M (level CTA): every reduced level, S1 up, top, S3 down
        if (level_cta) {
            stamp(a, step, ts);
            for (int l = 1; l <= nl - 2; ++l) {
                for (int t = threadIdx.x; t < views[l].P * kp; t += PS_NT) lv_block<1>(views[l], t / kp, t % kp, kp);
                __syncthreads();
                stamp(a, step, ts);
            }
            for (int j = threadIdx.x; j < kp; j += PS_NT) top_solve(views[nl - 1], j, kp);
            __syncthreads();
            stamp(a, step, ts);
            for (int l = nl - 2; l >= 1; --l) {
                for (int t = threadIdx.x; t < views[l].P * kp; t += PS_NT) lv_block<3>(views[l], t / kp, t % kp, kp);
                __syncthreads();
                stamp(a, step, ts);
            }
        }
        cl.sync();
        stamp(a, step, ts);
        // E (slice CTAs): level-0 S3 of the slice into the tile, row sums -> u_next
        if (!level_cta) {
            for (int it = threadIdx.x; it < nb * kp; it += PS_NT) l0_block<3>(a, sl, R, pb0, it / kp, it % kp);
            __syncthreads();
            for (int r = threadIdx.x; r < nb * TRI_M; r += PS_NT) {
                const int64_t row = r0 + r;
                if (row < a.n) {
                    const c128 v = row_sum(sl.tile + (size_t)r * kp, a.S, tpr);
                    un[row] = v;
                    if (a.snaps) a.snaps[(int64_t)step * a.n + row] = v;
                    if (a.final_out && step == a.n_steps - 1) a.final_out[row] = v;
                }
            }
        }
        cl.sync();
        stamp(a, step, ts);
        u = un;
    }
}

// level-0 blocks per slice CTA (CTA 0 of the cluster is the level CTA)
static int persist_bc(int64_t P0, int cs) { return (int)((P0 + (cs - 1) - 1) / (cs - 1)); }

static size_t persist_smem_bytes(const LevelDev *lv, int nl, int kp, int cs) {
    const size_t a = slice_bytes(persist_bc(lv[0].P, cs), kp), b = levels_bytes(lv, nl, kp);
    return a > b ? a : b;
}

// k_persist's dynamic shared-memory attribute as last set on this device
// (setting it costs ~1 us, a visible share of a ~20 us small-plan call)
// (per device; plans are created and stepped on their own device)
constexpr int PS_MAXDEV = 64;
static size_t g_persist_smem_attr[PS_MAXDEV] = {};
static bool g_persist_cluster_attr[PS_MAXDEV] = {};

static cudaError_t persist_set_smem(size_t sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= PS_MAXDEV) {
        cudaFuncSetAttribute(k_persist, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    }
    if (!g_persist_cluster_attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_persist, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        g_persist_cluster_attr[dev] = true;
    }
    if (sm == g_persist_smem_attr[dev]) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) g_persist_smem_attr[dev] = sm;
    return e;
}

// largest cluster this plan can run as (0: cannot run -- the slice must fit
// in shared memory and the cluster must be schedulable)
int persist_cluster_size(const LevelDev *lv, int nl, int kp) {
    for (int cs : {16, 8, 4}) {
        const size_t sm = persist_smem_bytes(lv, nl, kp, cs);
        if (sm > 200 * 1024) continue;
        persist_set_smem(sm);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(PS_NT);
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        const cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k_persist, &cfg);
        if (getenv("REXI_DEBUG"))
            fprintf(stderr, "[persist] cluster %d, %zu B smem: %s, %d active clusters\n", cs, sm,
                    cudaGetErrorString(e), nclusters);
        if (e == cudaSuccess && nclusters >= 1) return cs;
        cudaGetLastError();
    }
    return 0;
}

cudaError_t persist_launch(const L0Dev &z, const LevelDev *lv, int nl, const ShiftDev &S, int64_t n,
                           const c128 *u_in, c128 *ua, c128 *ub, c128 *snaps, int n_steps, int csize,
                           cudaStream_t st, c128 *final_out) {
    if (nl < 2 || nl > PS_MAXLV) return cudaErrorInvalidValue;
    PersistArgs a{};
    a.z = z;
    for (int l = 0; l < nl; ++l) a.lv[l] = lv[l];
    a.nl = nl;
    a.S = S;
    a.n = n;
    a.bc = persist_bc(lv[0].P, csize);
    a.u_in = u_in;
    a.ua = ua;
    a.ub = ub;
    a.snaps = snaps;
    a.final_out = final_out;
    a.n_steps = n_steps;
    static unsigned long long *tbuf = nullptr;
    const bool trace = getenv("REXI_PERSIST_TRACE") != nullptr;
    if (trace && !tbuf) cudaMalloc(&tbuf, 64 * sizeof(unsigned long long));
    if (trace) cudaMemsetAsync(tbuf, 0, 64 * sizeof(unsigned long long), st);
    a.tstamp = trace ? tbuf : nullptr;
    const size_t sm = persist_smem_bytes(lv, nl, S.kp, csize);
    {
        cudaError_t e = persist_set_smem(sm);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(PS_NT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_persist, a);
    if (trace && e == cudaSuccess) {
        unsigned long long h[64];
        cudaMemcpyAsync(h, tbuf, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "[persist] cluster %d, %d levels, %d blocks/CTA, steps %d\n", csize, nl, a.bc, n_steps);
        for (int step = 0; step < 3 && step < n_steps; ++step) {
            fprintf(stderr, "[persist] step %d:", step);
            for (int k = 1; k < 16 && h[step * 16 + k]; ++k)
                fprintf(stderr, " %.2f", (h[step * 16 + k] - h[step * 16 + k - 1]) * 1e-3);
            fprintf(stderr, " us\n");
        }
    }
    return e;
}

}  // namespace rexi
