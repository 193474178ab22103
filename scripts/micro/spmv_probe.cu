// What bounds the wide COCG spmv?  A 2D 7-point pattern (n_side = 1023, the
// cfg 3 interior grid), 64 complex128 shift lanes per row, the spmv's memory
// pattern: 7 z gathers, p and q read + written per row-lane.
//   GATHER : z gathered at the 7 stencil columns (the production pattern)
//   SELF   : all 7 "gathers" hit the row's own z segment (L1 hits)
//   NONE   : no gathers, the pointwise part only (the streaming bound)
//   WIN    : the claim's z rows (3 windows of 34 rows) copied to shared memory
//            by all threads first, gathers served from shared memory
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o spmv_probe spmv_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef double2 c128;
__device__ __forceinline__ c128 cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ c128 cadd(c128 a, c128 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ c128 cmul(c128 a, c128 b) { return cmk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

constexpr int NS = 1023;
constexpr int N = NS * NS;
constexpr int KP = 64;
constexpr int NNZ = 7;
__constant__ int OFF[NNZ] = {-NS, -NS + 1, -1, 0, 1, NS - 1, NS};

enum { GATHER = 0, SELF = 1, NONE = 2, WIN = 3, CSR = 4, RED = 5, STRIP = 6, STRIP2 = 7 };
// STRIP: each CTA walks a strip of claims 32 claims apart (one grid line
// down per claim), so the z rows of the line above were loaded into L1 by
// the CTA's previous claim; STRIP2 the same with segments of 64 lines

// 256 threads: 2 warps per row (64 lanes), 4 rows per pass, claims of 32 rows
template <int MODE>
__global__ void __launch_bounds__(256, 3) k_probe(const double *__restrict__ ta, const double *__restrict__ tb,
                                                  const int *__restrict__ ix, const c128 *__restrict__ z,
                                                  c128 *__restrict__ p, c128 *__restrict__ q, c128 beta, c128 sg,
                                                  int nclaims, c128 *part) {
    extern __shared__ c128 win[];   // WIN: [3][34][KP]
    __shared__ c128 sbp[8 * KP];
    const int lane = threadIdx.x & 63, slot = threadIdx.x >> 6;
    const int SEG = MODE == STRIP2 ? 64 : 16;
    const int nseg_lines = (nclaims / 32 + SEG - 1) / SEG;
    const int nwork = (MODE == STRIP || MODE == STRIP2) ? 32 * nseg_lines * SEG : nclaims;
    for (int w = blockIdx.x * ((MODE == STRIP || MODE == STRIP2) ? SEG : 1); w < nwork;
         w += ((MODE == STRIP || MODE == STRIP2) ? (w % SEG == SEG - 1 ? gridDim.x * SEG - SEG + 1 : 1) : gridDim.x)) {
        int claim = w;
        if (MODE == STRIP || MODE == STRIP2) {
            const int seg = w / SEG, j = w % SEG;          // segment = (strip, line block)
            const int strip = seg % 32, lb = seg / 32;
            claim = strip + 32 * (lb * SEG + j);
            if (claim >= nclaims) continue;
        }
        const int R0 = claim * 32;
        if (MODE == WIN) {
            __syncthreads();
            for (int w = 0; w < 3; ++w) {
                const int base = R0 - 1 + (w - 1) * NS;
                for (int t = threadIdx.x; t < 34 * KP; t += 256) {
                    const int r = base + t / KP;
                    win[(w * 34) * KP + t] = (r >= 0 && r < N) ? z[(size_t)r * KP + (t % KP)] : cmk(0.0, 0.0);
                }
            }
            __syncthreads();
        }
        c128 mu[2] = {cmk(0.0, 0.0), cmk(0.0, 0.0)};
        for (int k = 0; k < 8; ++k) {
            const int i = R0 + slot + 4 * k;
            if (i >= N) break;
            c128 acc = cmk(0.0, 0.0);
            if (MODE != NONE) {
                c128 zz[NNZ];
#pragma unroll
                for (int e = 0; e < NNZ; ++e) {
                    int c = i + OFF[e];
                    if (c < 0 || c >= N) c = i;
                    if (MODE == GATHER || MODE == STRIP || MODE == STRIP2) zz[e] = z[(size_t)c * KP + lane];
                    else if (MODE == SELF) zz[e] = z[(size_t)i * KP + lane];
                    else if (MODE == CSR) zz[e] = z[(size_t)__ldg(ix + (size_t)i * NNZ + e) * KP + lane];
                    else if (MODE == WIN) {
                        int w = OFF[e] < -1 ? 0 : OFF[e] > 1 ? 2 : 1;
                        if (c == i) w = 1;
                        const int rr = c - (R0 - 1 + (w - 1) * NS);
                        zz[e] = win[(w * 34 + rr) * KP + lane];
                    } else {
                        zz[e] = z[(size_t)c * KP + lane];
                    }
                }
#pragma unroll
                for (int e = 0; e < NNZ; ++e) {
                    const double a = __ldg(ta + (size_t)i * NNZ + e), b = __ldg(tb + (size_t)i * NNZ + e);
                    const c128 en = cmk(a + sg.y * b, -(sg.x * b));
                    acc = cadd(acc, cmul(en, zz[e]));
                }
            }
            const size_t o = (size_t)i * KP + lane;
            const c128 pi = cadd(z[o], cmul(beta, p[o]));
            const c128 qi = cadd(acc, cmul(beta, q[o]));
            p[o] = pi;
            q[o] = qi;
            if (MODE == RED) mu[k >> 2] = cadd(mu[k >> 2], cmul(pi, qi));
        }
        if (MODE == RED) {   // sub-block partials -> chunk partial, as the production kernel
            sbp[(slot * 2 + 0) * KP + lane] = mu[0];
            sbp[(slot * 2 + 1) * KP + lane] = mu[1];
            __syncthreads();
            if (threadIdx.x < KP) {
                c128 s = cmk(0.0, 0.0);
                for (int b = 0; b < 8; ++b) s = cadd(s, sbp[b * KP + threadIdx.x]);
                part[(size_t)claim * KP + threadIdx.x] = s;
            }
            __syncthreads();
        }
    }
}

// The recomputed-q iteration (no q vector): SPMV2 gathers z and p_old at the
// 7 columns (p_new = z + beta p_old formed per neighbour), writes p_new, mu;
// UPD2 gathers p_new again for q = S p_new, updates x and z.  UPD is today's
// update (x, z read + written, p, q read: 96 B per row-lane).
template <int MODE>
__global__ void __launch_bounds__(256, 3) k_iter(const double *__restrict__ ta, const double *__restrict__ tb,
                                                 const c128 *__restrict__ z, const c128 *__restrict__ pold,
                                                 c128 *__restrict__ pnew, c128 *__restrict__ x, c128 *__restrict__ zw,
                                                 const c128 *__restrict__ q, c128 beta, c128 alpha, c128 sg,
                                                 int nclaims, c128 *part) {
    __shared__ c128 sbp[8 * KP];
    const int lane = threadIdx.x & 63, slot = threadIdx.x >> 6;
    for (int claim = blockIdx.x; claim < nclaims; claim += gridDim.x) {
        const int R0 = claim * 32;
        c128 mu[2] = {cmk(0.0, 0.0), cmk(0.0, 0.0)};
        for (int k = 0; k < 8; ++k) {
            const int i = R0 + slot + 4 * k;
            if (i >= N) break;
            const size_t o = (size_t)i * KP + lane;
            c128 acc = cmk(0.0, 0.0);
            if (MODE != 2) {
                c128 zz[NNZ];
#pragma unroll
                for (int e = 0; e < NNZ; ++e) {
                    int c = i + OFF[e];
                    if (c < 0 || c >= N) c = i;
                    const size_t oc = (size_t)c * KP + lane;
                    zz[e] = MODE == 0 ? cadd(z[oc], cmul(beta, pold[oc])) : pnew[oc];
                }
#pragma unroll
                for (int e = 0; e < NNZ; ++e) {
                    const double a = __ldg(ta + (size_t)i * NNZ + e), b = __ldg(tb + (size_t)i * NNZ + e);
                    const c128 en = cmk(a + sg.y * b, -(sg.x * b));
                    acc = cadd(acc, cmul(en, zz[e]));
                }
            }
            if (MODE == 0) {
                const c128 pi = cadd(z[o], cmul(beta, pold[o]));
                pnew[o] = pi;
                mu[k >> 2] = cadd(mu[k >> 2], cmul(pi, acc));
            } else {
                const c128 pp = MODE == 1 ? pnew[o] : pold[o];
                const c128 qq = MODE == 1 ? acc : q[o];
                x[o] = cadd(x[o], cmul(alpha, pp));
                const c128 d = cmk(ta[(size_t)i * NNZ + 3] + sg.y, -sg.x);
                const double den = fma(d.x, d.x, d.y * d.y), r = 1.0 / den;
                const c128 di = cmk(d.x * r, -d.y * r);
                const c128 zn = cadd(zw[o], cmul(cmk(-alpha.x, -alpha.y), cmul(qq, di)));
                zw[o] = zn;
                mu[k >> 2] = cadd(mu[k >> 2], cmul(cmul(d, zn), zn));
            }
        }
        sbp[(slot * 2 + 0) * KP + lane] = mu[0];
        sbp[(slot * 2 + 1) * KP + lane] = mu[1];
        __syncthreads();
        if (threadIdx.x < KP) {
            c128 t = cmk(0.0, 0.0);
            for (int b = 0; b < 8; ++b) t = cadd(t, sbp[b * KP + threadIdx.x]);
            part[(size_t)claim * KP + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

template <int MODE>
static float run_iter(const double *ta, const double *tb, c128 *z, c128 *p, c128 *p2, c128 *x, c128 *q, c128 *part,
                      int sms) {
    const int nclaims = (N + 31) / 32;
    const int grid = sms * 3;
    const c128 beta = make_double2(0.3, 0.1), alpha = make_double2(0.2, -0.1), sg = make_double2(1.5, -2.0);
    auto go = [&] { k_iter<MODE><<<grid, 256>>>(ta, tb, z, p, p2, x, z, q, beta, alpha, sg, nclaims, part); };
    go();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        go();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

// work item = (32-row claim, 32-lane group); 8 warps = the 8 sub-blocks
// (rows w, w+8, w+16, w+24); the item's 3 z windows (row ranges) are copied to
// shared memory by bulk copies one item ahead (double buffered, one mbarrier
// per buffer); p, q own rows are register loads issued before the wait
constexpr int TW_ROWS = 3 * 34;
constexpr int LW = 32;
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_tmawin(const double *__restrict__ ta, const double *__restrict__ tb,
                                                  const c128 *__restrict__ z, c128 *__restrict__ p,
                                                  c128 *__restrict__ q, c128 beta, c128 sg, int nitems,
                                                  c128 *part) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    c128 *win = reinterpret_cast<c128 *>(sm + 128);       // [2][TW_ROWS][LW]
    __shared__ c128 sbp[8 * LW];
    constexpr int RPW = NT / 256;                          // warps per sub-block
    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int sb = warp / RPW, half = warp % RPW;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int item, int b) {
        const int claim = item >> 1, g = item & 1;
        const int R0 = claim * 32;
        uint32_t bytes = 0;
        for (int w = 0; w < 3; ++w) {
            const int base = R0 - 1 + (w - 1) * NS;
            for (int t = 0; t < 34; ++t) {
                const int r = base + t;
                if (r >= 0 && r < N) bytes += LW * 16;
            }
        }
        mbar_expect_tx(bar + b, bytes);
        for (int w = 0; w < 3; ++w) {
            const int base = R0 - 1 + (w - 1) * NS;
            for (int t = 0; t < 34; ++t) {
                const int r = base + t;
                if (r >= 0 && r < N)
                    bulk_g2s(win + ((size_t)b * TW_ROWS + w * 34 + t) * LW, z + (size_t)r * KP + g * LW, LW * 16, bar + b);
            }
        }
    };
    int item = blockIdx.x;
    if (threadIdx.x == 0 && item < nitems) issue(item, 0);
    uint32_t ph[2] = {0, 0};
    int b = 0;
    for (; item < nitems; item += gridDim.x, b ^= 1) {
        const int nxt = item + gridDim.x;
        if (threadIdx.x == 0 && nxt < nitems) issue(nxt, b ^ 1);
        const int claim = item >> 1, g = item & 1;
        const int R0 = claim * 32;
        const int lane = g * LW + l;
        // own-row loads before the wait
        c128 zo[4 / RPW], po[4 / RPW], qo[4 / RPW];
#pragma unroll
        for (int k = 0; k < 4 / RPW; ++k) {
            const int i = R0 + sb + 8 * (k * RPW + half);
            const size_t o = (size_t)i * KP + lane;
            po[k] = i < N ? p[o] : cmk(0.0, 0.0);
            qo[k] = i < N ? q[o] : cmk(0.0, 0.0);
            zo[k] = i < N ? z[o] : cmk(0.0, 0.0);
        }
        mbar_wait(bar + b, ph[b]);
        ph[b] ^= 1u;
        const c128 *wb = win + (size_t)b * TW_ROWS * LW;
        c128 mu = cmk(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < 4 / RPW; ++k) {
            const int i = R0 + sb + 8 * (k * RPW + half);
            if (i >= N) break;
            c128 acc = cmk(0.0, 0.0);
#pragma unroll
            for (int e = 0; e < NNZ; ++e) {
                int c = i + OFF[e];
                int w = OFF[e] < -1 ? 0 : OFF[e] > 1 ? 2 : 1;
                if (c < 0 || c >= N) { c = i; w = 1; }
                const int rr = c - (R0 - 1 + (w - 1) * NS);
                const c128 zz = wb[(w * 34 + rr) * LW + l];
                const double a = __ldg(ta + (size_t)i * NNZ + e), bb = __ldg(tb + (size_t)i * NNZ + e);
                const c128 en = cmk(a + sg.y * bb, -(sg.x * bb));
                acc = cadd(acc, cmul(en, zz));
            }
            const size_t o = (size_t)i * KP + lane;
            const c128 pi = cadd(zo[k], cmul(beta, po[k]));
            const c128 qi = cadd(acc, cmul(beta, qo[k]));
            p[o] = pi;
            q[o] = qi;
            mu = cadd(mu, cmul(pi, qi));
        }
        if (RPW == 1) sbp[sb * LW + l] = mu;
        __syncthreads();   // all warps done with buffer b (and sbp complete)
        if (threadIdx.x < LW) {
            c128 t = cmk(0.0, 0.0);
            for (int s2 = 0; s2 < 8; ++s2) t = cadd(t, sbp[s2 * LW + threadIdx.x]);
            part[(size_t)claim * KP + lane] = t;
        }
    }
}

// full-width windows (all 64 lanes: a window of 34 consecutive rows is ONE
// contiguous 34 KB range -> 3 bulk copies per claim), single buffer per CTA,
// 2 CTAs/SM; the next claim's copies are issued as soon as every warp is done
// reading the window (after the claim's last gather), overlapping this
// claim's p/q traffic and the other CTA's work
template <int DB>
__global__ void __launch_bounds__(256, DB ? 1 : 2) k_tma64(const double *__restrict__ ta, const double *__restrict__ tb,
                                                  const c128 *__restrict__ z, c128 *__restrict__ p,
                                                  c128 *__restrict__ q, c128 beta, c128 sg, int nclaims,
                                                  c128 *part) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    c128 *win = reinterpret_cast<c128 *>(sm + 128);       // [DB+1][3][34][KP]
    __shared__ c128 sbp[8 * KP];
    const int lane = threadIdx.x & 63, slot = threadIdx.x >> 6;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int claim, int b) {
        const int R0 = claim * 32;
        uint32_t bytes = 0;
        int lo[3], cnt[3];
        for (int w = 0; w < 3; ++w) {
            const int base = R0 - 1 + (w - 1) * NS;
            lo[w] = base < 0 ? 0 : base;
            const int hi = min(base + 34, N);
            cnt[w] = hi > lo[w] ? hi - lo[w] : 0;
            bytes += cnt[w] * KP * 16;
        }
        mbar_expect_tx(bar + b, bytes);
        for (int w = 0; w < 3; ++w) {
            const int base = R0 - 1 + (w - 1) * NS;
            if (cnt[w]) bulk_g2s(win + ((size_t)b * 3 * 34 + w * 34 + (lo[w] - base)) * KP, z + (size_t)lo[w] * KP,
                                 cnt[w] * KP * 16, bar + b);
        }
    };
    int claim = blockIdx.x;
    if (threadIdx.x == 0 && claim < nclaims) issue(claim, 0);
    uint32_t ph[2] = {0, 0};
    int b = 0;
    for (; claim < nclaims; claim += gridDim.x) {
        const int R0 = claim * 32;
        c128 po[8], qo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = R0 + slot + 4 * k;
            const size_t o = (size_t)min(i, N - 1) * KP + lane;
            po[k] = p[o];
            qo[k] = q[o];
        }
        if (DB && threadIdx.x == 0 && claim + (int)gridDim.x < nclaims) issue(claim + gridDim.x, b ^ 1);
        mbar_wait(bar + b, ph[b]);
        ph[b] ^= 1u;
        const c128 *wb = win + (size_t)b * 3 * 34 * KP;
        c128 mu[2] = {cmk(0.0, 0.0), cmk(0.0, 0.0)};
        c128 pi_[8], qi_[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = R0 + slot + 4 * k;
            c128 acc = cmk(0.0, 0.0);
            if (i < N) {
#pragma unroll
                for (int e = 0; e < NNZ; ++e) {
                    int c = i + OFF[e];
                    int w = OFF[e] < -1 ? 0 : OFF[e] > 1 ? 2 : 1;
                    if (c < 0 || c >= N) { c = i; w = 1; }
                    const int rr = c - (R0 - 1 + (w - 1) * NS);
                    const c128 zz = wb[(w * 34 + rr) * KP + lane];
                    const double a = __ldg(ta + (size_t)i * NNZ + e), bb = __ldg(tb + (size_t)i * NNZ + e);
                    const c128 en = cmk(a + sg.y * bb, -(sg.x * bb));
                    acc = cadd(acc, cmul(en, zz));
                }
            }
            const c128 zi = wb[(34 + (i - R0 + 1)) * KP + lane];
            pi_[k] = cadd(zi, cmul(beta, po[k]));
            qi_[k] = cadd(acc, cmul(beta, qo[k]));
            mu[k >> 2] = cadd(mu[k >> 2], cmul(pi_[k], qi_[k]));
        }
        __syncthreads();                 // window b fully read
        if (!DB && threadIdx.x == 0 && claim + (int)gridDim.x < nclaims) issue(claim + gridDim.x, b);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = R0 + slot + 4 * k;
            if (i < N) {
                const size_t o = (size_t)i * KP + lane;
                p[o] = pi_[k];
                q[o] = qi_[k];
            }
        }
        sbp[(slot * 2 + 0) * KP + lane] = mu[0];
        sbp[(slot * 2 + 1) * KP + lane] = mu[1];
        __syncthreads();
        if (threadIdx.x < KP) {
            c128 t = cmk(0.0, 0.0);
            for (int s2 = 0; s2 < 8; ++s2) t = cadd(t, sbp[s2 * KP + threadIdx.x]);
            part[(size_t)claim * KP + threadIdx.x] = t;
        }
        if (DB) b ^= 1;
    }
}

template <int DB>
static float run_t64(const double *ta, const double *tb, const c128 *z, c128 *p, c128 *q, c128 *part, int sms) {
    const int nclaims = (N + 31) / 32;
    const size_t sm = 128 + (DB + 1) * 3 * 34 * KP * sizeof(c128);
    cudaFuncSetAttribute(k_tma64<DB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const c128 beta = make_double2(0.3, 0.1), sg = make_double2(1.5, -2.0);
    const int grid = sms * (DB ? 1 : 2);
    k_tma64<DB><<<grid, 256, sm>>>(ta, tb, z, p, q, beta, sg, nclaims, part);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_tma64<DB><<<grid, 256, sm>>>(ta, tb, z, p, q, beta, sg, nclaims, part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

template <int NT>
static float run_tw(const double *ta, const double *tb, const c128 *z, c128 *p, c128 *q, c128 *part, int sms) {
    const int nitems = ((N + 31) / 32) * 2;
    const size_t sm = 128 + 2 * TW_ROWS * LW * sizeof(c128);
    cudaFuncSetAttribute(k_tmawin<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const c128 beta = make_double2(0.3, 0.1), sg = make_double2(1.5, -2.0);
    k_tmawin<NT><<<sms, NT, sm>>>(ta, tb, z, p, q, beta, sg, nitems, part);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_tmawin<NT><<<sms, NT, sm>>>(ta, tb, z, p, q, beta, sg, nitems, part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

template <int MODE>
static float run(const double *ta, const double *tb, const int *ix, const c128 *z, c128 *p, c128 *q, c128 *part,
                 int sms) {
    const int nclaims = (N + 31) / 32;
    const int grid = sms * 3;
    const size_t sm = MODE == WIN ? 3 * 34 * KP * sizeof(c128) : 0;
    if (MODE == WIN) cudaFuncSetAttribute(k_probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const c128 beta = make_double2(0.3, 0.1), sg = make_double2(1.5, -2.0);
    k_probe<MODE><<<grid, 256, sm>>>(ta, tb, ix, z, p, q, beta, sg, nclaims, part);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_probe<MODE><<<grid, 256, sm>>>(ta, tb, ix, z, p, q, beta, sg, nclaims, part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *ta, *tb;
    c128 *z, *p, *q;
    cudaMalloc(&ta, sizeof(double) * (size_t)N * NNZ);
    cudaMalloc(&tb, sizeof(double) * (size_t)N * NNZ);
    cudaMalloc(&z, sizeof(c128) * (size_t)N * KP);
    cudaMalloc(&p, sizeof(c128) * (size_t)N * KP);
    cudaMalloc(&q, sizeof(c128) * (size_t)N * KP);
    cudaMemset(ta, 0, sizeof(double) * (size_t)N * NNZ);
    cudaMemset(tb, 0, sizeof(double) * (size_t)N * NNZ);
    cudaMemset(z, 0, sizeof(c128) * (size_t)N * KP);
    cudaMemset(p, 0, sizeof(c128) * (size_t)N * KP);
    cudaMemset(q, 0, sizeof(c128) * (size_t)N * KP);
    int *ix;
    c128 *part;
    cudaMalloc(&ix, sizeof(int) * (size_t)N * NNZ);
    cudaMalloc(&part, sizeof(c128) * (size_t)(N / 32 + 1) * KP);
    {
        int *h = (int *)malloc(sizeof(int) * (size_t)N * NNZ);
        const int off[NNZ] = {-NS, -NS + 1, -1, 0, 1, NS - 1, NS};
        for (int i = 0; i < N; ++i)
            for (int e = 0; e < NNZ; ++e) {
                int c = i + off[e];
                h[(size_t)i * NNZ + e] = (c < 0 || c >= N) ? i : c;
            }
        cudaMemcpy(ix, h, sizeof(int) * (size_t)N * NNZ, cudaMemcpyHostToDevice);
        free(h);
    }
    const double bytes = (double)N * KP * 80.0 + (double)N * NNZ * 16.0;
    const char *names[8] = {"GATHER", "SELF", "NONE", "WIN", "CSR", "RED", "STRIP", "STRIP2"};
    float t[8];
    t[0] = run<GATHER>(ta, tb, ix, z, p, q, part, sms);
    t[1] = run<SELF>(ta, tb, ix, z, p, q, part, sms);
    t[2] = run<NONE>(ta, tb, ix, z, p, q, part, sms);
    t[3] = run<WIN>(ta, tb, ix, z, p, q, part, sms);
    t[4] = run<CSR>(ta, tb, ix, z, p, q, part, sms);
    t[5] = run<RED>(ta, tb, ix, z, p, q, part, sms);
    t[6] = run<STRIP>(ta, tb, ix, z, p, q, part, sms);
    t[7] = run<STRIP2>(ta, tb, ix, z, p, q, part, sms);
    {
        c128 *p2, *x;
        cudaMalloc(&p2, sizeof(c128) * (size_t)N * KP);
        cudaMalloc(&x, sizeof(c128) * (size_t)N * KP);
        cudaMemset(p2, 0, sizeof(c128) * (size_t)N * KP);
        cudaMemset(x, 0, sizeof(c128) * (size_t)N * KP);
        const float s2 = run_iter<0>(ta, tb, z, p, p2, x, q, part, sms);
        const float u2 = run_iter<1>(ta, tb, z, p, p2, x, q, part, sms);
        const float u0 = run_iter<2>(ta, tb, z, p, p2, x, q, part, sms);
        printf("SPMV2 (gather z+p_old, write p: 48 B) %.3f ms | UPD2 (gather p, x z r/w: 80 B) %.3f ms | "
               "UPD today (96 B) %.3f ms\n", s2, u2, u0);
        printf("recomputed-q iteration %.3f ms vs today's spmv (RED) + update %.3f ms\n", s2 + u2,
               run<RED>(ta, tb, ix, z, p, q, part, sms) + u0);
        cudaFree(p2);
        cudaFree(x);
    }
    const float t64 = run_t64<0>(ta, tb, z, p, q, part, sms);
    const float t64d = run_t64<1>(ta, tb, z, p, q, part, sms);
    printf("TMA64 single-buffer 2 CTA/SM %.3f ms | double-buffer 1 CTA/SM %.3f ms (vs RED %.3f)\n", t64, t64d,
           run<RED>(ta, tb, ix, z, p, q, part, sms));
    const float tw = run_tw<256>(ta, tb, z, p, q, part, sms);
    printf("%-7s %8.3f ms  %7.0f GB/s\n", "TMAWIN", tw, bytes / (tw * 1e-3) / 1e9);
    for (int m = 0; m < 8; ++m)
        printf("%-7s %8.3f ms  %7.0f GB/s (80 B per row-lane + matrix)\n", names[m], t[m], bytes / (t[m] * 1e-3) / 1e9);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
