// What bounds the wide COCG spmv?  A 2D 7-point pattern (n_side = 1023, the
// cfg 3 interior grid), 64 complex128 shift lanes per row, the spmv's memory
// pattern: 7 z gathers, p and q read + written per row-lane.
//   GATHER : z gathered at the 7 stencil columns (the production pattern)
//   SELF   : all 7 "gathers" hit the row's own z segment (L1 hits)
//   NONE   : no gathers, the pointwise part only (the streaming bound)
//   WIN    : the claim's z rows (3 windows of 34 rows) copied to shared memory
//            by all threads first, gathers served from shared memory
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o spmv_probe spmv_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef double2 c128;
__device__ __forceinline__ c128 cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ c128 cadd(c128 a, c128 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ c128 cmul(c128 a, c128 b) { return cmk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }

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
    for (int m = 0; m < 8; ++m)
        printf("%-7s %8.3f ms  %7.0f GB/s (80 B per row-lane + matrix)\n", names[m], t[m], bytes / (t[m] * 1e-3) / 1e9);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
