// screen.cu -- the reference's singularity screen of a banded shifted system.
//
// The reference factors every shifted matrix S_j = tau*A - (1j*sigma_j)*B with
// LAPACK zgbtrf when kl + ku + 1 <= 32 (solvers.py:25,108-115) and rejects
// the shift when the factorization hits an exact zero pivot (info > 0) or when
// the U diagonal of the PARTIALLY PIVOTED factor has min|U_ii| < 1e-14 max|U_ii|
// (solvers.py:52-69, RCOND_FLOOR).  The solvers here never form that factor
// (the 1D direct path factors without pivoting, COCG does not factor at all),
// so the verdict is recomputed on the device with zgbtf2's own algorithm
// (unblocked band LU, which zgbtrf runs for kl < its block size): per column,
// IZAMAX on |re| + |im| over the diagonal and the kl entries below it, swap,
// scale by the reciprocal pivot, rank-1 update of the active band.  One
// thread per shift walks the rows with a (kl+1) x (kl+ku+1) register window;
// the shared row data are warp-broadcast loads.  Only the U diagonal's
// extremes and the first zero pivot leave the kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"
#include "screen.cuh"

namespace rexi {

namespace {

constexpr int SCR_WR_MAX = 16;   // kl <= 15
constexpr int SCR_WC_MAX = 32;   // kl + ku + 1 <= 32

__device__ __forceinline__ double cabs1(c128 a) { return fabs(a.x) + fabs(a.y); }

// 1 / b without a division (the screen reproduces the reference's verdict, not
// its bits): the hardware reciprocal approximation of |b|^2 refined by two
// Newton steps (~full fp64 accuracy), times conj(b).  A division subroutine
// per row made the 1M-row chain of config 2 take 0.7 s.
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = r * fma(-d, r, 2.0);
    r = r * fma(-d, r, 2.0);
    return r;
}
__device__ __forceinline__ c128 crecip_smith(c128 b) {
    const double rd = rcp_nr(fma(b.x, b.x, b.y * b.y));   // |b| well inside 1e+-150 here
    return cmk(b.x * rd, -b.y * rd);
}

// band[(row * w + (d + kl)) * 3 + {0,1,2}] = fl(tau a), fl(tau a_im), b of entry
// (row, row + d), zero when absent; w = kl + ku + 1.  KL < 0: runtime extents
// (window in local memory); otherwise compile-time (window in registers).
// The row data are the same for every shift (thread): the warp stages chunks
// of CH rows in shared memory with cp.async, double buffered, so the
// sequential elimination never waits on a global load.
template <int KL, int KU>
__global__ void __launch_bounds__(32) k_band_screen(const double *__restrict__ band, int64_t n, int kl_rt, int ku_rt,
                                                    const c128 *__restrict__ sigma, int k, int CH,
                                                    double *umin_out, double *umax_out, long long *info_out) {
    extern __shared__ __align__(16) double sbuf[];           // [2][CH * w * 3]
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    constexpr bool RT = KL < 0;
    const int kl = RT ? kl_rt : KL, ku = RT ? ku_rt : KU;
    const int kv = kl + ku, w = kv + 1;
    const int per_row = w * 3;
    const int64_t nchunks = (n + CH - 1) / CH;
    auto stage = [&](int64_t c, int buf) {       // whole warp: rows [c*CH, c*CH + CH)
        const int64_t r0 = c * CH;
        const int rows = (int)min((int64_t)CH, n - r0);
        const int nd = rows * per_row;           // doubles; copy in 16-B pieces (+ a tail)
        const double *src = band + (size_t)r0 * per_row;
        double *dst = sbuf + (size_t)buf * CH * per_row;
        const bool al = ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
        if (al) {
            for (int t = threadIdx.x; t < nd / 2; t += 32) cp_async16(dst + 2 * t, src + 2 * t);
            if ((nd & 1) && threadIdx.x == 0) dst[nd - 1] = src[nd - 1];
        } else {
            for (int t = threadIdx.x; t < nd; t += 32) dst[t] = src[t];
        }
    };
    stage(0, 0);
    cp_async_wait_all();
    __syncwarp();
    const bool live = j < k;
    const c128 sg = live ? sigma[j] : cmk(0.0, 0.0);
    constexpr int WR = RT ? SCR_WR_MAX : (KL < 0 ? 1 : KL + 1);
    constexpr int WC = RT ? SCR_WC_MAX : (KL < 0 ? 1 : KL + KU + 1);
    c128 W[WR][WC];
    int64_t cur_chunk = 0;
    // the entering row's data: buffer eb, offset eo rows (advanced per row, no
    // 64-bit division on the dependent path)
    int eb = 0, eo = 0;
    auto next_row = [&]() {
        if (++eo == CH) {
            eo = 0;
            eb ^= 1;
        }
    };
    auto load_row = [&](int64_t r, int slot, int64_t col0) {
#pragma unroll
        for (int c = 0; c < WC; ++c)
            if (c <= kv) W[slot][c] = cmk(0.0, 0.0);
        if (r >= n) return;
        const double *e0 = sbuf + (size_t)eb * CH * per_row + (size_t)eo * per_row;
#pragma unroll
        for (int dd = 0; dd < WC; ++dd) {
            if (dd >= w) break;
            const int64_t col = r + dd - kl;
            const int64_t c = col - col0;
            if (col < 0 || col >= n || c < 0 || c > kv) continue;
            const double *e = e0 + dd * 3;
            W[slot][c] = form_entry(e[0], e[1], e[2], sg);
        }
    };
    // the window needs rows up to col + kl: keep chunks cur and cur + 1 staged
    if (nchunks > 1) stage(1, 1);
    cp_async_wait_all();
    __syncwarp();
#pragma unroll
    for (int s = 0; s < WR; ++s)
        if (s <= kl) {
            load_row(s, s, 0);
            next_row();
        }
    double umin = INFINITY, umax = 0.0;     // extremes of |U_ii|^2 (square roots at the end)
    long long info = 0;
    int col_off = 0;
    for (int64_t col = 0; col < n; ++col) {
        // entering chunk boundary: the row col + 1 + kl may sit in chunk cur + 1;
        // once col leaves chunk cur, refill its buffer with chunk cur + 2
        if (col_off == CH) {
            col_off = 0;
            __syncwarp();
            ++cur_chunk;
            if (cur_chunk + 1 < nchunks) stage(cur_chunk + 1, (int)((cur_chunk + 1) & 1));
            cp_async_wait_all();
            __syncwarp();
        }
        ++col_off;
        const int km = (int)min((int64_t)kl, n - 1 - col);
        int p = 0;
        double best = cabs1(W[0][0]);
#pragma unroll
        for (int s = 1; s < WR; ++s) {
            if (s > km) break;
            const double v = cabs1(W[s][0]);
            if (v > best) {
                best = v;
                p = s;
            }
        }
        bool zero = true;
#pragma unroll
        for (int s = 0; s < WR; ++s)
            if (s == p) zero = W[s][0].x == 0.0 && W[s][0].y == 0.0;
        if (!zero) {
            // row swap by selects (the shifts of a warp pivot differently)
#pragma unroll
            for (int s = 1; s < WR; ++s) {
                const bool sw = s == p;
#pragma unroll
                for (int c = 0; c < WC; ++c) {
                    const c128 a = W[0][c], b2 = W[s][c];
                    W[0][c] = sw ? b2 : a;
                    W[s][c] = sw ? a : b2;
                }
            }
            const c128 rp = crecip_smith(W[0][0]);
#pragma unroll
            for (int s = 1; s < WR; ++s) {
                if (s > km) break;
                const c128 m = cmul(rp, W[s][0]);
#pragma unroll
                for (int c = 1; c < WC; ++c)
                    if (c <= kv) W[s][c] = csub(W[s][c], cmul(m, W[0][c]));
            }
            const double u = fma(W[0][0].x, W[0][0].x, W[0][0].y * W[0][0].y);
            umin = fmin(umin, u);
            umax = isfinite(u) ? fmax(umax, u) : INFINITY;
        } else {
            if (info == 0) info = col + 1;
            umin = 0.0;
        }
#pragma unroll
        for (int s = 0; s + 1 < WR; ++s) {
            if (s >= kl) break;
#pragma unroll
            for (int c = 0; c + 1 < WC; ++c)
                if (c < kv) W[s][c] = W[s + 1][c + 1];
            W[s][kv] = cmk(0.0, 0.0);
        }
#pragma unroll
        for (int s = 0; s < WR; ++s)
            if (s == kl) load_row(col + 1 + kl, s, col + 1);
        next_row();
    }
    if (!live) return;
    umin_out[j] = sqrt(umin);
    umax_out[j] = sqrt(umax);
    info_out[j] = info;
}

}  // namespace

int ScreenJob::launch(const rexi_desc *d, int kl, int ku, const c128 *sigma_dev, cudaStream_t after,
                      std::string &err) {
    const int64_t n = d->n;
    k = d->k;
    const int w = kl + ku + 1;
    if (kl >= SCR_WR_MAX || w > SCR_WC_MAX) {
        err = "band screen: bandwidth above the reference's BAND_LIMIT";
        return REXI_ERR_UNSUPPORTED;
    }
    std::vector<double> band((size_t)n * w * 3, 0.0);
    for (int64_t r = 0; r < n; ++r)
        for (int32_t q = d->indptr[r]; q < d->indptr[r + 1]; ++q) {
            const int64_t dd = (int64_t)d->indices[q] - r + kl;
            double *e = &band[((size_t)r * w + dd) * 3];
            e[0] += d->tau * d->a_vals[q];          // duplicate entries add, as scipy's tocsr
            e[1] += d->a_imag ? d->tau * d->a_imag[q] : 0.0;
            e[2] += d->b_vals[q];
        }
#define SCK(expr)                                                     \
    do {                                                              \
        cudaError_t _e = (expr);                                      \
        if (_e != cudaSuccess) {                                      \
            err = std::string(#expr) + ": " + cudaGetErrorString(_e); \
            return REXI_ERR_CUDA;                                     \
        }                                                             \
    } while (0)
    // its own stream, ordered after the shifts' upload on the plan's stream:
    // the screen (a few SMs, sequential over the rows) overlaps the plan's
    // factorisation
    SCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t ev;
    SCK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SCK(cudaEventRecord(ev, after));
    SCK(cudaStreamWaitEvent(st, ev, 0));
    cudaEventDestroy(ev);
    SCK(cudaMalloc(&dband, sizeof(double) * band.size()));
    SCK(cudaMalloc(&dmin, sizeof(double) * k));
    SCK(cudaMalloc(&dmax, sizeof(double) * k));
    SCK(cudaMalloc(&dinfo, sizeof(long long) * k));
    SCK(rexi_poison(dband, sizeof(double) * band.size()));
    SCK(rexi_poison(dmin, sizeof(double) * k));
    SCK(rexi_poison(dmax, sizeof(double) * k));
    SCK(rexi_poison(dinfo, sizeof(long long) * k));
    // synchronous copy: the host staging vector goes out of scope on return
    SCK(cudaMemcpyAsync(dband, band.data(), sizeof(double) * band.size(), cudaMemcpyHostToDevice, st));
    SCK(cudaStreamSynchronize(st));
    const int grid = (k + 31) / 32;
    // rows per staged chunk: two chunks of row data in <= 96 KB of shared memory,
    // and at least kl + 2 rows so the window's entering row is always staged
    int CH = std::max(kl + 2, (int)std::min<int64_t>(1024, (96 * 1024) / (2 * (int64_t)w * 3 * 8)));
    CH = (CH + 1) & ~1;   // even: every chunk starts 16-B aligned (cp.async)
    const size_t smem = 2 * (size_t)CH * w * 3 * sizeof(double);
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, 32, smem, st>>>(dband, n, kl, ku, sigma_dev, k, CH, dmin, dmax, dinfo);
        return cudaGetLastError();
    };
    if (kl == 1 && ku == 1) SCK(go(k_band_screen<1, 1>));
    else if (kl == 2 && ku == 2) SCK(go(k_band_screen<2, 2>));
    else if (kl == 0 && ku == 0) SCK(go(k_band_screen<0, 0>));
    else SCK(go(k_band_screen<-1, -1>));
    return REXI_OK;
}

int ScreenJob::collect(std::vector<ScreenResult> &out, std::string &err) {
    std::vector<double> hmin(k), hmax(k);
    std::vector<long long> hinfo(k);
    SCK(cudaMemcpyAsync(hmin.data(), dmin, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(hmax.data(), dmax, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(hinfo.data(), dinfo, sizeof(long long) * k, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
#undef SCK
    out.resize(k);
    for (int j = 0; j < k; ++j) out[j] = ScreenResult{hmin[j], hmax[j], hinfo[j]};
    return REXI_OK;
}

ScreenJob::~ScreenJob() {
    if (st) cudaStreamSynchronize(st);
    cudaFree(dband);
    cudaFree(dmin);
    cudaFree(dmax);
    cudaFree(dinfo);
    if (st) cudaStreamDestroy(st);
}

// the reference's verdict and message for one shift (solvers.py:52-69); empty
// when the shift passes
std::string screen_verdict(const ScreenResult &r, int64_t n) {
    char buf[160];
    if (r.info > 0) {
        snprintf(buf, sizeof buf, "matrix is singular: zero pivot at index %lld", (long long)(r.info - 1));
        return buf;
    }
    if (n && (!(r.umin > 0.0) || r.umin < 1e-14 * r.umax)) {
        const double ratio = r.umax == 0.0 ? 0.0 : r.umin / r.umax;
        snprintf(buf, sizeof buf, "matrix is numerically singular (pivot ratio = %.3e)", ratio);
        return buf;
    }
    return std::string();
}

}  // namespace rexi
