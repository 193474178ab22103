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

// 1 / b, Smith's algorithm (the oracle's cdiv, oracle/rexi_oracle.c)
__device__ __forceinline__ c128 crecip_smith(c128 b) {
    if (fabs(b.x) >= fabs(b.y)) {
        const double r = b.y / b.x, den = b.x + r * b.y;
        return cmk(1.0 / den, -r / den);
    }
    const double r = b.x / b.y, den = b.y + r * b.x;
    return cmk(r / den, -1.0 / den);
}

// band[(row * w + (d + kl)) * 3 + {0,1,2}] = fl(tau a), fl(tau a_im), b of entry
// (row, row + d), zero when absent; w = kl + ku + 1.  KL < 0: runtime extents
// (window in local memory); otherwise compile-time (window in registers).
template <int KL, int KU>
__global__ void __launch_bounds__(32) k_band_screen(const double *__restrict__ band, int64_t n, int kl_rt, int ku_rt,
                                                    const c128 *__restrict__ sigma, int k, double *umin_out,
                                                    double *umax_out, long long *info_out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    constexpr bool RT = KL < 0;
    const int kl = RT ? kl_rt : KL, ku = RT ? ku_rt : KU;
    const int kv = kl + ku, w = kv + 1;
    constexpr int WR = RT ? SCR_WR_MAX : (KL < 0 ? 1 : KL + 1);
    constexpr int WC = RT ? SCR_WC_MAX : (KL < 0 ? 1 : KL + KU + 1);
    c128 W[WR][WC];
    const c128 sg = sigma[j];
    // matrix row r into window row `slot`, window column c = column - col0
    auto load_row = [&](int64_t r, int slot, int64_t col0) {
#pragma unroll
        for (int c = 0; c < WC; ++c)
            if (c <= kv) W[slot][c] = cmk(0.0, 0.0);
        if (r >= n) return;
#pragma unroll
        for (int dd = 0; dd < WC; ++dd) {
            if (dd >= w) break;
            const int64_t col = r + dd - kl;
            const int64_t c = col - col0;
            if (col < 0 || col >= n || c < 0 || c > kv) continue;
            const double *e = band + ((size_t)r * w + dd) * 3;
            W[slot][c] = form_entry(__ldg(e), __ldg(e + 1), __ldg(e + 2), sg);
        }
    };
#pragma unroll
    for (int s = 0; s < WR; ++s)
        if (s <= kl) load_row(s, s, 0);
    double umin = INFINITY, umax = 0.0;
    long long info = 0;
    for (int64_t col = 0; col < n; ++col) {
        const int km = (int)min((int64_t)kl, n - 1 - col);
        // IZAMAX over the diagonal and the km entries below it (first maximum)
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
            if (p != 0) {
#pragma unroll
                for (int s = 1; s < WR; ++s)
                    if (s == p)
#pragma unroll
                        for (int c = 0; c < WC; ++c) {
                            const c128 t = W[s][c];
                            W[s][c] = W[0][c];
                            W[0][c] = t;
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
            const double u = hypot(W[0][0].x, W[0][0].y);
            umin = fmin(umin, u);
            umax = fmax(umax, u);
        } else {
            if (info == 0) info = col + 1;
            umin = 0.0;
        }
        // slide the window one row down / one column right; the entering row
        // is the original row col + 1 + kl
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
    }
    umin_out[j] = umin;
    umax_out[j] = umax;
    info_out[j] = info;
}

}  // namespace

int band_screen(const rexi_desc *d, int kl, int ku, const c128 *sigma_dev, cudaStream_t st,
                std::vector<ScreenResult> &out, std::string &err) {
    const int64_t n = d->n;
    const int k = d->k;
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
    double *dband = nullptr, *dmin = nullptr, *dmax = nullptr;
    long long *dinfo = nullptr;
    auto cleanup = [&]() {
        cudaFree(dband);
        cudaFree(dmin);
        cudaFree(dmax);
        cudaFree(dinfo);
    };
#define SCK(expr)                                                   \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) {                                    \
            err = std::string(#expr) + ": " + cudaGetErrorString(_e); \
            cleanup();                                              \
            return REXI_ERR_CUDA;                                   \
        }                                                           \
    } while (0)
    SCK(cudaMalloc(&dband, sizeof(double) * band.size()));
    SCK(cudaMalloc(&dmin, sizeof(double) * k));
    SCK(cudaMalloc(&dmax, sizeof(double) * k));
    SCK(cudaMalloc(&dinfo, sizeof(long long) * k));
    SCK(rexi_poison(dband, sizeof(double) * band.size()));
    SCK(rexi_poison(dmin, sizeof(double) * k));
    SCK(rexi_poison(dmax, sizeof(double) * k));
    SCK(rexi_poison(dinfo, sizeof(long long) * k));
    SCK(cudaMemcpyAsync(dband, band.data(), sizeof(double) * band.size(), cudaMemcpyHostToDevice, st));
    const int grid = (k + 31) / 32;
    if (kl == 1 && ku == 1)
        k_band_screen<1, 1><<<grid, 32, 0, st>>>(dband, n, kl, ku, sigma_dev, k, dmin, dmax, dinfo);
    else if (kl == 2 && ku == 2)
        k_band_screen<2, 2><<<grid, 32, 0, st>>>(dband, n, kl, ku, sigma_dev, k, dmin, dmax, dinfo);
    else if (kl == 0 && ku == 0)
        k_band_screen<0, 0><<<grid, 32, 0, st>>>(dband, n, kl, ku, sigma_dev, k, dmin, dmax, dinfo);
    else
        k_band_screen<-1, -1><<<grid, 32, 0, st>>>(dband, n, kl, ku, sigma_dev, k, dmin, dmax, dinfo);
    SCK(cudaGetLastError());
    std::vector<double> hmin(k), hmax(k);
    std::vector<long long> hinfo(k);
    SCK(cudaMemcpyAsync(hmin.data(), dmin, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(hmax.data(), dmax, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(hinfo.data(), dinfo, sizeof(long long) * k, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
#undef SCK
    cleanup();
    out.resize(k);
    for (int j = 0; j < k; ++j) out[j] = ScreenResult{hmin[j], hmax[j], hinfo[j]};
    return REXI_OK;
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
