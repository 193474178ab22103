// assembly.cu -- P1 assembly of the pencil (A = 0.5 K + M_V, B = M) on a
// structured Kuhn mesh, on the GPU (the reference assembles
// on the host with scipy COO sums, spatial.py:143-223, and the builder's host
// fixture assembly restates that for P1: fixtures.py assemble_p1).
//
// Gather form, one thread per (interior row, stencil offset): the value is
// the sum of the element contributions whose (vertex a, vertex b) pair maps
// the row node to the column node, taken in the host's accumulation order
// (template t, then a, then b), starting from 0.0 -- so K and M come out
// bitwise identical to the host assembly.  The potential term uses the
// element potential matrices pot_e[t][cell][a][b] (computed on the device
// from the potential at the quadrature points).  Rows are stored with the
// offsets sorted by column delta (sorted CSR columns), boundary neighbours
// dropped.
#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

#include "../../include/rexi_b200.h"
#include "common.cuh"

namespace rexi {
void set_global_error(const std::string &msg);
}

namespace {

constexpr int AS_MAXOFF = 32;    // stencil offsets (3 / 7 / 15 for d = 1 / 2 / 3)
constexpr int AS_MAXC = 512;     // contributions

struct AsTable {
    int d, m, n_off, n_tmpl;
    int off[AS_MAXOFF][3];
    int cstart[AS_MAXOFF + 1];
    int ct[AS_MAXC], ca[AS_MAXC], cb[AS_MAXC];   // template, local row, local column
    int cva[AS_MAXC][3];                          // vertex a of template t (cell = node - cva)
    double cs[AS_MAXC], cm[AS_MAXC];              // stiffness, mass contribution
};

__constant__ AsTable g_tab;

__device__ __forceinline__ void node_coords(int64_t r, int d, int n1, int (&x)[3]) {
    // interior row r -> node coordinates in [1, m-1]^d (row-major, last axis fastest)
    x[0] = x[1] = x[2] = 0;
    for (int k = d - 1; k >= 0; --k) {
        x[k] = (int)(r % n1) + 1;
        r /= n1;
    }
}

__global__ void k_p1_count(int64_t n_int, int *counts) {
    const AsTable &T = g_tab;
    const int n1 = T.m - 1;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_int; r += (int64_t)gridDim.x * blockDim.x) {
        int x[3];
        node_coords(r, T.d, n1, x);
        int c = 0;
        for (int s = 0; s < T.n_off; ++s) {
            bool ok = true;
            for (int k = 0; k < T.d; ++k) {
                const int nb = x[k] + T.off[s][k];
                ok &= nb >= 1 && nb <= T.m - 1;
            }
            c += ok ? 1 : 0;
        }
        counts[r] = c;
    }
}

__global__ void k_p1_fill(int64_t n_int, const int *indptr, const double *pot_e, int *indices, double *a_vals,
                          double *b_vals) {
    const AsTable &T = g_tab;
    const int d = T.d, m = T.m, n1 = m - 1;
    const int64_t ncell = d == 1 ? m : (d == 2 ? (int64_t)m * m : (int64_t)m * m * m);
    const int dd = (d + 1) * (d + 1);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_int; r += (int64_t)gridDim.x * blockDim.x) {
        int x[3];
        node_coords(r, d, n1, x);
        int64_t w = indptr[r];
        for (int s = 0; s < T.n_off; ++s) {
            bool ok = true;
            int64_t delta = 0;
            for (int k = 0; k < d; ++k) {
                const int nb = x[k] + T.off[s][k];
                ok &= nb >= 1 && nb <= m - 1;
                delta = delta * n1 + T.off[s][k];
            }
            if (!ok) continue;
            double st = 0.0, ms = 0.0, pt = 0.0;
            for (int c = T.cstart[s]; c < T.cstart[s + 1]; ++c) {
                // element cell = node - vertex a of the template, inside [0, m)^d
                bool in = true;
                int64_t cell = 0;
                for (int k = 0; k < d; ++k) {
                    const int ck = x[k] - T.cva[c][k];
                    in &= ck >= 0 && ck < m;
                    cell = cell * m + ck;
                }
                if (!in) continue;
                st = __dadd_rn(st, T.cs[c]);
                ms = __dadd_rn(ms, T.cm[c]);
                pt = __dadd_rn(pt, pot_e[((int64_t)T.ct[c] * ncell + cell) * dd + T.ca[c] * (d + 1) + T.cb[c]]);
            }
            indices[w] = (int)(r + delta);
            a_vals[w] = __dadd_rn(__dmul_rn(0.5, st), pt);
            b_vals[w] = ms;
            ++w;
        }
    }
}

}  // namespace

extern "C" int rexi_assemble_p1(const rexi_p1_desc *desc, const double *pot_e, int32_t *indptr, int32_t *indices,
                                double *a_vals, double *b_vals) {
    auto fail = [](int code, const std::string &msg) {
        rexi::set_global_error(msg);
        return code;
    };
    if (!desc || !pot_e || !indptr || !indices || !a_vals || !b_vals) return fail(REXI_ERR_INVALID, "null argument");
    const rexi_p1_desc &D = *desc;
    if (D.d < 1 || D.d > 3 || D.m < 2) return fail(REXI_ERR_INVALID, "need 1 <= d <= 3 and m >= 2");
    if (D.n_off < 1 || D.n_off > AS_MAXOFF || D.n_contrib < 1 || D.n_contrib > AS_MAXC)
        return fail(REXI_ERR_UNSUPPORTED, "stencil table too large");
    AsTable T{};
    T.d = D.d;
    T.m = D.m;
    T.n_off = D.n_off;
    T.n_tmpl = D.n_templates;
    for (int s = 0; s < D.n_off; ++s)
        for (int k = 0; k < 3; ++k) T.off[s][k] = k < D.d ? D.offsets[s * D.d + k] : 0;
    for (int s = 0; s <= D.n_off; ++s) T.cstart[s] = D.contrib_start[s];
    for (int c = 0; c < D.n_contrib; ++c) {
        T.ct[c] = D.contrib_t[c];
        T.ca[c] = D.contrib_a[c];
        T.cb[c] = D.contrib_b[c];
        for (int k = 0; k < 3; ++k) T.cva[c][k] = k < D.d ? D.contrib_va[c * D.d + k] : 0;
        T.cs[c] = D.contrib_stiff[c];
        T.cm[c] = D.contrib_mass[c];
    }
    cudaError_t e = cudaSetDevice(D.device);
    cudaStream_t st = (cudaStream_t)D.stream;
    if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(g_tab, &T, sizeof T, 0, cudaMemcpyHostToDevice, st);
    int64_t n_int = 1;
    for (int k = 0; k < D.d; ++k) n_int *= (D.m - 1);
    const unsigned grid = (unsigned)std::min<int64_t>((n_int + 255) / 256, 65535);
    int *counts = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&counts, sizeof(int) * (n_int + 1), st);
    if (e == cudaSuccess) e = rexi_poison(counts, sizeof(int) * (n_int + 1), st);
    if (e == cudaSuccess) {
        k_p1_count<<<grid, 256, 0, st>>>(n_int, counts);
        e = cudaGetLastError();
    }
    // indptr: exclusive prefix sum of the row counts (host scan of an O(n) int array)
    std::vector<int> hc(n_int), hp(n_int + 1);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), counts, sizeof(int) * n_int, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
        hp[0] = 0;
        for (int64_t r = 0; r < n_int; ++r) hp[r + 1] = hp[r] + hc[r];
        e = cudaMemcpyAsync(indptr, hp.data(), sizeof(int) * (n_int + 1), cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) {
        k_p1_fill<<<grid, 256, 0, st>>>(n_int, indptr, pot_e, indices, a_vals, b_vals);
        e = cudaGetLastError();
    }
    if (counts) cudaFreeAsync(counts, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        char buf[256];
        snprintf(buf, sizeof buf, "CUDA error in rexi_assemble_p1: %s", cudaGetErrorString(e));
        return fail(e == cudaErrorMemoryAllocation ? REXI_ERR_NOMEM : REXI_ERR_CUDA, buf);
    }
    return REXI_OK;
}
