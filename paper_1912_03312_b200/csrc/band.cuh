// band.cuh -- direct solver for narrow banded pencils (P2 1D: pentadiagonal).
#pragma once
#include <string>
#include <vector>

#include "../../include/rexi_b200.h"
#include "cocg.cuh"
#include "common.cuh"
#include "tridiag.cuh"

namespace rexi {

constexpr int BAND_MIN = 2, BAND_MAX = 4;   // half bandwidths handled (1 is the TRIDIAG solver)

struct BandState {
    ProfHook *hook = nullptr;
    int B = 0;                  // half bandwidth (kl = ku = B; missing diagonals are zero)
    int64_t n = 0, npad = 0;    // rows, rows padded to P*M (decoupled unit rows)
    int M = 0, P = 0;           // rows per block, blocks
    int k = 0, kp = 0, refine = 0;
    double min_pivot_ratio = 1.0;
    std::vector<void *> allocs;
    int64_t bytes = 0;
    void *impl = nullptr;       // BandImpl (band.cu)
};

int band_create(BandState &bs, const rexi_desc *d, int B, const ShiftDev &S, int kp, int refine, cudaStream_t st,
                std::string &err);
// one step from device u: uout (rounded u1) or, with uout == nullptr, the
// double-double partial sum_j beta_j x_j into acc (SoA 4n)
int band_step(BandState &bs, const ShiftDev &S, cudaStream_t st, const c128 *u, c128 *uout, double *acc,
              int64_t *launches, std::string &err);
// per-shift solutions x (k*n, shift-major, device) of S_j x_j = rhs (device)
int band_solve_all(BandState &bs, const ShiftDev &S, cudaStream_t st, const c128 *rhs, c128 *x,
                   std::string &err);
void band_destroy(BandState &bs);

}  // namespace rexi
