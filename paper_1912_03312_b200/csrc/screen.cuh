// screen.cuh -- the reference's banded singularity screen (see screen.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/rexi_b200.h"
#include "common.cuh"

namespace rexi {

struct ScreenResult {
    double umin, umax;   // extremes of |U_ii| of the partially pivoted band LU
    long long info;      // zgbtrf info: first zero pivot (1-based), 0 if none
};

// zgbtf2 on every shifted system of the descriptor (kl + ku + 1 <= 32), on the
// device, on a stream of its own ordered after `after` (sigma_dev, the desc's
// k shifts, is uploaded there): launch() returns at once, collect() waits
struct ScreenJob {
    cudaStream_t st = nullptr;
    double *dband = nullptr, *dmin = nullptr, *dmax = nullptr;
    long long *dinfo = nullptr;
    int k = 0;
    int launch(const rexi_desc *d, int kl, int ku, const c128 *sigma_dev, cudaStream_t after, std::string &err);
    int collect(std::vector<ScreenResult> &out, std::string &err);
    ~ScreenJob();
};
// "" when the shift passes, else the reference's SolverError text
std::string screen_verdict(const ScreenResult &r, int64_t n);

}  // namespace rexi
