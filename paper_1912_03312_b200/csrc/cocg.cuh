// cocg.cuh -- lockstep-over-shifts Jacobi-COCG for general CSR pencils (2D/3D).
#pragma once
#include <string>
#include <vector>

#include "../../include/rexi_b200.h"
#include "common.cuh"
#include "tridiag.cuh"

namespace rexi {

// per-launch timing hook (implemented by the plan; begin/end bracket one launch)
struct ProfHook {
    virtual void begin(const char *name, double algorithmic_bytes) = 0;
    virtual void end() = 0;
    virtual ~ProfHook() {}
};

struct CocgState {
    ProfHook *hook = nullptr;
    int64_t n = 0, nnz = 0;
    int k = 0;
    int refine = 0;
    double tol = 1e-12;
    int max_iters = 20000;
    int64_t bytes = 0;
    int last_iters_max = 0;
    double last_iters_mean = 0.0;
    int shift_offset = 0;
    std::vector<int> gid;            // global index of each shift (error messages)
    std::vector<int> shift_iters;    // per-shift iterations of the last step (first solve + corrections)
    // phase timing of the rhs / accumulation kernels (stats rhs / reduce)
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bool ev_pending = false;
    double t_rhs_ms = 0.0, t_acc_ms = 0.0;
    std::vector<void *> allocs;
    void *impl = nullptr;   // CocgImpl (cocg.cu)
};

int cocg_create(CocgState &cg, const rexi_desc *d, const ShiftDev &S, int refine, cudaStream_t st,
                std::string &err);
int cocg_step(CocgState &cg, const ShiftDev &S, cudaStream_t st, const c128 *u, c128 *uout,
              double *acc, int64_t *launches, std::string &err);
int cocg_solve_all(CocgState &cg, const ShiftDev &S, cudaStream_t st, const c128 *rhs, bool rhs_host,
                   c128 *x, std::string &err);
void cocg_destroy(CocgState &cg);
// fold the last step's rhs / accumulation event times into t_rhs_ms / t_acc_ms
void cocg_collect_phase(CocgState &cg);
cudaError_t cocg_axpy_inplace(c128 *x, const c128 *y, int64_t n, cudaStream_t st);

}  // namespace rexi
