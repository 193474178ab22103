// cocg.cu -- placeholder until the lockstep COCG kernels land.
#include "cocg.cuh"

namespace rexi {

__global__ void k_axpy_inplace(c128 *x, const c128 *y, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = cadd(x[i], y[i]);
}

cudaError_t cocg_axpy_inplace(c128 *x, const c128 *y, int64_t n, cudaStream_t st) {
    k_axpy_inplace<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, y, n);
    return cudaGetLastError();
}

int cocg_create(CocgState &, const rexi_desc *, const ShiftDev &, int, cudaStream_t, std::string &err) {
    err = "COCG solver not built yet";
    return REXI_ERR_UNSUPPORTED;
}
int cocg_step(CocgState &, const ShiftDev &, cudaStream_t, const c128 *, c128 *, double *, int64_t *,
              std::string &err) {
    err = "COCG solver not built yet";
    return REXI_ERR_UNSUPPORTED;
}
int cocg_solve_all(CocgState &, const ShiftDev &, cudaStream_t, const c128 *, bool, c128 *, std::string &err) {
    err = "COCG solver not built yet";
    return REXI_ERR_UNSUPPORTED;
}
void cocg_destroy(CocgState &) {}

}  // namespace rexi
