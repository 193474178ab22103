// tridiag_launch.h -- host-callable launchers of the tridiagonal kernels.
#pragma once
#include "tridiag.cuh"

namespace rexi {

enum { TRI_OUT_X = 0, TRI_OUT_ACC = 1, TRI_OUT_X_ACC = 2 };

cudaError_t tri_launch_rhs(const L0Dev &z, int64_t n, const c128 *u, c128 *rhs, cudaStream_t st);
cudaError_t tri_launch_residual(const L0Dev &z, const LevelDev &L, const ShiftDev &S,
                                const c128 *rhs0, c128 *res, cudaStream_t st);
cudaError_t tri_launch_s1(const L0Dev &z, const LevelDev &L, const ShiftDev &S, int level,
                          const c128 *rhs0, const c128 *rst, const c128 *rin_a,
                          const c128 *rin_b, cudaStream_t st);
cudaError_t tri_launch_s3(const L0Dev &z, const LevelDev &L, const ShiftDev &S, int level,
                          const c128 *rhs0, const c128 *rst, const c128 *rin_a,
                          const c128 *rin_b, const c128 *Xnext, int out_mode, double *acc,
                          int acc_add, c128 *uout, cudaStream_t st);
cudaError_t tri_launch_top_solve(const LevelDev &L, const ShiftDev &S, const c128 *rin_a,
                                 const c128 *rin_b, cudaStream_t st);
cudaError_t tri_launch_factor(const L0Dev &z, const LevelDev &L, const LevelDev *next,
                              const ShiftDev &S, int level, unsigned long long *pmin,
                              unsigned long long *pmax, cudaStream_t st);
cudaError_t tri_launch_transpose(const c128 *X, int64_t n, int kp, int k, c128 *out, cudaStream_t st);
cudaError_t launch_combine(const double *parts, int g, int64_t n, c128 *out, cudaStream_t st);

// levels >= 1 reading the double-double reduced rhs of the correction pass
cudaError_t tri_launch_lv_dd(const LevelDev &L, const ShiftDev &S, int phase, const cdh *rdd_a,
                             const cdh *rdd_b, const c128 *Xnext, cudaStream_t st);
cudaError_t tri_launch_top_solve_dd(const LevelDev &L, const ShiftDev &S, const cdh *rdd_a,
                                    const cdh *rdd_b, cudaStream_t st);

// TMA-fed kernel for levels >= 1 of symmetric pencils (tridiag_l0.cu)
// one-launch multi-step loop for small 1D plans (tridiag_persist.cu)
constexpr int PS_MAXLV = 8;
int persist_cluster_size(const LevelDev *lv, int nl, int kp);
cudaError_t persist_launch(const L0Dev &z, const LevelDev *lv, int nl, const ShiftDev &S, int64_t n,
                           const c128 *u_in, c128 *ua, c128 *ub, c128 *snaps, int n_steps, int csize,
                           cudaStream_t st, c128 *final_out = nullptr);

inline int64_t lv_tma_ctas(int64_t n, int kp) {   // grid of lv_launch_tma
    const int64_t rows = (int64_t)(128 / kp) * TRI_M;
    return (n + rows - 1) / rows;
}
// rw (correction pass, dd rhs): phase 1 stores the rounded rhs rows there,
// phase 3 reads them back instead of re-combining the double-double halves
cudaError_t lv_launch_tma(const LevelDev &L, const ShiftDev &S, int phase, const c128 *rin_a, const c128 *rin_b,
                          const cdh *rdd_a, const cdh *rdd_b, const c128 *Xnext, cudaStream_t st,
                          c128 *rw = nullptr);

// level 1 of the refinement's correction pass in complex64 (tridiag_l0.cu)
cudaError_t lv32_launch(const LevelDev &L, const ShiftDev &S, int phase, const c64 *inv32, const c64 *sup32,
                        const cdh *rdd_a, const cdh *rdd_b, c64 *rw, const c128 *Xnext, cudaStream_t st);

// levels l0..top..l0 in one cluster launch (tridiag_l0.cu); lv_chain_start
// returns the first chained level (0: none) and the cluster size
int lv_chain_start(const LevelDev *lv, int nl, int kp, int *cs);
cudaError_t lv_launch_chain(const LevelDev *lv, int nl, int l0, int cs, const ShiftDev &S, cudaStream_t st);

// captured-step graph nodes (role 1: S1 reads u; role 2: the kernel that
// writes the rounded output) and their re-pointing (tridiag_l0.cu)
int l0_graph_role(cudaGraphNode_t node);
cudaError_t l0_graph_patch(cudaGraphExec_t exec, cudaGraphNode_t node, int role, const c128 *u, c128 *uout);

// TMA-fed level-0 kernels (tridiag_l0.cu)
bool l0v2_supported(int kp);
int64_t l0_row_padding();
cudaError_t l0_launch_s1(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *u, c128 *rhs0,
                         int64_t nout, cudaStream_t st);
cudaError_t l0_launch_s3acc(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                            const c128 *X1, double *acc, c128 *uout, int64_t nout, cudaStream_t st);
cudaError_t l0_launch_k2(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *rhs0,
                         const c128 *X1, double *acc, c64 *rres, const c64 *inv32, const float *const *r32,
                         const double2 *emax, int64_t nout, bool exact_residual, cudaStream_t st);
cudaError_t l0_launch_k3(const L0Dev &z, const LevelDev &L, const ShiftDev &S, const c128 *X1,
                         const c64 *inv32, const float *const *r32, const c64 *rres, double *acc, c128 *uout,
                         int64_t nout, cudaStream_t st);
cudaError_t launch_to_c64(const c128 *src, c64 *dst, int64_t n, cudaStream_t st);
cudaError_t launch_to_f32(const double *src, float *dst, int64_t n, cudaStream_t st);

}  // namespace rexi
