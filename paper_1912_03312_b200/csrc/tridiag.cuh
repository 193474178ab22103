// tridiag.cuh -- batched partitioned direct solver for tridiagonal shifted pencils
//
// Replaces LAPACK zgbtrf/zgbtrs on the K shifted systems
// S_j = tau*A - sigma_j*iB (reference solvers.py:42-80, integrate.py:169-222)
// for 1D P1 pencils.  See DESIGN.md "1D path" for the algorithm:
//
//  * every level splits its rows into blocks of M; the first row of each
//    block is an interface row, the other M-1 are interior rows;
//  * prepare factors every block interior (no-pivot LDU; the imaginary part
//    of S_j is the definite -Re(sigma_j) B, so no pivoting is needed) and
//    forms the Schur complement on the interface rows, which is again a
//    complex-symmetric tridiagonal system -> next level; a level with
//    <= TOP_MAX rows is solved directly (one thread per shift);
//  * a step runs S1 (interior solves with zero halos -> reduced rhs) up the
//    levels, the top solve, then S3 (interior solves with the interface
//    values known) down the levels; level-0 S3 fuses the beta-weighted,
//    double-double accumulation over shifts (fixed order, so the result does
//    not depend on how shifts are sharded).
//
// Layout: every per-shift array is [row][k_pad] complex128 ("shift index is
// the fast dimension"), so one warp = 32 shifts of one block reads 512
// contiguous bytes per row; the level-0 matrix is formed on the fly from the
// shared A/B diagonals (read once from HBM, broadcast from L1).
#pragma once
#include "common.cuh"

namespace rexi {

constexpr int TRI_M = 16;        // block size (rows per block, incl. the interface row)
constexpr int TRI_THREADS = 256; // CTA size
constexpr int TOP_MAX = 1;       // recurse until a single interface row remains

struct L0Dev {
    const double *ta_sub, *ta_sub_im, *b_sub;   // entry (i, i-1); row 0 holds 0
    const double *ta_dia, *ta_dia_im, *b_dia;   // entry (i, i)
    const double *ta_sup, *ta_sup_im, *b_sup;   // entry (i, i+1); row n-1 holds 0
    const double *b_sub_raw, *b_dia_raw, *b_sup_raw;  // B for the rhs (same as b_*)
};

struct LevelDev {
    int64_t n;        // rows of this level
    int64_t P;        // blocks (= rows of the next level)
    int top;          // 1: solved directly
    int sym;          // 1: symmetric pencil -> reduced levels store sup only
    c128 *sub, *dia, *sup;          // explicit coefficients, levels >= 1
    c128 *invd;                     // inverse pivots of interior rows
    c128 *ypart, *lc;               // S1 outputs: next-level rhs = ypart + lc  [P][kp]
    c128 *X;                        // solution  [n][kp]
    c128 *phiF, *phiL, *psiF, *psiL;// factor tips [P][kp]
    cdh *ypdd, *lcdd;               // refinement (level 0): dd reduced rhs of the correction (fp64 hi, fp32 lo)
};

struct ShiftDev {
    const c128 *sigma;   // [kp]
    const c128 *beta;    // [kp] (0 on padding lanes)
    int kp;
};

// ---- coefficient access ----
template <bool L0>
__device__ __forceinline__ c128 co_sub(const L0Dev &z, const LevelDev &L, const ShiftDev &S,
                                       int64_t i, int j, c128 sg) {
    if constexpr (L0) return form_entry(__ldg(z.ta_sub + i), __ldg(z.ta_sub_im + i), __ldg(z.b_sub + i), sg);
    // reduced levels of a symmetric pencil are complex symmetric: sub_i := sup_{i-1}
    // (one array, used consistently by the factorisation and the sweeps)
    else if (L.sym) return i > 0 ? L.sup[(i - 1) * S.kp + j] : cmk(0.0, 0.0);
    else return L.sub[i * S.kp + j];
}
template <bool L0>
__device__ __forceinline__ c128 co_sup(const L0Dev &z, const LevelDev &L, const ShiftDev &S,
                                       int64_t i, int j, c128 sg) {
    if constexpr (L0) return form_entry(__ldg(z.ta_sup + i), __ldg(z.ta_sup_im + i), __ldg(z.b_sup + i), sg);
    else return L.sup[i * S.kp + j];
}
template <bool L0>
__device__ __forceinline__ c128 co_dia(const L0Dev &z, const LevelDev &L, const ShiftDev &S,
                                       int64_t i, int j, c128 sg) {
    if constexpr (L0) return form_entry(__ldg(z.ta_dia + i), __ldg(z.ta_dia_im + i), __ldg(z.b_dia + i), sg);
    else return L.dia[i * S.kp + j];
}

}  // namespace rexi
