/*
 * rexi_b200.h -- C ABI of the B200-native REXI time step.
 *
 * One REXI step (reference rexiprop 0.1.0, pkg/src/rexiprop/integrate.py):
 *
 *     u1 = sum_j beta_j (tau*A - sigma_j*iB)^{-1} (iB u0)
 *
 * The reference has no FFI: its boundary is the Python function surface
 * rexi_prepare / rexi_step / rexi_run (integrate.py:143-245) over the
 * factorize()/solve() protocol of solvers.py:39-115.  These entry points
 * replace, one for one:
 *
 *   rexi_plan_create   <- rexi_prepare          integrate.py:143-190
 *                         (shifted-operator formation integrate.py:171,
 *                          factorize + zgbtrf   solvers.py:42-69,108-115)
 *   rexi_plan_step     <- rexi_step / rexi_run  integrate.py:193-245
 *   rexi_plan_run      <- rexi_run with an observer (every state kept)
 *                         (rhs integrate.py:203-206, K solves :208-222 via
 *                          zgbtrs solvers.py:76-80, Kahan reduce :59-68,224)
 *   rexi_plan_step_partial + rexi_combine_partials
 *                      <- the worker-pool split of the K solves and the
 *                         fixed-order reduction (integrate.py:114-120,
 *                         196-198, 215-224), across GPUs
 *   rexi_plan_solve    <- factorizations[j].solve(b)  solvers.py:76-80
 *   rexi_plan_destroy  <- RexiStepper.close()   integrate.py:131-140
 *
 * and, for the prepare/comparison paths around the step,
 * a pencil object holding (A, B) on one GPU:
 *
 *   rexi_pencil_create           <- factorize(sys.B)         solvers.py:108-115
 *   rexi_pencil_solve_b          <- factorize(sys.B).solve   solvers.py:76-80
 *   rexi_pencil_spectral_radius  <- spectral_radius_estimate spatial.py:314-344
 *   rexi_pencil_cheb_step        <- chebyshev_step / _run    integrate.py:333-377
 *   rexi_pencil_destroy
 *
 * Conventions: plain pointers and sizes only.  Complex values are
 * interleaved (re, im) doubles, layout-compatible with numpy complex128.
 * Every call returns a rexi_status; on failure rexi_plan_last_error() (or
 * rexi_last_error() when no plan exists) gives the message.  A plan is not
 * reentrant (reference SPEC.md: "rexi_run is not reentrant on a single
 * stepper"); distinct plans may run concurrently on distinct streams or
 * devices.  The plan owns device copies of everything in rexi_desc; the
 * caller keeps ownership of its host buffers.
 */
#ifndef REXI_B200_H
#define REXI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REXI_ABI_VERSION 3

typedef struct rexi_c128 { double re, im; } rexi_c128;
typedef struct rexi_plan rexi_plan;

typedef enum rexi_status {
    REXI_OK = 0,
    REXI_ERR_INVALID = 1,      /* -> ValueError                                  */
    REXI_ERR_SINGULAR = 2,     /* -> SolverError "shifted system j = ... singular" */
    REXI_ERR_NOCONV = 3,       /* -> SolverError (iterative solve did not converge) */
    REXI_ERR_BREAKDOWN = 4,    /* -> SolverError (COCG breakdown / non-finite)   */
    REXI_ERR_CUDA = 5,         /* -> DeviceError                                 */
    REXI_ERR_NOMEM = 6,        /* -> DeviceError (HBM exhausted)                 */
    REXI_ERR_UNSUPPORTED = 7   /* -> ValueError                                  */
} rexi_status;

typedef enum rexi_solver {
    REXI_SOLVER_AUTO = 0,      /* tridiagonal -> TRIDIAG, half band 2..4 -> BAND,
                                  else COCG                                      */
    REXI_SOLVER_TRIDIAG = 1,   /* batched partitioned direct solve (1D P1)       */
    REXI_SOLVER_COCG = 2,      /* lockstep Jacobi-COCG over shifts (2D/3D, any)  */
    REXI_SOLVER_BAND = 3       /* partitioned band LU, half bandwidth 2..4 (the
                                  reference's P2 1D pencils, bandwidth 5)        */
} rexi_solver;

typedef enum rexi_mem { REXI_MEM_HOST = 0, REXI_MEM_DEVICE = 1 } rexi_mem;

typedef struct rexi_desc {
    int32_t abi_version;       /* REXI_ABI_VERSION                                */
    int64_t n;                 /* n_dof                                           */
    int64_t nnz;               /* entries of the shared CSR pattern of A and B    */
    const int32_t *indptr;     /* host, n+1                                       */
    const int32_t *indices;    /* host, nnz, sorted within each row               */
    const double *a_vals;      /* host, nnz: A on the pattern (real part)         */
    const double *a_imag;      /* host, nnz or NULL: imaginary part of A          */
    const double *b_vals;      /* host, nnz: B on the pattern (real)              */
    int32_t k;                 /* number of shifts handled by this plan           */
    const rexi_c128 *shifts;   /* host, k: sigma_j                                */
    const rexi_c128 *weights;  /* host, k: beta_j                                 */
    int32_t shift_offset;      /* global index of shifts[0] (error messages)      */
    double tau;
    int32_t device;            /* CUDA ordinal                                    */
    int32_t solver;            /* rexi_solver                                     */
    int32_t refine;            /* residual-refinement rounds: -1 auto, 0..4       */
    double tol;                /* COCG relative residual target (0 -> 1e-12)      */
    int32_t max_iters;         /* COCG iteration cap per solve (0 -> 20000)       */
    void *stream;              /* cudaStream_t to run on, or NULL (plan-owned)    */
    double weight_ref;         /* COCG: reference |beta| for the per-shift tolerance
                                  weights (mean |beta| over ALL K shifts, so a shard
                                  converges exactly as in the unsharded run); 0 ->
                                  the mean over this plan's shifts                 */
    const int32_t *shift_ids;  /* host, k or NULL: global index of each shift (a
                                  cost-balanced shard is not contiguous); NULL ->
                                  shift_offset + i.  Error messages name these. */
} rexi_desc;

typedef struct rexi_stats {
    /* device time (CUDA events on the plan's stream) of the phases of the
     * reference timers rhs/local/reduce (integrate.py:110-112, 203-225):
     * rhs    = staging u onto the device + forming iB u where it is a kernel
     *          of its own (COCG); 0 when both are fused into the first solve
     *          kernel (1D zero-copy / device input),
     * local  = the shifted solves (and whatever is fused into them: the 1D
     *          level-0 kernels also form iB u and the beta-weighted sum),
     * reduce = the beta-weighted accumulation where it is a kernel of its own
     *          (COCG) + copying u1 back to the host.
     * A one-step call of a direct solver (TRIDIAG / BAND) fuses rhs and sum
     * into its kernels and is not event-timed (four timed events cost ~17 us,
     * a third of a config-1 step): t_local_ms is the host time of the call,
     * t_rhs_ms = t_reduce_ms = 0. */
    double t_rhs_ms;
    double t_local_ms;
    double t_reduce_ms;
    int64_t steps;             /* steps executed by this call                     */
    int64_t launches;          /* kernels launched by this call                   */
    int32_t iters_max;         /* COCG: max over shifts of the shift's iterations,
                                  first solve + corrections (last step)           */
    double iters_mean;         /* COCG: mean over shifts of the same (last step)  */
    int32_t refine_rounds;     /* refinement rounds applied per step              */
    int32_t bad_shift;         /* global index of a failing shift, -1 if none     */
} rexi_stats;

typedef struct rexi_info {
    int32_t solver;            /* resolved rexi_solver                            */
    int32_t bandwidth;         /* kl+ku+1 of the pattern (3 for 1D P1)            */
    int32_t k_pad;             /* lanes per block (padded shift count)            */
    int32_t levels;            /* TRIDIAG: partition levels (incl. top)           */
    int32_t refine;            /* resolved refinement rounds                      */
    int64_t device_bytes;      /* HBM held by the plan                            */
    double prepare_ms;         /* device time of rexi_plan_create                 */
    double min_pivot_ratio;    /* TRIDIAG: min over shifts of min|d|/max|d|       */
    int32_t persistent;        /* >0: small 1D plan, all steps of a call run in ONE
                                  launch of a thread-block cluster of this many CTAs */
    double screen_pivot_ratio; /* bandwidth <= 32: min over shifts of min|U_ii| /
                                  max|U_ii| of the partially pivoted band LU -- the
                                  reference's singularity screen (solvers.py:52-69),
                                  recomputed on the device at plan creation; 1 when
                                  the band is wider (the reference's dense LU) */
} rexi_info;

int rexi_plan_create(const rexi_desc *desc, rexi_plan **out);

/* n_steps REXI steps: u_out = step^n(u_in).  mem says whether u_in/u_out are
 * host (pinned or pageable) or device pointers.  u_in == u_out is allowed. */
int rexi_plan_step(rexi_plan *plan, const rexi_c128 *u_in, rexi_c128 *u_out,
                   int32_t n_steps, int32_t mem, rexi_stats *stats);

/* n_steps steps from u_in, writing the state after EVERY step into snaps
 * (n_steps * n complex, step-major): the on-device snapshots behind
 * rexi_run's observer (integrate.py:229-245, harness.py:220-225,330-336).
 * Small 1D plans run all steps in one launch; others chain device steps
 * without a host round trip.  mem applies to u_in and snaps. */
int rexi_plan_run(rexi_plan *plan, const rexi_c128 *u_in, rexi_c128 *snaps, int32_t n_steps, int32_t mem,
                  rexi_stats *stats);

/* One step for this plan's shard of shifts, leaving the double-double
 * partial sum sum_{j in shard} beta_j x_j in partial (device, 4*n doubles:
 * re_hi[n], re_lo[n], im_hi[n], im_lo[n]).  u_in is a device pointer.
 * On a caller-provided stream (desc.stream) a 1D plan's call is
 * stream-ordered: it returns once the step is enqueued, so the caller's
 * collective on that stream follows without a host round trip.  Otherwise
 * (own stream, COCG) it returns after the step completes. */
int rexi_plan_step_partial(rexi_plan *plan, const rexi_c128 *u_in, double *partial,
                           rexi_stats *stats);

/* out = round(sum_{g=0}^{G-1} partials[g]) in fixed g order (device pointers,
 * partials laid out as G consecutive 4*n blocks).  stream NULL: the legacy
 * stream, returns when done; otherwise stream-ordered on that stream. */
int rexi_combine_partials(const double *partials, int32_t g, int64_t n, rexi_c128 *out,
                          void *stream);

/* Per-shift solutions x_j = S_j^{-1} rhs for every shift of the plan
 * (x: k*n complex, shift-major).  mem applies to rhs and x. */
int rexi_plan_solve(rexi_plan *plan, const rexi_c128 *rhs, rexi_c128 *x, int32_t mem);

int rexi_plan_info(const rexi_plan *plan, rexi_info *info);

/* Order the plan's stream after all work enqueued so far on `stream` (e.g.
 * torch's current stream, which produced the device input): an event
 * recorded on `stream`, waited on by the plan's stream, no host sync.
 * Every rexi_plan_* call with device pointers returns only after its work
 * completed (except the stream-ordered 1D rexi_plan_step_partial on a
 * caller's stream), so outputs need no such wait. */
int rexi_plan_wait_stream(rexi_plan *plan, void *stream);

/* Per-shift COCG iterations of the last step (first solve + corrections),
 * iters: k entries in the plan's shift order; all 0 for the direct solver.
 * The cost model for balancing pole shards. */
int rexi_plan_shift_iters(const rexi_plan *plan, int32_t *iters);

/* Per-kernel device-time profiling with CUDA events on the plan's stream
 * (used by bench.py for the roofline).  enable resets the counters; the
 * report is text lines "<kernel> <launches> <total_ms>". */
int rexi_plan_profile(rexi_plan *plan, int32_t enable);
int rexi_plan_profile_report(rexi_plan *plan, char *buf, int64_t len);
int rexi_plan_destroy(rexi_plan *plan);
const char *rexi_plan_last_error(const rexi_plan *plan);
const char *rexi_last_error(void);
int rexi_device_count(int32_t *count);

/* ---- pencil (A, B): B-solves, spectral radius, Chebyshev stepping ---- */
typedef struct rexi_pencil rexi_pencil;

/* Uses n, nnz, indptr, indices, a_vals, a_imag, b_vals, device, stream and
 * tol / max_iters (CG on B: relative residual target, 0 -> 1e-14; iteration
 * cap, 0 -> 1000) of the descriptor; k, shifts, weights, tau are ignored.
 * B must be symmetric positive definite (the reference's mass matrix);
 * REXI_ERR_SINGULAR if a diagonal entry of B is not positive. */
int rexi_pencil_create(const rexi_desc *desc, rexi_pencil **out);

/* x = B^-1 rhs (Jacobi-preconditioned CG); mem applies to rhs and x. */
int rexi_pencil_solve_b(rexi_pencil *pencil, const rexi_c128 *rhs, rexi_c128 *x, int32_t mem,
                        int32_t *iterations);

/* Power iteration on B^-1 A from the host start vector v0 (normalised on
 * the device), Rayleigh quotient |v^H A v / v^H B v|, stop when two
 * successive quotients agree to tol relative (spatial.py:314-344).
 * iterations / converged as in SpectralRadiusEstimate (spatial.py:296-311). */
int rexi_pencil_spectral_radius(rexi_pencil *pencil, const rexi_c128 *v0, double tol, int32_t max_iters,
                                double *value, int32_t *iterations, int32_t *converged);

/* n_steps Chebyshev steps u <- p(tau M) u by the Clenshaw recurrence with
 * coefficients coeffs[0..degree] and scale = -tau/R (integrate.py:333-356):
 * b_k = a_k u + 2 scale B^-1 A b_{k+1} - b_{k+2}, out = a_0 u + scale B^-1 A b_1 - b_2.
 * mem applies to u_in / u_out; stats: device time, CG iterations (max and
 * mean per B-solve), launches. */
int rexi_pencil_cheb_step(rexi_pencil *pencil, const rexi_c128 *coeffs, int32_t degree, double scale,
                          const rexi_c128 *u_in, rexi_c128 *u_out, int32_t n_steps, int32_t mem,
                          rexi_stats *stats);
const char *rexi_pencil_last_error(const rexi_pencil *pencil);
/* as rexi_plan_wait_stream */
int rexi_pencil_wait_stream(rexi_pencil *pencil, void *stream);

/* ---- P1 assembly on a structured Kuhn mesh ----
 * Builds A = 0.5 K + M_V and B = M on the interior nodes of an m^d-cell grid
 * (d = 1, 2, 3; d! simplices per cell) directly in device memory, in the
 * builder's host assembly order (fixtures.py assemble_p1, restating the
 * reference's COO assembly spatial.py:193-223 for P1).  The caller supplies
 * the stencil/contribution table (host) and the element potential matrices
 * pot_e (device, [n_templates][m^d][(d+1)^2]); indptr (n_int+1), indices,
 * a_vals, b_vals (nnz = sum over offsets of prod_k (m-1-|o_k|)) are device
 * buffers the caller allocates. */
typedef struct rexi_p1_desc {
    int32_t d, m;                   /* dimension, cells per axis                     */
    int32_t n_templates;            /* simplices per cell (d!)                      */
    int32_t n_off;                  /* stencil offsets, sorted by column delta       */
    const int32_t *offsets;         /* host [n_off][d]                              */
    int32_t n_contrib;              /* element contributions, grouped by offset     */
    const int32_t *contrib_start;   /* host [n_off + 1]                             */
    const int32_t *contrib_t;       /* host [n_contrib] template index              */
    const int32_t *contrib_a;       /* host [n_contrib] local row (vertex a)        */
    const int32_t *contrib_b;       /* host [n_contrib] local column (vertex b)     */
    const int32_t *contrib_va;      /* host [n_contrib][d] vertex a offset in cells */
    const double *contrib_stiff;    /* host [n_contrib] K_e[a][b] (scaled by h)     */
    const double *contrib_mass;     /* host [n_contrib] M_e[a][b]                   */
    int32_t device;
    void *stream;
} rexi_p1_desc;
int rexi_assemble_p1(const rexi_p1_desc *desc, const double *pot_e, int32_t *indptr, int32_t *indices,
                     double *a_vals, double *b_vals);
int rexi_pencil_destroy(rexi_pencil *pencil);
int32_t rexi_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* REXI_B200_H */
