// plan.cu -- the C ABI of include/rexi_b200.h: plan creation (the analogue of
// rexi_prepare, reference integrate.py:143-190), stepping (rexi_step /
// rexi_run, integrate.py:193-245), per-shift solves and partial sums for the
// pole-sharded multi-GPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rexi_b200.h"
#include "band.cuh"
#include "cocg.cuh"
#include "screen.cuh"
#include "tridiag_launch.h"

using namespace rexi;

namespace {

thread_local std::string g_last_error;

struct TriState {
    int64_t n = 0;
    std::vector<LevelDev> lv;     // device pointers, one per level (last = top)
    L0Dev z{};
    c128 *rhs0 = nullptr, *rres = nullptr;
    c64 *inv32 = nullptr;         // refinement, TMA path: level-0 inverse pivots as complex64
    c64 *rres32 = nullptr;        // refinement, TMA path: complex64 residual (aliases rres)
    float *r32[6] = {};           // refinement, TMA path: level-0 sub/sup row data rounded to float
    c64 *l1_inv32 = nullptr, *l1_sup32 = nullptr, *l1_rw32 = nullptr;   // correction pass, level 1 (complex64)
    double *acc = nullptr;
    double2 *emax = nullptr;      // refinement, TMA path: per level-0 block max |fl(tau a)| and max |b| (K2's aligned residual)
    bool complex_a = false;       // A has an imaginary part: K2 keeps every residual product error-free
};

}  // namespace

namespace rexi {
void set_global_error(const std::string &msg) { g_last_error = msg; }
}  // namespace rexi

struct rexi_plan {
    int device = 0;
    int solver = REXI_SOLVER_AUTO;
    int64_t n = 0;
    int k = 0, kp = 0;
    int shift_offset = 0;
    std::vector<int> gid;         // global index of each shift (error messages)
    int refine = 0;
    int bandwidth = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    std::vector<void *> allocs;
    int64_t bytes = 0;
    ShiftDev S{};
    c128 *ubuf[2] = {nullptr, nullptr};
    TriState tri;
    CocgState cg;
    BandState band;
    double prepare_ms = 0.0;
    double min_pivot_ratio = 1.0;
    double screen_ratio = 1.0;    // min over shifts of min|U_ii| / max|U_ii| (pivoted band LU)
    cudaEvent_t phase_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // rexi_stats phases, reused per call
    std::vector<rexi_c128> shifts_host;
    int64_t launches = 0;
    // optional per-kernel CUDA-event profiling (rexi_plan_profile)
    bool prof = false;
    struct Rec { const char *name; cudaEvent_t a, b; double bytes; };
    struct Acc { int64_t count = 0; double ms = 0.0, bytes = 0.0; };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, Acc> prof_acc;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};   // 1D step replay (ubuf[g] -> ubuf[g^1])
    // the same step with its input/output kernels re-pointed per call at
    // page-locked host buffers (the last step of a host call)
    cudaGraph_t zc_src[2] = {nullptr, nullptr};
    cudaGraphExec_t zc_exec[2] = {nullptr, nullptr};
    cudaGraphNode_t zc_in_node[2] = {nullptr, nullptr}, zc_out_node[2] = {nullptr, nullptr};
    int persist_cs = 0;                               // >0: small 1D plan, all steps in one cluster launch
    c128 *pbuf[2] = {nullptr, nullptr};               // its state ping-pong
    int64_t graph_kernels = 0;
    // 1D shard step (rexi_plan_step_partial) replays, keyed by (u_in, partial)
    struct PartGraph { const void *u, *part; cudaGraphExec_t exec; int64_t kernels; };
    std::vector<PartGraph> part_graphs;
    struct Hook : rexi::ProfHook {
        rexi_plan *p = nullptr;
        cudaEvent_t a = nullptr;
        const char *name = nullptr;
        double bytes = 0.0;
        void begin(const char *n, double b) override;
        void end() override;
    } hook;
};

namespace {

cudaEvent_t prof_event(rexi_plan *p) {
    if (!p->pool.empty()) {
        cudaEvent_t e = p->pool.back();
        p->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    rexi_plan *p;
    const char *name;
    cudaEvent_t a = nullptr;
    ProfScope(rexi_plan *p_, const char *n) : p(p_), name(n) {
        ++p->launches;
        if (p->prof) {
            a = prof_event(p);
            cudaEventRecord(a, p->stream);
        }
    }
    ~ProfScope() {
        if (p->prof) {
            cudaEvent_t b = prof_event(p);
            cudaEventRecord(b, p->stream);
            p->pending.push_back({name, a, b, 0.0});
        }
    }
};

void prof_flush(rexi_plan *p) {
    if (p->pending.empty()) return;
    cudaStreamSynchronize(p->stream);
    for (auto &r : p->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto &acc = p->prof_acc[r.name];
        acc.count += 1;
        acc.ms += ms;
        acc.bytes += r.bytes;
        p->pool.push_back(r.a);
        p->pool.push_back(r.b);
    }
    p->pending.clear();
}

}  // namespace

void rexi_plan::Hook::begin(const char *n, double b) {
    if (!p->prof) return;
    name = n;
    bytes = b;
    a = prof_event(p);
    cudaEventRecord(a, p->stream);
}

void rexi_plan::Hook::end() {
    if (!p->prof) return;
    cudaEvent_t b = prof_event(p);
    cudaEventRecord(b, p->stream);
    p->pending.push_back({name, a, b, bytes});
}

namespace {

int set_err(rexi_plan *p, int code, const std::string &msg) {
    g_last_error = msg;
    if (p) p->err = msg;
    return code;
}

int cuda_err(rexi_plan *p, cudaError_t e, const char *what) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error in %s: %s (%s)", what, cudaGetErrorName(e),
             cudaGetErrorString(e));
    return set_err(p, e == cudaErrorMemoryAllocation ? REXI_ERR_NOMEM : REXI_ERR_CUDA, buf);
}

#define CK(expr)                                                   \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return cuda_err(plan, _e, #expr);   \
    } while (0)

template <typename T>
int dalloc(rexi_plan *plan, T **ptr, size_t count) {
    void *v = nullptr;
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&v, bytes);
    if (e != cudaSuccess) return cuda_err(plan, e, "cudaMalloc");
    e = rexi_poison(v, bytes);
    if (e != cudaSuccess) return cuda_err(plan, e, "poison");
    plan->allocs.push_back(v);
    plan->bytes += (int64_t)bytes;
    *ptr = (T *)v;
    return REXI_OK;
}

#define DALLOC(ptr, count)                          \
    do {                                            \
        int _rc = dalloc(plan, &(ptr), (count));    \
        if (_rc) return _rc;                        \
    } while (0)

int pick_kp(int k) {
    int kp = 1;
    while (kp < k) kp <<= 1;
    return kp;
}

// ------------------------------------------------------------------------
// tridiagonal path
// ------------------------------------------------------------------------
int tri_create(rexi_plan *plan, const rexi_desc *d) {
    const int64_t n = d->n;
    TriState &T = plan->tri;
    T.n = n;
    // diagonals of A (re, im) and B from the shared CSR pattern
    std::vector<double> a_sub(n, 0.0), a_dia(n, 0.0), a_sup(n, 0.0);
    std::vector<double> ai_sub(n, 0.0), ai_dia(n, 0.0), ai_sup(n, 0.0);
    std::vector<double> b_sub(n, 0.0), b_dia(n, 0.0), b_sup(n, 0.0);
    for (int64_t r = 0; r < n; ++r) {
        for (int32_t q = d->indptr[r]; q < d->indptr[r + 1]; ++q) {
            int64_t c = d->indices[q];
            double av = d->a_vals[q], ai = d->a_imag ? d->a_imag[q] : 0.0, bv = d->b_vals[q];
            if (ai != 0.0) T.complex_a = true;
            if (c == r - 1) { a_sub[r] = av; ai_sub[r] = ai; b_sub[r] = bv; }
            else if (c == r) { a_dia[r] = av; ai_dia[r] = ai; b_dia[r] = bv; }
            else if (c == r + 1) { a_sup[r] = av; ai_sup[r] = ai; b_sup[r] = bv; }
            else return set_err(plan, REXI_ERR_INVALID, "pattern is not tridiagonal");
        }
    }
    // fl(tau * a) exactly as numpy computes tau*A (integrate.py:171)
    auto scale = [&](std::vector<double> &v) { for (auto &x : v) x = d->tau * x; };
    scale(a_sub); scale(a_dia); scale(a_sup); scale(ai_sub); scale(ai_dia); scale(ai_sup);
    // TMA-fed level 0: pad to a multiple of the block size with decoupled unit
    // rows (zero couplings, diagonal 1, rhs 0) so every level-0 block is full
    int64_t n0 = n;
    if (l0v2_supported(plan->kp)) {
        n0 = (n + TRI_M - 1) / TRI_M * TRI_M;
        for (auto *v : {&a_sub, &a_dia, &a_sup, &ai_sub, &ai_dia, &ai_sup, &b_sub, &b_dia, &b_sup})
            v->resize(n0, 0.0);
        for (int64_t r = n; r < n0; ++r) a_dia[r] = 1.0;
    }
    double *dz[9];
    std::vector<double> *hz[9] = {&a_sub, &ai_sub, &b_sub, &a_dia, &ai_dia, &b_dia, &a_sup, &ai_sup, &b_sup};
    // padded so that the level-0 kernels' TMA row ranges never leave the allocation
    const int64_t pad = l0_row_padding();
    for (int q = 0; q < 9; ++q) {
        DALLOC(dz[q], (size_t)(n0 + pad));
        CK(cudaMemsetAsync(dz[q], 0, sizeof(double) * (n0 + pad), plan->stream));
        CK(cudaMemcpyAsync(dz[q], hz[q]->data(), sizeof(double) * n0, cudaMemcpyHostToDevice, plan->stream));
    }
    T.z = L0Dev{dz[0], dz[1], dz[2], dz[3], dz[4], dz[5], dz[6], dz[7], dz[8], dz[2], dz[5], dz[8]};
    if (plan->refine > 0 && l0v2_supported(plan->kp)) {
        // K2's aligned residual bounds |Re entry| <= max|fl(tau a)| + |Im sigma| max|b| per block
        const int64_t nb = n0 / TRI_M;
        std::vector<double2> em((size_t)nb);
        for (int64_t p = 0; p < nb; ++p) {
            double mt = 0.0, mb = 0.0;
            for (int64_t r = p * TRI_M; r < (p + 1) * TRI_M; ++r) {
                mt = std::max({mt, std::fabs(a_sub[r]), std::fabs(a_dia[r]), std::fabs(a_sup[r])});
                mb = std::max({mb, std::fabs(b_sub[r]), std::fabs(b_dia[r]), std::fabs(b_sup[r])});
            }
            em[(size_t)p] = make_double2(mt, mb);
        }
        DALLOC(T.emax, (size_t)nb);
        CK(cudaMemcpyAsync(T.emax, em.data(), sizeof(double2) * nb, cudaMemcpyHostToDevice, plan->stream));
        CK(cudaStreamSynchronize(plan->stream));
    }

    // symmetric pencil (the FEM case): reduced levels keep only sup
    bool sym = true;
    for (int64_t r = 0; r + 1 < n && sym; ++r)
        sym = a_sup[r] == a_sub[r + 1] && ai_sup[r] == ai_sub[r + 1] && b_sup[r] == b_sub[r + 1];
    // levels
    const int kp = plan->kp;
    int64_t nl = n0;
    for (;;) {
        LevelDev L{};
        L.n = nl;
        L.sym = sym ? 1 : 0;
        if (!T.lv.empty() && nl <= TOP_MAX) {
            L.top = 1;
            L.P = 0;
        } else {
            L.top = 0;
            L.P = (nl + TRI_M - 1) / TRI_M;
        }
        size_t rows = (size_t)nl * kp;
        DALLOC(L.invd, rows);
        DALLOC(L.X, rows);
        if (!T.lv.empty()) {
            if (!sym) DALLOC(L.sub, rows);
            DALLOC(L.dia, rows);
            DALLOC(L.sup, rows);
        }
        if (!L.top) {
            size_t pr = (size_t)L.P * kp;
            DALLOC(L.ypart, pr);
            DALLOC(L.lc, pr);
            DALLOC(L.phiF, pr);
            DALLOC(L.phiL, pr);
            DALLOC(L.psiF, pr);
            DALLOC(L.psiL, pr);
        }
        T.lv.push_back(L);
        if (L.top) break;
        nl = L.P;
    }
    DALLOC(T.rhs0, (size_t)(n0 + pad));
    CK(cudaMemsetAsync(T.rhs0, 0, sizeof(c128) * (n0 + pad), plan->stream));
    DALLOC(T.acc, (size_t)4 * n);
    if (plan->refine > 0) {
        DALLOC(T.rres, (size_t)n0 * kp);
        DALLOC(T.lv[0].ypdd, (size_t)T.lv[0].P * kp);
        DALLOC(T.lv[0].lcdd, (size_t)T.lv[0].P * kp);
    }

    // factor every level
    unsigned long long *pmin = nullptr, *pmax = nullptr;
    DALLOC(pmin, (size_t)kp);
    DALLOC(pmax, (size_t)kp);
    std::vector<unsigned long long> init_min(kp), init_max(kp, 0ull);
    double inf = INFINITY;
    unsigned long long inf_bits;
    memcpy(&inf_bits, &inf, sizeof inf_bits);
    std::fill(init_min.begin(), init_min.end(), inf_bits);
    CK(cudaMemcpyAsync(pmin, init_min.data(), sizeof(unsigned long long) * kp, cudaMemcpyHostToDevice, plan->stream));
    CK(cudaMemcpyAsync(pmax, init_max.data(), sizeof(unsigned long long) * kp, cudaMemcpyHostToDevice, plan->stream));
    for (size_t l = 0; l < T.lv.size(); ++l) {
        const LevelDev *next = l + 1 < T.lv.size() ? &T.lv[l + 1] : nullptr;
        CK(tri_launch_factor(T.z, T.lv[l], next, plan->S, (int)l, pmin, pmax, plan->stream));
    }
    std::vector<unsigned long long> hmin(kp), hmax(kp);
    CK(cudaMemcpyAsync(hmin.data(), pmin, sizeof(unsigned long long) * kp, cudaMemcpyDeviceToHost, plan->stream));
    CK(cudaMemcpyAsync(hmax.data(), pmax, sizeof(unsigned long long) * kp, cudaMemcpyDeviceToHost, plan->stream));
    CK(cudaStreamSynchronize(plan->stream));
    double worst = 1.0;
    for (int j = 0; j < plan->k; ++j) {
        double mn, mx;
        memcpy(&mn, &hmin[j], sizeof mn);
        memcpy(&mx, &hmax[j], sizeof mx);
        double ratio = mx > 0 ? mn / mx : 0.0;
        if (std::isinf(mn)) ratio = 1.0;  // no pivots at all (cannot happen: top level has >= 1 row)
        worst = std::min(worst, ratio);
        // the reference's verdict (pivoted zgbtrf screen) ran before this
        // factorization (rexi_plan_create); here only a no-pivot breakdown
        // the direct solver cannot run through is an error
        if (!(mn > 0.0) || !(mx < INFINITY)) {
            char buf[256];
            snprintf(buf, sizeof buf, "no-pivot block factorization broke down (pivot ratio = %.3e) [shift j = %d]",
                     ratio, plan->gid[j]);
            plan->min_pivot_ratio = ratio;
            return set_err(plan, REXI_ERR_SINGULAR, buf);
        }
    }
    plan->min_pivot_ratio = worst;
    if (plan->refine > 0 && l0v2_supported(kp)) {
        // the level-0 correction solve (K3) runs in complex64 (tridiag_l0.cu)
        DALLOC(T.inv32, (size_t)n0 * kp);
        CK(launch_to_c64(T.lv[0].invd, T.inv32, n0 * kp, plan->stream));
        const double *src32[6] = {T.z.ta_sub, T.z.ta_sub_im, T.z.b_sub, T.z.ta_sup, T.z.ta_sup_im, T.z.b_sup};
        const int64_t nrow = n0 + l0_row_padding();
        for (int q = 0; q < 6; ++q) {
            DALLOC(T.r32[q], (size_t)nrow);
            CK(launch_to_f32(src32[q], T.r32[q], nrow, plan->stream));
        }
        if (T.lv.size() >= 3 && T.lv[0].sym && !getenv("REXI_L1_FP64")) {
            // the correction pass's level 1 in complex64 (level 1 is not the top)
            const size_t e1 = (size_t)T.lv[1].n * kp;
            DALLOC(T.l1_inv32, e1);
            DALLOC(T.l1_sup32, e1);
            DALLOC(T.l1_rw32, e1);
            CK(launch_to_c64(T.lv[1].invd, T.l1_inv32, (int64_t)e1, plan->stream));
            CK(launch_to_c64(T.lv[1].sup, T.l1_sup32, (int64_t)e1, plan->stream));
        }
        T.rres32 = reinterpret_cast<c64 *>(T.rres);
        CK(cudaStreamSynchronize(plan->stream));
    }
    return REXI_OK;
}

// one pass of the level chain: S1 up, top solve, S3 down
int tri_chain(rexi_plan *plan, const c128 *rst, int out_mode, int acc_add, c128 *uout) {
    TriState &T = plan->tri;
    const size_t nl = T.lv.size();
    cudaStream_t st = plan->stream;
    for (size_t l = 0; l + 1 < nl; ++l) {
        const c128 *ra = l ? T.lv[l - 1].ypart : nullptr;
        const c128 *rb = l ? T.lv[l - 1].lc : nullptr;
        ProfScope ps(plan, l ? "s1_lv" : (rst ? "s1_l0_res" : "s1_l0"));
        CK(tri_launch_s1(T.z, T.lv[l], plan->S, (int)l, T.rhs0, l ? nullptr : rst, ra, rb, st));
    }
    {
        ProfScope ps(plan, "top");
        CK(tri_launch_top_solve(T.lv[nl - 1], plan->S, T.lv[nl - 2].ypart, T.lv[nl - 2].lc, st));
    }
    for (size_t l = nl - 1; l-- > 0;) {
        const c128 *ra = l ? T.lv[l - 1].ypart : nullptr;
        const c128 *rb = l ? T.lv[l - 1].lc : nullptr;
        const char *nm = l ? "s3_lv"
                           : (rst ? "s3_l0_res_acc"
                                  : (out_mode == TRI_OUT_ACC ? "s3_l0_acc"
                                                             : (out_mode == TRI_OUT_X ? "s3_l0_x" : "s3_l0_xacc")));
        ProfScope ps(plan, nm);
        CK(tri_launch_s3(T.z, T.lv[l], plan->S, (int)l, T.rhs0, l ? nullptr : rst, ra, rb,
                         T.lv[l + 1].X, l ? TRI_OUT_X : out_mode, T.acc, acc_add, l ? nullptr : uout,
                         st));
    }
    return REXI_OK;
}

// levels 1..top (S1 up, top solve, S3 down); level-1 rhs from level 0's
// ypart/lc, or from its double-double pieces in the correction pass
int tri_mid(rexi_plan *plan, bool dd) {
    TriState &T = plan->tri;
    const size_t nl = T.lv.size();
    cudaStream_t st = plan->stream;
    // TMA-staged kernel at every reduced level of a symmetric pencil (measured
    // faster than the plain kernel even for the few-CTA upper levels)
    const bool tma_ok = T.lv[0].sym && l0v2_supported(plan->kp);
    auto use_tma = [&](size_t) { return tma_ok; };
    // levels >= lc (one wave of <= 16 CTAs each) run as one cluster launch
    int ccs = 0;
    const int lc = tma_ok && !(nl == 2 && dd) ? lv_chain_start(T.lv.data(), (int)nl, plan->kp, &ccs) : 0;
    for (size_t l = 1; l + 1 < nl && (lc == 0 || (int)l < lc); ++l) {
        ProfScope ps(plan, "s1_lv");
        const bool d = l == 1 && dd;
        if (d && T.l1_inv32) CK(lv32_launch(T.lv[1], plan->S, 1, T.l1_inv32, T.l1_sup32, T.lv[0].ypdd, T.lv[0].lcdd,
                                            T.l1_rw32, nullptr, st));
        else if (use_tma(l)) CK(lv_launch_tma(T.lv[l], plan->S, 1, d ? nullptr : T.lv[l - 1].ypart, d ? nullptr : T.lv[l - 1].lc,
                                  d ? T.lv[0].ypdd : nullptr, d ? T.lv[0].lcdd : nullptr, nullptr, st,
                                  d ? T.lv[1].X : nullptr));
        else if (d) CK(tri_launch_lv_dd(T.lv[1], plan->S, 1, T.lv[0].ypdd, T.lv[0].lcdd, nullptr, st));
        else CK(tri_launch_s1(T.z, T.lv[l], plan->S, (int)l, nullptr, nullptr, T.lv[l - 1].ypart,
                              T.lv[l - 1].lc, st));
    }
    if (lc > 0) {
        ProfScope ps(plan, "lv_chain");
        CK(lv_launch_chain(T.lv.data(), (int)nl, lc, ccs, plan->S, st));
    } else {
        ProfScope ps(plan, "top");
        if (nl == 2 && dd) CK(tri_launch_top_solve_dd(T.lv[1], plan->S, T.lv[0].ypdd, T.lv[0].lcdd, st));
        else CK(tri_launch_top_solve(T.lv[nl - 1], plan->S, T.lv[nl - 2].ypart, T.lv[nl - 2].lc, st));
    }
    for (size_t l = lc > 0 ? (size_t)lc : nl - 1; l-- > 1;) {
        ProfScope ps(plan, "s3_lv");
        const bool d = l == 1 && dd;
        if (d && T.l1_inv32) CK(lv32_launch(T.lv[1], plan->S, 3, T.l1_inv32, T.l1_sup32, nullptr, nullptr,
                                            T.l1_rw32, T.lv[2].X, st));
        else if (use_tma(l)) CK(lv_launch_tma(T.lv[l], plan->S, 3, d ? nullptr : T.lv[l - 1].ypart, d ? nullptr : T.lv[l - 1].lc,
                                  d ? T.lv[0].ypdd : nullptr, d ? T.lv[0].lcdd : nullptr, T.lv[l + 1].X, st,
                                  d ? T.lv[1].X : nullptr));
        else if (d) CK(tri_launch_lv_dd(T.lv[1], plan->S, 3, T.lv[0].ypdd, T.lv[0].lcdd, T.lv[2].X, st));
        else CK(tri_launch_s3(T.z, T.lv[l], plan->S, (int)l, nullptr, nullptr, T.lv[l - 1].ypart,
                              T.lv[l - 1].lc, T.lv[l + 1].X, TRI_OUT_X, nullptr, 0, nullptr, st));
    }
    return REXI_OK;
}

// v2 step: TMA-fed level-0 kernels
int tri_step_v2(rexi_plan *plan, const c128 *u, c128 *uout) {
    TriState &T = plan->tri;
    cudaStream_t st = plan->stream;
    {
        ProfScope ps(plan, "l0_s1");   // rhs = iBu formed inside (no separate rhs kernel)
        CK(l0_launch_s1(T.z, T.lv[0], plan->S, u, T.rhs0, T.n, st));
    }
    int rc = tri_mid(plan, false);
    if (rc) return rc;
    if (plan->refine <= 0) {
        ProfScope ps(plan, "l0_s3acc");
        CK(l0_launch_s3acc(T.z, T.lv[0], plan->S, T.rhs0, T.lv[1].X, T.acc, uout, T.n, st));
        return REXI_OK;
    }
    {
        ProfScope ps(plan, "l0_k2");
        CK(l0_launch_k2(T.z, T.lv[0], plan->S, T.rhs0, T.lv[1].X, T.acc, T.rres32, T.inv32, T.r32, T.emax, T.n, T.complex_a, st));
    }
    rc = tri_mid(plan, true);
    if (rc) return rc;
    ProfScope ps(plan, "l0_k3");
    CK(l0_launch_k3(T.z, T.lv[0], plan->S, T.lv[1].X, T.inv32, T.r32, T.rres32, T.acc, uout, T.n, st));
    return REXI_OK;
}

// small unrefined 1D plans run every step of a call in ONE cluster launch
// (tridiag_persist.cu); REXI_PERSIST=0 disables it
int persist_setup(rexi_plan *plan) {
    TriState &T = plan->tri;
    const size_t nl = T.lv.size();
    if (const char *e = getenv("REXI_PERSIST"))
        if (atoi(e) == 0) return REXI_OK;
    if (plan->refine > 0 || nl < 2 || nl > (size_t)PS_MAXLV || plan->kp > 128 ||
        !l0v2_supported(plan->kp) || T.lv[nl - 2].P != 1)
        return REXI_OK;
    // the level-0 slices must fit in the shared memory of one cluster
    const int cs = persist_cluster_size(T.lv.data(), (int)nl, plan->kp);
    if (cs <= 0) return REXI_OK;
    int rc = dalloc(plan, &plan->pbuf[0], (size_t)plan->n);
    if (!rc) rc = dalloc(plan, &plan->pbuf[1], (size_t)plan->n);
    if (rc) return rc;
    plan->persist_cs = cs;
    return REXI_OK;
}

// one step from device u -> (uout rounded) or (T.acc partial when uout == nullptr)
int tri_step(rexi_plan *plan, const c128 *u, c128 *uout) {
    TriState &T = plan->tri;
    if (l0v2_supported(plan->kp)) return tri_step_v2(plan, u, uout);
    {
        ProfScope ps(plan, "rhs");
        CK(tri_launch_rhs(T.z, T.n, u, T.rhs0, plan->stream));
    }
    if (plan->refine <= 0) return tri_chain(plan, nullptr, TRI_OUT_ACC, 0, uout);
    int rc = tri_chain(plan, nullptr, TRI_OUT_X_ACC, 0, nullptr);
    if (rc) return rc;
    {
        ProfScope ps(plan, "residual");
        CK(tri_launch_residual(T.z, T.lv[0], plan->S, T.rhs0, T.rres, plan->stream));
    }
    return tri_chain(plan, T.rres, TRI_OUT_ACC, 1, uout);
}

// stats phases from the four events of a call (see rexi_plan_step) and the
// COCG rhs / accumulation kernel times; destroys the events
void fill_phases(rexi_plan *plan, cudaEvent_t ev[4], rexi_stats *stats) {
    float stage = 0.f, steps = 0.f, out = 0.f;
    cudaEventElapsedTime(&stage, ev[0], ev[1]);
    cudaEventElapsedTime(&steps, ev[1], ev[2]);
    cudaEventElapsedTime(&out, ev[2], ev[3]);
    (void)0;   // the events are the plan's (phase_ev), reused by every call
    cocg_collect_phase(plan->cg);
    const double cr = plan->cg.t_rhs_ms, ca = plan->cg.t_acc_ms;
    plan->cg.t_rhs_ms = plan->cg.t_acc_ms = 0.0;
    stats->t_rhs_ms = stage + cr;
    stats->t_local_ms = std::max(0.0, (double)steps - cr - ca);
    stats->t_reduce_ms = ca + out;
}

int plan_step_device(rexi_plan *plan, const c128 *u, c128 *uout) {
    if (plan->solver == REXI_SOLVER_TRIDIAG) return tri_step(plan, u, uout);
    if (plan->solver == REXI_SOLVER_BAND)
        return band_step(plan->band, plan->S, plan->stream, u, uout, plan->tri.acc, &plan->launches, plan->err);
    return cocg_step(plan->cg, plan->S, plan->stream, u, uout, plan->tri.acc, &plan->launches,
                     plan->err);
}

}  // namespace

extern "C" {

int32_t rexi_abi_version(void) { return REXI_ABI_VERSION; }

const char *rexi_last_error(void) { return g_last_error.c_str(); }

const char *rexi_plan_last_error(const rexi_plan *plan) {
    return plan ? plan->err.c_str() : g_last_error.c_str();
}

int rexi_device_count(int32_t *count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *count = 0;
        return cuda_err(nullptr, e, "cudaGetDeviceCount");
    }
    *count = c;
    return REXI_OK;
}

int rexi_plan_destroy(rexi_plan *plan) {
    if (!plan) return REXI_OK;
    cudaSetDevice(plan->device);
    if (plan->stream) cudaStreamSynchronize(plan->stream);
    for (void *p : plan->allocs) cudaFree(p);
    cocg_destroy(plan->cg);
    band_destroy(plan->band);
    for (auto &e : plan->phase_ev)
        if (e) cudaEventDestroy(e);
    for (auto &r : plan->pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto &g : plan->graph)
        if (g) cudaGraphExecDestroy(g);
    for (int g = 0; g < 2; ++g) {
        if (plan->zc_exec[g]) cudaGraphExecDestroy(plan->zc_exec[g]);
        if (plan->zc_src[g]) cudaGraphDestroy(plan->zc_src[g]);
    }
    for (auto &g : plan->part_graphs) cudaGraphExecDestroy(g.exec);
    for (auto e : plan->pool) cudaEventDestroy(e);
    if (plan->own_stream && plan->stream) cudaStreamDestroy(plan->stream);
    delete plan;
    return REXI_OK;
}

int rexi_plan_create(const rexi_desc *d, rexi_plan **out) {
    *out = nullptr;
    if (!d) return set_err(nullptr, REXI_ERR_INVALID, "null descriptor");
    if (d->abi_version != REXI_ABI_VERSION)
        return set_err(nullptr, REXI_ERR_INVALID, "ABI version mismatch");
    if (d->n < 1) return set_err(nullptr, REXI_ERR_INVALID, "n must be >= 1");
    if (d->k < 1) return set_err(nullptr, REXI_ERR_INVALID, "need at least one shift");
    if (!(d->tau > 0.0)) return set_err(nullptr, REXI_ERR_INVALID, "tau must be positive");
    if (!d->indptr || !d->indices || !d->a_vals || !d->b_vals || !d->shifts || !d->weights)
        return set_err(nullptr, REXI_ERR_INVALID, "null input array");
    rexi_plan *plan = new rexi_plan();
    plan->device = d->device;
    plan->n = d->n;
    plan->k = d->k;
    plan->shift_offset = d->shift_offset;
    plan->gid.resize(d->k);
    for (int j = 0; j < d->k; ++j) plan->gid[j] = d->shift_ids ? d->shift_ids[j] : d->shift_offset + j;
    plan->shifts_host.assign(d->shifts, d->shifts + d->k);
    // structure
    bool tri = true;
    int kl = 0, ku = 0;
    for (int64_t r = 0; r < d->n; ++r)
        for (int32_t q = d->indptr[r]; q < d->indptr[r + 1]; ++q) {
            int64_t c = d->indices[q];
            if (c < 0 || c >= d->n) {
                int rc = set_err(plan, REXI_ERR_INVALID, "column index out of range");
                rexi_plan_destroy(plan);
                return rc;
            }
            kl = std::max<int>(kl, (int)(r - c));
            ku = std::max<int>(ku, (int)(c - r));
        }
    tri = kl <= 1 && ku <= 1;
    plan->bandwidth = kl + ku + 1;
    int solver = d->solver;
    const int hb = std::max(kl, ku);
    const bool banded = hb >= BAND_MIN && hb <= BAND_MAX;
    // tridiagonal -> the partitioned 1D solver; half bandwidth 2..4 (the
    // reference's P2 pencils) -> the partitioned band LU; wider -> COCG
    if (solver == REXI_SOLVER_AUTO) solver = tri ? REXI_SOLVER_TRIDIAG : banded ? REXI_SOLVER_BAND : REXI_SOLVER_COCG;
    if (solver == REXI_SOLVER_BAND && !banded) {
        int rc = set_err(plan, REXI_ERR_UNSUPPORTED, "BAND solver needs a half bandwidth of 2..4");
        rexi_plan_destroy(plan);
        return rc;
    }
    if (solver == REXI_SOLVER_TRIDIAG && !tri) {
        int rc = set_err(plan, REXI_ERR_UNSUPPORTED, "TRIDIAG solver needs a tridiagonal pattern");
        rexi_plan_destroy(plan);
        return rc;
    }
    plan->solver = solver;
    plan->kp = pick_kp(d->k);
    // 1D: at least two lanes -- with one lane a level-0 CTA spans 2048 rows and
    // K2's staged row arrays exceed shared memory (the padding lane has beta = 0)
    if (solver == REXI_SOLVER_TRIDIAG && plan->kp < 2) plan->kp = 2;
    if (solver == REXI_SOLVER_TRIDIAG && plan->kp > 256) {
        int rc = set_err(plan, REXI_ERR_UNSUPPORTED, "TRIDIAG solver supports at most 256 shifts per plan");
        rexi_plan_destroy(plan);
        return rc;
    }
    // auto (-1): the direct 1D solve is refined only on request (the Python layer
    // decides by stiffness); COCG always gets one double-double refinement round
    const bool direct = solver == REXI_SOLVER_TRIDIAG || solver == REXI_SOLVER_BAND;
    if (d->refine < 0) plan->refine = direct ? 0 : 1;
    else plan->refine = std::min(d->refine, direct ? 1 : 4);

    cudaError_t e = cudaSetDevice(d->device);
    if (e != cudaSuccess) {
        int rc = cuda_err(plan, e, "cudaSetDevice");
        rexi_plan_destroy(plan);
        return rc;
    }
    if (d->stream) {
        plan->stream = (cudaStream_t)d->stream;
    } else {
        e = cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            int rc = cuda_err(plan, e, "cudaStreamCreate");
            rexi_plan_destroy(plan);
            return rc;
        }
        plan->own_stream = true;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, plan->stream);
    int rc = REXI_OK;
    {
        // shifts / weights, padded to kp lanes (padding: sigma_0 with beta = 0)
        const int kp = plan->kp;
        std::vector<rexi_c128> sg(kp), bt(kp);
        for (int j = 0; j < kp; ++j) {
            sg[j] = d->shifts[j < d->k ? j : 0];
            bt[j] = j < d->k ? d->weights[j] : rexi_c128{0.0, 0.0};
        }
        c128 *dsg = nullptr, *dbt = nullptr;
        rc = dalloc(plan, &dsg, kp);
        if (!rc) rc = dalloc(plan, &dbt, kp);
        if (!rc) {
            cudaMemcpyAsync(dsg, sg.data(), sizeof(c128) * kp, cudaMemcpyHostToDevice, plan->stream);
            cudaMemcpyAsync(dbt, bt.data(), sizeof(c128) * kp, cudaMemcpyHostToDevice, plan->stream);
            plan->S = ShiftDev{dsg, dbt, kp};
        }
        if (!rc) rc = dalloc(plan, &plan->ubuf[0], (size_t)d->n);
        if (!rc) rc = dalloc(plan, &plan->ubuf[1], (size_t)d->n);
        // the reference's singularity screen: it factors every shifted system
        // with partially pivoted zgbtrf when kl + ku + 1 <= 32 (solvers.py:25,
        // 108-115) and rejects the first shift j whose factor has a zero pivot
        // or min|U_ii| < 1e-14 max|U_ii| (solvers.py:52-69).  Same algorithm on
        // the device (screen.cu), same order, same messages; it runs beside
        // the plan's own factorisation and its verdict takes precedence.
        rexi::ScreenJob screen;
        bool screening = !rc && plan->bandwidth <= 32 && !getenv("REXI_NO_SCREEN");
        if (screening) {
            std::string serr;
            rc = screen.launch(d, kl, ku, plan->S.sigma, plan->stream, serr);
            if (rc) {
                set_err(plan, rc, serr);
                screening = false;
            }
        }
        auto screen_verdict_now = [&]() -> int {
            std::vector<rexi::ScreenResult> scr;
            std::string serr;
            int src = screen.collect(scr, serr);
            if (src) return set_err(plan, src, serr);
            for (int j = 0; j < d->k; ++j) {
                const std::string v = rexi::screen_verdict(scr[j], d->n);
                plan->screen_ratio = std::min(plan->screen_ratio, scr[j].umax > 0 ? scr[j].umin / scr[j].umax : 0.0);
                if (!v.empty())
                    return set_err(plan, REXI_ERR_SINGULAR, v + " [shift j = " + std::to_string(plan->gid[j]) + "]");
            }
            return REXI_OK;
        };
        if (!rc) {
            if (solver == REXI_SOLVER_TRIDIAG) {
                rc = tri_create(plan, d);
                if (!rc) rc = persist_setup(plan);
            } else if (solver == REXI_SOLVER_BAND) {
                rc = dalloc(plan, &plan->tri.acc, (size_t)4 * d->n);
                if (!rc) rc = band_create(plan->band, d, std::max(hb, BAND_MIN), plan->S, plan->kp, plan->refine,
                                          plan->stream, plan->err);
                if (rc) set_err(plan, rc, plan->err);
                else plan->min_pivot_ratio = plan->band.min_pivot_ratio;
            } else {
                rc = dalloc(plan, &plan->tri.acc, (size_t)4 * d->n);
                if (!rc) rc = cocg_create(plan->cg, d, plan->S, plan->refine, plan->stream, plan->err);
                if (rc) set_err(plan, rc, plan->err);
            }
        }
        if (screening) {
            // the screen's verdict first (the reference raises it from its
            // factorisation), then whatever the plan's own creation reported
            const std::string own_err = plan->err;
            const int src = screen_verdict_now();
            if (src) rc = src;
            else if (rc) set_err(plan, rc, own_err);
        }
    }
    if (rc) {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        std::string msg = plan->err;
        rexi_plan_destroy(plan);
        g_last_error = msg;
        return rc;
    }
    cudaEventRecord(e1, plan->stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    plan->prepare_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        int rc2 = cuda_err(plan, e, "prepare");
        std::string msg = plan->err;
        rexi_plan_destroy(plan);
        g_last_error = msg;
        return rc2;
    }
    *out = plan;
    return REXI_OK;
}

int rexi_plan_profile(rexi_plan *plan, int32_t enable) {
    if (!plan) return set_err(nullptr, REXI_ERR_INVALID, "null plan");
    prof_flush(plan);
    plan->prof = enable != 0;
    plan->prof_acc.clear();
    plan->hook.p = plan;
    plan->cg.hook = &plan->hook;
    plan->band.hook = plan->prof ? &plan->hook : nullptr;
    return REXI_OK;
}

int rexi_plan_profile_report(rexi_plan *plan, char *buf, int64_t len) {
    if (!plan || !buf || len <= 0) return set_err(plan, REXI_ERR_INVALID, "bad arguments");
    prof_flush(plan);
    std::string s;
    char line[256];
    for (auto &kv : plan->prof_acc) {
        snprintf(line, sizeof line, "%s %lld %.6f %.0f\n", kv.first.c_str(), (long long)kv.second.count,
                 kv.second.ms, kv.second.bytes);
        s += line;
    }
    if ((int64_t)s.size() + 1 > len) return set_err(plan, REXI_ERR_INVALID, "buffer too small");
    memcpy(buf, s.c_str(), s.size() + 1);
    return REXI_OK;
}

int rexi_plan_info(const rexi_plan *plan, rexi_info *info) {
    if (!plan || !info) return set_err(nullptr, REXI_ERR_INVALID, "null argument");
    info->solver = plan->solver;
    info->bandwidth = plan->bandwidth;
    info->k_pad = plan->kp;
    info->levels = (int32_t)plan->tri.lv.size();
    info->refine = plan->refine;
    info->device_bytes = plan->bytes + plan->cg.bytes + plan->band.bytes;
    info->prepare_ms = plan->prepare_ms;
    info->min_pivot_ratio = plan->min_pivot_ratio;
    info->persistent = plan->persist_cs;
    info->screen_pivot_ratio = plan->screen_ratio;
    return REXI_OK;
}

int rexi_plan_wait_stream(rexi_plan *plan, void *stream) {
    if (!plan) return set_err(nullptr, REXI_ERR_INVALID, "null plan");
    if ((cudaStream_t)stream == plan->stream) return REXI_OK;
    CK(cudaSetDevice(plan->device));
    cudaEvent_t e = nullptr;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaError_t r = cudaEventRecord(e, (cudaStream_t)stream);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(plan->stream, e, 0);
    cudaEventDestroy(e);   // released once the wait is satisfied
    if (r != cudaSuccess) return cuda_err(plan, r, "rexi_plan_wait_stream");
    return REXI_OK;
}

int rexi_plan_shift_iters(const rexi_plan *plan, int32_t *iters) {
    if (!plan || !iters) return set_err(nullptr, REXI_ERR_INVALID, "null argument");
    for (int j = 0; j < plan->k; ++j)
        iters[j] = plan->solver == REXI_SOLVER_COCG && j < (int)plan->cg.shift_iters.size()
                       ? plan->cg.shift_iters[j] : 0;
    return REXI_OK;
}

int rexi_plan_step(rexi_plan *plan, const rexi_c128 *u_in, rexi_c128 *u_out, int32_t n_steps,
                   int32_t mem, rexi_stats *stats) {
    if (!plan) return set_err(nullptr, REXI_ERR_INVALID, "null plan");
    if (n_steps < 0) return set_err(plan, REXI_ERR_INVALID, "n_steps must be >= 0");
    CK(cudaSetDevice(plan->device));
    const int64_t n = plan->n;
    cudaStream_t st = plan->stream;
    plan->launches = 0;
    // phase events: [0] before staging u, [1] after it (rhs), [2] after the
    // steps (local), [3] after copying u1 out (reduce)
    // A one-step call of a direct solver fuses the rhs into its first kernel
    // and the sum into its last: its phases are all "local", timed on the
    // host (four timed events cost ~17 us per call, a third of a cfg-1 step)
    const bool phase_ev = stats && !(n_steps <= 1 && plan->solver != REXI_SOLVER_COCG);
    const auto host_t0 = std::chrono::steady_clock::now();
    cudaEvent_t *ev = plan->phase_ev;
    if (phase_ev) {
        for (int i = 0; i < 4; ++i)
            if (!ev[i]) CK(cudaEventCreate(&ev[i]));
        cocg_collect_phase(plan->cg);
        plan->cg.t_rhs_ms = plan->cg.t_acc_ms = 0.0;
        CK(cudaEventRecord(ev[0], st));
    }
    // zero-copy output: when u_out is page-locked host memory, the last step's
    // final kernel writes u1 straight into it over PCIe (overlapped with the
    // kernel) instead of a separate device-to-host copy afterwards
    auto mapped = [](const void *p) -> c128 * {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
            return (c128 *)pa.devicePointer;
        cudaGetLastError();
        return nullptr;
    };
    c128 *zc_out = nullptr;
    const bool persist = n_steps > 0 && plan->persist_cs > 0 && !plan->prof;
    // (the band solver's step has no re-pointable output node: its last step
    // replays the graph and copies u1 out instead of running its kernels one
    // by one into the mapped buffer)
    const bool zc_ok = mem == REXI_MEM_HOST && n_steps > 0 && plan->solver != REXI_SOLVER_BAND &&
                       !getenv("REXI_NO_ZEROCOPY");
    if (zc_ok) zc_out = mapped(u_out);
    // zero-copy input: a one-step host call of a TMA-path 1D plan reads u from
    // page-locked host memory inside the level-0 S1 kernel (which forms rhs =
    // iBu itself), so the host->device transfer overlaps that kernel's HBM
    // traffic instead of preceding it
    const c128 *zc_in = nullptr;
    if (zc_ok && zc_out && (persist || (n_steps == 1 && plan->solver == REXI_SOLVER_TRIDIAG &&
                                        l0v2_supported(plan->kp))))
        zc_in = mapped(u_in);
    // the persistent loop reads its input once and writes its last state
    // once: both straight over the link when the host buffers are page-locked
    if (persist && !zc_in) zc_out = nullptr;
    const c128 *src;
    if (zc_in) {
        src = zc_in;
    } else if (mem == REXI_MEM_HOST) {
        CK(cudaMemcpyAsync(plan->ubuf[0], u_in, sizeof(c128) * n, cudaMemcpyHostToDevice, st));
        src = plan->ubuf[0];
    } else {
        src = (const c128 *)u_in;
    }
    if (phase_ev) CK(cudaEventRecord(ev[1], st));
    int cur = (src == plan->ubuf[0]) ? 0 : 1;
    if (n_steps > 0 && plan->persist_cs > 0 && !plan->prof) {
        TriState &T = plan->tri;
        CK(persist_launch(T.z, T.lv.data(), (int)T.lv.size(), plan->S, n, src, plan->pbuf[0], plan->pbuf[1],
                          nullptr, n_steps, plan->persist_cs, st, zc_out));
        plan->launches += 1;
        src = plan->pbuf[(n_steps - 1) & 1];
        n_steps = -n_steps;    // steps done; restored below
    } else if (n_steps > 0 && (plan->solver == REXI_SOLVER_TRIDIAG || plan->solver == REXI_SOLVER_BAND) &&
               !plan->prof) {
        // a direct step is a fixed kernel sequence: replay it as a CUDA graph
        // (two graphs, ping-ponging between the plan's state buffers)
        if (src != plan->ubuf[0] && src != plan->ubuf[1] && !zc_in) {
            CK(cudaMemcpyAsync(plan->ubuf[0], src, sizeof(c128) * n, cudaMemcpyDeviceToDevice, st));
            cur = 0;
        }
        for (int g = 0; g < 2; ++g) {
            if (plan->graph[g]) continue;
            cudaGraph_t graph = nullptr;
            const int64_t l0 = plan->launches;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            int rc = plan_step_device(plan, plan->ubuf[g], plan->ubuf[g ^ 1]);
            cudaError_t ce = cudaStreamEndCapture(st, &graph);
            if (rc) return rc;
            if (ce != cudaSuccess) return cuda_err(plan, ce, "cudaStreamEndCapture");
            CK(cudaGraphInstantiate(&plan->graph[g], graph, 0));
            // a second instance whose S1 / output kernels get re-pointed per
            // host call (the source graph stays alive for the node handles)
            size_t nn = 0;
            CK(cudaGraphGetNodes(graph, nullptr, &nn));
            std::vector<cudaGraphNode_t> nodes(nn);
            CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
            for (cudaGraphNode_t nd : nodes) {
                const int role = l0_graph_role(nd);
                if (role == 1) plan->zc_in_node[g] = nd;
                if (role == 2) plan->zc_out_node[g] = nd;
            }
            if (plan->zc_in_node[g] && plan->zc_out_node[g]) {
                CK(cudaGraphInstantiate(&plan->zc_exec[g], graph, 0));
                plan->zc_src[g] = graph;
            } else {
                cudaGraphDestroy(graph);
            }
            plan->graph_kernels = plan->launches - l0;
            plan->launches = l0;
        }
        const int graph_steps = zc_out ? n_steps - 1 : n_steps;
        for (int s = 0; s < graph_steps; ++s) {
            CK(cudaGraphLaunch(plan->graph[cur], st));
            plan->launches += plan->graph_kernels;
            cur ^= 1;
        }
        if (!(zc_in && graph_steps == 0)) src = plan->ubuf[cur];
        if (zc_out && plan->zc_exec[cur] && !getenv("REXI_NO_ZC_GRAPH")) {
            // last step straight into the page-locked output: the captured
            // step with its S1 (input) and output kernels re-pointed
            CK(l0_graph_patch(plan->zc_exec[cur], plan->zc_in_node[cur], 1, src, nullptr));
            CK(l0_graph_patch(plan->zc_exec[cur], plan->zc_out_node[cur], 2, nullptr, zc_out));
            CK(cudaGraphLaunch(plan->zc_exec[cur], st));
            plan->launches += plan->graph_kernels;
        } else if (zc_out) {   // last step straight into the page-locked output
            int rc = plan_step_device(plan, src, zc_out);
            if (rc) return rc;
        }
        n_steps = -n_steps;    // steps done; restored below
    }
    for (int s = 0; s < n_steps; ++s) {
        c128 *dst;
        bool last = s == n_steps - 1;
        if (last && mem == REXI_MEM_DEVICE) dst = (c128 *)u_out;
        else if (last && zc_out) dst = zc_out;
        else dst = plan->ubuf[src == plan->ubuf[0] ? 1 : 0];
        if (dst == src) dst = plan->ubuf[cur ^ 1];   // in-place device call
        int rc = plan_step_device(plan, src, dst);
        if (rc) {
            if (rc == REXI_ERR_NOCONV || rc == REXI_ERR_BREAKDOWN) return set_err(plan, rc, plan->err);
            return rc;
        }
        src = dst;
        cur = (src == plan->ubuf[0]) ? 0 : 1;
    }
    if (n_steps < 0) n_steps = -n_steps;
    if (phase_ev) CK(cudaEventRecord(ev[2], st));
    if (n_steps == 0) {
        if (mem == REXI_MEM_HOST) {
            if (u_out != u_in) memcpy(u_out, u_in, sizeof(c128) * n);
        } else if (u_out != u_in) {
            CK(cudaMemcpyAsync(u_out, u_in, sizeof(c128) * n, cudaMemcpyDeviceToDevice, st));
        }
    } else if (mem == REXI_MEM_HOST) {
        if (!zc_out) CK(cudaMemcpyAsync(u_out, src, sizeof(c128) * n, cudaMemcpyDeviceToHost, st));
    } else if ((const void *)src != (const void *)u_out) {
        CK(cudaMemcpyAsync(u_out, src, sizeof(c128) * n, cudaMemcpyDeviceToDevice, st));
    }
    if (phase_ev) CK(cudaEventRecord(ev[3], st));
    CK(cudaStreamSynchronize(st));
    prof_flush(plan);
    if (stats) {
        if (phase_ev) {
            fill_phases(plan, ev, stats);
        } else {
            stats->t_rhs_ms = stats->t_reduce_ms = 0.0;
            stats->t_local_ms =
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
        }
        stats->steps = n_steps;
        stats->launches = plan->launches;
        stats->iters_max = plan->cg.last_iters_max;
        stats->iters_mean = plan->cg.last_iters_mean;
        stats->refine_rounds = plan->refine;
        stats->bad_shift = -1;
    }
    return REXI_OK;
}

int rexi_plan_run(rexi_plan *plan, const rexi_c128 *u_in, rexi_c128 *snaps, int32_t n_steps, int32_t mem,
                  rexi_stats *stats) {
    if (!plan) return set_err(nullptr, REXI_ERR_INVALID, "null plan");
    if (!u_in || !snaps) return set_err(plan, REXI_ERR_INVALID, "null argument");
    if (n_steps < 0) return set_err(plan, REXI_ERR_INVALID, "n_steps must be >= 0");
    if (n_steps == 0) return REXI_OK;
    CK(cudaSetDevice(plan->device));
    const int64_t n = plan->n;
    cudaStream_t st = plan->stream;
    plan->launches = 0;
    cudaEvent_t *ev = plan->phase_ev;
    for (int i = 0; i < 4; ++i)
        if (!ev[i]) CK(cudaEventCreate(&ev[i]));
    cocg_collect_phase(plan->cg);
    plan->cg.t_rhs_ms = plan->cg.t_acc_ms = 0.0;
    CK(cudaEventRecord(ev[0], st));
    c128 *dsnap = (c128 *)snaps, *tmp = nullptr;
    if (mem == REXI_MEM_HOST) {
        CK(cudaMallocAsync((void **)&tmp, sizeof(c128) * n * (size_t)n_steps, st));
        CK(rexi_poison(tmp, sizeof(c128) * n * (size_t)n_steps, st));
        dsnap = tmp;
    }
    const c128 *src = (const c128 *)u_in;
    if (mem == REXI_MEM_HOST) {
        CK(cudaMemcpyAsync(plan->ubuf[0], u_in, sizeof(c128) * n, cudaMemcpyHostToDevice, st));
        src = plan->ubuf[0];
    }
    CK(cudaEventRecord(ev[1], st));
    int rc = REXI_OK;
    if (plan->persist_cs > 0 && !plan->prof) {
        TriState &T = plan->tri;
        CK(persist_launch(T.z, T.lv.data(), (int)T.lv.size(), plan->S, n, src, plan->pbuf[0], plan->pbuf[1], dsnap,
                          n_steps, plan->persist_cs, st));
        plan->launches += 1;
    } else {
        for (int s = 0; s < n_steps && !rc; ++s)
            rc = plan_step_device(plan, s == 0 ? src : dsnap + (size_t)(s - 1) * n, dsnap + (size_t)s * n);
    }
    CK(cudaEventRecord(ev[2], st));
    if (!rc && mem == REXI_MEM_HOST)
        CK(cudaMemcpyAsync(snaps, dsnap, sizeof(c128) * n * (size_t)n_steps, cudaMemcpyDeviceToHost, st));
    if (tmp) cudaFreeAsync(tmp, st);
    CK(cudaEventRecord(ev[3], st));
    CK(cudaStreamSynchronize(st));
    prof_flush(plan);
    rexi_stats local_stats{};
    fill_phases(plan, ev, &local_stats);
    if (rc) {
        if (rc == REXI_ERR_NOCONV || rc == REXI_ERR_BREAKDOWN) return set_err(plan, rc, plan->err);
        return rc;
    }
    if (stats) {
        *stats = local_stats;
        stats->steps = n_steps;
        stats->launches = plan->launches;
        stats->iters_max = plan->cg.last_iters_max;
        stats->iters_mean = plan->cg.last_iters_mean;
        stats->refine_rounds = plan->refine;
        stats->bad_shift = -1;
    }
    return REXI_OK;
}

int rexi_plan_step_partial(rexi_plan *plan, const rexi_c128 *u_in, double *partial,
                           rexi_stats *stats) {
    if (!plan) return set_err(nullptr, REXI_ERR_INVALID, "null plan");
    CK(cudaSetDevice(plan->device));
    plan->launches = 0;
    // the step accumulates its double-double partial straight into the
    // caller's buffer (same SoA layout as the plan's accumulator)
    double *const acc_saved = plan->tri.acc;
    plan->tri.acc = partial;
    int rc = REXI_OK;
    if (plan->solver == REXI_SOLVER_TRIDIAG && !plan->prof && !getenv("REXI_NO_GRAPH")) {
        // the 1D step is a fixed kernel sequence: capture it once per
        // (u_in, partial) pair and replay (a sharded run alternates two)
        cudaStream_t st = plan->stream;
        auto it = std::find_if(plan->part_graphs.begin(), plan->part_graphs.end(),
                               [&](const rexi_plan::PartGraph &g) { return g.u == u_in && g.part == partial; });
        if (it == plan->part_graphs.end()) {
            if (plan->part_graphs.size() >= 4) {
                cudaGraphExecDestroy(plan->part_graphs.front().exec);
                plan->part_graphs.erase(plan->part_graphs.begin());
            }
            cudaGraph_t graph = nullptr;
            const int64_t l0 = plan->launches;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            rc = tri_step(plan, (const c128 *)u_in, nullptr);
            cudaError_t ce = cudaStreamEndCapture(st, &graph);
            if (rc) {
                plan->tri.acc = acc_saved;
                if (graph) cudaGraphDestroy(graph);
                return rc;
            }
            if (ce != cudaSuccess) {
                plan->tri.acc = acc_saved;
                return cuda_err(plan, ce, "cudaStreamEndCapture");
            }
            rexi_plan::PartGraph g{u_in, partial, nullptr, plan->launches - l0};
            cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ie != cudaSuccess) {
                plan->tri.acc = acc_saved;
                return cuda_err(plan, ie, "cudaGraphInstantiate");
            }
            plan->launches = l0;
            plan->part_graphs.push_back(g);
            it = plan->part_graphs.end() - 1;
        }
        const cudaError_t le = cudaGraphLaunch(it->exec, st);
        plan->launches += it->kernels;
        plan->tri.acc = acc_saved;
        if (le != cudaSuccess) return cuda_err(plan, le, "cudaGraphLaunch");
    } else {
        rc = plan_step_device(plan, (const c128 *)u_in, nullptr);
        plan->tri.acc = acc_saved;
    }
    if (rc) return rc == REXI_ERR_NOCONV || rc == REXI_ERR_BREAKDOWN ? set_err(plan, rc, plan->err) : rc;
    // stream-ordered on a caller's stream (1D: nothing to check on the host;
    // COCG has synchronised for its convergence checks already)
    if (plan->own_stream || plan->prof || plan->solver != REXI_SOLVER_TRIDIAG) CK(cudaStreamSynchronize(plan->stream));
    else CK(cudaGetLastError());
    prof_flush(plan);
    if (stats) {
        memset(stats, 0, sizeof *stats);
        cocg_collect_phase(plan->cg);
        stats->t_rhs_ms = plan->cg.t_rhs_ms;
        stats->t_reduce_ms = plan->cg.t_acc_ms;
        plan->cg.t_rhs_ms = plan->cg.t_acc_ms = 0.0;
        stats->steps = 1;
        stats->launches = plan->launches;
        stats->iters_max = plan->cg.last_iters_max;
        stats->iters_mean = plan->cg.last_iters_mean;
        stats->refine_rounds = plan->refine;
        stats->bad_shift = -1;
    }
    return REXI_OK;
}

int rexi_combine_partials(const double *partials, int32_t g, int64_t n, rexi_c128 *out, void *stream) {
    rexi_plan *plan = nullptr;
    CK(launch_combine(partials, g, n, (c128 *)out, (cudaStream_t)stream));
    if (!stream) CK(cudaStreamSynchronize((cudaStream_t)stream));
    return REXI_OK;
}

int rexi_plan_solve(rexi_plan *plan, const rexi_c128 *rhs, rexi_c128 *x, int32_t mem) {
    if (!plan) return set_err(nullptr, REXI_ERR_INVALID, "null plan");
    CK(cudaSetDevice(plan->device));
    const int64_t n = plan->n;
    cudaStream_t st = plan->stream;
    c128 *xd = nullptr;
    c128 *tmp = nullptr;
    if (mem == REXI_MEM_HOST) {
        CK(cudaMallocAsync((void **)&tmp, sizeof(c128) * n * plan->k, st));
        xd = tmp;
    } else {
        xd = (c128 *)x;
    }
    if (plan->solver == REXI_SOLVER_TRIDIAG) {
        TriState &T = plan->tri;
        CK(cudaMemcpyAsync(T.rhs0, rhs, sizeof(c128) * n,
                           mem == REXI_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
        int rc = tri_chain(plan, nullptr, TRI_OUT_X, 0, nullptr);
        if (rc) return rc;
        if (plan->refine > 0) {
            // refine the per-shift solutions: x += S^-1 (rhs - S x); keep x_hi only
            CK(tri_launch_residual(T.z, T.lv[0], plan->S, T.rhs0, T.rres, st));
            c128 *x0 = nullptr;
            CK(cudaMallocAsync((void **)&x0, sizeof(c128) * n * plan->kp, st));
            CK(cudaMemcpyAsync(x0, T.lv[0].X, sizeof(c128) * n * plan->kp, cudaMemcpyDeviceToDevice, st));
            rc = tri_chain(plan, T.rres, TRI_OUT_X, 0, nullptr);
            if (rc) return rc;
            CK(cocg_axpy_inplace(T.lv[0].X, x0, (int64_t)n * plan->kp, st));
            CK(cudaFreeAsync(x0, st));
        }
        CK(tri_launch_transpose(T.lv[0].X, n, plan->kp, plan->k, xd, st));
    } else if (plan->solver == REXI_SOLVER_BAND) {
        c128 *rd = (c128 *)rhs;
        if (mem == REXI_MEM_HOST) {
            CK(cudaMemcpyAsync(plan->ubuf[0], rhs, sizeof(c128) * n, cudaMemcpyHostToDevice, st));
            rd = plan->ubuf[0];
        }
        int rc = band_solve_all(plan->band, plan->S, st, rd, xd, plan->err);
        if (rc) return set_err(plan, rc, plan->err);
    } else {
        int rc = cocg_solve_all(plan->cg, plan->S, st, (const c128 *)rhs, mem == REXI_MEM_HOST, xd, plan->err);
        if (rc) return set_err(plan, rc, plan->err);
    }
    if (mem == REXI_MEM_HOST) {
        CK(cudaMemcpyAsync(x, xd, sizeof(c128) * n * plan->k, cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(tmp, st));
    }
    CK(cudaStreamSynchronize(st));
    return REXI_OK;
}

}  // extern "C"
