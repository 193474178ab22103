// common.cuh -- complex128 / double-double device helpers for the REXI path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

typedef double2 c128;   // (x = re, y = im), layout-compatible with numpy complex128

// REXI_POISON=1 (test hygiene, tests/test_gpu_hygiene.py): every device
// allocation is filled with 0xFF bytes (NaN doubles, -1 integers) before use,
// so a kernel that reads memory nothing wrote first changes the results
// instead of silently reading the zeros a fresh allocation usually holds
// (the stand-in for compute-sanitizer initcheck, closed on this pool).
#include <cstdlib>
inline cudaError_t rexi_poison(void *p, size_t bytes, cudaStream_t st = 0) {
    static const bool on = std::getenv("REXI_POISON") != nullptr;
    if (!on || !p || !bytes) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(p, 0xFF, bytes, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
}

__device__ __forceinline__ c128 cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ c128 cadd(c128 a, c128 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ c128 csub(c128 a, c128 b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ c128 cneg(c128 a) { return cmk(-a.x, -a.y); }
__device__ __forceinline__ c128 cmul(c128 a, c128 b) {
    return cmk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a - b*c
__device__ __forceinline__ c128 cfnma(c128 a, c128 b, c128 c) {
    return cmk(fma(-b.x, c.x, fma(b.y, c.y, a.x)), fma(-b.x, c.y, fma(-b.y, c.x, a.y)));
}
__device__ __forceinline__ c128 crcp(c128 d) {
    double den = fma(d.x, d.x, d.y * d.y);
    double r = 1.0 / den;
    return cmk(d.x * r, -d.y * r);
}
__device__ __forceinline__ double cabs2(c128 a) { return fma(a.x, a.x, a.y * a.y); }

// complex64 helpers (the level-0 correction solve of the refined 1D step)
typedef float2 c64;
__device__ __forceinline__ c64 c64mk(float r, float i) { return make_float2(r, i); }
__device__ __forceinline__ c64 to_c64(c128 a) { return make_float2(__double2float_rn(a.x), __double2float_rn(a.y)); }
__device__ __forceinline__ c128 to_c128(c64 a) { return make_double2((double)a.x, (double)a.y); }
__device__ __forceinline__ c64 fmul(c64 a, c64 b) {
    return c64mk(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a - b*c
__device__ __forceinline__ c64 ffnma(c64 a, c64 b, c64 c) {
    return c64mk(fmaf(-b.x, c.x, fmaf(b.y, c.y, a.x)), fmaf(-b.x, c.y, fmaf(-b.y, c.x, a.y)));
}

// Shifted-operator entry with the reference's rounding (integrate.py:171):
// tau*A - (1j*sigma)*B  ->  re = fl(fl(tau*a) + fl(Im(sigma)*b)),  im = -fl(Re(sigma)*b)
// ta = fl(tau*a) is precomputed on the host side of the plan; no FMA contraction here.
__device__ __forceinline__ c128 form_entry(double ta, double ta_im, double b, c128 s) {
    double re = __dadd_rn(ta, __dmul_rn(s.y, b));
    double im = __dsub_rn(ta_im, __dmul_rn(s.x, b));
    return cmk(re, im);
}

// ---- double-double (error-free transforms) ----
struct dd { double hi, lo; };
__device__ __forceinline__ dd two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {   // |a| >= |b|
    double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = fast_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
    dd s = two_sum(a.hi, b);
    s.lo = __dadd_rn(s.lo, a.lo);
    return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }

// complex double-double accumulator
struct cdd { dd re, im; };
__device__ __forceinline__ cdd cdd_zero() { return {{0.0, 0.0}, {0.0, 0.0}}; }
// acc += w * x with the complex product formed exactly (4 two_prods)
__device__ __forceinline__ cdd cdd_fma(cdd acc, c128 w, c128 x) {
    dd p1 = two_prod(w.x, x.x), p2 = two_prod(-w.y, x.y);
    dd p3 = two_prod(w.x, x.y), p4 = two_prod(w.y, x.x);
    acc.re = dd_add(acc.re, dd_add(p1, p2));
    acc.im = dd_add(acc.im, dd_add(p3, p4));
    return acc;
}
__device__ __forceinline__ cdd cdd_add(cdd a, cdd b) {
    return {dd_add(a.re, b.re), dd_add(a.im, b.im)};
}
// a complex double-double stored as (fp64 hi, fp32 lo): 24 instead of 32 B.
// The refined 1D step keeps the correction's interface halves in it: they
// only need to cancel to ~1e-13 of hi and then be accurate to ~1e-5.  The
// pair is renormalised first (the accumulators' low words also carry whole
// small products), so rounding lo to fp32 costs ~2^-77 of |hi|.
struct cdh { double hr, hi; float lr, li; };
__device__ __forceinline__ cdh cdh_pack(cdd a) {
    const dd r = two_sum(a.re.hi, a.re.lo), i = two_sum(a.im.hi, a.im.lo);
    return {r.hi, i.hi, __double2float_rn(r.lo), __double2float_rn(i.lo)};
}
__device__ __forceinline__ cdd cdh_unpack(cdh h) { return {{h.hr, (double)h.lr}, {h.hi, (double)h.li}}; }
__device__ __forceinline__ c128 cdd_round(cdd a) {
    return cmk(__dadd_rn(a.re.hi, a.re.lo), __dadd_rn(a.im.hi, a.im.lo));
}
// r -= e*x exactly (e, x complex doubles) into a complex dd accumulator
__device__ __forceinline__ cdd cdd_sub_prod(cdd acc, c128 e, c128 x) {
    dd p1 = two_prod(e.x, x.x), p2 = two_prod(-e.y, x.y);
    dd p3 = two_prod(e.x, x.y), p4 = two_prod(e.y, x.x);
    acc.re = dd_add(acc.re, dd_neg(dd_add(p1, p2)));
    acc.im = dd_add(acc.im, dd_neg(dd_add(p3, p4)));
    return acc;
}

#define REXI_CUDA_CHECK(expr)                                                     \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return rexi_fail_cuda(plan_for_err, _e, #expr, __FILE__, __LINE__); \
    } while (0)

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers (sm_90+/sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy, completion signalled on bar (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// global -> L2 bulk prefetch (no completion tracking; bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 16-byte global -> shared copy that does not block the issuing thread
// (cp.async, completion by cp_async_wait_all + a barrier): a staging loop
// keeps all its copies in flight instead of one load round trip each
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// ---- sloppy double-double accumulation of fp64 terms (error-free TwoSum) ----
struct ddacc { double hi, lo; };
__device__ __forceinline__ void ddacc_add(ddacc &s, double t) {
    dd r = two_sum(s.hi, t);
    s.hi = r.hi;
    s.lo = __dadd_rn(s.lo, r.lo);
}
