// lx_common.cuh -- shared device helpers for the B200 LAPLEX kernels (sm_100a).
//
// Precision policy: every floating-point operation that feeds an output is
// written with an explicit-rounding intrinsic (__fmaf_rn, __fmul_rn, ...), so
// ptxas never re-contracts it.  That pins three bitwise contracts of the
// reference: batch row r == single-row matvec (tests/test_operator.cpp:120-132),
// op(a,b,t) == op(a/t,b/t,1) (tests/test_operator.cpp:98-108), and the x_bar of
// matvec_vjp == matvec_transpose.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lx {

constexpr unsigned FULL = 0xffffffffu;

template <class R>
struct Traits;

template <>
struct Traits<float> {
    using Key = uint32_t;
    static constexpr int kPasses = 4;  // 8-bit digits
    static constexpr Key kSign = 0x80000000u;
};

template <>
struct Traits<double> {
    using Key = unsigned long long;
    static constexpr int kPasses = 8;
    static constexpr Key kSign = 0x8000000000000000ull;
};

// exp for the scan/carry exponents (all arguments are anchor differences <= 0):
// ex2.approx on x*log2(e).  Relative error ~2^-22 + |x|*2^-24, i.e. < 1e-6 on
// every term that is not already below 1e-8 of the diagonal; fp64 uses exp().
__device__ __forceinline__ float xexp(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(x, 1.4426950408889634f)));
    return y;
}
__device__ __forceinline__ double xexp(double x) { return exp(x); }
__device__ __forceinline__ float xfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double xfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float xdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float xcos(float a) { return cosf(a); }
__device__ __forceinline__ double xcos(double a) { return cos(a); }
__device__ __forceinline__ float xsin(float a) { return sinf(a); }
__device__ __forceinline__ double xsin(double a) { return sin(a); }

__device__ __forceinline__ uint32_t as_bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ unsigned long long as_bits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ float from_bits(uint32_t b, float) { return __uint_as_float(b); }
__device__ __forceinline__ double from_bits(unsigned long long b, double) {
    return __longlong_as_double((long long)b);
}

// Order-preserving radix key of an IEEE value.  -0 is canonicalised to +0 so
// that the two zeros compare equal (std::stable_sort with operator<, reference
// scan.hpp:36-37) and keep input order; the sign of the zero is carried in the
// index payload's top bit and restored when the sorted values are written.
template <class R>
__device__ __forceinline__ typename Traits<R>::Key radix_key(R v) {
    using K = typename Traits<R>::Key;
    K b = as_bits(v);
    if (b == Traits<R>::kSign) b = 0;
    return (b & Traits<R>::kSign) ? ~b : (b | Traits<R>::kSign);
}

template <class R>
__device__ __forceinline__ R radix_value(typename Traits<R>::Key k, bool neg_zero) {
    using K = typename Traits<R>::Key;
    K b = (k & Traits<R>::kSign) ? (k & ~Traits<R>::kSign) : ~k;
    if (neg_zero) b = Traits<R>::kSign;
    return from_bits(b, R(0));
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- Blackwell async-copy helpers (TMA bulk copy + mbarrier, cp.async) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait with a hardware suspend hint: the waiting warp is descheduled until the
// phase completes (or the hint expires) instead of polling, so a lane that
// only waits (the main pass's producer) takes no issue slots from compute warps
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// 1-D TMA bulk copy global -> shared (16-byte aligned, size % 16 == 0), completes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// order this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) accesses of the same bytes (buffer refills)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// element-wise async gather global -> shared (LDGSTS)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) {
    return __shfl_up_sync(FULL, v, d);
}
template <class T>
__device__ __forceinline__ T shfl_down(T v, int d) {
    return __shfl_down_sync(FULL, v, d);
}

}  // namespace lx
