// common.cuh -- shared device helpers for the specsense-b200 kernels (sm_100a).
//
// Bit-exact arithmetic: every floating-point expression on the parity path is
// written with explicit-rounding intrinsics (__dadd_rn / __dmul_rn / __fma_rn,
// __fadd_rn / __fmul_rn / __fdiv_rn) so nvcc's default FMA contraction cannot
// change the rounding sequence the reference's GCC build performs
// (DESIGN.md §5 lists the contracted sites of the reference build).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ssb {

struct cd {
    double re, im;
};

__device__ __forceinline__ cd c_add(cd a, cd b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }
__device__ __forceinline__ cd c_sub(cd a, cd b) { return {__dsub_rn(a.re, b.re), __dsub_rn(a.im, b.im)}; }
// SSFFT-1 complex multiply: (fma(a.re, w.re, -(a.im*w.im)), fma(a.re, w.im, a.im*w.re))
__device__ __forceinline__ cd c_mul(cd a, cd w) {
    const double t1 = __dmul_rn(a.im, w.im);
    const double t2 = __dmul_rn(a.im, w.re);
    return {__fma_rn(a.re, w.re, -t1), __fma_rn(a.re, w.im, t2)};
}
// a * (-i)
__device__ __forceinline__ cd c_mi(cd a) { return {a.im, -a.re}; }

constexpr double kR2 = 0x1.6a09e667f3bcdp-1; // sqrt(2)/2
constexpr double kC1 = 0x1.d906bcf328d46p-1; // cos(pi/8)
constexpr double kS1 = 0x1.87de2a6aea963p-2; // sin(pi/8)

// a * W8 = a * (1 - i)/sqrt2
__device__ __forceinline__ cd c_w8(cd a) {
    return {__dmul_rn(__dadd_rn(a.re, a.im), kR2), __dmul_rn(__dsub_rn(a.im, a.re), kR2)};
}
// a * W8^3 = a * (-1 - i)/sqrt2
__device__ __forceinline__ cd c_w83(cd a) {
    return {__dmul_rn(__dsub_rn(a.im, a.re), kR2), -__dmul_rn(__dadd_rn(a.re, a.im), kR2)};
}

// ---------------------------------------------------------------- PTX wrappers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// TMA 1-D bulk copy global -> shared, completion counted on `bar` (bytes).
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------ misc helpers

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Inclusive warp scan.
__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

} // namespace ssb
