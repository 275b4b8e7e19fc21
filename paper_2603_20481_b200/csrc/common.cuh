// common.cuh -- shared device helpers for the specsense-b200 kernels (sm_100a).
//
// Bit-exact arithmetic: every floating-point expression on the parity path is
// written with explicit-rounding intrinsics (__dadd_rn / __dmul_rn / __fma_rn,
// __fadd_rn / __fmul_rn / __fdiv_rn) so nvcc's default FMA contraction cannot
// change the rounding sequence the reference's GCC build performs
// (DESIGN.md §5 lists the contracted sites of the reference build).
#pragma once

#include <atomic>
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

// ---------------------------------------------------------------- TMEM
// Tensor memory as plain per-thread storage: 128 lanes x 512 columns of 32 bit
// per SM.  Warp w of a CTA reaches lanes 32*(w%4) .. +31 only; with the
// 32x32b shape lane i of the warp moves TMEM lane (base + i), .x32 = 32
// consecutive columns into 32 registers.  Address = (lane << 16) | column.

// One warp allocates NCOLS columns (power of two >= 32) and writes the base
// address to *slot; the caller then fences + barriers before anyone reads it.
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 consecutive 32-bit columns of this thread's lane <-> r[0..31]
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// Kernel attributes (e.g. the dynamic shared-memory limit) belong to the
// function's instance on one device: set once per device and function.  `done`
// holds one bit per device ordinal; races only repeat the (idempotent) call.
template <class F>
inline cudaError_t set_attr_once(std::atomic<unsigned long long>& done, F&& set) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = set();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
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
