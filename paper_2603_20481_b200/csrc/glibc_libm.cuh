// glibc_libm.cuh -- device restatement of glibc 2.39's x86_64 log10f and
// powf(10, y), the libm calls that define the reference's floor stage
// (proj/src/detector.cpp:217 `10.0f*std::log10(float)`, :222
// `std::pow(10.0f, float)`).  Third-party dependency: glibc 2.39
// (Ubuntu 2.39-0ubuntu8.5), sysdeps/ieee754/flt-32/{e_log10f,e_logf,e_powf}.c
// with the x86_64 FMA ifunc variants (e_logf-fma.c, e_powf-fma.c) that glibc
// selects on FMA+AVX2 hosts -- the GPU box's Xeon and this image's.  A non-FMA
// host would select the SSE2 builds; kSse2 variants are kept for that case and
// chosen at ss_open() from CPUID exactly as glibc's ifunc resolver does.
//
// Table / polynomial constants: this image's libm.so.6 .rodata (__logf_data,
// __powf_log2_data, __exp2f_data).  Every operation uses an explicit-rounding
// intrinsic so nvcc cannot re-contract it.  Verified bit-exact against the live
// glibc on the GPU over strided sweeps of all 2^32 inputs
// (tests/test_gpu_libm.py); the CPU restatement oracle/libm_port.c matches
// glibc on the full 2^32 sweep (tools/libm_exhaustive.c).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ssb {

__constant__ double c_logf_tab[16][2] = {
    {0x1.661ec79f8f3bep+0, -0x1.57bf7808caadep-2}, {0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2},
    {0x1.49539f0f010bp+0, -0x1.01eae7f513a67p-2},  {0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3},
    {0x1.30d190c8864a5p+0, -0x1.6574f0ac07758p-3}, {0x1.25e227b0b8eap+0, -0x1.1aa2bc79c81p-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.a4e76ce8c0e5ep-4}, {0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4},
    {0x1.0953f419900a7p+0, -0x1.252f438e10c1ep-5}, {0x1p+0, 0x0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.aa5aa5df25984p-5},  {0x1.ca4b31f026aap-1, 0x1.c5e53aa362eb4p-4},
    {0x1.b2036576afce6p-1, 0x1.526e57720db08p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.bc2860d22477p-3},
    {0x1.886e6037841edp-1, 0x1.1058bc8a07ee1p-2},  {0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2},
};

__constant__ double c_powf_tab[16][2] = {
    {0x1.661ec79f8f3bep+0, -0x1.efec65b963019p-2}, {0x1.571ed4aaf883dp+0, -0x1.b0b6832d4fca4p-2},
    {0x1.49539f0f010bp+0, -0x1.7418b0a1fb77bp-2},  {0x1.3c995b0b80385p+0, -0x1.39de91a6dcf7bp-2},
    {0x1.30d190c8864a5p+0, -0x1.01d9bf3f2b631p-2}, {0x1.25e227b0b8eap+0, -0x1.97c1d1b3b7afp-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.2f9e393af3c9fp-3}, {0x1.12358f08ae5bap+0, -0x1.960cbbf788d5cp-4},
    {0x1.0953f419900a7p+0, -0x1.a6f9db6475fcep-5}, {0x1p+0, 0x0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.338ca9f24f53dp-4},  {0x1.ca4b31f026aap-1, 0x1.476a9543891bap-3},
    {0x1.b2036576afce6p-1, 0x1.e840b4ac4e4d2p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.40645f0c6651cp-2},
    {0x1.886e6037841edp-1, 0x1.88e9c2c1b9ff8p-2},  {0x1.767dcf5534862p-1, 0x1.ce0a44eb17bccp-2},
};

__constant__ unsigned long long c_exp2f_tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

// logf(x) for the operands log10f passes (positive finite, normalised by the caller).
__device__ __forceinline__ float glibc_logf(float x, bool fma_variant) {
    constexpr double kLn2 = 0x1.62e42fefa39efp-1;
    constexpr double A0 = -0x1.00ea348b88334p-2, A1 = 0x1.5575b0be00b6ap-2, A2 = -0x1.ffffef20a4123p-2;
    uint32_t ix = __float_as_uint(x);
    if (ix == 0x3f800000u) return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        if (ix * 2 == 0) return -__int_as_float(0x7f800000);
        if (ix == 0x7f800000u) return x;
        if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u) return __int_as_float(0x7fc00000);
        ix = __float_as_uint(__fmul_rn(x, 0x1p23f));
        ix -= 23u << 23;
    }
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = static_cast<int>((tmp >> 19) & 15u);
    const int k = static_cast<int32_t>(tmp) >> 23;
    const uint32_t iz = ix - (tmp & 0xff800000u);
    const double invc = c_logf_tab[i][0], logc = c_logf_tab[i][1];
    const double z = static_cast<double>(__uint_as_float(iz));
    double out;
    if (fma_variant) {
        const double r = __fma_rn(z, invc, -1.0);
        const double y0 = __fma_rn(static_cast<double>(k), kLn2, logc);
        const double r2 = __dmul_rn(r, r);
        double y = __fma_rn(r, A1, A2);
        y = __fma_rn(r2, A0, y);
        out = __fma_rn(r2, y, __dadd_rn(r, y0));
    } else {
        const double r = __dsub_rn(__dmul_rn(z, invc), 1.0);
        const double y0 = __dadd_rn(logc, __dmul_rn(static_cast<double>(k), kLn2));
        const double r2 = __dmul_rn(r, r);
        double y = __dadd_rn(__dmul_rn(A1, r), A2);
        y = __dadd_rn(__dmul_rn(A0, r2), y);
        out = __dadd_rn(__dmul_rn(y, r2), __dadd_rn(y0, r));
    }
    return __double2float_rn(out);
}

// e_log10f.c: float composition over logf (no fused operations).
__device__ __forceinline__ float glibc_log10f(float x, bool fma_variant) {
    const float two25 = 3.3554432000e+07f;
    const float ivln10 = __uint_as_float(0x3ede5bd9u);
    const float log10_2hi = __uint_as_float(0x3e9a2080u);
    const float log10_2lo = __uint_as_float(0x355427dbu);
    int32_t hx = __float_as_int(x);
    int32_t k = 0;
    if (hx < 0x00800000) {
        if ((hx & 0x7fffffff) == 0) return -__int_as_float(0x7f800000);
        if (hx < 0) return __int_as_float(0x7fc00000);
        k -= 25;
        x = __fmul_rn(x, two25);
        hx = __float_as_int(x);
    }
    if (hx >= 0x7f800000) return __fadd_rn(x, x);
    k += (hx >> 23) - 127;
    const int32_t i = static_cast<int32_t>((static_cast<uint32_t>(k) & 0x80000000u) >> 31);
    hx = (hx & 0x007fffff) | ((0x7f - i) << 23);
    const float y = static_cast<float>(k + i);
    x = __int_as_float(hx);
    const float lo = __fmul_rn(y, log10_2lo);
    const float z = __fadd_rn(__fmul_rn(ivln10, glibc_logf(x, fma_variant)), lo);
    return __fadd_rn(z, __fmul_rn(y, log10_2hi));
}

// powf(10.0f, y) (e_powf.c with x = 10: positive normal base, sign_bias 0).
__device__ __forceinline__ float glibc_powf10(float y, bool fma_variant) {
    constexpr double A[5] = {0x1.27616c9496e0bp-2, -0x1.71969a075c67ap-2, 0x1.ec70a6ca7baddp-2,
                             -0x1.7154748bef6c8p-1, 0x1.71547652ab82bp+0};
    constexpr double SHIFT = 0x1.8p+47;
    constexpr double C0 = 0x1.c6af84b912394p-5, C1 = 0x1.ebfce50fac4f3p-3, C2 = 0x1.62e42ff0c52d6p-1;
    const uint32_t iy = __float_as_uint(y);
    if (2 * iy - 1 >= 2u * 0x7f800000u - 1) {
        if (2 * iy == 0) return 1.0f;
        if (2 * iy > 2u * 0x7f800000u) return __fadd_rn(10.0f, y);  // NaN
        return (iy & 0x80000000u) ? 0.0f : __int_as_float(0x7f800000);  // -inf -> 0, +inf -> inf
    }
    // log2(10): ix = 0x41200000 -> tmp = 0x01ed0000, i = 13, k = 3, z = 1.25f
    constexpr uint32_t ix = 0x41200000u;
    constexpr uint32_t tmp = ix - 0x3f330000u;
    constexpr int i = static_cast<int>((tmp >> 19) & 15u);
    constexpr int k = static_cast<int32_t>(tmp & 0xff800000u) >> 23;
    const double invc = c_powf_tab[i][0], logc = c_powf_tab[i][1];
    const double z = static_cast<double>(__uint_as_float(ix - (tmp & 0xff800000u)));
    double logx;
    if (fma_variant) {
        const double r = __fma_rn(z, invc, -1.0);
        const double y0 = __dadd_rn(logc, static_cast<double>(k));
        const double yy = __fma_rn(r, A[0], A[1]);
        const double p = __fma_rn(r, A[2], A[3]);
        const double r2 = __dmul_rn(r, r);
        double q = __fma_rn(r, A[4], y0);
        const double r4 = __dmul_rn(r2, r2);
        q = __fma_rn(r2, p, q);
        logx = __fma_rn(r4, yy, q);
    } else {
        const double r = __dsub_rn(__dmul_rn(z, invc), 1.0);
        const double y0 = __dadd_rn(logc, static_cast<double>(k));
        const double r2 = __dmul_rn(r, r);
        const double yy = __dadd_rn(__dmul_rn(A[0], r), A[1]);
        const double p = __dadd_rn(__dmul_rn(A[2], r), A[3]);
        const double r4 = __dmul_rn(r2, r2);
        double q = __dadd_rn(__dmul_rn(A[4], r), y0);
        q = __dadd_rn(__dmul_rn(p, r2), q);
        logx = __dadd_rn(__dmul_rn(yy, r4), q);
    }
    const double ylogx = __dmul_rn(static_cast<double>(y), logx);
    const unsigned long long yb = static_cast<unsigned long long>(__double_as_longlong(ylogx));
    constexpr unsigned long long k126 = 0x405F800000000000ull >> 47;  // asuint64(126.0) >> 47
    if (((yb >> 47) & 0xffff) >= k126) {
        if (ylogx > 0x1.fffffffd1d571p+6) return __int_as_float(0x7f800000);
        if (ylogx <= -150.0) return 0.0f;
        if (ylogx < -149.0) return __fmul_rn(0x1.4p-75f, 0x1.4p-75f);  // __math_may_uflowf
    }
    double kd = __dadd_rn(ylogx, SHIFT);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, SHIFT);
    const double r = __dsub_rn(ylogx, kd);
    unsigned long long t = c_exp2f_tab[ki % 32];
    t += ki << (52 - 5);
    const double s = __longlong_as_double(static_cast<long long>(t));
    double out;
    if (fma_variant) {
        const double zz = __fma_rn(r, C0, C1);
        const double r2 = __dmul_rn(r, r);
        double yy = __fma_rn(r, C2, 1.0);
        yy = __fma_rn(zz, r2, yy);
        out = __dmul_rn(yy, s);
    } else {
        const double zz = __dadd_rn(__dmul_rn(C0, r), C1);
        const double r2 = __dmul_rn(r, r);
        double yy = __dadd_rn(__dmul_rn(C2, r), 1.0);
        yy = __dadd_rn(__dmul_rn(zz, r2), yy);
        out = __dmul_rn(yy, s);
    }
    return __double2float_rn(out);
}

} // namespace ssb
