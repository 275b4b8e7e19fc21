/*
 * oracle/libm_port.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The detector's floor stage is defined by glibc's float libm
 * (proj/src/detector.cpp:217 `10.0f * std::log10(float)` -> log10f and
 * :222 `std::pow(10.0f, float)` -> powf).  Third-party
 * dependency: glibc 2.39 (Ubuntu 2.39-0ubuntu8.5, this image and the GPU box),
 * x86_64 build.  This file restates its published algorithms:
 *
 *   log10f  : sysdeps/ieee754/flt-32/e_log10f.c (fdlibm-derived float
 *             composition over logf; no FMA: baseline x86-64 code);
 *   logf    : sysdeps/ieee754/flt-32/e_logf.c (16-entry table + degree-3
 *             polynomial in double), ifunc'ed on x86_64 between an FMA build
 *             (e_logf-fma.c, selected when FMA+AVX2 are usable) and SSE2;
 *   powf    : sysdeps/ieee754/flt-32/e_powf.c (log2 via 16-entry table +
 *             degree-5 polynomial, exp2 via 32-entry table + degree-3
 *             polynomial), same FMA/SSE2 ifunc pair.
 *
 * The table and polynomial constants are the ones in this image's
 * libm.so.6 .rodata (__logf_data, __powf_log2_data, __exp2f_data), read at
 * the addresses the disassembly of log10f / __logf_fma / __powf_fma
 * references; the operation order (and which products fuse in the FMA build)
 * follows that disassembly.  tests/test_libm_port.py checks both variants
 * against the live glibc on strided sweeps of all 2^32 float bit patterns;
 * tools/libm_exhaustive.c runs the full sweep (DESIGN.md records the result).
 * The device port (paper_2603_20481_b200/csrc/glibc_libm.cuh) is written
 * independently from the same description and checked against glibc on the
 * GPU (tests/test_gpu_libm.py).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint32_t asu32(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float asf32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint64_t asu64(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double asf64(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

static const double LOGF_T[16][2] = {
    {0x1.661ec79f8f3bep+0, -0x1.57bf7808caadep-2}, {0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2},
    {0x1.49539f0f010bp+0, -0x1.01eae7f513a67p-2},  {0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3},
    {0x1.30d190c8864a5p+0, -0x1.6574f0ac07758p-3}, {0x1.25e227b0b8eap+0, -0x1.1aa2bc79c81p-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.a4e76ce8c0e5ep-4}, {0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4},
    {0x1.0953f419900a7p+0, -0x1.252f438e10c1ep-5}, {0x1p+0, 0x0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.aa5aa5df25984p-5},  {0x1.ca4b31f026aap-1, 0x1.c5e53aa362eb4p-4},
    {0x1.b2036576afce6p-1, 0x1.526e57720db08p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.bc2860d22477p-3},
    {0x1.886e6037841edp-1, 0x1.1058bc8a07ee1p-2},  {0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2},
};
static const double LOGF_LN2 = 0x1.62e42fefa39efp-1;
static const double LOGF_A[3] = {-0x1.00ea348b88334p-2, 0x1.5575b0be00b6ap-2, -0x1.ffffef20a4123p-2};

/* logf for positive normal/subnormal finite x (the only inputs log10f hands it). */
static float logf_port(float x, int fma_variant) {
    uint32_t ix = asu32(x);
    if (ix == 0x3f800000u) return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        if (ix * 2 == 0) return -INFINITY;
        if (ix == 0x7f800000u) return x;
        if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u) return NAN;
        ix = asu32(x * 0x1p23f);
        ix -= 23u << 23;
    }
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) % 16);
    const int k = (int32_t)tmp >> 23;
    const uint32_t iz = ix - (tmp & 0xff800000u);
    const double invc = LOGF_T[i][0], logc = LOGF_T[i][1];
    const double z = (double)asf32(iz);
    if (fma_variant) {
        const double r = fma(z, invc, -1.0);
        const double y0 = fma((double)k, LOGF_LN2, logc);
        const double r2 = r * r;
        double y = fma(r, LOGF_A[1], LOGF_A[2]);
        y = fma(r2, LOGF_A[0], y);
        return (float)fma(r2, y, r + y0);
    } else {
        const double r = z * invc - 1.0;
        const double y0 = logc + (double)k * LOGF_LN2;
        const double r2 = r * r;
        double y = LOGF_A[1] * r + LOGF_A[2];
        y = LOGF_A[0] * r2 + y;
        return (float)(y * r2 + (y0 + r));
    }
}

/* e_log10f.c: float composition over logf, no fusion. */
float oracle_log10f(float x, int fma_variant) {
    const float two25 = 3.3554432000e+07f;
    const float ivln10 = asf32(0x3ede5bd9u);
    const float log10_2hi = asf32(0x3e9a2080u);
    const float log10_2lo = asf32(0x355427dbu);
    int32_t hx = (int32_t)asu32(x);
    int32_t k = 0;
    if (hx < 0x00800000) {
        if ((hx & 0x7fffffff) == 0) return -two25 / fabsf(x);
        if (hx < 0) return (x - x) / (x - x);
        k -= 25;
        x *= two25;
        hx = (int32_t)asu32(x);
    }
    if (hx >= 0x7f800000) return x + x;
    k += (hx >> 23) - 127;
    const int32_t i = (int32_t)(((uint32_t)k & 0x80000000u) >> 31);
    hx = (hx & 0x007fffff) | ((0x7f - i) << 23);
    const float y = (float)(k + i);
    x = asf32((uint32_t)hx);
    const float lo = y * log10_2lo;
    const float z = ivln10 * logf_port(x, fma_variant) + lo;
    return z + y * log10_2hi;
}

static const double POWF_T[16][2] = {
    {0x1.661ec79f8f3bep+0, -0x1.efec65b963019p-2}, {0x1.571ed4aaf883dp+0, -0x1.b0b6832d4fca4p-2},
    {0x1.49539f0f010bp+0, -0x1.7418b0a1fb77bp-2},  {0x1.3c995b0b80385p+0, -0x1.39de91a6dcf7bp-2},
    {0x1.30d190c8864a5p+0, -0x1.01d9bf3f2b631p-2}, {0x1.25e227b0b8eap+0, -0x1.97c1d1b3b7afp-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.2f9e393af3c9fp-3}, {0x1.12358f08ae5bap+0, -0x1.960cbbf788d5cp-4},
    {0x1.0953f419900a7p+0, -0x1.a6f9db6475fcep-5}, {0x1p+0, 0x0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.338ca9f24f53dp-4},  {0x1.ca4b31f026aap-1, 0x1.476a9543891bap-3},
    {0x1.b2036576afce6p-1, 0x1.e840b4ac4e4d2p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.40645f0c6651cp-2},
    {0x1.886e6037841edp-1, 0x1.88e9c2c1b9ff8p-2},  {0x1.767dcf5534862p-1, 0x1.ce0a44eb17bccp-2},
};
static const double POWF_A[5] = {0x1.27616c9496e0bp-2, -0x1.71969a075c67ap-2, 0x1.ec70a6ca7baddp-2,
                                 -0x1.7154748bef6c8p-1, 0x1.71547652ab82bp+0};
static const uint64_t EXP2F_T[32] = {
    0x3ff0000000000000, 0x3fefd9b0d3158574, 0x3fefb5586cf9890f, 0x3fef9301d0125b51,
    0x3fef72b83c7d517b, 0x3fef54873168b9aa, 0x3fef387a6e756238, 0x3fef1e9df51fdee1,
    0x3fef06fe0a31b715, 0x3feef1a7373aa9cb, 0x3feedea64c123422, 0x3feece086061892d,
    0x3feebfdad5362a27, 0x3feeb42b569d4f82, 0x3feeab07dd485429, 0x3feea47eb03a5585,
    0x3feea09e667f3bcd, 0x3fee9f75e8ec5f74, 0x3feea11473eb0187, 0x3feea589994cce13,
    0x3feeace5422aa0db, 0x3feeb737b0cdc5e5, 0x3feec49182a3f090, 0x3feed503b23e255d,
    0x3feee89f995ad3ad, 0x3feeff76f2fb5e47, 0x3fef199bdd85529c, 0x3fef3720dcef9069,
    0x3fef5818dcfba487, 0x3fef7c97337b9b5f, 0x3fefa4afa2a490da, 0x3fefd0765b6e4540,
};
static const double EXP2F_SHIFT = 0x1.8p+47;
static const double EXP2F_C[3] = {0x1.c6af84b912394p-5, 0x1.ebfce50fac4f3p-3, 0x1.62e42ff0c52d6p-1};

/*
 * powf(x, y) for x a positive normal float (the detector only ever raises
 * 10.0f), all y.  Returns the same value as glibc, errno/flags aside.
 */
float oracle_powf(float x, float y, int fma_variant) {
    const uint32_t ix = asu32(x), iy = asu32(y);
    /* zeroinfnan(iy) */
    if (2 * iy - 1 >= 2u * 0x7f800000u - 1) {
        if (2 * iy == 0) return 1.0f;
        if (ix == 0x3f800000u) return (2 * iy <= 2u * 0x7fc00000u) ? 1.0f : x + y;
        if (2 * ix > 2u * 0x7f800000u || 2 * iy > 2u * 0x7f800000u) return x + y;
        if (2 * ix == 2 * 0x3f800000u) return 1.0f;
        if ((2 * ix < 2 * 0x3f800000u) == !(iy & 0x80000000u)) return 0.0f;
        return y * y;
    }
    /* log2 */
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) % 16);
    const uint32_t top = tmp & 0xff800000u;
    const uint32_t iz = ix - top;
    const int k = (int32_t)top >> 23;
    const double invc = POWF_T[i][0], logc = POWF_T[i][1];
    const double z = (double)asf32(iz);
    double logx;
    if (fma_variant) {
        const double r = fma(z, invc, -1.0);
        const double y0 = logc + (double)k;
        const double yy = fma(r, POWF_A[0], POWF_A[1]);
        const double p = fma(r, POWF_A[2], POWF_A[3]);
        const double r2 = r * r;
        double q = fma(r, POWF_A[4], y0);
        const double r4 = r2 * r2;
        q = fma(r2, p, q);
        logx = fma(r4, yy, q);
    } else {
        const double r = z * invc - 1.0;
        const double y0 = logc + (double)k;
        const double r2 = r * r;
        const double yy = POWF_A[0] * r + POWF_A[1];
        const double p = POWF_A[2] * r + POWF_A[3];
        const double r4 = r2 * r2;
        double q = POWF_A[4] * r + y0;
        q = p * r2 + q;
        logx = yy * r4 + q;
    }
    const double ylogx = (double)y * logx;
    if (((asu64(ylogx) >> 47) & 0xffff) >= (asu64(126.0) >> 47)) {
        if (ylogx > 0x1.fffffffd1d571p+6) return INFINITY;
        /* round-to-nearest: the 0x1.fffffffa3aae2p+6 band does not overflow */
        if (ylogx <= -150.0) return 0.0f;
        if (ylogx < -149.0) {
            /* __math_may_uflowf: 0x1.4p-75f * 0x1.4p-75f */
            volatile float t = 0x1.4p-75f;
            return t * t;
        }
    }
    /* exp2 */
    double kd = ylogx + EXP2F_SHIFT;
    const uint64_t ki = asu64(kd);
    kd -= EXP2F_SHIFT;
    const double r = ylogx - kd;
    uint64_t t = EXP2F_T[ki % 32];
    t += ki << (52 - 5);
    const double s = asf64(t);
    double out;
    if (fma_variant) {
        const double zz = fma(r, EXP2F_C[0], EXP2F_C[1]);
        const double r2 = r * r;
        double yy = fma(r, EXP2F_C[2], 1.0);
        yy = fma(zz, r2, yy);
        out = yy * s;
    } else {
        const double zz = EXP2F_C[0] * r + EXP2F_C[1];
        const double r2 = r * r;
        double yy = EXP2F_C[2] * r + 1.0;
        yy = zz * r2 + yy;
        out = yy * s;
    }
    return (float)out;
}

/* Batch helpers for ctypes. */
void oracle_log10f_batch(const float* x, long long n, int fma_variant, float* out) {
    for (long long i = 0; i < n; ++i) out[i] = oracle_log10f(x[i], fma_variant);
}
void oracle_powf10_batch(const float* y, long long n, int fma_variant, float* out) {
    for (long long i = 0; i < n; ++i) out[i] = oracle_powf(10.0f, y[i], fma_variant);
}
/* The live glibc, for comparison (log10f / powf as the reference calls them). */
void oracle_glibc_log10f_batch(const float* x, long long n, float* out) {
    for (long long i = 0; i < n; ++i) out[i] = log10f(x[i]);
}
void oracle_glibc_powf10_batch(const float* y, long long n, float* out) {
    for (long long i = 0; i < n; ++i) out[i] = powf(10.0f, y[i]);
}
