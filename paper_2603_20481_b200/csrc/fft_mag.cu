// fft_mag.cu -- K1: IQ rows -> DC-centred FFT-magnitude TF rows (+ exact PSD).
//
// Replaces frontend::fft_row / make_plot / make_plots
// (proj/src/frontend.cpp:127-183) and, fused, the column sum of
// detector::estimate_psd_into (proj/src/detector.cpp:170-184).
//
// Arithmetic: the SSFFT-2 specification -- FP64 Stockham DIT
// autosort, radix-16 passes + one radix-2^(log2N mod 4) pass, one table
// twiddle per butterfly and its powers by a fixed product tree,
// explicit-rounding butterflies -- then out[k] = float(sqrt(fma(re, re,
// im*im))) of bin (k + N/2) mod N, exactly the expression GCC emits for
// proj/src/frontend.cpp:147 (vmulsd im*im; vfmadd re*re+.; vsqrtsd; cvtsd2ss).
// The oracle's FFTW shim (oracle/fftw_shim.c) implements the same spec on the
// CPU, so TF plots are bit-identical.
//
// Layout / schedule (B200): row groups of 256 threads (512 for N = 8192), two
// per CTA for N <= 4096, 16 complex doubles per thread in registers;
// G = 256/(N/16) rows per group iteration.  The next iteration's raw IQ rows
// (contiguous, G*N samples) are fetched by one TMA 1-D bulk copy into the
// group's shared stage behind an mbarrier while the current rows transform;
// the inter-pass exchanges go through a padded shared buffer (idx + idx/16:
// conflict-free), whole complex values for N >= 4096 with the next pass's
// twiddle tree computed in the barrier wait.  In PSD mode a group owns one
// whole plot and walks its rows in order, so the per-column sum of x^2 runs in
// the reference's exact row order (acc = fma(x, x, acc): x^2 is exact, fusion
// is bit-neutral) -- in registers for N <= 2048, in tensor memory (TMEM,
// tcgen05.ld/st) for N >= 4096.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

namespace ssb {

// ---------------------------------------------------------------- butterflies

__device__ __forceinline__ void dft2(cd* v) {
    const cd a = v[0], b = v[1];
    v[0] = c_add(a, b);
    v[1] = c_sub(a, b);
}

template <int S>
__device__ __forceinline__ void dft4s(cd* v) {
    const cd t0 = c_add(v[0], v[2 * S]);
    const cd t1 = c_sub(v[0], v[2 * S]);
    const cd t2 = c_add(v[S], v[3 * S]);
    const cd t3 = c_sub(v[S], v[3 * S]);
    v[0] = c_add(t0, t2);
    v[2 * S] = c_sub(t0, t2);
    v[S] = {__dadd_rn(t1.re, t3.im), __dsub_rn(t1.im, t3.re)};
    v[3 * S] = {__dsub_rn(t1.re, t3.im), __dadd_rn(t1.im, t3.re)};
}

__device__ __forceinline__ void dft8(cd* v) {
    cd e[4] = {v[0], v[2], v[4], v[6]};
    cd o[4] = {v[1], v[3], v[5], v[7]};
    dft4s<1>(e);
    dft4s<1>(o);
    o[1] = c_w8(o[1]);
    o[2] = c_mi(o[2]);
    o[3] = c_w83(o[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = c_add(e[k], o[k]);
        v[k + 4] = c_sub(e[k], o[k]);
    }
}

// 4x4 decomposition; y[n1*4+k2] after the first DFT4 layer.
__device__ __forceinline__ void dft16_tail(cd* y, cd* v);

__device__ __forceinline__ void dft16(cd* v) {
    cd y[16];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
        cd t[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
        dft4s<1>(t);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) y[n1 * 4 + k2] = t[k2];
    }
    dft16_tail(y, v);
}

// The first DFT4 layer of a DFT16 on integer samples (int16 IQ): every sum is
// an integer below 2^17, exact in int32 as in double, so this layer leaves the
// FP64 pipe; y[n1*4+k2] as dft16 forms it.
__device__ __forceinline__ void dft16_layer1_int(const int* re, const int* im, cd* y) {
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
        const int t0r = re[n1] + re[n1 + 8], t0i = im[n1] + im[n1 + 8];
        const int t1r = re[n1] - re[n1 + 8], t1i = im[n1] - im[n1 + 8];
        const int t2r = re[n1 + 4] + re[n1 + 12], t2i = im[n1 + 4] + im[n1 + 12];
        const int t3r = re[n1 + 4] - re[n1 + 12], t3i = im[n1 + 4] - im[n1 + 12];
        y[n1 * 4 + 0] = {static_cast<double>(t0r + t2r), static_cast<double>(t0i + t2i)};
        y[n1 * 4 + 2] = {static_cast<double>(t0r - t2r), static_cast<double>(t0i - t2i)};
        y[n1 * 4 + 1] = {static_cast<double>(t1r + t3i), static_cast<double>(t1i - t3r)};
        y[n1 * 4 + 3] = {static_cast<double>(t1r - t3i), static_cast<double>(t1i + t3r)};
    }
}

// internal W16 twiddles + second DFT4 layer: y -> v (natural order)
__device__ __forceinline__ void dft16_tail(cd* y, cd* v) {
    const cd w1 = {kC1, -kS1};
    const cd w3 = {kS1, -kC1};
    const cd w9 = {-kC1, kS1};
    y[5] = c_mul(y[5], w1);
    y[6] = c_w8(y[6]);
    y[7] = c_mul(y[7], w3);
    y[9] = c_w8(y[9]);
    y[10] = c_mi(y[10]);
    y[11] = c_w83(y[11]);
    y[13] = c_mul(y[13], w3);
    y[14] = c_w83(y[14]);
    y[15] = c_mul(y[15], w9);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
        cd t[4] = {y[k2], y[4 + k2], y[8 + k2], y[12 + k2]};
        dft4s<1>(t);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = t[k1];
    }
}

template <int R>
__device__ __forceinline__ void dft_r(cd* v) {
    if constexpr (R == 2) dft2(v);
    else if constexpr (R == 4) dft4s<1>(v);
    else if constexpr (R == 8) dft8(v);
    else dft16(v);
}

// ------------------------------------------------------------------ plan

template <int LOGN>
struct FftPlan {
    static constexpr int N = 1 << LOGN;
    static constexpr int P = N >= 16 ? 16 : N;      // points per thread
    static constexpr int TPR = N / P;               // threads per row
    static constexpr int NT = TPR > 256 ? TPR : 256; // threads per CTA
    static constexpr int G = NT / TPR;              // rows per iteration
    static constexpr int NP = (LOGN == 3) ? 1 : (LOGN / 4 + (LOGN % 4 ? 1 : 0));
    static constexpr int SROW = N + N / 16;          // padded smem row (elements)
    __host__ __device__ static constexpr int radix(int p) {
        return (LOGN == 3) ? 8 : (p < LOGN / 4 ? 16 : (1 << (LOGN % 4)));
    }
    __host__ __device__ static constexpr int ns(int p) {
        int s = 1;
        for (int q = 0; q < p; ++q) s *= radix(q);
        return s;
    }
    // Twiddle block of pass p >= 1 (Ns > 1): (R-1)*Ns entries, tw[r*k*s] at
    // (r-1)*Ns + k with s = N/(Ns*R) -- a pass-major re-layout of the
    // canonical table so a warp's 32 lanes read 32 consecutive entries.
    __host__ __device__ static constexpr int tw_block(int p) { return (radix(p) - 1) * ns(p); }
    __host__ __device__ static constexpr int tw_off(int p) {
        int o = 0;
        for (int q = 1; q < p; ++q) o += tw_block(q);
        return o;
    }
    __host__ __device__ static constexpr int tw_size() { return tw_off(NP); }
};

__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 4); }

// SSFFT-2 twiddles of pass PASS for this thread's butterflies b_u = j + TPR*u:
// w1 from the table, higher powers by a fixed product tree -- one table load
// per butterfly instead of R-1 (the loads, not the multiplies, were the cost:
// DESIGN.md §4).  w[u*R + r] = w1^r (r >= 1).
template <int LOGN, int PASS, bool TWS>
__device__ __forceinline__ void pass_twiddles(int j, const double2* __restrict__ tw, cd* w) {
    // tw points at the CTA's shared-memory copy of the pass tables (plain
    // loads -> LDS.128) or, for N >= 4096, at the global table (L1)
    using PL = FftPlan<LOGN>;
    constexpr int R = PL::radix(PASS);
    constexpr int NS = PL::ns(PASS);
    constexpr int U = PL::P / R;
    if constexpr (NS > 1) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int b = j + PL::TPR * u;
            const int k = b % NS;
            const double2* t = tw + PL::tw_off(PASS) + k;
            const double2 w1t = TWS ? t[0] : __ldg(t);
            cd* x = w + u * R;
            x[1] = cd{w1t.x, w1t.y};
            if constexpr (R > 2) x[2] = c_mul(x[1], x[1]);
            if constexpr (R > 3) x[3] = c_mul(x[2], x[1]);
            if constexpr (R > 4) {
                x[4] = c_mul(x[2], x[2]);
                x[5] = c_mul(x[4], x[1]);
                x[6] = c_mul(x[4], x[2]);
                x[7] = c_mul(x[4], x[3]);
            }
            if constexpr (R > 8) {
                x[8] = c_mul(x[4], x[4]);
#pragma unroll
                for (int q = 9; q < 16; ++q) x[q] = c_mul(x[8], x[q - 8]);
            }
        }
    }
}

// Twiddle + butterflies of pass p on register data already holding this
// pass's inputs: butterfly b_u = j + TPR*u owns v[u*R .. u*R+R-1]; w from
// pass_twiddles.
template <int LOGN, int PASS>
__device__ __forceinline__ void run_pass(cd* v, const cd* w) {
    using PL = FftPlan<LOGN>;
    constexpr int R = PL::radix(PASS);
    constexpr int NS = PL::ns(PASS);
    constexpr int U = PL::P / R;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) v[u * R + r] = c_mul(v[u * R + r], w[u * R + r]);
        }
        dft_r<R>(v + u * R);
    }
}

__device__ __forceinline__ void group_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Next-iteration TMA issue, handed to the first exchange: once every thread of
// the group has passed its first barrier, every thread has consumed the stage.
struct StageIssue {
    void* stage;
    const void* src;
    uint32_t bytes;
    uint64_t* bar;
    bool go;
    bool leader;
    __device__ __forceinline__ void operator()() const {
        if (go && leader) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, bytes);
            bulk_g2s(stage, src, bytes, bar);
        }
    }
};

// Store pass PASS's outputs into smem (padded), then load pass PASS+1's
// inputs.  CX = false: real parts then imaginary parts through one N-double
// buffer (half the shared memory of a complex exchange, 4 barriers).  CX =
// true: whole complex values, 16-byte STS/LDS, 2 barriers (the padding keeps
// both the pass-0 strided stores and the lane-contiguous loads conflict-free).
// Barriers are the group's named barrier, so the row groups of a CTA never
// wait on each other.
template <int LOGN, int PASS, bool CX, bool TWS>
__device__ __forceinline__ void exchange(cd* v, int j, double* buf, int bar_id, const StageIssue& nxt,
                                         const double2* tw, cd* wn) {
    using PL = FftPlan<LOGN>;
    constexpr int R = PL::radix(PASS);
    constexpr int NS = PL::ns(PASS);
    constexpr int U = PL::P / R;
    constexpr int R2 = PL::radix(PASS + 1);
    constexpr int U2 = PL::P / R2;
    if constexpr (CX) {
        double2* cbuf = reinterpret_cast<double2*>(buf);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int b = j + PL::TPR * u;
            const int k = b % NS;
            const int base = (b - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) cbuf[pad_idx(base + r * NS)] = make_double2(v[u * R + r].re, v[u * R + r].im);
        }
        // the data registers are free until the loads: the next pass's
        // twiddle tree fills the wait for the slowest warp of the group
        pass_twiddles<LOGN, PASS + 1, TWS>(j, tw, wn);
        group_sync(bar_id, PL::NT);
        if (PASS == 0) nxt();
#pragma unroll
        for (int u = 0; u < U2; ++u) {
            const int b = j + PL::TPR * u;
#pragma unroll
            for (int r = 0; r < R2; ++r) {
                const double2 x = cbuf[pad_idx(b + r * (PL::N / R2))];
                v[u * R2 + r] = {x.x, x.y};
            }
        }
        group_sync(bar_id, PL::NT);
    } else {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int b = j + PL::TPR * u;
                const int k = b % NS;
                const int base = (b - k) * R + k;
#pragma unroll
                for (int r = 0; r < R; ++r) buf[pad_idx(base + r * NS)] = half ? v[u * R + r].im : v[u * R + r].re;
            }
            group_sync(bar_id, PL::NT);
            if (PASS == 0 && half == 0) nxt();
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int b = j + PL::TPR * u;
#pragma unroll
                for (int r = 0; r < R2; ++r) {
                    const double x = buf[pad_idx(b + r * (PL::N / R2))];
                    if (half) v[u * R2 + r].im = x;
                    else v[u * R2 + r].re = x;
                }
            }
            group_sync(bar_id, PL::NT);
        }
        pass_twiddles<LOGN, PASS + 1, TWS>(j, tw, wn);
    }
}

// Y0: pass 0's inputs are already through the first DFT4 layer (int16 path)
template <int LOGN, int PASS, bool TWS, bool CX, bool Y0 = false>
__device__ __forceinline__ void passes_from(cd* v, int j, const double2* tw, double* buf, int bar_id,
                                            const StageIssue& nxt, const cd* w) {
    using PL = FftPlan<LOGN>;
    if constexpr (Y0) {
        static_assert(PASS == 0 && PL::radix(0) == 16 && PL::P == 16, "Y0: one radix-16 butterfly in pass 0");
        cd y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) y[i] = v[i];
        dft16_tail(y, v);
    } else {
        run_pass<LOGN, PASS>(v, w);
    }
    if constexpr (PASS + 1 < PL::NP) {
        cd wn[16];
        exchange<LOGN, PASS, CX, TWS>(v, j, buf, bar_id, nxt, tw, wn);
        passes_from<LOGN, PASS + 1, TWS, CX>(v, j, tw, buf, bar_id, nxt, wn);
    }
}

__device__ __forceinline__ double rsqrt_seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

// |X| rounded to float, bit-identical to float(sqrt(fma(re, re, im*im))).
// Fast path (every point, branch-free): MUFU.RSQ64H seed + one Newton step in
// double gives sqrt(q) within 11,681 double ulps (bound below); when that
// estimate is further than kMidMargin ulps from a float rounding midpoint
// (low 29 mantissa bits vs 2^28), rounding it to float equals rounding the
// correctly rounded double sqrt -- no midpoint lies between them; the
// rounding itself is one F2F.F32.F64 (conversion unit, off the FP64 pipe).  A
// normal float result also proves q far from the seed's flush range and from
// overflow.  Otherwise (2^-15.4 of the points, or zero / subnormal / huge
// magnitudes) the warp takes a uniform branch in which the flagged lanes redo
// theirs with the IEEE __dsqrt_rn + F2F.  That branch delays the whole row
// group at its next barrier, so its rate matters: with the former 2^16-ulp
// margin 64 % of the rows had a flagged point and K1 lost 0.9 of 12.9 ms
// (measured with the branch disabled); a second Newton level ahead of
// __dsqrt_rn spilled registers in the row loop (14.5 ms).
// SH: the transform ran on inputs scaled by 2^SH (int16 IQ without its exact
// 2^-15 decode factor); power-of-two scaling commutes with every rounding of
// the FFT, so the true magnitude is the computed one times 2^-SH, applied as
// an exponent offset (fast path) or an exact multiply (slow path).
//
// kMidMargin: tools/rsq_probe.cu evaluates the seed on every high word of
// [1,4) (it depends on the high word only) at both ends of the low word:
// relative error e <= 2^-20.037, so the Newton estimate is within 1.5 e^2 =
// 11,680.2 ulps of sqrt(q), + 0.5 for its own rounding (11,589.7 observed);
// the reference's s = RN_d(sqrt(q)) is within 0.5 ulp of sqrt(q).  The Newton
// error is one-sided: s1 - sqrt(q) = -sqrt(q) (1.5 e^2 + 2 e d1 + ..), d1 the
// 2^-53 rounding of s0, so s1 exceeds sqrt(q) by at most its own rounding
// (probe: +0.5 ulp) and s - s1 lies in [-1.01, 11,681.7].  A float midpoint m
// can separate s1 from s, or equal s, only if m - s1 is in that interval: a
// point is flagged iff m - s1 is in [-kMidAbove, kMidMargin] = [-4, 12288].
#ifndef K1_MID_MARGIN
#define K1_MID_MARGIN 12288
#endif
constexpr uint32_t kMidMargin = K1_MID_MARGIN;
constexpr uint32_t kMidAbove = 4;

template <int P, int SH>
__device__ __forceinline__ void mags(const cd* v, float* m) {
    uint32_t slow = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const double q = __fma_rn(v[i].re, v[i].re, __dmul_rn(v[i].im, v[i].im));
        // Newton step s1 = s0 + (q - s0^2) y/2, s0 = q y.  Only h = y/2 is kept
        // (an exponent decrement of the seed, integer pipe) and s0 = 2 (q h) by
        // an exponent increment: power-of-two scalings commute with the
        // roundings, so s0 and s1 are the same doubles, with one register pair
        // and two integer instructions less per point than holding y and h.
        // (q = 0 or non-finite: the increments yield finite garbage or NaN,
        // the float is not normal, and the point is flagged.)
        const double y = rsqrt_seed(q);
        const double h = __hiloint2double(__double2hiint(y) - (1 << 20), __double2loint(y));
        const double w = __dmul_rn(q, h);
        const double s0 = __hiloint2double(__double2hiint(w) + (1 << 20), __double2loint(w));
        const double d = __fma_rn(-s0, s0, q);
        const double s1 = __fma_rn(d, h, s0);
        const uint32_t hi = static_cast<uint32_t>(__double2hiint(s1));
        const uint32_t lo = static_cast<uint32_t>(__double2loint(s1));
        // float rounding by F2F.F32.F64 (the conversion unit); 2^-SH as an
        // exponent decrement first
        const float mf = __double2float_rn(SH ? __hiloint2double(static_cast<int>(hi - (SH << 20)), static_cast<int>(lo)) : s1);
        // dist = low 29 bits - 2^28 (ulps from the midpoint); flagged iff
        // -margin <= dist <= above, tested on 8 * (low 29 bits) (one IMAD
        // drops the three high bits and subtracts the window's start)
        const uint32_t mid8 = lo * 8u - 8u * ((1u << 28) - kMidMargin);
        const bool normal = __float_as_uint(mf) >= 0x00800000u && __float_as_uint(mf) < 0x7f800000u;
        m[i] = mf;
        if (!(normal && mid8 > 8u * (kMidMargin + kMidAbove) + 7u)) slow |= 1u << i;
    }
    if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
        for (int i = 0; i < P; ++i)
            if ((slow >> i) & 1u)
                m[i] = __double2float_rn(__dmul_rn(
                    __dsqrt_rn(__fma_rn(v[i].re, v[i].re, __dmul_rn(v[i].im, v[i].im))), 1.0 / (1 << SH)));
    }
}

// ------------------------------------------------------------------ kernel

struct FftArgs {
    const void* iq;      // n_rows_total * N samples, f32 or i16 interleaved
    float* tf;           // n_rows_total * N floats, may be null in PSD mode
    float* psd;          // n_plots * N (PSD mode)
    float* col_lo;       // n_plots * N column minima / maxima of the plot (PSD mode, TMEM shapes) or null
    float* col_hi;
    const double2* tw;   // per-N pass twiddle table (global)
    long long total_rows;
    int rows_per_plot;   // PSD mode: T
    int n_plots;
    int hop;             // samples between consecutive rows (N: rectangular, no overlap)
    const double* win;   // N window weights (WIN mode), x_w = double(x) * w[n]
};

// CTA = GROUPS independent row groups of NT threads.  Each group owns one plot
// (PSD mode) or a strided set of row iterations, its own exchange buffer, TMA
// stage, mbarrier and named barrier.  One-row-per-iteration shapes (N >= 4096)
// exchange whole complex values (CX) and keep the per-column PSD accumulators
// in tensor memory (TMEM, otherwise idle here): shared memory holds only the
// exchange buffer and the IQ stage, registers stay free for butterfly ILP,
// and the pass twiddles come through L1.  Multi-row shapes (N <= 2048)
// accumulate in registers and share an smem copy of the twiddles.
template <int LOGN>
struct K1Shape {
    using PL = FftPlan<LOGN>;
    static constexpr int GROUPS = LOGN >= 13 ? 1 : 2;
    static constexpr bool TW_SMEM = PL::G > 1;
    static constexpr bool CX = PL::G == 1;
    static constexpr bool ACC_TMEM = PL::G == 1;
    static constexpr int XW = CX ? 2 : 1;  // doubles per exchange element
    static constexpr int THREADS = PL::NT * GROUPS;
    static constexpr int WARPS = THREADS / 32;
    // TMEM: warp w uses lanes 32*(w%4).., columns 32*(w/4) .. +31 (16 doubles)
    static constexpr int TMEM_COLS = WARPS <= 4 ? 32 : WARPS <= 8 ? 64 : WARPS <= 16 ? 128 : 256;
    // column extremes (fminf / fmaxf of the plot's magnitudes, for K4) in a
    // second block of TMEM_COLS columns: 16 minima + 16 maxima per thread
    // blocks of TMEM_COLS columns: PSD sums, [column extremes], [window weights]; the allocation is a power of two
    __host__ __device__ static constexpr int tmem_alloc_cols(bool ext, bool wint = false) {
        const int nb = 1 + (ext ? 1 : 0) + (wint ? 1 : 0);
        return (nb == 1 ? 1 : nb == 2 ? 2 : 4) * TMEM_COLS;
    }
    static_assert(!ACC_TMEM || PL::P == 16, "one 32-column TMEM slot holds 16 double accumulators");
    __host__ __device__ static constexpr size_t tw_bytes() { return TW_SMEM ? sizeof(double2) * (PL::tw_size() > 0 ? PL::tw_size() : 1) : 0; }
    __host__ __device__ static constexpr size_t group_bytes(int sample_bytes) {
        return sizeof(double) * XW * PL::G * PL::SROW + static_cast<size_t>(sample_bytes) * PL::G * PL::N +
               (PL::G > 1 ? sizeof(float) * PL::G * PL::N : 0);
    }
    __host__ __device__ static constexpr size_t smem(int sample_bytes) { return tw_bytes() + GROUPS * group_bytes(sample_bytes); }
};

template <int LOGN, int FMT, bool PSD, bool WIN, bool EXT>
__global__ void __launch_bounds__(K1Shape<LOGN>::THREADS, 1)
fft_mag_kernel(FftArgs a) {
    using PL = FftPlan<LOGN>;
    using KS = K1Shape<LOGN>;
    constexpr int N = PL::N;
    constexpr int G = PL::G;
    constexpr int SAMPLE_BYTES = FMT == 0 ? 8 : 4;
    // STFT window weights of this thread's 16 samples (the same every row) in a
    // third block of TMEM columns: one tcgen05.ld per row, issued ahead of the
    // stage wait, instead of 16 L1 loads at the start of the row
    constexpr bool WINT = WIN && PSD && KS::ACC_TMEM && PL::radix(0) == 16 && PL::P == 16;
    constexpr int WOFF = KS::TMEM_COLS * (EXT ? 2 : 1);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[KS::GROUPS];

    const int gi = static_cast<int>(threadIdx.x) / PL::NT;  // row group
    const int lt = static_cast<int>(threadIdx.x) % PL::NT;  // thread within the group
    const int g = lt / PL::TPR;
    const int j = lt % PL::TPR;
    const int bar_id = 1 + gi;

    // shared twiddle tables (N <= 4096)
    const double2* tw = a.tw;
    if constexpr (KS::TW_SMEM) {
        double2* st = reinterpret_cast<double2*>(smem_raw);
        for (int e = threadIdx.x; e < PL::tw_size(); e += KS::THREADS) st[e] = a.tw[e];
        tw = st;
    }
    unsigned char* gbase = smem_raw + KS::tw_bytes() + gi * KS::group_bytes(SAMPLE_BYTES);
    double* xbuf = reinterpret_cast<double*>(gbase);                                   // G * SROW
    unsigned char* stage = gbase + sizeof(double) * KS::XW * G * PL::SROW;             // G*N samples
    float* magbuf = reinterpret_cast<float*>(stage + SAMPLE_BYTES * G * N);           // G*N (G > 1)
    double* mybuf = xbuf + KS::XW * g * PL::SROW;
    uint64_t* bar = &bars[gi];

    // iteration space of this group
    long long it_begin, it_end, it_step, row_base;
    if constexpr (PSD) {
        const long long plot = static_cast<long long>(blockIdx.x) * KS::GROUPS + gi;
        row_base = plot * a.rows_per_plot;
        it_begin = 0;
        it_end = plot < a.n_plots ? (a.rows_per_plot + G - 1) / G : 0;
        it_step = 1;
    } else {
        row_base = 0;
        it_begin = static_cast<long long>(blockIdx.x) * KS::GROUPS + gi;
        it_end = (a.total_rows + G - 1) / G;
        it_step = static_cast<long long>(gridDim.x) * KS::GROUPS;
    }
    const long long row_limit = PSD ? row_base + a.rows_per_plot : a.total_rows;
    auto chunk = [&](long long it, const void** src, uint32_t* bytes) {
        const long long r0 = row_base + it * G;
        long long nr = row_limit - r0;
        if (nr > G) nr = G;
        // rows (frames) start every `hop` samples; rectangular mode: hop == N
        const int hop = WIN ? a.hop : N;
        *src = static_cast<const unsigned char*>(a.iq) + r0 * hop * SAMPLE_BYTES;
        *bytes = static_cast<uint32_t>(((nr - 1) * hop + N) * SAMPLE_BYTES);
    };

    if (lt == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    // PSD accumulators in TMEM: this thread's 16 columns k(i) are 16 doubles =
    // 32 consecutive 32-bit TMEM columns of its lane
    __shared__ uint32_t tmem_slot;
    const int wid = static_cast<int>(threadIdx.x) >> 5;
    if constexpr (PSD && KS::ACC_TMEM) {
        if (wid == 0) tmem_alloc<KS::tmem_alloc_cols(EXT, WINT)>(&tmem_slot);
        tmem_fence_before();
    }
    __syncthreads();  // twiddle copy + mbarrier init (+ TMEM address) visible to all groups
    uint32_t taddr = 0;
    if constexpr (PSD && KS::ACC_TMEM) {
        tmem_fence_after();
        taddr = tmem_slot + (static_cast<uint32_t>(32 * (wid & 3)) << 16) + static_cast<uint32_t>(32 * (wid >> 2));
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0u;  // +0.0 in both halves of every double
        tmem_st32(taddr, z);
        if constexpr (EXT) {
            uint32_t ext[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                ext[i] = 0x7f800000u;       // +inf: minima
                ext[16 + i] = 0xff800000u;  // -inf: maxima
            }
            tmem_st32(taddr + KS::TMEM_COLS, ext);
        }
        if constexpr (WINT) {
            uint32_t wb[32];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const double w = __ldg(a.win + j + r * (N / 16));
                wb[2 * r] = static_cast<uint32_t>(__double2loint(w));
                wb[2 * r + 1] = static_cast<uint32_t>(__double2hiint(w));
            }
            tmem_st32(taddr + WOFF, wb);
            tmem_wait_st();
        }
    }
    if (lt == 0 && it_begin < it_end) {
        StageIssue first{stage, nullptr, 0u, bar, true, true};
        chunk(it_begin, &first.src, &first.bytes);
        first();
    }

    constexpr int NACC = (PSD && !KS::ACC_TMEM) ? (G == 1 ? PL::P : (N >= PL::NT ? N / PL::NT : 1)) : 1;
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;

    constexpr int RL = PL::radix(PL::NP - 1);
    constexpr int NSL = PL::ns(PL::NP - 1);
    constexpr int UL = PL::P / RL;
    uint32_t phase = 0;
    for (long long it = it_begin; it < it_end; it += it_step) {
        const long long r0 = row_base + it * G;
        const long long row = r0 + g;
        const bool valid = G == 1 || row < row_limit;  // G == 1: the iteration space is exactly the rows

        uint32_t wb[WINT ? 32 : 1];
        if constexpr (WINT) tmem_ld32(taddr + WOFF, wb);
        mbar_wait(bar, phase);
        phase ^= 1;
        if constexpr (WINT) tmem_wait_ld();

        // pass-0 inputs from the stage
        cd v[16];
        // int16 IQ, no window: pass 0's first DFT4 layer in integer arithmetic
        constexpr bool INT_L1 = FMT == 1 && !WIN && PL::radix(0) == 16 && PL::P == 16;
        if constexpr (INT_L1) {
            int re[16], im[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int sidx = g * N + j + r * (N / 16);
                const short2 x = valid ? reinterpret_cast<const short2*>(stage)[sidx] : make_short2(0, 0);
                re[r] = x.x;
                im[r] = x.y;
            }
            dft16_layer1_int(re, im, v);  // v holds y
        } else {
            constexpr int R0 = PL::radix(0);
            constexpr int U0 = PL::P / R0;
#pragma unroll
            for (int u = 0; u < U0; ++u) {
                const int b = j + PL::TPR * u;
#pragma unroll
                for (int r = 0; r < R0; ++r) {
                    const int n = b + r * (N / R0);  // sample position within the frame
                    const int s = (WIN ? g * a.hop : g * N) + n;
                    if constexpr (FMT == 0) {
                        const float2 x = valid ? reinterpret_cast<const float2*>(stage)[s] : make_float2(0.f, 0.f);
                        v[u * R0 + r] = {static_cast<double>(x.x), static_cast<double>(x.y)};
                    } else {
                        const short2 x = valid ? reinterpret_cast<const short2*>(stage)[s] : make_short2(0, 0);
                        // frontend.cpp:383: raw * (1.0f/32768) is exact; the 2^-15 is applied
                        // to the magnitudes instead (mags<P, 15>), bit-identically
                        v[u * R0 + r] = {static_cast<double>(x.x), static_cast<double>(x.y)};
                    }
                    if constexpr (WIN) {  // STFT extension: one rounded product per component
                        const double w = WINT ? __hiloint2double(static_cast<int>(wb[WINT ? 2 * r + 1 : 0]), static_cast<int>(wb[WINT ? 2 * r : 0]))
                                              : __ldg(a.win + n);
                        v[u * R0 + r] = {__dmul_rn(v[u * R0 + r].re, w), __dmul_rn(v[u * R0 + r].im, w)};
                    }
                }
            }
        }
        StageIssue nxt{stage, nullptr, 0u, bar, it + it_step < it_end, lt == 0};
        if (nxt.go) chunk(it + it_step, &nxt.src, &nxt.bytes);
        if constexpr (PL::NP == 1) {  // no exchange barrier to piggy-back on
            group_sync(bar_id, PL::NT);
            nxt();
        }
        cd w0[16];  // pass 0 has no twiddles (Ns = 1)
        passes_from<LOGN, 0, KS::TW_SMEM, KS::CX, INT_L1>(v, j, tw, mybuf, bar_id, nxt, w0);

        // epilogue: outputs of the last pass, index q = b + r*NS_last
        float m[PL::P];
        // G == 1 PSD: the TMEM load of this thread's column sums is issued
        // before the magnitudes, so its latency overlaps them (measured:
        // -1 % vs after the stores)
        uint32_t t[32];
        if constexpr (G == 1 && PSD) {
            tmem_wait_st();  // the previous row's update has landed
            tmem_ld32(taddr, t);
        }
        mags<PL::P, FMT == 1 ? 15 : 0>(v, m);
        if constexpr (G == 1) {
            float* out = a.tf ? a.tf + row * N : nullptr;
#pragma unroll
            for (int u = 0; u < UL; ++u) {
#pragma unroll
                for (int r = 0; r < RL; ++r) {
                    const int q = j + PL::TPR * u + r * NSL;
                    // j < TPR and every other term is a multiple of TPR: the DC shift is a constant offset
                    const int k = j + ((q - j + N / 2) & (N - 1));
                    if (valid && out) out[k] = m[u * RL + r];
                }
            }
            if constexpr (PSD) {
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < PL::P; ++i) {
                    const double md = static_cast<double>(m[i]);
                    const double s = __fma_rn(md, md, __hiloint2double(static_cast<int>(t[2 * i + 1]), static_cast<int>(t[2 * i])));
                    t[2 * i] = static_cast<uint32_t>(__double2loint(s));
                    t[2 * i + 1] = static_cast<uint32_t>(__double2hiint(s));
                }
                tmem_st32(taddr, t);
                if constexpr (EXT) {  // column extremes for K4 (order-free, exact)
                    uint32_t e[32];
                    tmem_ld32(taddr + KS::TMEM_COLS, e);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < PL::P; ++i) {
                        e[i] = __float_as_uint(fminf(__uint_as_float(e[i]), m[i]));
                        e[16 + i] = __float_as_uint(fmaxf(__uint_as_float(e[16 + i]), m[i]));
                    }
                    tmem_st32(taddr + KS::TMEM_COLS, e);
                }
            }
        } else {
            // stage magnitudes so stores are row-contiguous and PSD runs in row order
            float* mrow = magbuf + g * N;
#pragma unroll
            for (int u = 0; u < UL; ++u) {
#pragma unroll
                for (int r = 0; r < RL; ++r) {
                    const int q = j + PL::TPR * u + r * NSL;
                    // j < TPR and every other term is a multiple of TPR: the DC shift is a constant offset
                    const int k = j + ((q - j + N / 2) & (N - 1));
                    mrow[k] = m[u * RL + r];
                }
            }
            group_sync(bar_id, PL::NT);
            long long nvalid = row_limit - r0;
            if (nvalid > G) nvalid = G;
            if (a.tf) {
                float* out = a.tf + r0 * N;
                const int total = static_cast<int>(nvalid) * N;
                for (int e = lt; e < total; e += PL::NT) out[e] = magbuf[e];
            }
            if constexpr (PSD) {
#pragma unroll
                for (int i = 0; i < NACC; ++i) {
                    const int c = lt + PL::NT * i;
                    if (c < N) {
                        for (int gg = 0; gg < nvalid; ++gg) {
                            const double md = static_cast<double>(magbuf[gg * N + c]);
                            acc[i] = __fma_rn(md, md, acc[i]);
                        }
                    }
                }
            }
            group_sync(bar_id, PL::NT);
        }
    }

    if constexpr (PSD) {
        const long long plot = static_cast<long long>(blockIdx.x) * KS::GROUPS + gi;
        if (plot < a.n_plots) {
            const double inv_rows = __ddiv_rn(1.0, static_cast<double>(a.rows_per_plot));
            float* psd = a.psd + plot * N;
            if constexpr (G == 1) {
                uint32_t t[32];
                tmem_wait_st();
                tmem_ld32(taddr, t);
                tmem_wait_ld();
#pragma unroll
                for (int u = 0; u < UL; ++u)
#pragma unroll
                    for (int r = 0; r < RL; ++r) {
                        const int i = u * RL + r;
                        const int q = j + PL::TPR * u + r * NSL;
                        // j < TPR and every other term is a multiple of TPR: the DC shift is a constant offset
                    const int k = j + ((q - j + N / 2) & (N - 1));
                        const double sum = __hiloint2double(static_cast<int>(t[2 * i + 1]), static_cast<int>(t[2 * i]));
                        psd[k] = __double2float_rn(__dmul_rn(sum, inv_rows));
                    }
                if constexpr (EXT) {
                    tmem_ld32(taddr + KS::TMEM_COLS, t);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < UL; ++u)
#pragma unroll
                        for (int r = 0; r < RL; ++r) {
                            const int i = u * RL + r;
                            const int k = j + ((PL::TPR * u + r * NSL + N / 2) & (N - 1));
                            a.col_lo[plot * N + k] = __uint_as_float(t[i]);
                            a.col_hi[plot * N + k] = __uint_as_float(t[16 + i]);
                        }
                }
            } else {
#pragma unroll
                for (int i = 0; i < NACC; ++i) {
                    const int c = lt + PL::NT * i;
                    if (c < N) psd[c] = __double2float_rn(__dmul_rn(acc[i], inv_rows));
                }
            }
        }
        if constexpr (KS::ACC_TMEM) {
            tmem_wait_st();
            tmem_fence_before();
            __syncthreads();  // every warp is done with its columns
            tmem_fence_after();
            if (wid == 0) tmem_dealloc<KS::tmem_alloc_cols(EXT, WINT)>(tmem_slot);
        }
    }
}

} // namespace ssb

// ------------------------------------------------------------------ host side


namespace ssb {

// SSFFT-1 canonical twiddles tw[e] = (cos t, -sin t), t = (2 pi e)/N, expanded
// into the per-pass layout the kernel reads: pass p (Ns > 1) block holds
// tw[r*k*N/(Ns*R)] at (r-1)*Ns + k.
template <int LOGN>
static void build_tw(std::vector<double2>& out) {
    using PL = FftPlan<LOGN>;
    constexpr int N = PL::N;
    std::vector<double2> canon(N);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int e = 0; e < N; ++e) {
        const double t = (two_pi * static_cast<double>(e)) / static_cast<double>(N);
        canon[e] = make_double2(std::cos(t), -std::sin(t));
    }
    out.assign(PL::tw_size() > 0 ? PL::tw_size() : 1, make_double2(0, 0));
    for (int p = 1; p < PL::NP; ++p) {
        const int R = PL::radix(p), NS = PL::ns(p);
        const size_t s = static_cast<size_t>(N / (NS * R));
        double2* blk = out.data() + PL::tw_off(p);
        for (int r = 1; r < R; ++r)
            for (int k = 0; k < NS; ++k) blk[(r - 1) * NS + k] = canon[r * k * s];
    }
}

template <int LOGN, int FMT, bool PSD, bool WIN, bool EXT = false>
static cudaError_t ensure_smem_attr() {
    static std::atomic<unsigned long long> attr_done;  // per instantiation, one bit per device
    return set_attr_once(attr_done, [] {
        return cudaFuncSetAttribute(fft_mag_kernel<LOGN, FMT, PSD, WIN, EXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(K1Shape<LOGN>::smem(FMT == 0 ? 8 : 4)));
    });
}

// plots the fused-PSD grid processes concurrently per SM (one plot per row group)
template <int LOGN, int FMT, bool WIN>
static int psd_slots_one() {
    if (ensure_smem_attr<LOGN, FMT, true, WIN>() != cudaSuccess) return 0;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fft_mag_kernel<LOGN, FMT, true, WIN, false>,
                                                      K1Shape<LOGN>::THREADS,
                                                      K1Shape<LOGN>::smem(FMT == 0 ? 8 : 4)) != cudaSuccess)
        return 0;
    return blocks * K1Shape<LOGN>::GROUPS;
}

template <int LOGN, int FMT, bool PSD, bool WIN, bool EXT = false>
static cudaError_t launch_one(const FftLaunch& L, cudaStream_t st) {
    using PL = FftPlan<LOGN>;
    using KS = K1Shape<LOGN>;
    auto kern = fft_mag_kernel<LOGN, FMT, PSD, WIN, EXT>;
    const size_t smem = KS::smem(FMT == 0 ? 8 : 4);
    cudaError_t e = ensure_smem_attr<LOGN, FMT, PSD, WIN, EXT>();
    if (e != cudaSuccess) return e;
    FftArgs a;
    a.iq = L.iq;
    a.tf = L.tf;
    a.psd = L.psd_out;
    a.col_lo = EXT ? L.col_lo : nullptr;
    a.col_hi = EXT ? L.col_hi : nullptr;
    a.tw = L.tw;
    a.total_rows = L.total_rows;
    a.rows_per_plot = L.rows_per_plot;
    a.n_plots = L.n_plots;
    a.hop = L.hop > 0 ? L.hop : PL::N;
    a.win = L.win;
    long long grid;
    if (PSD) {
        grid = (L.n_plots + KS::GROUPS - 1) / KS::GROUPS;
    } else {
        const long long iters = (L.total_rows + PL::G - 1) / PL::G;
        const long long groups = (iters + KS::GROUPS - 1) / KS::GROUPS;
        grid = groups < L.num_sms ? groups : L.num_sms;
    }
    if (grid <= 0) return cudaSuccess;
    kern<<<static_cast<unsigned>(grid), KS::THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

template <int LOGN>
static cudaError_t dispatch_fmt(const FftLaunch& L, cudaStream_t st) {
    if constexpr (K1Shape<LOGN>::ACC_TMEM) {  // fused PSD + column extremes (K4's cluster form)
        if (L.psd && L.col_lo) {
            if (L.win) return L.fmt == 0 ? launch_one<LOGN, 0, true, true, true>(L, st) : launch_one<LOGN, 1, true, true, true>(L, st);
            return L.fmt == 0 ? launch_one<LOGN, 0, true, false, true>(L, st) : launch_one<LOGN, 1, true, false, true>(L, st);
        }
    }
    if (L.win) {
        if (L.fmt == 0) return L.psd ? launch_one<LOGN, 0, true, true>(L, st) : launch_one<LOGN, 0, false, true>(L, st);
        return L.psd ? launch_one<LOGN, 1, true, true>(L, st) : launch_one<LOGN, 1, false, true>(L, st);
    }
    if (L.fmt == 0) return L.psd ? launch_one<LOGN, 0, true, false>(L, st) : launch_one<LOGN, 0, false, false>(L, st);
    return L.psd ? launch_one<LOGN, 1, true, false>(L, st) : launch_one<LOGN, 1, false, false>(L, st);
}

// STFT extension window (BASELINE config 5: "4096-pt Hann STFT with 50%
// overlap"; no reference oracle -- SURVEY.md §8(f) F2): periodic Hann,
// w[n] = 0.5 * (1 - cos(t)), t = (2 pi n) / N, glibc cos in double.
void fft_window(int n_fft, int kind, std::vector<double>& out) {
    out.assign(static_cast<size_t>(n_fft), 1.0);
    if (kind != 1) return;
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int n = 0; n < n_fft; ++n) {
        const double t = (two_pi * static_cast<double>(n)) / static_cast<double>(n_fft);
        out[static_cast<size_t>(n)] = 0.5 * (1.0 - std::cos(t));
    }
}

cudaError_t fft_mag_launch(const FftLaunch& L, cudaStream_t st) {
    switch (L.logn) {
    case 3: return dispatch_fmt<3>(L, st);
    case 4: return dispatch_fmt<4>(L, st);
    case 5: return dispatch_fmt<5>(L, st);
    case 6: return dispatch_fmt<6>(L, st);
    case 7: return dispatch_fmt<7>(L, st);
    case 8: return dispatch_fmt<8>(L, st);
    case 9: return dispatch_fmt<9>(L, st);
    case 10: return dispatch_fmt<10>(L, st);
    case 11: return dispatch_fmt<11>(L, st);
    case 12: return dispatch_fmt<12>(L, st);
    case 13: return dispatch_fmt<13>(L, st);
    default: return cudaErrorInvalidValue;
    }
}

template <int LOGN>
static int psd_slots_fmt(int fmt, bool win) {
    if (win) return fmt == 0 ? psd_slots_one<LOGN, 0, true>() : psd_slots_one<LOGN, 1, true>();
    return fmt == 0 ? psd_slots_one<LOGN, 0, false>() : psd_slots_one<LOGN, 1, false>();
}

bool fft_psd_extremes(int logn) { return logn == 12 || logn == 13; }  // the TMEM (one row per group) shapes

int fft_psd_slots_per_sm(int logn, int fmt, bool win) {
    switch (logn) {
    case 3: return psd_slots_fmt<3>(fmt, win);
    case 4: return psd_slots_fmt<4>(fmt, win);
    case 5: return psd_slots_fmt<5>(fmt, win);
    case 6: return psd_slots_fmt<6>(fmt, win);
    case 7: return psd_slots_fmt<7>(fmt, win);
    case 8: return psd_slots_fmt<8>(fmt, win);
    case 9: return psd_slots_fmt<9>(fmt, win);
    case 10: return psd_slots_fmt<10>(fmt, win);
    case 11: return psd_slots_fmt<11>(fmt, win);
    case 12: return psd_slots_fmt<12>(fmt, win);
    case 13: return psd_slots_fmt<13>(fmt, win);
    default: return 0;
    }
}

// ------------------------------------------------------------- large N
// n_fft = 2^14 .. 2^20 (one row no longer fits one CTA's shared memory): the
// same SSFFT-2 passes, one kernel per pass over global double2 scratch,
// then a magnitude kernel with the reference's exact expression.  Slower than
// K1, but the arithmetic -- and so every output bit -- is identical.
struct RtPlan {
    int logn, n, np;
    int radix[8], ns[8];
    long long w1off[8];  // offset of pass p's w1 block (Ns entries) in the compact table
    long long w1size;
};

static RtPlan rt_plan(int logn) {
    RtPlan P{};
    P.logn = logn;
    P.n = 1 << logn;
    P.np = logn / 4 + (logn % 4 ? 1 : 0);
    int ns = 1;
    long long off = 0;
    for (int p = 0; p < P.np; ++p) {
        P.radix[p] = p < logn / 4 ? 16 : (1 << (logn % 4));
        P.ns[p] = ns;
        P.w1off[p] = off;
        if (p > 0) off += ns;
        ns *= P.radix[p];
    }
    P.w1size = off > 0 ? off : 1;
    return P;
}

// w1 of pass p (Ns > 1), butterfly class k: canonical tw[k * N / (Ns * R)]
static void build_w1(const RtPlan& P, std::vector<double2>& out) {
    out.assign(static_cast<size_t>(P.w1size), make_double2(0, 0));
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int p = 1; p < P.np; ++p) {
        const long long s = P.n / (static_cast<long long>(P.ns[p]) * P.radix[p]);
        for (int k = 0; k < P.ns[p]; ++k) {
            const double t = (two_pi * static_cast<double>(k * s)) / static_cast<double>(P.n);
            out[static_cast<size_t>(P.w1off[p] + k)] = make_double2(std::cos(t), -std::sin(t));
        }
    }
}

template <int R>
__device__ __forceinline__ void twiddle_tree(cd* v, cd w1) {
    // SSFFT-2 powers of w1, applied in the spec's product order (run_pass)
    cd w[16];
    w[1] = w1;
    if constexpr (R > 2) w[2] = c_mul(w[1], w[1]);
    if constexpr (R > 3) w[3] = c_mul(w[2], w[1]);
    if constexpr (R > 4) {
        w[4] = c_mul(w[2], w[2]);
        w[5] = c_mul(w[4], w[1]);
        w[6] = c_mul(w[4], w[2]);
        w[7] = c_mul(w[4], w[3]);
    }
    if constexpr (R > 8) {
        w[8] = c_mul(w[4], w[4]);
#pragma unroll
        for (int q = 9; q < 16; ++q) w[q] = c_mul(w[8], w[q - 8]);
    }
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = c_mul(v[r], w[r]);
}

// One Stockham pass.  FIRST: read the IQ rows (frames every hop samples,
// optional window) instead of the scratch.
template <int R, bool FIRST, int FMT>
__global__ void large_pass_kernel(const void* __restrict__ src, double2* __restrict__ dst, int n, int ns, int hop,
                                  const double* __restrict__ win, const double2* __restrict__ w1, long long rows) {
    const int nb = n / R;
    const long long total = rows * nb;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = idx / nb;
        const int j = static_cast<int>(idx % nb);
        cd v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = j + r * nb;
            if constexpr (FIRST) {
                const long long at = row * hop + e;
                if constexpr (FMT == 0) {
                    const float2 x = static_cast<const float2*>(src)[at];
                    v[r] = {static_cast<double>(x.x), static_cast<double>(x.y)};
                } else {
                    const short2 x = static_cast<const short2*>(src)[at];
                    v[r] = {__dmul_rn(static_cast<double>(x.x), 0x1p-15), __dmul_rn(static_cast<double>(x.y), 0x1p-15)};
                }
                if (win) {
                    const double w = __ldg(win + e);
                    v[r] = {__dmul_rn(v[r].re, w), __dmul_rn(v[r].im, w)};
                }
            } else {
                const double2 x = static_cast<const double2*>(src)[row * n + e];
                v[r] = {x.x, x.y};
            }
        }
        const int k = j % ns;
        if (ns > 1) {
            const double2 t = __ldg(w1 + k);
            twiddle_tree<R>(v, cd{t.x, t.y});
        }
        dft_r<R>(v);
        const long long base = row * n + static_cast<long long>(j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[base + static_cast<long long>(r) * ns] = make_double2(v[r].re, v[r].im);
    }
}

// out[row][k] = float(sqrt(fma(re, re, im * im))) of X[(k + N/2) mod N]
__global__ void large_mag_kernel(const double2* __restrict__ x, float* __restrict__ out, int n, long long rows) {
    const long long total = rows * n;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = idx / n;
        const int k = static_cast<int>(idx % n);
        const double2 v = x[row * n + ((k + n / 2) & (n - 1))];
        out[idx] = __double2float_rn(__dsqrt_rn(__fma_rn(v.x, v.x, __dmul_rn(v.y, v.y))));
    }
}

template <bool FIRST, int FMT>
static void large_pass(int R, const void* src, double2* dst, int n, int ns, int hop, const double* win,
                       const double2* w1, long long rows, int num_sms, cudaStream_t st) {
    const long long work = rows * (n / R);
    const unsigned grid = static_cast<unsigned>(std::min<long long>((work + 255) / 256, 32LL * num_sms));
    switch (R) {
    case 16: large_pass_kernel<16, FIRST, FMT><<<grid, 256, 0, st>>>(src, dst, n, ns, hop, win, w1, rows); break;
    case 8: large_pass_kernel<8, FIRST, FMT><<<grid, 256, 0, st>>>(src, dst, n, ns, hop, win, w1, rows); break;
    case 4: large_pass_kernel<4, FIRST, FMT><<<grid, 256, 0, st>>>(src, dst, n, ns, hop, win, w1, rows); break;
    default: large_pass_kernel<2, FIRST, FMT><<<grid, 256, 0, st>>>(src, dst, n, ns, hop, win, w1, rows); break;
    }
}

size_t fft_large_w1_count(int logn) { return static_cast<size_t>(rt_plan(logn).w1size); }
void fft_large_w1(int logn, std::vector<double2>& out) { build_w1(rt_plan(logn), out); }

// rows of frames -> TF rows, in row chunks that keep the two double2 scratch
// buffers (a, b: chunk_rows * n each) bounded.  Returns the kernels launched.
cudaError_t fft_large_launch(const FftLaunch& L, const double2* w1, double2* a, double2* b, long long chunk_rows,
                             cudaStream_t st, int* launches) {
    const RtPlan P = rt_plan(L.logn);
    const int hop = L.hop > 0 ? L.hop : P.n;
    const size_t sb = L.fmt == 0 ? sizeof(float2) : sizeof(short2);
    int nl = 0;
    for (long long r0 = 0; r0 < L.total_rows; r0 += chunk_rows) {
        const long long rows = std::min(chunk_rows, L.total_rows - r0);
        const void* src = static_cast<const unsigned char*>(L.iq) + r0 * hop * sb;
        double2* in = a;
        double2* out = b;
        for (int pidx = 0; pidx < P.np; ++pidx) {
            const double2* wp = w1 + P.w1off[pidx];
            if (pidx == 0) {
                if (L.fmt == 0) large_pass<true, 0>(P.radix[0], src, out, P.n, 1, hop, L.win, wp, rows, L.num_sms, st);
                else large_pass<true, 1>(P.radix[0], src, out, P.n, 1, hop, L.win, wp, rows, L.num_sms, st);
            } else {
                large_pass<false, 0>(P.radix[pidx], in, out, P.n, P.ns[pidx], hop, nullptr, wp, rows, L.num_sms, st);
            }
            ++nl;
            double2* t = in;
            in = out;
            out = t;
        }
        const unsigned grid = static_cast<unsigned>(std::min<long long>((rows * P.n + 255) / 256, 32LL * L.num_sms));
        large_mag_kernel<<<grid, 256, 0, st>>>(in, L.tf + r0 * P.n, P.n, rows);
        ++nl;
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (launches) *launches = nl;
    return cudaSuccess;
}

void fft_twiddles(int logn, std::vector<double2>& out) {
    switch (logn) {
    case 3: build_tw<3>(out); break;
    case 4: build_tw<4>(out); break;
    case 5: build_tw<5>(out); break;
    case 6: build_tw<6>(out); break;
    case 7: build_tw<7>(out); break;
    case 8: build_tw<8>(out); break;
    case 9: build_tw<9>(out); break;
    case 10: build_tw<10>(out); break;
    case 11: build_tw<11>(out); break;
    case 12: build_tw<12>(out); break;
    case 13: build_tw<13>(out); break;
    default: out.clear();
    }
}

} // namespace ssb
