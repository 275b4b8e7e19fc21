// binarize.cu -- K4: per-column Otsu binarisation over the active columns.
//
// Replaces detector::binarize_columns / binarize / otsu_threshold
// (proj/src/detector.cpp:273-341, helpers :22-73).  One CTA per (plot,
// 32-column mask word).  Words with no active column write background and
// exit.  Otherwise three row sweeps over the word's 32 columns (one 128-byte
// line per row, so every warp load is a single coalesced line):
//   A  column min / max over all rows             (:284-293)
//   B  256-bin histograms in shared memory         (:314-320)
//      -> Otsu split per column, one warp per column: integer prefix sums,
//         between-class variance ((w0*w1)*(mu0-mu1))*(mu0-mu1) in double
//         per split, first-maximum argmax (:43-67); threshold (:69-73)
//   C  mask = v > thr, packed with __ballot_sync into the word  (:328-334)
// Sweep A streams from HBM; B and C re-read the same 32 x T block, which the
// 126 MB L2 still holds (DESIGN.md §4 K4).
#include "common.cuh"
#include "internal.h"

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

namespace cg = cooperative_groups;

namespace ssb {

constexpr int kBinThreads = 256;
constexpr int kBinWarps = kBinThreads / 32;
constexpr int kHistStride = 257;  // padded so column l, bin b hits bank (l + b) % 32

// bin_of (detector.cpp:36-39): trunc(fl(fl(v - lo) * scale)) clamped to 255.
// y >= 0 here, so trunc = floor, taken as the low mantissa bits of
// fl_rd(y + 2^23) -- an FP32 add instead of an F2I on the XU pipe.  The
// unsigned clamp also sends NaN / +inf (only from non-finite input, undefined
// behaviour in the reference) to bin 255, in bounds.
__device__ __forceinline__ int bin_index(float v, float lo, float scale) {
    const float y = __fmul_rn(__fsub_rn(v, lo), scale);
    return static_cast<int>(min(static_cast<uint32_t>(__float_as_int(__fadd_rd(y, 8388608.0f))) - 0x4B000000u, 255u));
}

__device__ __forceinline__ double rcp_newton(double p) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
#pragma unroll
    for (int k = 0; k < 2; ++k) r = __fma_rn(r, __fma_rn(-p, r, 1.0), r);
    return r;
}

// otsu_split (detector.cpp:43-67) for one column, one warp: lane owns bins
// 8*lane .. 8*lane+7 (hq).  Counts and bin-weighted sums are integers below
// 2^53, so their prefix sums are exact in double, in any order.
//
// The reference evaluates var_i = ((w0*w1)*(mu0-mu1))*(mu0-mu1) with two
// divides per split.  Here every split first gets a cheap estimate of the
// exact rational it rounds, X_i = D^2 / (w0 w1), D = sum0*w1 - sum1*w0
// (exact in double: |D| < 2^50), with a Newton reciprocal (rel. err. < 2^-38).
// Rounding analysis of the reference's expression: |var_i - X_i| <= w0 w1
// 2^-34.4 + 2^-52 X_i (mu's <= 255 carry 2^-53 relative error, the difference
// at most 3*255 ulps of 2^-53, two rounded products).  So every split whose
// var_i equals the maximum has estimate >= M - tol with M the largest
// estimate and tol = M 2^-30 + total^2 2^-34; only those candidates (nearly
// always one) run the reference's exact divides, and the first maximum among
// them is the reference's split.  Empty bins i > 0 repeat bin i-1's
// (w0, sum0), so they can never be the first maximum and are skipped.
__device__ __forceinline__ int otsu_split_warp(const uint32_t* hq, int lane) {
    double cnt[8], wsum[8];
    double lc = 0.0, ls = 0.0;
    uint32_t nz = 0;  // bins whose count is non-zero (or bin 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int bin = lane * 8 + q;
        const double h = static_cast<double>(hq[q]);
        lc = __dadd_rn(lc, h);
        ls = __fma_rn(static_cast<double>(bin), h, ls);
        cnt[q] = lc;
        wsum[q] = ls;
        nz |= (hq[q] != 0u || bin == 0) ? (1u << q) : 0u;
    }
    // exclusive prefix over lanes of (lc, ls)
    double pc = lc, ps = ls;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double tc = __shfl_up_sync(0xffffffffu, pc, o);
        const double ts = __shfl_up_sync(0xffffffffu, ps, o);
        if (lane >= o) {
            pc = __dadd_rn(pc, tc);
            ps = __dadd_rn(ps, ts);
        }
    }
    const double total = __shfl_sync(0xffffffffu, pc, 31);
    const double sum_all = __shfl_sync(0xffffffffu, ps, 31);
    pc = __dsub_rn(pc, lc);
    ps = __dsub_rn(ps, ls);

    // estimates
    double est[8];
    double m = -1.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double w0 = __dadd_rn(pc, cnt[q]);
        const double w1 = __dsub_rn(total, w0);
        double e = ((nz >> q) & 1u) ? 0.0 : -1.0;
        if (((nz >> q) & 1u) && w0 > 0.0 && w1 > 0.0) {
            const double s0 = __dadd_rn(ps, wsum[q]);
            const double s1 = __dsub_rn(sum_all, s0);
            const double d = __fma_rn(s0, w1, -__dmul_rn(s1, w0));
            const double p = __dmul_rn(w0, w1);
            e = __dmul_rn(__dmul_rn(d, d), rcp_newton(p));
        }
        est[q] = e;
        m = fmax(m, e);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double floor_v = m - (m * 0x1p-30 + total * total * 0x1p-34);

    double best_v = -1.0;
    int best_i = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (est[q] >= floor_v && est[q] >= 0.0) {
            const double w0 = __dadd_rn(pc, cnt[q]);
            const double w1 = __dsub_rn(total, w0);
            double var = 0.0;
            if (w0 > 0.0 && w1 > 0.0) {
                const double sum0 = __dadd_rn(ps, wsum[q]);
                const double mu0 = __ddiv_rn(sum0, w0);
                const double mu1 = __ddiv_rn(__dsub_rn(sum_all, sum0), w1);
                const double d = __dsub_rn(mu0, mu1);
                var = __dmul_rn(__dmul_rn(__dmul_rn(w0, w1), d), d);
            }
            if (var > best_v) {
                best_v = var;
                best_i = lane * 8 + q;
            }
        }
    }
    // first maximum across lanes (ties -> lowest split index)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best_v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (ov > best_v || (ov == best_v && oi < best_i)) {
            best_v = ov;
            best_i = oi;
        }
    }
    return best_i;
}

// Tile path (<= 2 * kTileMaxRows rows per column): the same search with the
// prefix sums in uint32.
__device__ __forceinline__ int otsu_split_warp_u32(const uint32_t* hq, int lane) {
    // counts and bin-weighted sums are integers below 2^32 (<= 12288 rows of
    // one column, bins <= 255): their prefix sums are exact in uint32, in any
    // order, and convert exactly to the doubles the reference accumulates
    uint32_t cnt[8], wsum[8];
    uint32_t lc = 0u, ls = 0u;
    uint32_t nz = 0;  // bins whose count is non-zero (or bin 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t bin = static_cast<uint32_t>(lane * 8 + q);
        lc += hq[q];
        ls += bin * hq[q];
        cnt[q] = lc;
        wsum[q] = ls;
        nz |= (hq[q] != 0u || bin == 0u) ? (1u << q) : 0u;
    }
    // exclusive prefix over lanes of (lc, ls)
    uint32_t pcu = lc, psu = ls;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t tc = __shfl_up_sync(0xffffffffu, pcu, o);
        const uint32_t ts = __shfl_up_sync(0xffffffffu, psu, o);
        if (lane >= o) {
            pcu += tc;
            psu += ts;
        }
    }
    const uint32_t total_u = __shfl_sync(0xffffffffu, pcu, 31);
    const uint32_t sum_all_u = __shfl_sync(0xffffffffu, psu, 31);
    pcu -= lc;
    psu -= ls;
    const double total = static_cast<double>(total_u);
    const double sum_all = static_cast<double>(sum_all_u);

    // estimates X_i = D^2 / p, D = sum0*w1 - sum1*w0 exactly in int64
    // (|D| < 2^37), p = w0*w1 < 2^26.  First in FP32 for every split
    // (relative error < 2^-21: D and p rounded once, rcp.approx within an ulp,
    // two rounded products), then in double only for the splits that can
    // still be candidates.  With f the float and e the double estimates
    // (|e - X| <= 2^-37 X), every candidate i (e_i >= M_e - tol, below) has
    // f_i >= (1 - 2^-18) M_f - total^2 2^-34, M_f = max f (the argmax of e is a
    // candidate itself, so M_e is the maximum over the kept splits).  Bins
    // with a count but no split (w0 or w1 = 0) have X = 0 exactly; empty bins
    // none (-1).
    float fe[8];
    uint32_t cls0 = 0, cls2 = 0;  // splits with X = 0 exactly / with an estimate
    long long dds[8];
    uint32_t ps[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t w0 = pcu + cnt[q];
        const uint32_t w1 = total_u - w0;
        const uint32_t s0 = psu + wsum[q];
        const uint32_t s1 = sum_all_u - s0;
        dds[q] = static_cast<long long>(s0) * w1 - static_cast<long long>(s1) * w0;
        ps[q] = w0 * w1;
        fe[q] = 0.0f;
        if ((nz >> q) & 1u) {
            if (w0 > 0u && w1 > 0u) {
                const float df = __ll2float_rn(dds[q]);
                float r;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint2float_rn(ps[q])));
                fe[q] = __fmul_rn(__fmul_rn(df, df), r);
                cls2 |= 1u << q;
            } else {
                cls0 |= 1u << q;
            }
        }
    }
    float mfl = 0.0f;
#pragma unroll
    for (int q = 0; q < 8; ++q) mfl = fmaxf(mfl, fe[q]);
    const float mf = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mfl)));  // f >= 0: bit order
    const double thr = static_cast<double>(mf) * (1.0 - 0x1p-17) - total * total * 0x1p-33;  // 2x margins
    uint32_t kept = cls0 & (thr <= 0.0 ? 0xffu : 0u);
#pragma unroll
    for (int q = 0; q < 8; ++q) kept |= ((cls2 >> q) & 1u) && static_cast<double>(fe[q]) >= thr ? (1u << q) : 0u;

    double est[8];
    double m = -1.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        double e = -1.0;
        if (__any_sync(0xffffffffu, (kept >> q) & 1u)) {  // nearly always one or two q of the eight
            if ((kept >> q) & 1u) {
                e = 0.0;
                if ((cls2 >> q) & 1u) {
                    const double d = static_cast<double>(dds[q]);
                    e = __dmul_rn(__dmul_rn(d, d), rcp_newton(static_cast<double>(ps[q])));
                }
            }
        }
        est[q] = e;
        m = fmax(m, e);
    }
    // warp maximum of the estimates, exactly, by two 32-bit REDUX steps on the
    // bit patterns (order-preserving for the non-negative doubles; the -1
    // placeholders map to +0; the kept set is never empty)
    {
        const unsigned long long key = m > 0.0 ? static_cast<unsigned long long>(__double_as_longlong(m)) : 0ull;
        const uint32_t khi = static_cast<uint32_t>(key >> 32);
        const uint32_t mhi = __reduce_max_sync(0xffffffffu, khi);
        const uint32_t mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? static_cast<uint32_t>(key) : 0u);
        m = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
    }
    const double floor_v = m - (m * 0x1p-30 + total * total * 0x1p-34);

    // the reference's split is among the candidates (estimate >= floor_v);
    // when there is exactly one -- nearly always -- it is the split, and the
    // exact divides and the first-maximum reduction are not needed
    uint32_t cand = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) cand |= (est[q] >= floor_v && est[q] >= 0.0) ? (1u << q) : 0u;
    const uint32_t n_cand = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(__popc(cand)));
    if (n_cand == 1u) {
        const uint32_t holders = __ballot_sync(0xffffffffu, cand != 0u);
        const int src = __ffs(static_cast<int>(holders)) - 1;
        return __shfl_sync(0xffffffffu, lane * 8 + __ffs(static_cast<int>(cand)) - 1, src);
    }

    double best_v = -1.0;
    int best_i = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if ((cand >> q) & 1u) {
            const uint32_t w0u = pcu + cnt[q];
            const double w0 = static_cast<double>(w0u);
            const double w1 = static_cast<double>(total_u - w0u);
            double var = 0.0;
            if (w0 > 0.0 && w1 > 0.0) {
                const double sum0 = static_cast<double>(psu + wsum[q]);
                const double mu0 = __ddiv_rn(sum0, w0);
                const double mu1 = __ddiv_rn(__dsub_rn(sum_all, sum0), w1);
                const double d = __dsub_rn(mu0, mu1);
                var = __dmul_rn(__dmul_rn(__dmul_rn(w0, w1), d), d);
            }
            if (var > best_v) {
                best_v = var;
                best_i = lane * 8 + q;
            }
        }
    }
    // first maximum across lanes (ties -> lowest split index)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best_v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (ov > best_v || (ov == best_v && oi < best_i)) {
            best_v = ov;
            best_i = oi;
        }
    }
    return best_i;
}

__global__ void __launch_bounds__(kBinThreads) binarize_kernel(BinarizeLaunch a) {
    __shared__ uint32_t hist[32 * kHistStride];
    __shared__ float s_lo[kBinWarps][32], s_hi[kBinWarps][32];
    __shared__ float c_lo[32], c_scale[32], c_thr[32];
    __shared__ double c_span[32];
    __shared__ int c_use[32];

    const int wd = blockIdx.x;
    const int p = blockIdx.y;
    const int W = (a.cols + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int col = wd * 32 + lane;
    const bool in_image = col < a.cols;
    const int rows = a.rows;
    const float* tf = a.tf + static_cast<long long>(p) * rows * a.cols;
    const uint32_t abits = a.active_bits[static_cast<long long>(p) * W + wd];
    const bool u8 = a.mask_u8 != nullptr;
    const bool col_out = in_image && (!u8 || (col >= a.c0 && col < a.c1));

    if (abits == 0) {
        if (u8) {
            for (int r = warp; r < rows; r += kBinWarps)
                if (col_out) a.mask_u8[static_cast<long long>(r) * a.cols + col] = 0;
        } else if (a.mask_bits) {
            uint32_t* mb = a.mask_bits + (static_cast<long long>(p) * W + wd) * mask_rs(rows);  // word-major
            for (int r = threadIdx.x; r < rows; r += kBinThreads) mb[r] = 0;
        }
        if (a.col_thr && threadIdx.x < 32 && in_image)
            a.col_thr[static_cast<long long>(p) * a.cols + col] = INFINITY;
        if (a.col_valid && threadIdx.x < 32 && in_image)
            a.col_valid[static_cast<long long>(p) * a.cols + col] = 0;
        return;
    }
    const bool active = in_image && ((abits >> lane) & 1u);

    // ---- sweep A: min / max (std::min / std::max semantics: NaN never taken)
    float lo = INFINITY, hi = -INFINITY;
    if (in_image) {
        int r = warp;
        for (; r + 3 * kBinWarps < rows; r += 4 * kBinWarps) {
            float x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = __ldg(tf + static_cast<long long>(r + q * kBinWarps) * a.cols + col);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                lo = (x[q] < lo) ? x[q] : lo;
                hi = (hi < x[q]) ? x[q] : hi;
            }
        }
        for (; r < rows; r += kBinWarps) {
            const float x = __ldg(tf + static_cast<long long>(r) * a.cols + col);
            lo = (x < lo) ? x : lo;
            hi = (hi < x) ? x : hi;
        }
    }
    s_lo[warp][lane] = lo;
    s_hi[warp][lane] = hi;
    for (int i = threadIdx.x; i < 32 * kHistStride; i += kBinThreads) hist[i] = 0;
    __syncthreads();
    if (warp == 0) {
        float l = s_lo[0][lane], h = s_hi[0][lane];
        for (int q = 1; q < kBinWarps; ++q) {
            l = (s_lo[q][lane] < l) ? s_lo[q][lane] : l;
            h = (h < s_hi[q][lane]) ? s_hi[q][lane] : h;
        }
        const float scale = __fdiv_rn(256.0f, __fsub_rn(h, l));
        const bool valid = h > l && isfinite(scale);
        c_lo[lane] = l;
        c_scale[lane] = scale;
        c_span[lane] = __dsub_rn(static_cast<double>(h), static_cast<double>(l));
        c_use[lane] = (active && valid) ? 1 : 0;
        c_thr[lane] = INFINITY;
    }
    __syncthreads();

    // ---- sweep B: histograms of the active, non-constant columns
    const bool use = c_use[lane] != 0;
    if (__any_sync(0xffffffffu, use)) {
        const float clo = c_lo[lane], csc = c_scale[lane];
        uint32_t* h = hist + lane * kHistStride;
        int r = warp;
        for (; r + 3 * kBinWarps < rows; r += 4 * kBinWarps) {
            float x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                x[q] = use ? __ldg(tf + static_cast<long long>(r + q * kBinWarps) * a.cols + col) : 0.0f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (use) {
                    atomicAdd(h + bin_index(x[q], clo, csc), 1u);
                }
            }
        }
        for (; r < rows; r += kBinWarps) {
            if (use) {
                atomicAdd(h + bin_index(__ldg(tf + static_cast<long long>(r) * a.cols + col), clo, csc), 1u);
            }
        }
    }
    __syncthreads();

    // ---- Otsu split: one warp per column, lane owns bins 8*lane .. 8*lane+7
    for (int c = warp; c < 32; c += kBinWarps) {
        if (!c_use[c]) continue;
        uint32_t hq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) hq[q] = hist[c * kHistStride + lane * 8 + q];
        const int best_i = otsu_split_warp(hq, lane);
        if (lane == 0) {
            const double lod = static_cast<double>(c_lo[c]);
            // /256 as *2^-8: the same correctly rounded value (a power of two), no DDIV
            const double e = __dmul_rn(__dmul_rn(static_cast<double>(best_i) + 1.0, c_span[c]), 0x1p-8);
            c_thr[c] = __double2float_rn(__dadd_rn(lod, e));
        }
    }
    __syncthreads();

    if (a.col_thr && threadIdx.x < 32 && in_image)
        a.col_thr[static_cast<long long>(p) * a.cols + col] = c_thr[lane];
    if (a.col_valid && threadIdx.x < 32 && in_image)
        a.col_valid[static_cast<long long>(p) * a.cols + col] = c_use[lane];
    if (!u8 && a.mask_bits == nullptr) return;

    // ---- sweep C: threshold, packed
    const float thr = c_thr[lane];
    if (u8) {
        for (int r = warp; r < rows; r += kBinWarps) {
            if (!col_out) continue;
            const float x = in_image ? __ldg(tf + static_cast<long long>(r) * a.cols + col) : 0.0f;
            a.mask_u8[static_cast<long long>(r) * a.cols + col] = x > thr ? 1 : 0;
        }
    } else {
        uint32_t* mb = a.mask_bits + (static_cast<long long>(p) * W + wd) * mask_rs(rows);  // word-major
        int r = warp;
        for (; r + 3 * kBinWarps < rows; r += 4 * kBinWarps) {
            float x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                x[q] = in_image ? __ldg(tf + static_cast<long long>(r + q * kBinWarps) * a.cols + col) : 0.0f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t word = __ballot_sync(0xffffffffu, in_image && x[q] > thr);
                if (lane == 0) mb[r + q * kBinWarps] = word;
            }
        }
        for (; r < rows; r += kBinWarps) {
            const float x = in_image ? __ldg(tf + static_cast<long long>(r) * a.cols + col) : 0.0f;
            const uint32_t word = __ballot_sync(0xffffffffu, in_image && x > thr);
            if (lane == 0) mb[r] = word;
        }
    }
}

cudaError_t binarize_tile_launch(const BinarizeLaunch& L, cudaStream_t st);

cudaError_t binarize_launch(const BinarizeLaunch& L, cudaStream_t st) {
    if (L.n_plots <= 0 || L.rows <= 0 || L.cols <= 0) return cudaSuccess;
    if (L.mask_bytes) return binarize_tile_launch(L, st);  // caller checked binarize_tile_ok
    const int W = (L.cols + 31) / 32;
    dim3 grid(W, L.n_plots);
    binarize_kernel<<<grid, kBinThreads, 0, st>>>(L);
    return cudaGetLastError();
}

} // namespace ssb

// ---------------------------------------------------------------------------
// binarize_tile_kernel: the batch path for plots of <= kTileMaxRows rows.
// One CTA per (plot, 8-column group): the group's T x 8 values (32 bytes per
// row) are pulled into shared memory once by TMA (a 3-D tensor map over the
// TF batch, one 8 x 256-row box per mbarrier, all boxes in flight at once,
// issued by one thread), and sweeps A/B/C run from shared memory -- one HBM
// read of the active columns in total; sweep A consumes each box as it lands.
// The output byte (8 mask bits) lands in the bit-packed mask word in place
// (little-endian: byte g of word w = columns 32w + 8g .. +7).
constexpr int kTileCols = 8;
// tile histograms: 260 words per column (a multiple of 4, so Otsu reads each
// lane's 8 bins as two 128-bit loads); an atomic instruction's lanes hit
// columns q and q + 4 (banks 16 apart for the same bin)
constexpr int kTileHistStride = 260;
constexpr int kTileMaxRows = 6144;
constexpr int kBox = 256;  // rows per TMA box (the box-dimension limit)
static_assert(kTileMaxRows % kBox == 0, "whole boxes");

namespace ssb {

// TMA tile load of box (8 columns x kBox rows x 1 plot) at (c0, r0, p) of the
// [plots][rows][cols] fp32 TF tensor, completion counted on `bar`
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map, int c0, int r0, int p, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(p), "r"(smem_u32(bar))
        : "memory");
}

// NSPLIT = 2: a 2-CTA cluster shares one column group, each CTA holding half
// of the rows (tall plots, e.g. the 4881-row Hann STFT, keep 2 CTAs per SM);
// column extremes are pushed into the partner (DSMEM stores), each CTA
// pushes its partial histograms into the partner's shared memory before the
// second (last) cluster barrier, and both run the same Otsu locally.
template <int NSPLIT>
__global__ void __launch_bounds__(kBinThreads, 2) binarize_tile_kernel(BinarizeLaunch a, const __grid_constant__ CUtensorMap tmap) {
    static_assert(NSPLIT == 1 || NSPLIT == 2, "pairs: the partner is rank ^ 1");
    extern __shared__ __align__(128) float bt_vals[];     // (rows / NSPLIT, rounded up to kBox) x 8
    __shared__ __align__(8) uint64_t box_bar[kTileMaxRows / kBox];
    __shared__ __align__(16) uint32_t hist[kTileCols * kTileHistStride];
    __shared__ __align__(16) uint32_t hist_peer[NSPLIT > 1 ? kTileCols * kTileHistStride : 4];  // the partner's partials
    __shared__ float s_lo[kBinWarps][kTileCols], s_hi[kBinWarps][kTileCols];
    __shared__ float part_lo[kTileCols], part_hi[kTileCols], peer_lo[kTileCols], peer_hi[kTileCols];
    __shared__ float c_lo[kTileCols], c_scale[kTileCols], c_thr[kTileCols];
    __shared__ double c_span[kTileCols];
    __shared__ int c_use[kTileCols];

    // one column group of plot p; par = this CTA's use count of the box
    // barriers (parity), first = initialise them
    auto run_group = [&](int p, int grp, uint32_t par, bool first) {
        const int rank = NSPLIT == 1 ? 0 : static_cast<int>(cg::this_cluster().block_rank());
        const int rows_all = a.rows, cols = a.cols;
        const int half = (rows_all + NSPLIT - 1) / NSPLIT;
        const int rbase = rank * half;
        const int rows = max(0, min(rows_all, rbase + half) - rbase);  // this CTA's rows
        const int W = (cols + 31) / 32;
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        const uint32_t abyte = (a.active_bits[static_cast<long long>(p) * W + grp / 4] >> (8 * (grp & 3))) & 0xffu;
        // byte (grp & 3) of the word-major mask words (grp >> 2, r): the tile path
        // writes the packed mask K5 reads, 4 bytes apart per row
        uint8_t* plane = a.mask_bytes + ((static_cast<long long>(p) * W + (grp >> 2)) * mask_rs(rows_all) + rbase) * 4 + (grp & 3);
        const int col0 = grp * kTileCols;
        if (abyte == 0) {  // both CTAs of a cluster see the same byte and leave together
            if (!a.skip_empty)
                for (int r = tid; r < rows; r += kBinThreads) plane[4 * r] = 0;
            return;
        }
        // ---- load the block: one TMA box per kBox rows (32 B x kBox), each on its
        // own mbarrier, so sweep A starts on the first box while the rest land
        const int nbox = (rows + kBox - 1) / kBox;
        if (tid < nbox) {  // thread b issues box b: the boxes leave in parallel
            if (first) {  // persistent CTAs reuse the barriers: one phase per group
                mbar_init(&box_bar[tid], 1);
                fence_mbar_init();
            }
            mbar_arrive_expect_tx(&box_bar[tid], kBox * kTileCols * sizeof(float));
            tma_load_box(bt_vals + tid * kBox * kTileCols, &tmap, col0, rbase + tid * kBox, p, &box_bar[tid]);
        }
        // per-column binning constants from the column extremes (bin_of,
        // detector.cpp:28-39); thread tid < 8 owns column col0 + tid
        auto set_col = [&](float l, float h) {
            const float scale = __fdiv_rn(256.0f, __fsub_rn(h, l));
            const bool valid = h > l && isfinite(scale);
            const bool act = (col0 + tid < cols) && ((abyte >> tid) & 1u);
            c_lo[tid] = l;
            c_scale[tid] = scale;
            c_span[tid] = __dsub_rn(static_cast<double>(h), static_cast<double>(l));
            c_use[tid] = (act && valid) ? 1 : 0;
            c_thr[tid] = INFINITY;
        };
        // extremes supplied by the fused K1 (exact: order-free min / max of the
        // same floats): no min / max sweep, and each box is binned as it lands
        const bool ext = a.col_lo != nullptr;
        for (int i = tid; i < kTileCols * kTileHistStride; i += kBinThreads) hist[i] = 0;
        if (ext && tid < kTileCols) {
            const long long ci = static_cast<long long>(p) * cols + col0 + tid;
            set_col(a.col_lo[ci], a.col_hi[ci]);
        }
        __syncthreads();  // mbarrier init (+ the constants) visible

        if (!ext) {
            // ---- sweep A: two threads per row, one float4 (4 columns) each; fminf /
            // fmaxf equal std::min / std::max here (NaN is never taken by either, and
            // the sign of a zero extreme never reaches an output)
            {
                const int hh = tid & 1;
                float lo4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
                float hi4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
                // exactly two rows of each box per thread, branch-free: rows past the
                // CTA's last row re-read that row (a repeated value changes no extreme)
                static_assert(kBox == 2 * (kBinThreads / 2), "two rows of a box per thread");
                const int last = rows - 1;
                for (int b = 0; b < nbox; ++b) {
                    mbar_wait(&box_bar[b], par);
                    const int r0 = min(b * kBox + (tid >> 1), last);
                    const int r1 = min(b * kBox + kBinThreads / 2 + (tid >> 1), last);
                    const float4 x = *reinterpret_cast<const float4*>(bt_vals + r0 * kTileCols + 4 * hh);
                    const float4 y = *reinterpret_cast<const float4*>(bt_vals + r1 * kTileCols + 4 * hh);
                    lo4[0] = fminf(lo4[0], fminf(x.x, y.x)); hi4[0] = fmaxf(hi4[0], fmaxf(x.x, y.x));
                    lo4[1] = fminf(lo4[1], fminf(x.y, y.y)); hi4[1] = fmaxf(hi4[1], fmaxf(x.y, y.y));
                    lo4[2] = fminf(lo4[2], fminf(x.z, y.z)); hi4[2] = fmaxf(hi4[2], fmaxf(x.z, y.z));
                    lo4[3] = fminf(lo4[3], fminf(x.w, y.w)); hi4[3] = fmaxf(hi4[3], fmaxf(x.w, y.w));
                }
        #pragma unroll
                for (int o = 2; o < 32; o <<= 1)
        #pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        lo4[q] = fminf(lo4[q], __shfl_xor_sync(0xffffffffu, lo4[q], o));
                        hi4[q] = fmaxf(hi4[q], __shfl_xor_sync(0xffffffffu, hi4[q], o));
                    }
                if (lane < 2) {
        #pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        s_lo[warp][4 * lane + q] = lo4[q];
                        s_hi[warp][4 * lane + q] = hi4[q];
                    }
                }
            }
            __syncthreads();
            if constexpr (NSPLIT > 1) {
                if (tid < kTileCols) {
                    float l = s_lo[0][tid], h = s_hi[0][tid];
                    for (int q = 1; q < kBinWarps; ++q) {
                        l = fminf(l, s_lo[q][tid]);
                        h = fmaxf(h, s_hi[q][tid]);
                    }
                    part_lo[tid] = l;
                    part_hi[tid] = h;
                    // push into the partner too (peer slot): after the barrier both
                    // read only local shared memory
                    cg::cluster_group cl = cg::this_cluster();
                    *cl.map_shared_rank(&peer_lo[tid], rank ^ 1) = l;
                    *cl.map_shared_rank(&peer_hi[tid], rank ^ 1) = h;
                }
                cg::this_cluster().sync();
            }
            if (tid < kTileCols) {
                float l, h;
                if constexpr (NSPLIT > 1) {
                    // min / max are order-free: every CTA of the cluster derives the same extremes
                    l = fminf(part_lo[tid], peer_lo[tid]);
                    h = fmaxf(part_hi[tid], peer_hi[tid]);
                } else {
                    l = s_lo[0][tid];
                    h = s_hi[0][tid];
                    for (int q = 1; q < kBinWarps; ++q) {
                        l = fminf(l, s_lo[q][tid]);
                        h = fmaxf(h, s_hi[q][tid]);
                    }
                }
                set_col(l, h);
            }
            __syncthreads();

            // ---- sweep B: histograms from shared memory.  Two threads per row, one
            // float4 (4 columns) each, as in sweep A: one LDS.128 per 4 values and
            // the per-column constants in registers.  Branch-free: a column that is
            // not binarised (inactive or constant) still counts into its own
            // histogram (bin_index stays in [0, 255] for any input), which Otsu then
            // ignores
            {
                const int hh = tid & 1;
                float clo[4], csc[4];
                uint32_t* hc[4];
                bool any = false;
        #pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int cc = 4 * hh + q;
                    clo[q] = c_lo[cc];
                    csc[q] = c_scale[cc];
                    hc[q] = hist + cc * kTileHistStride;
                    any |= c_use[cc] != 0;
                }
                if (any) {
                    constexpr int RS = kBinThreads / 2;  // row stride
                    int r = tid >> 1;
                    for (; r + RS < rows; r += 2 * RS) {
                        const float4 x0 = *reinterpret_cast<const float4*>(bt_vals + r * kTileCols + 4 * hh);
                        const float4 x1 = *reinterpret_cast<const float4*>(bt_vals + (r + RS) * kTileCols + 4 * hh);
                        const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        #pragma unroll
                        for (int q = 0; q < 8; ++q) atomicAdd(hc[q & 3] + bin_index(xv[q], clo[q & 3], csc[q & 3]), 1u);
                    }
                    if (r < rows) {
                        const float4 x0 = *reinterpret_cast<const float4*>(bt_vals + r * kTileCols + 4 * hh);
                        const float xv[4] = {x0.x, x0.y, x0.z, x0.w};
        #pragma unroll
                        for (int q = 0; q < 4; ++q) atomicAdd(hc[q] + bin_index(xv[q], clo[q], csc[q]), 1u);
                    }
                }
            }
        } else {
            // ---- sweep B, streaming: two rows of each box per thread (one float4
            // of 4 columns each) as soon as the box lands; every thread waits for
            // every box, since sweep C reads them all
            const int hh = tid & 1;
            float clo[4], csc[4];
            uint32_t* hc[4];
            bool any = false;
    #pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int cc = 4 * hh + q;
                clo[q] = c_lo[cc];
                csc[q] = c_scale[cc];
                hc[q] = hist + cc * kTileHistStride;
                any |= c_use[cc] != 0;
            }
            for (int b = 0; b < nbox; ++b) {
                mbar_wait(&box_bar[b], par);
                const int ra = b * kBox + (tid >> 1), rb = ra + kBinThreads / 2;
                if (any && ra < rows) {
                    const float4 x = *reinterpret_cast<const float4*>(bt_vals + ra * kTileCols + 4 * hh);
                    const float xv[4] = {x.x, x.y, x.z, x.w};
    #pragma unroll
                    for (int q = 0; q < 4; ++q) atomicAdd(hc[q] + bin_index(xv[q], clo[q], csc[q]), 1u);
                }
                if (any && rb < rows) {
                    const float4 x = *reinterpret_cast<const float4*>(bt_vals + rb * kTileCols + 4 * hh);
                    const float xv[4] = {x.x, x.y, x.z, x.w};
    #pragma unroll
                    for (int q = 0; q < 4; ++q) atomicAdd(hc[q] + bin_index(xv[q], clo[q], csc[q]), 1u);
                }
            }
        }
        __syncthreads();

        // cluster: each CTA pushes its partial histograms into its partner's
        // hist_peer (DSMEM stores) before the one barrier; afterwards both hold
        // the full histograms locally, run all 8 Otsu splits themselves and touch
        // no remote memory again, so no second barrier is needed
        if constexpr (NSPLIT > 1) {
            cg::cluster_group cl = cg::this_cluster();
            uint32_t* peer = cl.map_shared_rank(hist_peer, rank ^ 1);
            for (int i = tid; i < kTileCols * kTileHistStride; i += kBinThreads) peer[i] = hist[i];
            cl.sync();
        }
        if (warp < kTileCols && c_use[warp]) {
            const int cc = warp;
            uint32_t hq[8];
            {
                const uint4* h4 = reinterpret_cast<const uint4*>(hist + cc * kTileHistStride + lane * 8);
                const uint4 a0 = h4[0], a1 = h4[1];
                hq[0] = a0.x; hq[1] = a0.y; hq[2] = a0.z; hq[3] = a0.w;
                hq[4] = a1.x; hq[5] = a1.y; hq[6] = a1.z; hq[7] = a1.w;
            }
            if constexpr (NSPLIT > 1) {
                const uint4* h4 = reinterpret_cast<const uint4*>(hist_peer + cc * kTileHistStride + lane * 8);
                const uint4 a0 = h4[0], a1 = h4[1];
                hq[0] += a0.x; hq[1] += a0.y; hq[2] += a0.z; hq[3] += a0.w;
                hq[4] += a1.x; hq[5] += a1.y; hq[6] += a1.z; hq[7] += a1.w;
            }
            const int best_i = otsu_split_warp_u32(hq, lane);
            if (lane == 0) {
                const double lod = static_cast<double>(c_lo[cc]);
                // /256 as *2^-8: the same correctly rounded value (a power of two), no DDIV
                const double e = __dmul_rn(__dmul_rn(static_cast<double>(best_i) + 1.0, c_span[cc]), 0x1p-8);
                c_thr[cc] = __double2float_rn(__dadd_rn(lod, e));
            }
        }
        __syncthreads();
        if (a.col_thr && tid < kTileCols && col0 + tid < cols && rank == 0)
            a.col_thr[static_cast<long long>(p) * cols + col0 + tid] = c_thr[tid];

        // ---- sweep C: one row per thread, 8 compares -> one mask byte
        float thr[kTileCols];
    #pragma unroll
        for (int q = 0; q < kTileCols; ++q) thr[q] = c_thr[q];
        for (int r = tid; r < rows; r += kBinThreads) {
            const float4 x0 = *reinterpret_cast<const float4*>(bt_vals + r * kTileCols);
            const float4 x1 = *reinterpret_cast<const float4*>(bt_vals + r * kTileCols + 4);
            const uint32_t b = (x0.x > thr[0] ? 1u : 0u) | (x0.y > thr[1] ? 2u : 0u) | (x0.z > thr[2] ? 4u : 0u) |
                               (x0.w > thr[3] ? 8u : 0u) | (x1.x > thr[4] ? 16u : 0u) | (x1.y > thr[5] ? 32u : 0u) |
                               (x1.z > thr[6] ? 64u : 0u) | (x1.w > thr[7] ? 128u : 0u);
            plane[4 * r] = static_cast<uint8_t>(b);
        }
    };
    if constexpr (NSPLIT == 1) {
        if (a.group_list) {
            // persistent: the CTA walks the active column groups (K3's list, in
            // plot and group order), so empty groups cost no CTA at all
            const int G = a.cols / kTileCols;
            const int count = *a.group_count;
            uint32_t par = 0;
            for (int it = blockIdx.x; it < count; it += gridDim.x) {
                const int e = a.group_list[it];
                run_group(e / G, e % G, par, it == static_cast<int>(blockIdx.x));
                par ^= 1u;
                __syncthreads();  // the block buffer and histograms are reused
            }
            return;
        }
    }
    run_group(blockIdx.y, blockIdx.x / NSPLIT, 0u, true);
}

// one CTA per column group while its block leaves room for 2 CTAs per SM,
// else a 2-CTA cluster per group (rows split in halves)
constexpr int kTileSplitRows = 3264;

bool binarize_tile_ok(int rows, int cols) { return cols % 32 == 0 && rows <= 2 * kTileMaxRows && rows > 0; }

// The 2-CTA cluster form (rows > kTileSplitRows) gains from the fused K1's
// column extremes (no min / max sweep, no extremes exchange, histograms built
// as boxes land: Hann K4 7.43 -> 5.97 ms per step against +1.0 ms of K1); the
// single-CTA form's min / max sweep already hides under its box loads, so
// there the extremes cost K1 more than they save (C5r: K1 +0.49, K4 -0.43).
bool binarize_wants_extremes(int rows) { return rows > kTileSplitRows; }

bool binarize_tile_persistent(int rows, int cols) { return binarize_tile_ok(rows, cols) && rows <= kTileSplitRows; }

// The [plots][rows][cols] fp32 TF tensor as a TMA tensor map with 8 x kBox x 1
// boxes (rows past the end of a plot read as zeros and are never used).
static cudaError_t make_tf_map(const BinarizeLaunch& L, CUtensorMap* map) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(L.cols), static_cast<cuuint64_t>(L.rows),
                                static_cast<cuuint64_t>(L.n_plots)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(L.cols) * sizeof(float),
                                   static_cast<cuuint64_t>(L.rows) * L.cols * sizeof(float)};
    const cuuint32_t box[3] = {kTileCols, kBox, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(L.tf), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t binarize_tile_launch(const BinarizeLaunch& L, cudaStream_t st) {
    const int split = L.rows > kTileSplitRows ? 2 : 1;
    const int rows_cta = (L.rows + split - 1) / split;
    const size_t smem = sizeof(float) * kTileCols * static_cast<size_t>((rows_cta + kBox - 1) / kBox * kBox);
    static std::atomic<unsigned long long> attr_set[2];
    const cudaError_t ae = set_attr_once(attr_set[split - 1], [&] {
        const int lim = kTileCols * kTileMaxRows * static_cast<int>(sizeof(float));
        return split == 1 ? cudaFuncSetAttribute(binarize_tile_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim)
                          : cudaFuncSetAttribute(binarize_tile_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    });
    if (ae != cudaSuccess) return ae;
    CUtensorMap map;
    const cudaError_t me = make_tf_map(L, &map);
    if (me != cudaSuccess) return me;
    if (split == 1) {
        if (L.group_list) {  // persistent: 2 CTAs per SM walk the active groups
            static int sms[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (!sms[dev & 63]) cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
            binarize_tile_kernel<1><<<2 * sms[dev & 63], kBinThreads, smem, st>>>(L, map);
            return cudaGetLastError();
        }
        dim3 grid(L.cols / kTileCols, L.n_plots);
        binarize_tile_kernel<1><<<grid, kBinThreads, smem, st>>>(L, map);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (L.cols / kTileCols), L.n_plots);
    cfg.blockDim = dim3(kBinThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, binarize_tile_kernel<2>, L, map);
}

} // namespace ssb
