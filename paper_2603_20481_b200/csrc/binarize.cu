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

namespace ssb {

constexpr int kBinThreads = 256;
constexpr int kBinWarps = kBinThreads / 32;
constexpr int kHistStride = 257;  // padded so column l, bin b hits bank (l + b) % 32

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
            uint32_t* mb = a.mask_bits + static_cast<long long>(p) * rows * W + wd;
            for (int r = threadIdx.x; r < rows; r += kBinThreads) mb[static_cast<long long>(r) * W] = 0;
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
                    int b = __float2int_rz(__fmul_rn(__fsub_rn(x[q], clo), csc));
                    b = b > 255 ? 255 : b;
                    atomicAdd(h + b, 1u);
                }
            }
        }
        for (; r < rows; r += kBinWarps) {
            if (use) {
                const float x = __ldg(tf + static_cast<long long>(r) * a.cols + col);
                int b = __float2int_rz(__fmul_rn(__fsub_rn(x, clo), csc));
                b = b > 255 ? 255 : b;
                atomicAdd(h + b, 1u);
            }
        }
    }
    __syncthreads();

    // ---- Otsu split: one warp per column, lane owns bins 8*lane .. 8*lane+7
    for (int c = warp; c < 32; c += kBinWarps) {
        if (!c_use[c]) continue;
        const uint32_t* h = hist + c * kHistStride;
        unsigned long long cnt[8], wsum[8];
        unsigned long long lc = 0, ls = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int bin = lane * 8 + q;
            lc += h[bin];
            ls += static_cast<unsigned long long>(bin) * h[bin];
            cnt[q] = lc;
            wsum[q] = ls;
        }
        // exclusive prefix over lanes of (lc, ls)
        unsigned long long pc = lc, ps = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long tc = __shfl_up_sync(0xffffffffu, pc, o);
            const unsigned long long ts = __shfl_up_sync(0xffffffffu, ps, o);
            if (lane >= o) {
                pc += tc;
                ps += ts;
            }
        }
        const unsigned long long total = __shfl_sync(0xffffffffu, pc, 31);
        const double sum_all = static_cast<double>(__shfl_sync(0xffffffffu, ps, 31));
        pc -= lc;
        ps -= ls;
        double best_v = -1.0;
        int best_i = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned long long w0 = pc + cnt[q];
            const unsigned long long w1 = total - w0;
            const double sum0 = static_cast<double>(ps + wsum[q]);
            double var = 0.0;
            if (w0 > 0 && w1 > 0) {
                const double mu0 = __ddiv_rn(sum0, static_cast<double>(w0));
                const double mu1 = __ddiv_rn(__dsub_rn(sum_all, sum0), static_cast<double>(w1));
                const double d = __dsub_rn(mu0, mu1);
                var = __dmul_rn(__dmul_rn(__dmul_rn(static_cast<double>(w0), static_cast<double>(w1)), d), d);
            }
            if (var > best_v) {
                best_v = var;
                best_i = lane * 8 + q;
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
        if (lane == 0) {
            const double lod = static_cast<double>(c_lo[c]);
            const double e = __ddiv_rn(__dmul_rn(static_cast<double>(best_i) + 1.0, c_span[c]), 256.0);
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
        uint32_t* mb = a.mask_bits + static_cast<long long>(p) * rows * W + wd;
        int r = warp;
        for (; r + 3 * kBinWarps < rows; r += 4 * kBinWarps) {
            float x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                x[q] = in_image ? __ldg(tf + static_cast<long long>(r + q * kBinWarps) * a.cols + col) : 0.0f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t word = __ballot_sync(0xffffffffu, in_image && x[q] > thr);
                if (lane == 0) mb[static_cast<long long>(r + q * kBinWarps) * W] = word;
            }
        }
        for (; r < rows; r += kBinWarps) {
            const float x = in_image ? __ldg(tf + static_cast<long long>(r) * a.cols + col) : 0.0f;
            const uint32_t word = __ballot_sync(0xffffffffu, in_image && x > thr);
            if (lane == 0) mb[static_cast<long long>(r) * W] = word;
        }
    }
}

cudaError_t binarize_launch(const BinarizeLaunch& L, cudaStream_t st) {
    if (L.n_plots <= 0 || L.rows <= 0 || L.cols <= 0) return cudaSuccess;
    const int W = (L.cols + 31) / 32;
    dim3 grid(W, L.n_plots);
    binarize_kernel<<<grid, kBinThreads, 0, st>>>(L);
    return cudaGetLastError();
}

} // namespace ssb
