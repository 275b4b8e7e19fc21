// morph.cu -- K5: binary morphology on bit-packed TF masks.
//
// Replaces detector::consolidate (proj/src/detector.cpp:482-492) and the
// morphology primitives it composes (:345-480).  Masks are bit-packed,
// 32 columns per uint32 word (bit b of word w = column 32w+b) and stored
// WORD-MAJOR: bits[p][w][r], rows contiguous -- 1/32 of the reference's byte
// mask, and every kernel that walks it has consecutive lanes on consecutive
// rows (coalesced global access, conflict-free shared access).
//
// consolidate_kernel fuses the whole chain close3x3 -> open3x3 -> open1x3
// (3x1 when one_d_opening_along_time) in registers (see below).
#include "common.cuh"
#include "internal.h"

namespace ssb {


// byte mask [p][rows][cols] -> word-major bits [p][W][rows]
__global__ void pack_u8_kernel(const uint8_t* __restrict__ m, int rows, int cols, uint32_t* __restrict__ bits) {
    const int W = (cols + 31) / 32;
    const int p = blockIdx.y;
    const long long nwords = static_cast<long long>(rows) * W;
    const int lane = threadIdx.x & 31;
    const long long warp_global = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const uint8_t* mp = m + static_cast<long long>(p) * rows * cols;
    uint32_t* bp = bits + static_cast<long long>(p) * mask_rs(rows) * W;
    for (long long wi = warp_global; wi < nwords; wi += nwarps) {
        const long long r = wi / W;
        const int w = static_cast<int>(wi % W);
        const int c = w * 32 + lane;
        const bool b = c < cols && mp[r * cols + c] != 0;
        const uint32_t word = __ballot_sync(0xffffffffu, b);
        if (lane == 0) bp[static_cast<long long>(w) * mask_rs(rows) + r] = word;
    }
}

cudaError_t pack_u8_launch(const uint8_t* m, int n_plots, int rows, int cols, uint32_t* bits, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    dim3 grid(256, n_plots);
    pack_u8_kernel<<<grid, 256, 0, st>>>(m, rows, cols, bits);
    return cudaGetLastError();
}

__global__ void unpack_kernel(const uint32_t* __restrict__ bits, int rows, int cols, uint8_t* __restrict__ m) {
    const int W = (cols + 31) / 32;
    const int p = blockIdx.y;
    const long long npx = static_cast<long long>(rows) * cols;
    const uint32_t* bp = bits + static_cast<long long>(p) * mask_rs(rows) * W;
    uint8_t* mp = m + static_cast<long long>(p) * npx;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < npx;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = i / cols;
        const int c = static_cast<int>(i % cols);
        mp[i] = (bp[static_cast<long long>(c >> 5) * mask_rs(rows) + r] >> (c & 31)) & 1u;
    }
}

cudaError_t unpack_launch(const uint32_t* bits, int n_plots, int rows, int cols, uint8_t* m, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    dim3 grid(512, n_plots);
    unpack_kernel<<<grid, 256, 0, st>>>(bits, rows, cols, m);
    return cudaGetLastError();
}

// ------------------------------------------------------------- fused chain
// Register-resident form: a warp owns a band of 16 output rows x 30 mask
// words.  Lane l holds word (band*30 + l - 1) for kRegNR = 16 + 2*HALO
// consecutive rows in registers; lanes 0 and 31 are halo words.  Vertical
// erode/dilate is register-to-register (rows i-1, i, i+1 of the same lane),
// horizontal is a funnel shift with the neighbouring lanes' words
// (__shfl_up/down).  Each step moves information at most one row / column,
// so HALO rows (the chain's vertical reach: 4 for close3x3 + open3x3 + the
// 1x3 line, 6 with the 3x1 line) and one halo word per side (horizontal
// reach <= 6 columns) absorb the invalid margin: no shared memory, no
// barriers.  Out-of-image rows and words are zeroed and the last word masked
// after every step (out-of-image = background for erode and dilate,
// detector.cpp:359-362, 393-410).
constexpr int kRegOwnRows = 16;  // 16 owned rows beat 24 (0.634 vs 0.718 ms per C5r step: occupancy)
constexpr int kRegOwn = 30;      // owned words per warp

template <int HALO>
struct RegBand {
    static constexpr int OWN = kRegOwnRows;
    static constexpr int kRegNR = OWN + 2 * HALO;
    uint32_t x[kRegNR];
    int lo, hi;        // buffer rows [lo, hi) lie inside the image
    uint32_t wmask;    // 0 outside the image's words; last word: valid columns only

    __device__ __forceinline__ void clip() {
#pragma unroll
        for (int i = 0; i < kRegNR; ++i) x[i] = (i >= lo && i < hi) ? (x[i] & wmask) : 0u;
    }
    __device__ __forceinline__ void vert(bool erode) {
        uint32_t prev = x[0];
#pragma unroll
        for (int i = 1; i < kRegNR - 1; ++i) {
            const uint32_t cur = x[i];
            x[i] = erode ? (prev & cur & x[i + 1]) : (prev | cur | x[i + 1]);
            prev = cur;
        }
    }
    __device__ __forceinline__ void horiz(bool erode) {
#pragma unroll
        for (int i = 0; i < kRegNR; ++i) {
            const uint32_t v = x[i];
            const uint32_t prev = __shfl_up_sync(0xffffffffu, v, 1);    // word w-1 (lane 0: its own, halo)
            const uint32_t next = __shfl_down_sync(0xffffffffu, v, 1);  // word w+1 (lane 31: its own, halo)
            // funnel shifts written as shifts: the __funnelshift intrinsics are
            // volatile asm, which pins their order against the shuffles
            const uint32_t left = (v << 1) | (prev >> 31);
            const uint32_t right = (v >> 1) | (next << 31);
            x[i] = erode ? (v & left & right) : (v | left | right);
        }
    }
    // two horizontal erosions at once (1x5, radius 2): the same two shuffles
    __device__ __forceinline__ void horiz_erode2() {
#pragma unroll
        for (int i = 0; i < kRegNR; ++i) {
            const uint32_t v = x[i];
            const uint32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
            const uint32_t next = __shfl_down_sync(0xffffffffu, v, 1);
            x[i] = v & ((v << 1) | (prev >> 31)) & ((v << 2) | (prev >> 30)) & ((v >> 1) | (next << 31)) &
                   ((v >> 2) | (next << 30));
        }
    }
    // one erosion / dilation: 3x3 (vert then horiz), 3x1 (vert), 1x3 (horiz);
    // CLIP = false for bands with every row and word inside the image
    template <bool CLIP>
    __device__ __forceinline__ void step(bool erode, bool v, bool h) {
        if (v) vert(erode);
        if (h) horiz(erode);
        if (CLIP) clip();
    }
    // close3x3 -> open3x3 -> open with the line element.  Erosions (and
    // dilations) with zero padding commute with each other, and a 3x3 step is
    // its vertical and horizontal passes in either order, so the erode of the
    // close and the erode of the open -- adjacent -- run as one vertical
    // radius-2 pass plus one horizontal radius-2 pass: 5 horizontal passes
    // (shuffles) instead of 6, same mask (clipping after each of them is
    // exact: an erosion's out-of-image output is 0 anyway)
    template <bool CLIP>
    __device__ __forceinline__ void chain(bool along_time) {
        if (CLIP) clip();
        step<CLIP>(false, true, true);  // close 3x3: dilate
        vert(true);                     // close's erode + open's erode: 5x5 erosion
        vert(true);
        horiz_erode2();
        if (CLIP) clip();
        step<CLIP>(false, true, true);  // open 3x3: dilate
        step<CLIP>(true, along_time, !along_time);  // open with the line element
        step<CLIP>(false, along_time, !along_time);
    }
};

// in/out: word-major bits [p][W][rows].  One warp per (row band, word band).
template <int HALO>
__global__ void __launch_bounds__(128, 7) consolidate_kernel(const uint32_t* __restrict__ in, int rows, int cols,
                                                          int wbands, long long bands, bool along_time,
                                                          uint32_t* __restrict__ out,
                                                          const uint32_t* __restrict__ active_bits) {
    using RB = RegBand<HALO>;
    const int W = (cols + 31) / 32;
    const int lane = threadIdx.x & 31;
    const long long gwarp = blockIdx.x * 4LL + (threadIdx.x >> 5);
    if (gwarp >= bands) return;  // uniform per warp
    const int p = blockIdx.y;
    const int rb = static_cast<int>(gwarp / wbands), wb = static_cast<int>(gwarp % wbands);
    const int r0 = rb * RB::OWN, row0 = r0 - HALO;
    const int gw = wb * kRegOwn + lane - 1;
    const bool wvalid = gw >= 0 && gw < W;
    constexpr int kRegNR = RB::kRegNR;
    RB t;
    t.lo = max(0, -row0);
    t.hi = min(kRegNR, rows - row0);
    t.wmask = !wvalid ? 0u : ((gw == W - 1 && (cols & 31)) ? ((1u << (cols & 31)) - 1u) : 0xffffffffu);
    uint32_t keep = 0xffffffffu;  // bytes K4 wrote (groups with an active column)
    if (active_bits && wvalid) {
        const uint32_t ab = __ldg(active_bits + static_cast<long long>(p) * W + gw);
        keep = ((ab & 0xffu) ? 0xffu : 0u) | ((ab & 0xff00u) ? 0xff00u : 0u) | ((ab & 0xff0000u) ? 0xff0000u : 0u) |
               ((ab & 0xff000000u) ? 0xff000000u : 0u);
    }
    const int rs = mask_rs(rows);
    const uint32_t* src = in + (static_cast<long long>(p) * W + (wvalid ? gw : 0)) * rs + row0;
    if (HALO % 4 == 0 && row0 >= 0 && row0 + kRegNR <= rs) {
        // 16-byte aligned (row0 and rs are multiples of 4): 128-bit loads;
        // rows past the image (padding) are cleared below
#pragma unroll
        for (int i = 0; i < kRegNR; i += 4) {
            const uint4 q = wvalid ? __ldg(reinterpret_cast<const uint4*>(src + i)) : make_uint4(0u, 0u, 0u, 0u);
            t.x[i] = q.x;
            t.x[i + 1] = q.y;
            t.x[i + 2] = q.z;
            t.x[i + 3] = q.w;
        }
#pragma unroll
        for (int i = 0; i < kRegNR; ++i) t.x[i] = (i < t.hi) ? (t.x[i] & keep) : 0u;
    } else {
#pragma unroll
        for (int i = 0; i < kRegNR; ++i) t.x[i] = (wvalid && i >= t.lo && i < t.hi) ? (__ldg(src + i) & keep) : 0u;
    }
    // interior bands (most of a plot) skip the out-of-image clipping entirely
    const bool interior = t.lo == 0 && t.hi == kRegNR && t.wmask == 0xffffffffu;
    if (__all_sync(0xffffffffu, interior)) t.template chain<false>(along_time);
    else t.template chain<true>(along_time);
    if (!wvalid || lane == 0 || lane == 31) return;
    uint32_t* dst = out + (static_cast<long long>(p) * W + gw) * rs + r0;
    if (r0 + RB::OWN <= rs) {  // r0 is a multiple of 16: 128-bit stores (padding rows may take garbage)
#pragma unroll
        for (int i = 0; i < RB::OWN; i += 4)
            *reinterpret_cast<uint4*>(dst + i) = make_uint4(t.x[HALO + i], t.x[HALO + i + 1], t.x[HALO + i + 2],
                                                            t.x[HALO + i + 3]);
    } else {
        const int nrow = min(RB::OWN, rows - r0);
#pragma unroll
        for (int i = 0; i < RB::OWN; ++i)
            if (i < nrow) dst[i] = t.x[HALO + i];
    }
}

cudaError_t consolidate_bits_launch(const uint32_t* in, int n_plots, int rows, int cols, bool along_time,
                                    uint32_t* out, cudaStream_t st, const uint32_t* active_bits) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    const int W = (cols + 31) / 32;
    const int wbands = (W + kRegOwn - 1) / kRegOwn;
    // vertical reach of the chain: 4 rows (1x3 line), 6 (3x1 line)
    const int own = along_time ? RegBand<6>::OWN : RegBand<4>::OWN;
    const long long bands = static_cast<long long>((rows + own - 1) / own) * wbands;
    dim3 grid(static_cast<unsigned>((bands + 3) / 4), n_plots);
    if (along_time)
        consolidate_kernel<6><<<grid, 128, 0, st>>>(in, rows, cols, wbands, bands, along_time, out, active_bits);
    else
        consolidate_kernel<4><<<grid, 128, 0, st>>>(in, rows, cols, wbands, bands, along_time, out, active_bits);
    return cudaGetLastError();
}

// ------------------------------------------------- generic u8 (stage API)

// One erosion/dilation with an (sr x sc) all-ones element, out-of-image =
// background, for columns [e0, e1) of every row.
__global__ void morph_u8_kernel(const uint8_t* __restrict__ src, int rows, int cols, bool erode, int hr, int hc,
                                int e0, int e1, uint8_t* __restrict__ dst) {
    const int w = e1 - e0;
    const long long n = static_cast<long long>(rows) * w;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / w);
        const int c = e0 + static_cast<int>(i % w);
        bool acc = erode;
        for (int dr = -hr; dr <= hr; ++dr) {
            const int rr = r + dr;
            for (int dc = -hc; dc <= hc; ++dc) {
                const int cc = c + dc;
                const bool v = rr >= 0 && rr < rows && cc >= 0 && cc < cols &&
                               src[static_cast<long long>(rr) * cols + cc] != 0;
                acc = erode ? (acc && v) : (acc || v);
            }
        }
        dst[static_cast<long long>(r) * cols + c] = acc ? 1 : 0;
    }
}

cudaError_t morph_u8_launch(const uint8_t* src, int rows, int cols, int op, int se_rows, int se_cols, int c0,
                            int c1, uint8_t* tmp, uint8_t* dst, cudaStream_t st) {
    const int hr = (se_rows - 1) / 2, hc = (se_cols - 1) / 2;
    auto one = [&](const uint8_t* s, uint8_t* d, bool erode, int a0, int a1) {
        if (a1 <= a0) return cudaSuccess;
        morph_u8_kernel<<<512, 256, 0, st>>>(s, rows, cols, erode, hr, hc, a0, a1, d);
        return cudaGetLastError();
    };
    if (op == 0) return one(src, dst, true, c0, c1);
    if (op == 1) return one(src, dst, false, c0, c1);
    const int e0 = c0 - hc < 0 ? 0 : c0 - hc;
    const int e1 = c1 + hc > cols ? cols : c1 + hc;
    const bool first_erodes = op == 2;
    cudaError_t e = one(src, tmp, first_erodes, e0, e1);
    if (e != cudaSuccess) return e;
    return one(tmp, dst, !first_erodes, c0, c1);
}

} // namespace ssb
