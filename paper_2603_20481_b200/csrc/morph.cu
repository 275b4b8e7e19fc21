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
// (3x1 when one_d_opening_along_time) in shared memory: one CTA owns a tile of
// 64 buffer rows (56 output rows + 4 halo rows each side; 52 + 6 for the
// vertical line) across all W words, column-major in smem (a[w][i]), and
// applies the six erode/dilate steps as separable vertical (row AND/OR) and
// horizontal (shift/carry AND/OR across neighbouring words) passes.  Outside
// the image counts as background for erosion and dilation alike (:359-362,
// :393-410): out-of-image rows are re-zeroed after every step and bits past
// the last column are masked, so each step sees the reference's clipped
// neighbourhood.  The two buffer edge rows are never recomputed; the invalid
// band grows one row per vertical step and the halo absorbs it.
#include "common.cuh"
#include "internal.h"

namespace ssb {

constexpr int kMorphThreads = 256;
constexpr int kTileNR = 64;  // buffer rows per CTA (a power of two: thread -> (word, row) is shifts)

// byte mask [p][rows][cols] -> word-major bits [p][W][rows]
__global__ void pack_u8_kernel(const uint8_t* __restrict__ m, int rows, int cols, uint32_t* __restrict__ bits) {
    const int W = (cols + 31) / 32;
    const int p = blockIdx.y;
    const long long nwords = static_cast<long long>(rows) * W;
    const int lane = threadIdx.x & 31;
    const long long warp_global = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const uint8_t* mp = m + static_cast<long long>(p) * rows * cols;
    uint32_t* bp = bits + static_cast<long long>(p) * nwords;
    for (long long wi = warp_global; wi < nwords; wi += nwarps) {
        const long long r = wi / W;
        const int w = static_cast<int>(wi % W);
        const int c = w * 32 + lane;
        const bool b = c < cols && mp[r * cols + c] != 0;
        const uint32_t word = __ballot_sync(0xffffffffu, b);
        if (lane == 0) bp[static_cast<long long>(w) * rows + r] = word;
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
    const uint32_t* bp = bits + static_cast<long long>(p) * rows * W;
    uint8_t* mp = m + static_cast<long long>(p) * npx;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < npx;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = i / cols;
        const int c = static_cast<int>(i % cols);
        mp[i] = (bp[static_cast<long long>(c >> 5) * rows + r] >> (c & 31)) & 1u;
    }
}

cudaError_t unpack_launch(const uint32_t* bits, int n_plots, int rows, int cols, uint8_t* m, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    dim3 grid(512, n_plots);
    unpack_kernel<<<grid, 256, 0, st>>>(bits, rows, cols, m);
    return cudaGetLastError();
}

// ------------------------------------------------------------- fused chain

struct MTile {
    uint32_t* a;       // [W][kTileNR] current image (column-major)
    uint32_t* b;       // [W][kTileNR] scratch
    int W;
    uint32_t last_mask;
    int out_top, out_bot;  // buffer rows [0,out_top) and [out_bot,kTileNR) lie outside the image

    // every thread visits (w, i) for i in [1, NR-1): e = w*NR + i
    __device__ __forceinline__ void vpass(bool erode) const {
        for (int e = threadIdx.x; e < W * kTileNR; e += kMorphThreads) {
            const int i = e & (kTileNR - 1);
            if (i == 0 || i == kTileNR - 1) continue;
            const uint32_t u = a[e - 1], c = a[e], d = a[e + 1];
            b[e] = erode ? (u & c & d) : (u | c | d);
        }
    }
    __device__ __forceinline__ void hpass(const uint32_t* src, uint32_t* dst, bool erode) const {
        for (int e = threadIdx.x; e < W * kTileNR; e += kMorphThreads) {
            const int w = e >> 6;  // kTileNR == 64
            const uint32_t x = src[e];
            const uint32_t prev = w > 0 ? src[e - kTileNR] : 0u;
            const uint32_t next = w + 1 < W ? src[e + kTileNR] : 0u;
            const uint32_t left = (x << 1) | (prev >> 31);   // column c-1 at bit c
            const uint32_t right = (x >> 1) | (next << 31);  // column c+1 at bit c
            uint32_t y = erode ? (x & left & right) : (x | left | right);
            if (w == W - 1) y &= last_mask;
            dst[e] = y;
        }
    }
    __device__ __forceinline__ void clip() const {
        if (out_top == 0 && out_bot == kTileNR) return;
        for (int e = threadIdx.x; e < W * kTileNR; e += kMorphThreads) {
            const int i = e & (kTileNR - 1);
            if (i < out_top || i >= out_bot) a[e] = 0u;
        }
    }
    // one erosion / dilation: 3x3 (vert && horiz), 3x1 (vert), 1x3 (horiz)
    __device__ __forceinline__ void step(bool erode, bool vert, bool horiz) {
        if (vert) {
            vpass(erode);
            __syncthreads();
            if (horiz) {
                hpass(b, a, erode);
            } else {
                uint32_t* t = a;  // result is in b (edge rows: stale, invalid anyway)
                a = b;
                b = t;
            }
        } else {
            hpass(a, b, erode);
            uint32_t* t = a;
            a = b;
            b = t;
        }
        __syncthreads();
        clip();
        __syncthreads();
    }
};

// in_bits: word-major bits [p][W][rows], or in_planes: byte planes [p][4W][rows].
__global__ void __launch_bounds__(kMorphThreads)
consolidate_kernel(const uint32_t* __restrict__ in_bits, const uint8_t* __restrict__ in_planes, int rows, int cols,
                   int halo, bool along_time, uint32_t* __restrict__ out) {
    extern __shared__ uint32_t mo_smem[];
    const int W = (cols + 31) / 32;
    const int p = blockIdx.y;
    const int tile_rows = kTileNR - 2 * halo;
    const int r0 = blockIdx.x * tile_rows;
    const int row0 = r0 - halo;  // global row of buffer row 0
    MTile t;
    t.W = W;
    t.a = mo_smem;
    t.b = mo_smem + W * kTileNR;
    t.last_mask = (cols & 31) ? ((1u << (cols & 31)) - 1u) : 0xffffffffu;
    t.out_top = row0 < 0 ? -row0 : 0;
    t.out_bot = rows - row0 < kTileNR ? rows - row0 : kTileNR;
    for (int e = threadIdx.x; e < W * kTileNR; e += kMorphThreads) {
        const int w = e >> 6, i = e & (kTileNR - 1);
        const int g = row0 + i;
        uint32_t word = 0u;
        if (g >= 0 && g < rows) {
            if (in_planes) {
                const uint8_t* bp = in_planes + (static_cast<long long>(p) * 4 * W + 4 * w) * rows + g;
                word = static_cast<uint32_t>(bp[0]) | (static_cast<uint32_t>(bp[rows]) << 8) |
                       (static_cast<uint32_t>(bp[2 * static_cast<long long>(rows)]) << 16) |
                       (static_cast<uint32_t>(bp[3 * static_cast<long long>(rows)]) << 24);
            } else {
                word = in_bits[(static_cast<long long>(p) * W + w) * rows + g];
            }
        }
        t.a[e] = word;
    }
    __syncthreads();
    t.step(false, true, true);  // close 3x3: dilate, erode
    t.step(true, true, true);
    t.step(true, true, true);   // open 3x3: erode, dilate
    t.step(false, true, true);
    t.step(true, along_time, !along_time);  // open with the line element
    t.step(false, along_time, !along_time);
    const int nrow = min(tile_rows, rows - r0);
    for (int e = threadIdx.x; e < W * kTileNR; e += kMorphThreads) {
        const int w = e >> 6, i = e & (kTileNR - 1);
        if (i >= halo && i < halo + nrow) out[(static_cast<long long>(p) * W + w) * rows + r0 + (i - halo)] = t.a[e];
    }
}

cudaError_t consolidate_bits_launch(const uint32_t* in, const uint8_t* planes, int n_plots, int rows, int cols,
                                    bool along_time, uint32_t* out, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    const int W = (cols + 31) / 32;
    const int halo = along_time ? 6 : 4;
    const int tile_rows = kTileNR - 2 * halo;
    const size_t smem = sizeof(uint32_t) * 2 * static_cast<size_t>(W) * kTileNR;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;  // cols > 14,000: not on the device path
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(consolidate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((rows + tile_rows - 1) / tile_rows, n_plots);
    consolidate_kernel<<<grid, kMorphThreads, smem, st>>>(in, planes, rows, cols, halo, along_time, out);
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
