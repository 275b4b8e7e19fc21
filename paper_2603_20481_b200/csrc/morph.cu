// morph.cu -- K5: binary morphology on bit-packed TF masks.
//
// Replaces detector::consolidate (proj/src/detector.cpp:482-492) and the
// morphology primitives it composes (:345-480).  Masks are bit-packed,
// 32 columns per uint32 word (bit b of word w = column 32w+b), rows
// contiguous -- 1/32 of the reference's byte mask (2441 x 4096 -> 1.25 MB).
//
// consolidate_bits_kernel fuses the whole chain close3x3 -> open3x3 ->
// open1x3 (3x1 when one_d_opening_along_time) in shared memory: one CTA owns a
// tile of TR output rows across all words, loads TR + 2H rows (H = 4, or 6
// with the vertical line), and applies the six erode/dilate steps as
// separable vertical (row AND/OR) + horizontal (shift/carry AND/OR) word ops.
// Outside the image counts as background for erosion and dilation alike
// (:359-362, :393-410): out-of-image rows are re-zeroed after every step and
// bits past the last column are masked, so each step sees exactly the
// reference's clipped neighbourhood.
#include "common.cuh"
#include "internal.h"

namespace ssb {

constexpr int kMorphThreads = 256;

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
        if (lane == 0) bp[wi] = word;
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
        mp[i] = (bp[r * W + (c >> 5)] >> (c & 31)) & 1u;
    }
}

cudaError_t unpack_launch(const uint32_t* bits, int n_plots, int rows, int cols, uint8_t* m, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    dim3 grid(512, n_plots);
    unpack_kernel<<<grid, 256, 0, st>>>(bits, rows, cols, m);
    return cudaGetLastError();
}

// ------------------------------------------------------------- fused chain

struct MorphTile {
    uint32_t* a;   // [NR][W] current image
    uint32_t* b;   // [NR][W] vertical-pass temp
    int NR, W, cols, rows, row0;  // row0: global row of buffer row 0
    uint32_t last_mask;           // valid bits of the last word
};

// Vertical pass a -> b over buffer rows [1, NR-1).
__device__ __forceinline__ void vpass(const MorphTile& t, bool erode) {
    const int n = (t.NR - 2) * t.W;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = 1 + e / t.W, w = e % t.W;
        const uint32_t u = t.a[(i - 1) * t.W + w], c = t.a[i * t.W + w], d = t.a[(i + 1) * t.W + w];
        t.b[i * t.W + w] = erode ? (u & c & d) : (u | c | d);
    }
}

// Horizontal pass src -> dst over buffer rows [1, NR-1), out-of-image columns 0.
__device__ __forceinline__ void hpass(const MorphTile& t, const uint32_t* src, uint32_t* dst, bool erode) {
    const int n = (t.NR - 2) * t.W;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = 1 + e / t.W, w = e % t.W;
        const uint32_t* row = src + i * t.W;
        const uint32_t x = row[w];
        const uint32_t prev = w > 0 ? row[w - 1] : 0u;
        const uint32_t next = w + 1 < t.W ? row[w + 1] : 0u;
        const uint32_t left = (x << 1) | (prev >> 31);   // column c-1 at bit c
        uint32_t right = (x >> 1) | (next << 31);         // column c+1 at bit c
        if (w == t.W - 1) right &= t.last_mask >> 1;      // column `cols` is off-image
        uint32_t y = erode ? (x & left & right) : (x | left | right);
        if (w == t.W - 1) y &= t.last_mask;
        dst[i * t.W + w] = y;
    }
}

// Re-zero buffer rows outside the image (and the two buffer edge rows, whose
// neighbourhoods were not available).
__device__ __forceinline__ void clip_rows(const MorphTile& t, uint32_t* img) {
    const int n = t.NR * t.W;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = e / t.W;
        const int g = t.row0 + i;
        if (g < 0 || g >= t.rows || i == 0 || i == t.NR - 1) img[e] = 0u;
    }
}

// one erosion / dilation with a 3x3 (vert && horiz), 3x1 (vert) or 1x3 (horiz) element
__device__ __forceinline__ void step(const MorphTile& t, bool erode, bool vert, bool horiz) {
    if (vert && horiz) {
        vpass(t, erode);
        __syncthreads();
        hpass(t, t.b, t.a, erode);
    } else if (vert) {
        vpass(t, erode);
        __syncthreads();
        const int n = (t.NR - 2) * t.W;
        for (int e = threadIdx.x; e < n; e += blockDim.x) t.a[t.W + e] = t.b[t.W + e];
    } else {
        hpass(t, t.a, t.b, erode);
        __syncthreads();
        const int n = (t.NR - 2) * t.W;
        for (int e = threadIdx.x; e < n; e += blockDim.x) t.a[t.W + e] = t.b[t.W + e];
    }
    __syncthreads();
    clip_rows(t, t.a);
    __syncthreads();
}

__global__ void __launch_bounds__(kMorphThreads)
consolidate_bits_kernel(const uint32_t* __restrict__ in, int rows, int cols, int tile_rows, int halo,
                        bool along_time, uint32_t* __restrict__ out) {
    extern __shared__ uint32_t mo_smem[];
    const int W = (cols + 31) / 32;
    const int p = blockIdx.y;
    const int r0 = blockIdx.x * tile_rows;
    if (r0 >= rows) return;
    MorphTile t;
    t.NR = tile_rows + 2 * halo;
    t.W = W;
    t.cols = cols;
    t.rows = rows;
    t.row0 = r0 - halo;
    t.last_mask = (cols & 31) ? ((1u << (cols & 31)) - 1u) : 0xffffffffu;
    t.a = mo_smem;
    t.b = mo_smem + t.NR * W;
    const uint32_t* src = in + static_cast<long long>(p) * rows * W;
    for (int e = threadIdx.x; e < t.NR * W; e += blockDim.x) {
        const int g = t.row0 + e / W;
        t.a[e] = (g >= 0 && g < rows) ? src[static_cast<long long>(g) * W + (e % W)] : 0u;
        t.b[e] = 0u;
    }
    __syncthreads();
    // close 3x3: dilate, erode
    step(t, false, true, true);
    step(t, true, true, true);
    // open 3x3: erode, dilate
    step(t, true, true, true);
    step(t, false, true, true);
    // open with the line element: 1x3 along frequency, or 3x1 along time
    step(t, true, along_time, !along_time);
    step(t, false, along_time, !along_time);
    uint32_t* dst = out + static_cast<long long>(p) * rows * W;
    const int nout = min(tile_rows, rows - r0) * W;
    for (int e = threadIdx.x; e < nout; e += blockDim.x)
        dst[static_cast<long long>(r0) * W + e] = t.a[(halo + e / W) * W + (e % W)];
}

cudaError_t consolidate_bits_launch(const uint32_t* in, int n_plots, int rows, int cols, bool along_time,
                                    uint32_t* out, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    const int W = (cols + 31) / 32;
    const int halo = along_time ? 6 : 4;
    int tile_rows = W <= 64 ? 128 : (W <= 128 ? 64 : 32);
    if (tile_rows > rows) tile_rows = rows;
    const size_t smem = sizeof(uint32_t) * 2 * (tile_rows + 2 * halo) * W;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(consolidate_bits_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((rows + tile_rows - 1) / tile_rows, n_plots);
    consolidate_bits_kernel<<<grid, kMorphThreads, smem, st>>>(in, rows, cols, tile_rows, halo, along_time, out);
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
