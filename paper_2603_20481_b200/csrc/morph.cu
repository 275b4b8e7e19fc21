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

// One CTA: TR output rows x all W words, buffers of NR = TR + 2H rows.
// W is a template parameter so the (row, word) decomposition of the thread
// index is shifts, not divisions.  The two buffer edge rows are never
// recomputed: the invalid band grows one row per vertical step, which the H
// halo rows absorb (H = number of vertical steps).  Rows outside the image
// are re-zeroed after every step (only tiles at the image edges have any).
template <int WC>
struct Tile {
    int Wr;  // runtime word count when WC == 0
    __device__ __forceinline__ int W() const { return WC ? WC : Wr; }
    __device__ __forceinline__ int RPI() const { return W() >= kMorphThreads ? 1 : kMorphThreads / W(); }
    uint32_t* a;
    uint32_t* b;
    int NR, row0, rows;
    uint32_t last_mask;
    int out_top, out_bot;  // buffer rows [0,out_top) and [out_bot,NR) lie outside the image

    __device__ __forceinline__ void vpass(bool erode) const {
        const int w = threadIdx.x % W();
        for (int i = 1 + static_cast<int>(threadIdx.x) / W(); i < NR - 1; i += RPI()) {
            const uint32_t u = a[(i - 1) * W() + w], c = a[i * W() + w], d = a[(i + 1) * W() + w];
            b[i * W() + w] = erode ? (u & c & d) : (u | c | d);
        }
    }
    __device__ __forceinline__ void hpass(const uint32_t* src, uint32_t* dst, bool erode) const {
        const int w = threadIdx.x % W();
        for (int i = 1 + static_cast<int>(threadIdx.x) / W(); i < NR - 1; i += RPI()) {
            const uint32_t* row = src + i * W();
            const uint32_t x = row[w];
            const uint32_t prev = w > 0 ? row[w - 1] : 0u;
            const uint32_t next = w + 1 < W() ? row[w + 1] : 0u;
            const uint32_t left = (x << 1) | (prev >> 31);  // column c-1 at bit c
            const uint32_t right = (x >> 1) | (next << 31); // column c+1 at bit c
            uint32_t y = erode ? (x & left & right) : (x | left | right);
            if (w == W() - 1) y &= last_mask;
            dst[i * W() + w] = y;
        }
    }
    __device__ __forceinline__ void copy_back() const {
        const int w = threadIdx.x % W();
        for (int i = 1 + static_cast<int>(threadIdx.x) / W(); i < NR - 1; i += RPI()) a[i * W() + w] = b[i * W() + w];
    }
    __device__ __forceinline__ void clip() const {
        if (out_top == 0 && out_bot == NR) return;
        const int w = threadIdx.x % W();
        for (int i = static_cast<int>(threadIdx.x) / W(); i < NR; i += RPI())
            if (i < out_top || i >= out_bot) a[i * W() + w] = 0u;
    }
    // one erosion / dilation: 3x3 (vert && horiz), 3x1 (vert), 1x3 (horiz)
    __device__ __forceinline__ void step(bool erode, bool vert, bool horiz) const {
        if (vert) {
            vpass(erode);
            __syncthreads();
            if (horiz) hpass(b, a, erode);
            else copy_back();
        } else {
            hpass(a, b, erode);
            __syncthreads();
            copy_back();
        }
        __syncthreads();
        clip();
        __syncthreads();
    }
};

template <int WC>
__global__ void __launch_bounds__(kMorphThreads)
consolidate_bits_kernel(const uint32_t* __restrict__ in, const uint8_t* __restrict__ planes, int rows, int cols,
                        int tile_rows, int halo, bool along_time, uint32_t* __restrict__ out) {
    extern __shared__ uint32_t mo_smem[];
    const int p = blockIdx.y;
    const int r0 = blockIdx.x * tile_rows;
    if (r0 >= rows) return;
    Tile<WC> t;
    t.Wr = (cols + 31) / 32;
    const int W = t.W();
    t.NR = tile_rows + 2 * halo;
    t.row0 = r0 - halo;
    t.rows = rows;
    t.last_mask = (cols & 31) ? ((1u << (cols & 31)) - 1u) : 0xffffffffu;
    t.out_top = t.row0 < 0 ? -t.row0 : 0;
    t.out_bot = rows - t.row0 < t.NR ? rows - t.row0 : t.NR;
    t.a = mo_smem;
    t.b = mo_smem + t.NR * W;
    const int w = threadIdx.x % W;
    if (planes) {
        // byte planes [p][4W][rows]: lanes walk rows so each plane read is contiguous
        const uint8_t* pl = planes + static_cast<long long>(p) * 4 * W * rows;
        for (int e = threadIdx.x; e < W * t.NR; e += kMorphThreads) {
            const int ww = e / t.NR, i = e - ww * t.NR;
            const int g = t.row0 + i;
            uint32_t word = 0u;
            if (g >= 0 && g < rows) {
                const uint8_t* b = pl + static_cast<long long>(4 * ww) * rows + g;
                word = static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[rows]) << 8) |
                       (static_cast<uint32_t>(b[2 * static_cast<long long>(rows)]) << 16) |
                       (static_cast<uint32_t>(b[3 * static_cast<long long>(rows)]) << 24);
            }
            t.a[i * W + ww] = word;
        }
    } else {
        const uint32_t* src = in + static_cast<long long>(p) * rows * W;
        for (int i = static_cast<int>(threadIdx.x) / W; i < t.NR; i += t.RPI()) {
            const int g = t.row0 + i;
            t.a[i * W + w] = (g >= 0 && g < rows) ? src[static_cast<long long>(g) * W + w] : 0u;
        }
    }
    __syncthreads();
    t.step(false, true, true);  // close 3x3: dilate, erode
    t.step(true, true, true);
    t.step(true, true, true);   // open 3x3: erode, dilate
    t.step(false, true, true);
    t.step(true, along_time, !along_time);  // open with the line element
    t.step(false, along_time, !along_time);
    uint32_t* dst = out + static_cast<long long>(p) * rows * W;
    const int nrow = min(tile_rows, rows - r0);
    for (int i = static_cast<int>(threadIdx.x) / W; i < nrow; i += t.RPI())
        dst[static_cast<long long>(r0 + i) * W + w] = t.a[(halo + i) * W + w];
}

template <int WC>
static cudaError_t consolidate_w(const uint32_t* in, const uint8_t* planes, int n_plots, int rows, int cols,
                                 bool along_time, uint32_t* out, cudaStream_t st) {
    const int W = WC ? WC : (cols + 31) / 32;
    const int halo = along_time ? 6 : 4;
    // ~128 output rows per CTA for narrow masks, 32 for the widest
    int tile_rows = W <= 32 ? 128 : (W <= 128 ? 64 : 32);
    if (tile_rows > rows) tile_rows = rows;
    const size_t smem = sizeof(uint32_t) * 2 * (tile_rows + 2 * halo) * W;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(consolidate_bits_kernel<WC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((rows + tile_rows - 1) / tile_rows, n_plots);
    consolidate_bits_kernel<WC><<<grid, kMorphThreads, smem, st>>>(in, planes, rows, cols, tile_rows, halo, along_time,
                                                                 out);
    return cudaGetLastError();
}

cudaError_t consolidate_bits_launch(const uint32_t* in, const uint8_t* planes, int n_plots, int rows, int cols,
                                    bool along_time, uint32_t* out, cudaStream_t st) {
    if (n_plots <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    switch ((cols + 31) / 32) {
    case 1: return consolidate_w<1>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 2: return consolidate_w<2>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 4: return consolidate_w<4>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 8: return consolidate_w<8>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 16: return consolidate_w<16>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 32: return consolidate_w<32>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 64: return consolidate_w<64>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 128: return consolidate_w<128>(in, planes, n_plots, rows, cols, along_time, out, st);
    case 256: return consolidate_w<256>(in, planes, n_plots, rows, cols, along_time, out, st);
    default: return consolidate_w<0>(in, planes, n_plots, rows, cols, along_time, out, st);  // any width
    }
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
