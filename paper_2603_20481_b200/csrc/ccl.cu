// ccl.cu -- K6: 4-connected component extents on bit-packed masks.
//
// Replaces detector::resolve_components / component_extents /
// label_components and the box conversion (proj/src/detector.cpp:494-635).
// Run-based union-find, batched over plots:
//   1 count   : runs starting per row (start bits = x & ~(x<<1 | carry)),
//               one thread per row over the word-major mask
//   2 scan    : per-plot exclusive row offsets; 3 per-plot pool bases
//   4 emit    : runs in row-major order of their start pixel -> pool
//   5 union   : each run unites with the overlapping runs of the row above
//               (4-connectivity = shared column, :543-555); lock-free
//               union-by-min (CAS on roots), so every root is the smallest run
//               index of its component = its first row-major pixel.  First
//               within 16-row blocks in shared memory, then across the block
//               boundaries in global memory
//   6 flatten : parent -> root; area, max_t, min_f, max_f by atomics
//   7 compact : roots with area >= min_area, numbered densely in root order
//               (= first-pixel order, area filter before numbering: :570-593)
//               -> extents, half-open bin boxes (:622-624) and physical boxes
//               in double (:626-635)
// Capacity: the run pool is sized by the caller; a plot whose runs do not fit
// is flagged (plot_ok = 0, *overflow = 1) and the host re-runs it alone with
// an exact-size pool (capi.cu).
#include "common.cuh"
#include "internal.h"

#include <climits>

namespace ssb {

// Masks are word-major (bits[p][w][r]).  A CTA covers 32 consecutive rows x
// kSeg word segments: warp k walks segment k of each row (lane = row, so a
// warp reads 32 consecutive rows of a word: coalesced).  Starts and ends of
// runs are counted per segment; a run's index is the number of starts before
// its start bit in the row, its end the number of ends before its end bit,
// so segments emit independently once their prefix counts are known.
constexpr int kSeg = kCclSeg;

struct SegRange {
    int w0, w1;
};
__device__ __forceinline__ SegRange seg_range(int W, int k) {
    const int per = (W + kSeg - 1) / kSeg;
    const int w0 = min(W, k * per);
    return {w0, min(W, w0 + per)};
}

// carry into word w0: bit 31 of the row's previous word
__device__ __forceinline__ uint32_t seg_carry(const uint32_t* col, int rs, int w0) {
    return w0 > 0 ? (col[static_cast<long long>(w0 - 1) * rs] >> 31) : 0u;
}

// Also records each segment's exclusive start / end offsets within its row
// (seg_off[p][r][k] = {starts, ends} before segment k), so emit_runs walks
// the mask once.
__global__ void __launch_bounds__(32 * kSeg) count_runs_kernel(const uint32_t* __restrict__ bits, int rows, int W,
                                                               int* row_runs, int2* seg_off) {
    __shared__ int st_s[kSeg][32], en_s[kSeg][32];
    const int p = blockIdx.y;
    const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
    const int r = blockIdx.x * 32 + lane;
    int ns = 0, ne = 0;
    if (r < rows) {
        const int rs = mask_rs(rows);
        const uint32_t* col = bits + static_cast<long long>(p) * W * rs + r;
        const SegRange g = seg_range(W, k);
        uint32_t carry = seg_carry(col, rs, g.w0);
        int w = g.w0;
        for (; w + 8 <= g.w1; w += 8) {  // eight word loads in flight
            uint32_t xs[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) xs[q] = __ldg(col + static_cast<long long>(w + q) * rs);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t sh = (xs[q] << 1) | carry;
                ns += __popc(xs[q] & ~sh);
                ne += __popc(~xs[q] & sh);
                carry = xs[q] >> 31;
            }
        }
        for (; w < g.w1; ++w) {
            const uint32_t x = __ldg(col + static_cast<long long>(w) * rs);
            const uint32_t sh = (x << 1) | carry;
            ns += __popc(x & ~sh);
            ne += __popc(~x & sh);
            carry = x >> 31;
        }
    }
    st_s[k][lane] = ns;
    en_s[k][lane] = ne;
    __syncthreads();
    if (r < rows) {
        int s0 = 0, e0 = 0;
        for (int q = 0; q < k; ++q) {
            s0 += st_s[q][lane];
            e0 += en_s[q][lane];
        }
        seg_off[(static_cast<long long>(p) * rows + r) * kSeg + k] = make_int2(s0, e0);
        if (k == kSeg - 1) row_runs[static_cast<long long>(p) * rows + r] = s0 + ns;
    }
}

__global__ void scan_rows_kernel(const int* row_runs, int rows, int* row_off) {
    __shared__ int red[32];
    __shared__ int carry_s;
    const int p = blockIdx.x;
    const int* in = row_runs + static_cast<long long>(p) * rows;
    int* out = row_off + static_cast<long long>(p) * (rows + 1);
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < rows; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < rows ? in[i] : 0;
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        const int inc = warp_incl_scan(v);
        if (l == 31) red[w] = inc;
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            int x = l < nw ? red[l] : 0;
            x = warp_incl_scan(x);
            if (l < nw) red[l] = x;
        }
        __syncthreads();
        const int carry = carry_s;
        const int excl = carry + (w > 0 ? red[w - 1] : 0) + inc - v;
        if (i < rows) out[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry_s = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[rows] = carry_s;
}

// Pool base of every plot: exclusive prefix of the plots' run totals; a plot
// whose runs would pass pool_cap is flagged (the host then re-runs every plot
// alone with an exact pool, capi.cu).  One 1024-thread block, chunked scan.
__global__ void __launch_bounds__(1024) plot_base_kernel(const int* row_off, int n_plots, int rows, long long pool_cap,
                                                         long long* plot_base, int* plot_ok, int* overflow) {
    __shared__ long long red[32];
    __shared__ long long carry_s;
    __shared__ int of_s;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        carry_s = 0;
        of_s = 0;
    }
    __syncthreads();
    for (int c0 = 0; c0 < n_plots; c0 += blockDim.x) {
        const int p = c0 + threadIdx.x;
        const long long v = p < n_plots ? row_off[static_cast<long long>(p) * (rows + 1) + rows] : 0;
        long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, inc, o);
            if (l >= o) inc += t;
        }
        if (l == 31) red[w] = inc;
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            long long x = l < nw ? red[l] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, x, o);
                if (l >= o) x += t;
            }
            if (l < nw) red[l] = x;
        }
        __syncthreads();
        const long long base = carry_s + (w > 0 ? red[w - 1] : 0) + inc - v;
        if (p < n_plots) {
            plot_base[p] = base;
            const int ok = base + v <= pool_cap ? 1 : 0;
            plot_ok[p] = ok;
            if (!ok) of_s = 1;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry_s = base + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *overflow = of_s;
}

// Runs of one row in column order (start bits x & ~(x<<1|carry), end bits
// ~x & (x<<1|carry)), appended at the row's offset in the pool; segment k of
// the row writes the starts / ends that fall in its words.
__global__ void __launch_bounds__(32 * kSeg) emit_runs_kernel(const uint32_t* __restrict__ bits, int rows, int cols,
                                                              const int* row_off, const int2* __restrict__ seg_off,
                                                              const long long* plot_base, const int* plot_ok,
                                                              CclWorkspace ws) {
    const int W = (cols + 31) / 32;
    const int p = blockIdx.y;
    const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
    const int r = blockIdx.x * 32 + lane;
    if (r >= rows || !plot_ok[p]) return;
    const int rs = mask_rs(rows);
    const uint32_t* col = bits + static_cast<long long>(p) * W * rs + r;
    const SegRange g = seg_range(W, k);
    const int2 so = seg_off[(static_cast<long long>(p) * rows + r) * kSeg + k];
    const long long row0 = plot_base[p] + row_off[static_cast<long long>(p) * (rows + 1) + r];
    long long si = row0 + so.x, ei = row0 + so.y;
    uint32_t carry = seg_carry(col, rs, g.w0);
    auto emit_word = [&](int w, uint32_t x) {
        const uint32_t sh = (x << 1) | carry;
        uint32_t starts = x & ~sh, ends = ~x & sh;
        carry = x >> 31;
        while (starts) {
            const int bpos = __ffs(starts) - 1;
            starts &= starts - 1;
            ws.run_begin[si] = 32 * w + bpos;
            ws.run_row[si] = r;
            ws.parent[si] = static_cast<int>(si);
            ++si;
        }
        while (ends) {
            const int bpos = __ffs(ends) - 1;
            ends &= ends - 1;
            ws.run_end[ei++] = 32 * w + bpos;
        }
    };
    int w = g.w0;
    for (; w + 8 <= g.w1; w += 8) {  // eight word loads in flight
        uint32_t xs[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xs[q] = __ldg(col + static_cast<long long>(w + q) * rs);
#pragma unroll
        for (int q = 0; q < 8; ++q) emit_word(w + q, xs[q]);
    }
    for (; w < g.w1; ++w) emit_word(w, __ldg(col + static_cast<long long>(w) * rs));
    if (k == kSeg - 1 || g.w1 == W) {
        // a run still open after the last word reaches the last column (cols % 32 == 0)
        if (g.w1 == W && g.w0 < g.w1 && carry) ws.run_end[ei] = cols;
    }
}

__device__ __forceinline__ int uf_find(int* parent, int x) {
    for (;;) {
        const int p = __ldcg(parent + x);
        if (p == x) return x;
        const int gp = __ldcg(parent + p);
        if (gp != p) parent[x] = gp;  // path halving; any ancestor is a valid parent
        x = p;
    }
}

// Read-only find for the flatten pass: every thread writes only its own
// parent entry there, so no path-halving store can overwrite a finished one.
__device__ __forceinline__ int uf_root(const int* parent, int x) {
    for (;;) {
        const int p = __ldcg(parent + x);
        if (p == x) return x;
        x = p;
    }
}

__device__ __forceinline__ void uf_unite(int* parent, int a, int b) {
    for (;;) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(parent + a, a, b);  // hook the larger root under the smaller
        if (old == a) return;
        a = old;
    }
}

// Unite the runs of row r with the overlapping runs of row r - 1 (global
// union-find); lanes stride over the row's runs.
__device__ __forceinline__ void unite_row_global(int r, const int* off, long long base, CclWorkspace& ws, int lane,
                                                 int nlanes) {
    const long long prev_b = base + off[r - 1], cur_b = base + off[r], cur_e = base + off[r + 1];
    for (long long i = cur_b + lane; i < cur_e; i += nlanes) {
        const int b = ws.run_begin[i], e = ws.run_end[i];
        long long lo = prev_b, hi = cur_b;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (ws.run_end[mid] > b) hi = mid;
            else lo = mid + 1;
        }
        for (long long q = lo; q < cur_b && ws.run_begin[q] < e; ++q)
            uf_unite(ws.parent, static_cast<int>(i), static_cast<int>(q));
    }
}

// Shared-memory union-find on local run indices (union-by-min: the root is
// the smallest index, i.e. the earliest run in row-major order).
__device__ __forceinline__ int sm_find(int* par, int x) {
    for (;;) {
        const int p = par[x];
        if (p == x) return x;
        const int gp = par[p];
        if (gp != p) par[x] = gp;
        x = p;
    }
}
__device__ __forceinline__ void sm_unite(int* par, int a, int b) {
    for (;;) {
        a = sm_find(par, a);
        b = sm_find(par, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(par + a, a, b);
        if (old == a) return;
        a = old;
    }
}

// Union within blocks of kUB rows: the block's runs (contiguous in the pool)
// are united in shared memory, then every run's parent is set to its
// block-local root and each block-local root gets its block-local component's
// statistics (area, max row, min / max column; area = 0 marks the other runs),
// so the global flatten walks and updates one entry per block-local
// component instead of one per run.  Blocks whose runs exceed kUCap unite in
// global memory and give every run its own statistics.  Rows r0 (a block's
// first row) are joined to the row above by union_boundary_kernel afterwards.
// Launched for every plot, one row included (rows == 1: each run alone).
constexpr int kUB = 16;  // 16 beat 32 (0.78 ms per C5r step) and 64 (1.02)
#ifndef K6_UCAP
#define K6_UCAP 1024
#endif
constexpr int kUCap = K6_UCAP;
#ifndef K6_UTHREADS
#define K6_UTHREADS 256
#endif
constexpr int kUThreads = K6_UTHREADS;  // warp-per-row-pair form: 256 beat 128 (0.72 ms per C5r step), 64 (0.96), 32 (1.27)

__global__ void __launch_bounds__(kUThreads) union_block_kernel(int rows, const int* row_off, const long long* plot_base,
                                                          const int* plot_ok, CclWorkspace ws) {
    __shared__ int sb[kUCap], se[kUCap], sp[kUCap];
    __shared__ int s_area[kUCap], s_maxt[kUCap], s_minf[kUCap], s_maxf[kUCap];
    __shared__ int roff[kUB + 1];
    const int p = blockIdx.y;
    const int r0 = blockIdx.x * kUB, r1 = min(rows, r0 + kUB);
    if (!plot_ok[p] || r0 >= rows) return;
    const int* off = row_off + static_cast<long long>(p) * (rows + 1);
    const long long base = plot_base[p];
    const int g0 = off[r0], n = off[r1] - g0;
    const int lane = threadIdx.x & 31;
    if (n > kUCap) {  // dense block: rows r0+1 .. r1-1 in global memory, one warp per row
        for (int r = r0 + 1 + (threadIdx.x >> 5); r < r1; r += blockDim.x >> 5)
            unite_row_global(r, off, base, ws, lane, 32);
        for (int r = r0 + (threadIdx.x >> 5); r < r1; r += blockDim.x >> 5)
            for (long long i = base + off[r] + lane; i < base + off[r + 1]; i += 32) {
                const int b = ws.run_begin[i], e = ws.run_end[i];
                ws.area[i] = static_cast<unsigned long long>(e - b);
                ws.max_t[i] = r;
                ws.min_f[i] = b;
                ws.max_f[i] = e - 1;
            }
        return;
    }
    const long long gb = base + g0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sb[i] = ws.run_begin[gb + i];
        se[i] = ws.run_end[gb + i];
        sp[i] = i;
        s_area[i] = 0;
        s_maxt[i] = -1;
        s_minf[i] = INT_MAX;
        s_maxf[i] = -1;
    }
    for (int j = threadIdx.x; j <= r1 - r0; j += blockDim.x) roff[j] = off[r0 + j] - g0;
    __syncthreads();
    // one thread per run (a block holds ~70 runs on a C5r plot: a warp per row
    // pair left most lanes idle and walked the pairs in turn); the run's row
    // is the last j with roff[j] <= i
    auto row_of = [&](int i) {
        int lo = 0, hi = r1 - r0 - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (roff[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    for (int i = roff[1] + threadIdx.x; i < n; i += blockDim.x) {
        const int j = row_of(i);
        const int pb = roff[j - 1], cb = roff[j];
        const int b = sb[i], e = se[i];
        int lo = pb, hi = cb;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (se[mid] > b) hi = mid;
            else lo = mid + 1;
        }
        for (int q = lo; q < cb && sb[q] < e; ++q) sm_unite(sp, i, q);
    }
    __syncthreads();
    // parents and block-local statistics
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int x = i;
        while (sp[x] != x) x = sp[x];
        ws.parent[gb + i] = static_cast<int>(gb + x);
        atomicAdd(&s_area[x], se[i] - sb[i]);
        atomicMax(&s_maxt[x], r0 + row_of(i));
        atomicMin(&s_minf[x], sb[i]);
        atomicMax(&s_maxf[x], se[i] - 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int a = s_area[i];  // > 0 exactly for the block-local roots
        ws.area[gb + i] = static_cast<unsigned long long>(a);
        if (a > 0) {
            ws.max_t[gb + i] = s_maxt[i];
            ws.min_f[gb + i] = s_minf[i];
            ws.max_f[gb + i] = s_maxf[i];
        }
    }
}

// Block boundaries: row k*kUB joins row k*kUB - 1 (global union-find).
__global__ void union_boundary_kernel(int rows, const int* row_off, const long long* plot_base, const int* plot_ok,
                                      CclWorkspace ws) {
    const int p = blockIdx.y;
    const int r = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) + 1) * kUB;
    if (r >= rows || !plot_ok[p]) return;
    const int* off = row_off + static_cast<long long>(p) * (rows + 1);
    unite_row_global(r, off, plot_base[p], ws, threadIdx.x & 31, 32);
}

// Entries with statistics (area > 0: block-local roots, or every run of a
// dense block) hook onto their global root and add their statistics to it.
// Only those entries change; a run's component is its block-local root's.
__global__ void flatten_kernel(int rows, const int* row_off, const long long* plot_base, const int* plot_ok,
                               CclWorkspace ws) {
    const int p = blockIdx.y;
    if (!plot_ok[p]) return;
    const long long base = plot_base[p];
    const long long n = row_off[static_cast<long long>(p) * (rows + 1) + rows];
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = base + k;
        const unsigned long long a = ws.area[i];
        if (a == 0ull) continue;
        const int root = uf_root(ws.parent, static_cast<int>(i));
        if (root == static_cast<int>(i)) continue;
        ws.parent[i] = root;
        atomicAdd(ws.area + root, a);
        atomicMax(ws.max_t + root, ws.max_t[i]);
        atomicMin(ws.min_f + root, ws.min_f[i]);
        atomicMax(ws.max_f + root, ws.max_f[i]);
    }
}

__global__ void compact_kernel(int rows, int cols, const int* row_off, const long long* plot_base,
                               const int* plot_ok, CclWorkspace ws, CclLaunch L) {
    __shared__ int red[32];
    __shared__ int carry_s;
    const int p = blockIdx.x;
    if (!plot_ok[p]) {
        if (threadIdx.x == 0) L.n_comp[p] = -1;
        return;
    }
    const long long base = plot_base[p];
    const long long n = row_off[static_cast<long long>(p) * (rows + 1) + rows];
    const double fs = L.fs;
    // TFPlotView::dt_s = cols / fs (frontend.hpp:61); STFT extension: hop / fs
    const double dt = __ddiv_rn(static_cast<double>(L.time_bins > 0 ? L.time_bins : cols), fs);
    const double df = __ddiv_rn(fs, static_cast<double>(cols));
    const double seq = L.start_seq ? static_cast<double>(L.start_seq[p]) : 0.0;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (long long c0 = 0; c0 < n; c0 += blockDim.x) {
        const long long k = c0 + threadIdx.x;
        const long long i = base + k;
        int flag = 0;
        if (k < n) flag = (ws.parent[i] == static_cast<int>(i) && ws.area[i] >= static_cast<unsigned long long>(L.min_area)) ? 1 : 0;
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        const int inc = warp_incl_scan(flag);
        if (l == 31) red[w] = inc;
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            int x = l < nw ? red[l] : 0;
            x = warp_incl_scan(x);
            if (l < nw) red[l] = x;
        }
        __syncthreads();
        const int carry = carry_s;
        const int id = carry + (w > 0 ? red[w - 1] : 0) + inc - flag;
        if (k < n && ws.parent[i] == static_cast<int>(i)) ws.dense[i] = flag ? id : -1;  // read per root only
        if (flag) {
            if (id < L.cap) {
                const long long o = static_cast<long long>(p) * L.cap + id;
                const int min_t = ws.run_row[i], max_t = ws.max_t[i];
                const int min_f = ws.min_f[i], max_f = ws.max_f[i];
                if (L.extents) {
                    long long* e = L.extents + 5 * o;
                    e[0] = min_t;
                    e[1] = max_t;
                    e[2] = min_f;
                    e[3] = max_f;
                    e[4] = static_cast<long long>(ws.area[i]);
                }
                if (L.bin_boxes) {
                    int* bb = L.bin_boxes + 4 * o;
                    bb[0] = min_t;
                    bb[1] = max_t + 1;
                    bb[2] = min_f;
                    bb[3] = max_f + 1;
                }
                if (L.boxes) {
                    double* bx = L.boxes + 4 * o;
                    bx[0] = __dmul_rn(static_cast<double>(min_f - cols / 2), df);
                    bx[1] = __dmul_rn(static_cast<double>(max_f + 1 - cols / 2), df);
                    bx[2] = __dmul_rn(__dadd_rn(seq, static_cast<double>(min_t)), dt);
                    bx[3] = __dmul_rn(__dadd_rn(seq, static_cast<double>(max_t + 1)), dt);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry_s = id + flag;
        __syncthreads();
    }
    if (threadIdx.x == 0) L.n_comp[p] = carry_s;
}

__global__ void labels_kernel(int rows, int cols, const int* row_off, CclWorkspace ws, int32_t* labels) {
    const long long n = row_off[rows];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int id = ws.dense[uf_root(ws.parent, static_cast<int>(i))];
        if (id < 0) continue;
        int32_t* row = labels + static_cast<long long>(ws.run_row[i]) * cols;
        for (int c = ws.run_begin[i]; c < ws.run_end[i]; ++c) row[c] = id + 1;
    }
}

cudaError_t ccl_launch(const CclLaunch& L, cudaStream_t st) {
    if (L.n_plots <= 0 || L.rows <= 0 || L.cols <= 0) return cudaSuccess;
    const int W = (L.cols + 31) / 32;
    const CclWorkspace& ws = L.ws;
    dim3 tgrid((L.rows + 31) / 32, L.n_plots);
    count_runs_kernel<<<tgrid, 32 * kSeg, 0, st>>>(L.bits, L.rows, W, ws.row_runs, ws.seg_off);
    scan_rows_kernel<<<L.n_plots, 1024, 0, st>>>(ws.row_runs, L.rows, ws.row_off);
    plot_base_kernel<<<1, 1024, 0, st>>>(ws.row_off, L.n_plots, L.rows, ws.pool_cap, ws.plot_base, ws.plot_ok,
                                         ws.overflow);
    emit_runs_kernel<<<tgrid, 32 * kSeg, 0, st>>>(L.bits, L.rows, L.cols, ws.row_off, ws.seg_off, ws.plot_base,
                                                  ws.plot_ok, ws);
    {
        const int nblk = (L.rows + kUB - 1) / kUB;
        union_block_kernel<<<dim3(nblk, L.n_plots), kUThreads, 0, st>>>(L.rows, ws.row_off, ws.plot_base, ws.plot_ok, ws);
        if (nblk > 1) {
            dim3 bgrid((nblk - 1 + 7) / 8, L.n_plots);
            union_boundary_kernel<<<bgrid, 256, 0, st>>>(L.rows, ws.row_off, ws.plot_base, ws.plot_ok, ws);
        }
    }
    int per_plot = 4096 / (L.n_plots > 0 ? L.n_plots : 1);
    if (per_plot < 2) per_plot = 2;
    if (per_plot > 64) per_plot = 64;
    dim3 fgrid(per_plot, L.n_plots);
    flatten_kernel<<<fgrid, 256, 0, st>>>(L.rows, ws.row_off, ws.plot_base, ws.plot_ok, ws);
    compact_kernel<<<L.n_plots, 512, 0, st>>>(L.rows, L.cols, ws.row_off, ws.plot_base, ws.plot_ok, ws, L);
    if (L.labels) {
        cudaMemsetAsync(L.labels, 0, sizeof(int32_t) * static_cast<size_t>(L.rows) * L.cols, st);
        // single-plot use: plot 0's runs start at pool index 0
        labels_kernel<<<256, 256, 0, st>>>(L.rows, L.cols, ws.row_off, ws, L.labels);
    }
    return cudaGetLastError();
}

} // namespace ssb
