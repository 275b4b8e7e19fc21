// floor.cu -- K2 column PSD (stage form) and K3 noise floor + column pruning.
//
// K3 replaces detector::smooth_and_floor + prune_columns
// (proj/src/detector.cpp:210-255), one CTA per plot:
//   db[k]   = raw > 0 ? 10.0f * log10f(raw) : -3000.0f        (glibc log10f port)
//   sdb[i]  = float( sum_{j=-h..h} acc + w_j * (double)db[mirror(i+j)] )
//             -- a rounded multiply then a rounded add, in j order (:203-204)
//   s[i]    = powf(10.0f, sdb[i] / 10.0f)                      (glibc powf port)
//   floor   = lowest strict local minimum (plateau counted once at its first
//             index, :229-242), else the global minimum (:243)
//   thr     = float(double(floor) * pow(10, margin/10))        (:246-247)
//   active  = { k : raw[k] >= thr } ascending                  (:250-255)
// The SG weights come from the host (host_consts.cpp restates :84-142 with the
// three fused updates GCC emits); pow(10, margin/10) is a host-libm constant.
#include "common.cuh"
#include "glibc_libm.cuh"
#include "internal.h"

#include <cfloat>

namespace ssb {

constexpr int kFloorThreads = 512;

__device__ __forceinline__ int mirror_index(int i, int n) {
    if (i < 0) return -i;
    if (i >= n) return 2 * (n - 1) - i;
    return i;
}

__device__ __forceinline__ float block_min(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    v = (threadIdx.x < nw) ? red[threadIdx.x] : INFINITY;
    if (w == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    const float r = red[0];
    __syncthreads();
    return r;
}

// Exclusive block scan of one int per thread; returns the exclusive prefix and
// writes the total to *total.
__device__ __forceinline__ int block_excl_scan(int v, int* red, int* total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int inc = warp_incl_scan(v);
    __syncthreads();
    if (l == 31) red[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        int x = l < nw ? red[l] : 0;
        x = warp_incl_scan(x);
        if (l < nw) red[l] = x;
    }
    __syncthreads();
    const int before = (w > 0 ? red[w - 1] : 0) + inc - v;
    *total = red[((blockDim.x + 31) >> 5) - 1];
    __syncthreads();
    return before;
}

__device__ __forceinline__ double fir_at(const float* db, const double* w, int i, int n, int h) {
    double acc = 0.0;
    for (int j = -h; j <= h; ++j)
        acc = __dadd_rn(acc, __dmul_rn(w[j + h], static_cast<double>(db[mirror_index(i + j, n)])));
    return acc;
}

__global__ void __launch_bounds__(kFloorThreads) floor_kernel(FloorLaunch a) {
    extern __shared__ double fl_smem[];
    const int n = a.n;
    const int h = (a.window - 1) / 2;
    double* w = fl_smem;
    const int p = blockIdx.x;
    // dB and smoothed rows: shared memory, or global scratch for very wide plots
    float* db = a.scratch ? a.scratch + 2LL * p * n : reinterpret_cast<float*>(w + a.window);
    float* s = db + n;
    __shared__ float red_f[32];
    __shared__ int red_i[32];

    const float* raw = a.raw + static_cast<long long>(p) * n;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int i = tid; i < a.window; i += nt) w[i] = a.weights[i];
    for (int k = tid; k < n; k += nt) {
        const float r = raw[k];
        db[k] = r > 0.0f ? __fmul_rn(10.0f, glibc_log10f(r, a.fma_variant)) : -3000.0f;
    }
    __syncthreads();
    bool my_nan = false;
    for (int i = tid; i < n; i += nt) {
        const float sdb = __double2float_rn(fir_at(db, w, i, n, h));
        const float sv = glibc_powf10(__fdiv_rn(sdb, 10.0f), a.fma_variant);
        s[i] = sv;
        a.smoothed[static_cast<long long>(p) * n + i] = sv;
        my_nan |= (sv != sv);
    }
    const bool any_nan = __syncthreads_or(my_nan);

    // strict local minima, plateaus counted once at their first index
    float best = INFINITY;
    for (int i = 1 + tid; i < n - 1; i += nt) {
        const float si = s[i];
        const bool visited = (i == 1) || !(si == s[i - 1]);
        if (!visited) continue;
        int j = i;
        while (j + 1 < n && s[j + 1] == si) ++j;
        const bool left_up = s[i - 1] > si;
        const bool right_up = (j + 1 < n) && s[j + 1] > si;
        if (left_up && right_up && si < best) best = si;
    }
    float fl = block_min(best, red_f);
    if (!(fl < INFINITY)) {
        // no strict local minimum: std::min_element (first smallest under '<')
        if (!any_nan) {
            float m = INFINITY;
            for (int i = tid; i < n; i += nt) m = fminf(m, s[i]);
            fl = block_min(m, red_f);
        } else {
            __shared__ float seq_min;
            if (tid == 0) {
                float m = s[0];
                for (int i = 1; i < n; ++i)
                    if (s[i] < m) m = s[i];
                seq_min = m;
            }
            __syncthreads();
            fl = seq_min;
        }
    }
    const float thr = __double2float_rn(__dmul_rn(static_cast<double>(fl), a.pow10_margin));
    if (tid == 0) {
        a.floor_thr[2 * p + 0] = fl;
        a.floor_thr[2 * p + 1] = thr;
    }

    // prune: contiguous chunk per thread, block scan for the ascending compaction
    const int chunk = (n + nt - 1) / nt;
    const int k0 = tid * chunk;
    const int k1 = min(n, k0 + chunk);
    int cnt = 0;
    for (int k = k0; k < k1; ++k) cnt += raw[k] >= thr ? 1 : 0;
    int total = 0;
    int off = block_excl_scan(cnt, red_i, &total);
    int* act = a.active + static_cast<long long>(p) * n;
    for (int k = k0; k < k1; ++k)
        if (raw[k] >= thr) act[off++] = k;
    if (tid == 0) a.n_active[p] = total;
    if (a.active_bits) {
        const int W = (n + 31) / 32;
        uint32_t* bits = a.active_bits + static_cast<long long>(p) * W;
        for (int wd = tid; wd < W; wd += nt) {
            uint32_t b = 0;
            for (int q = 0; q < 32; ++q) {
                const int k = wd * 32 + q;
                if (k < n && raw[k] >= thr) b |= 1u << q;
            }
            bits[wd] = b;
        }
    }
    if (a.group_list) {
        // K4's work list: the plot's 8-column groups with an active column, in
        // group order, in one block of the batch list reserved by one atomic
        const int G = (n + 7) / 8;
        auto active_group = [&](int g) {
            bool any = false;
            for (int k = 8 * g; k < min(n, 8 * g + 8); ++k) any |= raw[k] >= thr;
            return any ? 1 : 0;
        };
        int mine = 0;
        for (int g = tid; g < G; g += nt) mine += active_group(g);
        int total_g = 0;
        (void)block_excl_scan(mine, red_i, &total_g);
        __shared__ int base_s;
        if (tid == 0) base_s = atomicAdd(a.group_count, total_g);
        __syncthreads();
        int base = base_s;
        for (int g0 = 0; g0 < G; g0 += nt) {
            const int g = g0 + tid;
            const int f = g < G ? active_group(g) : 0;
            int round_total = 0;
            const int o = block_excl_scan(f, red_i, &round_total);
            if (f) a.group_list[base + o] = p * G + g;
            base += round_total;
        }
    }
}

cudaError_t floor_launch(const FloorLaunch& L, cudaStream_t st) {
    if (L.n_plots <= 0) return cudaSuccess;
    if (floor_needs_scratch(L.n, L.window) && !L.scratch) return cudaErrorInvalidValue;
    const size_t smem = sizeof(double) * L.window + (L.scratch ? 0 : sizeof(float) * 2 * L.n);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(floor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    floor_kernel<<<L.n_plots, kFloorThreads, smem, st>>>(L);
    return cudaGetLastError();
}

// Stage form of savgol_smooth (detector.cpp:192-208): one CTA.
__global__ void __launch_bounds__(kFloorThreads) savgol_kernel(const float* v, int n, int window,
                                                               const double* weights, float* out) {
    extern __shared__ double sg_smem[];
    double* w = sg_smem;
    float* vals = reinterpret_cast<float*>(w + window);
    for (int i = threadIdx.x; i < window; i += blockDim.x) w[i] = weights[i];
    for (int i = threadIdx.x; i < n; i += blockDim.x) vals[i] = v[i];
    __syncthreads();
    const int h = (window - 1) / 2;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = __double2float_rn(fir_at(vals, w, i, n, h));
}

cudaError_t savgol_launch(const float* v, int n, int window, const double* weights, float* out,
                          cudaStream_t st) {
    const size_t smem = sizeof(double) * window + sizeof(float) * n;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(savgol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    savgol_kernel<<<1, kFloorThreads, smem, st>>>(v, n, window, weights, out);
    return cudaGetLastError();
}

// Stage form of estimate_psd_into (detector.cpp:170-184): one thread per
// column, rows in order, 8 loads in flight.
__global__ void psd_cols_kernel(const float* __restrict__ tf, int rows, int cols, int c0, int c1,
                                float* __restrict__ out) {
    const int p = blockIdx.y;
    const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= c1) return;
    const float* base = tf + static_cast<long long>(p) * rows * cols + c;
    double acc = 0.0;
    int r = 0;
    for (; r + 8 <= rows; r += 8) {
        float x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = __ldg(base + static_cast<long long>(r + q) * cols);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double d = static_cast<double>(x[q]);
            acc = __fma_rn(d, d, acc);
        }
    }
    for (; r < rows; ++r) {
        const double d = static_cast<double>(__ldg(base + static_cast<long long>(r) * cols));
        acc = __fma_rn(d, d, acc);
    }
    const double inv = __ddiv_rn(1.0, static_cast<double>(rows));
    out[static_cast<long long>(p) * (c1 - c0) + (c - c0)] = __double2float_rn(__dmul_rn(acc, inv));
}

// Tiled form for 8-column groups (16-byte aligned rows): one CTA per (plot,
// 8 columns).  All 256 threads stream row chunks (256 rows x 32 B) into a
// 4-deep shared ring with cp.async; the 8 owning threads then run each
// column's sum in row order out of shared memory.  Keeps ~24 KB per CTA in
// flight, so even one plot (F/8 CTAs) streams its TF plot at a useful rate
// where the thread-per-column form is bound by 8 loads in flight per column.
constexpr int kPsdTileCols = 8;
constexpr int kPsdTileRows = 256;
constexpr int kPsdStages = 4;

__device__ __forceinline__ void psd_cp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}

__global__ void __launch_bounds__(kPsdTileRows) psd_tile_kernel(const float* __restrict__ tf, int rows, int cols,
                                                               int c0, int c1, float* __restrict__ out) {
    __shared__ __align__(16) float ring[kPsdStages][kPsdTileRows * kPsdTileCols];
    const int g = blockIdx.x, p = blockIdx.y, t = threadIdx.x;
    const float* base = tf + static_cast<long long>(p) * rows * cols + c0 + g * kPsdTileCols;
    const int nchunks = (rows + kPsdTileRows - 1) / kPsdTileRows;
    auto load = [&](int chunk) {
        if (chunk < nchunks) {
            const int r = chunk * kPsdTileRows + t;
            if (r < rows) {
                float* dst = &ring[chunk % kPsdStages][t * kPsdTileCols];
                const float* src = base + static_cast<long long>(r) * cols;
                psd_cp16(dst, src);
                psd_cp16(dst + 4, src + 4);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int c = 0; c < kPsdStages - 1; ++c) load(c);
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        load(c + kPsdStages - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(kPsdStages - 1) : "memory");
        __syncthreads();
        if (t < kPsdTileCols) {
            const float* v = &ring[c % kPsdStages][t];
            const int nr = min(kPsdTileRows, rows - c * kPsdTileRows);
            int r = 0;
            for (; r + 8 <= nr; r += 8) {
                float x[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) x[q] = v[(r + q) * kPsdTileCols];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double d = static_cast<double>(x[q]);
                    acc = __fma_rn(d, d, acc);
                }
            }
            for (; r < nr; ++r) {
                const double d = static_cast<double>(v[r * kPsdTileCols]);
                acc = __fma_rn(d, d, acc);
            }
        }
        __syncthreads();  // slot c % stages is refilled by the load at c + 1
    }
    if (t < kPsdTileCols) {
        const double inv = __ddiv_rn(1.0, static_cast<double>(rows));
        out[static_cast<long long>(p) * (c1 - c0) + g * kPsdTileCols + t] = __double2float_rn(__dmul_rn(acc, inv));
    }
}

// Batch form: one warp per 32-column stripe of a plot (lane = column, every
// row read is one 128-byte line), 16 rows of loads in flight per lane, then
// the 16 sums in row order.  No shared memory, no barriers: with enough
// plots there are far more column chains than the FP64 pipe needs, so the
// kernel streams the TF plot at HBM rate.
constexpr int kPsdStripeRows = 16;

__global__ void __launch_bounds__(256) psd_stripe_kernel(const float* __restrict__ tf, int n_plots, int rows, int cols,
                                                         int c0, int c1, int stripes, float* __restrict__ out) {
    const long long gw = blockIdx.x * 8LL + (threadIdx.x >> 5);  // global warp = (plot, stripe)
    const int p = static_cast<int>(gw / stripes), sidx = static_cast<int>(gw % stripes);
    const int c = c0 + sidx * 32 + (threadIdx.x & 31);
    if (p >= n_plots || c >= c1) return;
    const float* base = tf + static_cast<long long>(p) * rows * cols + c;
    double acc = 0.0;
    int r = 0;
    for (; r + kPsdStripeRows <= rows; r += kPsdStripeRows) {
        float x[kPsdStripeRows];
#pragma unroll
        for (int q = 0; q < kPsdStripeRows; ++q) x[q] = __ldcs(base + static_cast<long long>(r + q) * cols);
#pragma unroll
        for (int q = 0; q < kPsdStripeRows; ++q) {
            const double d = static_cast<double>(x[q]);
            acc = __fma_rn(d, d, acc);
        }
    }
    for (; r < rows; ++r) {
        const double d = static_cast<double>(__ldcs(base + static_cast<long long>(r) * cols));
        acc = __fma_rn(d, d, acc);
    }
    const double inv = __ddiv_rn(1.0, static_cast<double>(rows));
    out[static_cast<long long>(p) * (c1 - c0) + (c - c0)] = __double2float_rn(__dmul_rn(acc, inv));
}

cudaError_t psd_cols_launch(const float* tf, int n_plots, int rows, int cols, int c0, int c1,
                            float* out, cudaStream_t st) {
    const int w = c1 - c0;
    if (w <= 0 || n_plots <= 0) return cudaSuccess;
    const bool aligned = reinterpret_cast<uintptr_t>(tf) % 16 == 0 && cols % 4 == 0 && c0 % 4 == 0;
    // enough column chains to keep every SM's FP64 pipe busy: warp stripes
    if (static_cast<long long>(n_plots) * w >= 148LL * 512) {
        const int stripes = (w + 31) / 32;
        const long long warps = static_cast<long long>(stripes) * n_plots;
        psd_stripe_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, st>>>(tf, n_plots, rows, cols, c0, c1,
                                                                                  stripes, out);
        return cudaGetLastError();
    }
    if (aligned && w % kPsdTileCols == 0) {
        dim3 grid(w / kPsdTileCols, n_plots);
        psd_tile_kernel<<<grid, kPsdTileRows, 0, st>>>(tf, rows, cols, c0, c1, out);
        return cudaGetLastError();
    }
    dim3 grid((w + 127) / 128, n_plots);
    psd_cols_kernel<<<grid, 128, 0, st>>>(tf, rows, cols, c0, c1, out);
    return cudaGetLastError();
}

// prune_columns (detector.cpp:250-255) against a given threshold: one CTA,
// ascending compaction by block scan.
__global__ void __launch_bounds__(kFloorThreads) prune_kernel(const float* raw, int n, float thr, int* active,
                                                               int* n_active) {
    __shared__ int red_i[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int chunk = (n + nt - 1) / nt;
    const int k0 = tid * chunk;
    const int k1 = min(n, k0 + chunk);
    int cnt = 0;
    for (int k = k0; k < k1; ++k) cnt += raw[k] >= thr ? 1 : 0;
    int total = 0;
    int off = block_excl_scan(cnt, red_i, &total);
    for (int k = k0; k < k1; ++k)
        if (raw[k] >= thr) active[off++] = k;
    if (tid == 0) *n_active = total;
}

cudaError_t prune_launch(const float* raw, int n, float thr, int* active, int* n_active, cudaStream_t st) {
    prune_kernel<<<1, kFloorThreads, 0, st>>>(raw, n, thr, active, n_active);
    return cudaGetLastError();
}

__global__ void libm_test_kernel(const float* x, long long n, int which, bool fma_variant, float* out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = which == 0 ? glibc_log10f(x[i], fma_variant) : glibc_powf10(x[i], fma_variant);
}

cudaError_t libm_test_launch(const float* x, long long n, int which, bool fma_variant, float* out,
                             cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    libm_test_kernel<<<148 * 8, 256, 0, st>>>(x, n, which, fma_variant, out);
    return cudaGetLastError();
}

} // namespace ssb
