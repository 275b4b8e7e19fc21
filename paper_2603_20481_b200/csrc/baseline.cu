// baseline.cu -- device part of the Searchlight-style baseline detector
// (baseline::baseline_detect, proj/src/baseline.cpp:103-176).
//
// The reference's cost is the dyadic kernel bank: for every kernel size
// (2^i x 2^j, up to 121 at 2000 x 1024) it evaluates the summed-area mean of
// the window around every cell.  Here the summed-area table (SAT) and the
// per-size candidate bitmaps (mean > seed threshold) are built on the GPU;
// the greedy walk over candidates, box growth and merging -- inherently
// sequential, a few dependent lookups per step -- stay on the host
// (csrc/baseline_host.cpp) with the same double arithmetic.
//
// SAT arithmetic (baseline.cpp:15-38): per row a running double sum of x^2
// (x float, x*x exact in double), then s[t+1][f+1] = s[t][f+1] + row_acc[f]:
// two sequential chains, kept sequential (thread per row, then thread per
// column) so every partial sum rounds exactly as the reference's loop does.
#include "common.cuh"
#include "internal.h"

namespace ssb {

// R[t][f] = sum_{g <= f} x[t][g]^2 in g order.  Thread per row; rows of 32
// threads read 32 different rows per instruction, so stage 32 x 32 tiles
// through shared memory to keep the global reads coalesced.
__global__ void __launch_bounds__(256) sat_rows_kernel(const float* __restrict__ tf, int rows, int cols,
                                                       double* __restrict__ racc) {
    __shared__ float tile[8][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = (blockIdx.x * 8 + warp) * 32;  // this warp's 32 rows
    double acc = 0.0;
    const int my_row = r0 + lane;
    for (int c0 = 0; c0 < cols; c0 += 32) {
        // coalesced: lane reads column c0 + lane of each of the 32 rows
        for (int i = 0; i < 32; ++i) {
            const int r = r0 + i, c = c0 + lane;
            tile[warp][i][lane] = (r < rows && c < cols) ? tf[static_cast<long long>(r) * cols + c] : 0.0f;
        }
        __syncwarp();
        if (my_row < rows) {
            const int nc = min(32, cols - c0);
            for (int j = 0; j < nc; ++j) {
                const double x = static_cast<double>(tile[warp][lane][j]);
                acc = __fma_rn(x, x, acc);  // x*x exact: the same as the reference's rounded add
                racc[static_cast<long long>(my_row) * cols + c0 + j] = acc;
            }
        }
        __syncwarp();
    }
}

// s[(t+1)(cols+1) + f+1] = s[t(cols+1) + f+1] + R[t][f]; row 0 and column 0 are 0.
__global__ void sat_cols_kernel(const double* __restrict__ racc, int rows, int cols, double* __restrict__ sat) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    const long long w = cols + 1;
    if (f > cols) return;
    sat[f] = 0.0;
    if (f == 0) {
        for (int t = 1; t <= rows; ++t) sat[t * w] = 0.0;
        return;
    }
    double s = 0.0;
    for (int t = 0; t < rows; ++t) {
        s = __dadd_rn(s, racc[static_cast<long long>(t) * cols + (f - 1)]);
        sat[(t + 1) * w + f] = s;
    }
}

// Candidate bitmaps: bit (k, t, f) = !(mean(window_k(t, f)) <= seed), the
// reference's test before a cell seeds a box (baseline.cpp:130-137).  One
// thread per (size, row, 32-column word).
__global__ void cand_kernel(const double* __restrict__ sat, int rows, int cols, const int* __restrict__ sizes,
                            int n_sizes, const float* __restrict__ noise_floor, double p10, double conv,
                            uint32_t* __restrict__ bits) {
    // seed threshold (baseline.cpp:116-119): conv * (double(floor) * 10^(offset/10))
    const double seed = __dmul_rn(conv, __dmul_rn(static_cast<double>(*noise_floor), p10));
    const int W = (cols + 31) / 32;
    const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long total = static_cast<long long>(n_sizes) * rows * W;
    if (idx >= total) return;
    const int wd = static_cast<int>(idx % W);
    const int t = static_cast<int>((idx / W) % rows);
    const int k = static_cast<int>(idx / (static_cast<long long>(W) * rows));
    const int kr = sizes[2 * k], kc = sizes[2 * k + 1];
    const int t0 = max(0, t - (kr - 1) / 2), t1 = min(rows, t + kr / 2 + 1);
    const long long w = cols + 1;
    const double* a = sat + t0 * w;
    const double* b = sat + t1 * w;
    const long long nr = t1 - t0;
    uint32_t word = 0;
    const int fbeg = wd * 32, fend = min(cols, fbeg + 32);
    for (int f = fbeg; f < fend; ++f) {
        const int f0 = max(0, f - (kc - 1) / 2), f1 = min(cols, f + kc / 2 + 1);
        const double sum = __dadd_rn(__dsub_rn(__dsub_rn(b[f1], a[f1]), b[f0]), a[f0]);
        const double mean = __ddiv_rn(sum, static_cast<double>(nr * (f1 - f0)));
        if (!(mean <= seed)) word |= 1u << (f - fbeg);
    }
    bits[idx] = word;
}

cudaError_t baseline_sat_launch(const float* tf, int rows, int cols, double* racc, double* sat, cudaStream_t st) {
    const int row_blocks = (rows + 255) / 256;
    sat_rows_kernel<<<row_blocks, 256, 0, st>>>(tf, rows, cols, racc);
    sat_cols_kernel<<<(cols + 1 + 127) / 128, 128, 0, st>>>(racc, rows, cols, sat);
    return cudaGetLastError();
}

cudaError_t baseline_cand_launch(const double* sat, int rows, int cols, const int* sizes, int n_sizes,
                                 const float* noise_floor, double p10, double conv, uint32_t* bits, cudaStream_t st) {
    const long long total = static_cast<long long>(n_sizes) * rows * ((cols + 31) / 32);
    if (total == 0) return cudaSuccess;
    cand_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(sat, rows, cols, sizes, n_sizes, noise_floor,
                                                                            p10, conv, bits);
    return cudaGetLastError();
}

} // namespace ssb
