// internal.h -- launcher interfaces shared by the specsense-b200 translation
// units (not part of the public C ABI; see include/specsense_b200.h).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

namespace ssb {

// ---- K1 fft_mag.cu
struct FftLaunch {
    int logn = 0;
    int fmt = 0;          // 0 f32 IQ, 1 i16 IQ
    bool psd = false;     // fused exact-order PSD, one CTA per plot
    const void* iq = nullptr;
    float* tf = nullptr;  // may be null when psd
    float* psd_out = nullptr;
    float* col_lo = nullptr;     // fused PSD, n_fft >= 4096: the plots' column extremes (K4's sweep A) or null
    float* col_hi = nullptr;
    const double2* tw = nullptr;
    long long total_rows = 0;
    int rows_per_plot = 0;
    int n_plots = 0;
    int num_sms = 148;
    int hop = 0;                 // STFT extension: frame step (0 = n_fft, the reference's rectangular hop)
    const double* win = nullptr; // STFT extension: device window weights (null = rectangular)
};
cudaError_t fft_mag_launch(const FftLaunch& L, cudaStream_t st);
// plots per SM the fused-PSD K1 grid runs concurrently (one plot per row group)
int fft_psd_slots_per_sm(int logn, int fmt, bool win);
// the fused-PSD K1 also writes column extremes (FftLaunch::col_lo / col_hi) for this size
bool fft_psd_extremes(int logn);
void fft_window(int n_fft, int kind, std::vector<double>& out);  // kind 0 rect, 1 periodic Hann
// n_fft = 2^14 .. 2^20: global-memory SSFFT-2 passes + magnitudes (no PSD)
constexpr int kLargeLogNMax = 20;
size_t fft_large_w1_count(int logn);
void fft_large_w1(int logn, std::vector<double2>& out);
cudaError_t fft_large_launch(const FftLaunch& L, const double2* w1, double2* a, double2* b, long long chunk_rows,
                             cudaStream_t st, int* launches);
void fft_twiddles(int logn, std::vector<double2>& out);

// ---- K2/K3 floor.cu
// PSD of a plot-major batch of TF plots, columns [c0, c1) (one thread per column,
// rows in order): detector.cpp:170-184.
cudaError_t psd_cols_launch(const float* tf, int n_plots, int rows, int cols, int c0, int c1,
                            float* out, cudaStream_t st);

struct FloorLaunch {
    const float* raw = nullptr;   // n_plots x n
    int n_plots = 0;
    int n = 0;
    int window = 31;
    const double* weights = nullptr;  // device, window doubles
    double pow10_margin = 0.0;        // pow(10.0, margin_db / 10.0), host libm
    bool fma_variant = true;
    float* smoothed = nullptr;    // n_plots x n
    float* floor_thr = nullptr;   // n_plots x 2
    int* active = nullptr;        // n_plots x n (compacted, ascending)
    int* n_active = nullptr;      // n_plots
    uint32_t* active_bits = nullptr;  // n_plots x W (W = ceil(n/32)), may be null
    int* group_list = nullptr;    // optional: p * ceil(n/8) + g for every 8-column group g with an active column
    int* group_count = nullptr;   // ... appended per plot at *group_count (zeroed by the caller)
    float* scratch = nullptr;     // n_plots x 2n floats: the dB / smoothed rows when they exceed shared memory
};
// true when the floor stage needs FloorLaunch::scratch (rows of n floats do not fit shared memory)
inline bool floor_needs_scratch(int n, int window) { return 8ull * window + 8ull * n > 200ull * 1024; }
cudaError_t floor_launch(const FloorLaunch& L, cudaStream_t st);
cudaError_t prune_launch(const float* raw, int n, float thr, int* active, int* n_active, cudaStream_t st);
cudaError_t savgol_launch(const float* v, int n, int window, const double* weights, float* out,
                          cudaStream_t st);
cudaError_t libm_test_launch(const float* x, long long n, int which, bool fma_variant, float* out,
                             cudaStream_t st);

// host constants (host_consts.cpp)
bool savgol_weights_host(int window, int order, std::vector<double>& w);
bool host_has_fma_avx2();

// ---- K4 binarize.cu
// Word-major bit masks [p][w][rs] keep each word's rows at a stride padded to
// a multiple of 4 (16 bytes): row bands of 4-aligned rows load and store as
// 128-bit vectors (K5).  Rows rows .. rs-1 are padding, never read as data.
__host__ __device__ inline int mask_rs(int rows) { return (rows + 3) & ~3; }

struct BinarizeLaunch {
    const float* tf = nullptr;          // n_plots x rows x cols
    int n_plots = 0;
    int rows = 0;
    int cols = 0;
    const uint32_t* active_bits = nullptr;  // n_plots x W
    const int* group_list = nullptr;    // optional (single-CTA tile path): the active 8-column groups, p * (cols/8) + g,
    const int* group_count = nullptr;   // and their count (device): persistent CTAs walk them
    const float* col_lo = nullptr;      // optional n_plots x cols column extremes (from K1): the tile path
    const float* col_hi = nullptr;      // then skips its min / max sweep and bins boxes as they land
    uint32_t* mask_bits = nullptr;      // n_plots x W x rows word-major bits (bit mode) or null
    uint8_t* mask_bytes = nullptr;     // tile path: the word-major bit mask as bytes (byte k of word w = columns 32w+8k..+7) or null
    bool skip_empty = false;           // tile path: groups with no active column write nothing (K5 masks them)
    uint8_t* mask_u8 = nullptr;         // rows x cols (u8 mode, columns [c0,c1)) or null
    int c0 = 0, c1 = 0;                 // u8 mode column range
    float* col_thr = nullptr;           // optional n_plots x cols thresholds (+inf inactive)
    int* col_valid = nullptr;           // optional n_plots x cols: active && non-constant
};
cudaError_t binarize_launch(const BinarizeLaunch& L, cudaStream_t st);
// true when the smem-resident tile kernel (bytewise writes into the bit mask) handles this shape
bool binarize_tile_ok(int rows, int cols);
// true when the tile path should take column extremes from the fused K1 (BinarizeLaunch::col_lo)
bool binarize_wants_extremes(int rows);
// true when the tile path runs as persistent CTAs over a list of active groups (FloorLaunch::group_list)
bool binarize_tile_persistent(int rows, int cols);

// ---- K5 morph.cu
cudaError_t pack_u8_launch(const uint8_t* m, int n_plots, int rows, int cols, uint32_t* bits,
                           cudaStream_t st);
cudaError_t unpack_launch(const uint32_t* bits, int n_plots, int rows, int cols, uint8_t* m,
                          cudaStream_t st);
// close 3x3 -> open 3x3 -> open 1x3 (3x1 if along_time), bit-packed, fused in
// registers.  in / out: word-major bit masks [p][ceil(cols/32)][rows].
// active_bits (optional, [p][W]): bytes of `in` whose 8-column group has no
// active column are read as background (the tile K4 leaves them unwritten).
cudaError_t consolidate_bits_launch(const uint32_t* in, int n_plots, int rows,
                                    int cols, bool along_time, uint32_t* out, cudaStream_t st,
                                    const uint32_t* active_bits = nullptr);
// Generic single-plot u8 morphology of columns [c0, c1) (stage API): op 0 erode,
// 1 dilate, 2 open, 3 close; tmp: rows x cols scratch.
cudaError_t morph_u8_launch(const uint8_t* src, int rows, int cols, int op, int se_rows, int se_cols,
                            int c0, int c1, uint8_t* tmp, uint8_t* dst, cudaStream_t st);

// ---- K6 ccl.cu
constexpr int kCclSeg = 4;  // word segments per row in the run kernels (ccl.cu)
struct CclWorkspace {
    int* row_runs = nullptr;      // n_plots x rows: runs starting in each row
    int2* seg_off = nullptr;      // n_plots x rows x kCclSeg: {starts, ends} before each row segment
    int* row_off = nullptr;       // n_plots x (rows + 1): exclusive prefix within the plot
    long long* plot_base = nullptr;  // n_plots: first pool index of the plot's runs
    int* plot_ok = nullptr;       // n_plots: 1 if the plot's runs fit the pool
    int* overflow = nullptr;      // 1 flag: some plot did not fit
    // run pool (capacity pool_cap), runs in row-major order of their start pixel
    int* run_begin = nullptr;
    int* run_end = nullptr;
    int* run_row = nullptr;
    int* parent = nullptr;
    unsigned long long* area = nullptr;
    int* min_f = nullptr;
    int* max_f = nullptr;
    int* max_t = nullptr;
    int* dense = nullptr;         // dense component id per root run (-1: dropped)
    long long pool_cap = 0;
};
struct CclLaunch {
    const uint32_t* bits = nullptr;  // n_plots x rows x W
    int n_plots = 0, rows = 0, cols = 0;
    int min_area = 4;
    CclWorkspace ws;
    // outputs
    int* n_comp = nullptr;            // n_plots (true count, may exceed cap)
    long long cap = 0;                // per plot capacity of the record arrays
    long long* extents = nullptr;     // n_plots x cap x 5 (min_t,max_t,min_f,max_f,area) or null
    int* bin_boxes = nullptr;         // n_plots x cap x 4 (t0,t1,f0,f1) or null
    double* boxes = nullptr;          // n_plots x cap x 4 (f0,f1,t0,t1) or null
    const unsigned long long* start_seq = nullptr;  // n_plots (boxes)
    double fs = 0.0;
    int time_bins = 0;                // samples per row step for t: cols (reference) or the STFT hop
    int32_t* labels = nullptr;        // rows x cols label raster (single plot) or null
};
cudaError_t ccl_launch(const CclLaunch& L, cudaStream_t st);

// ---- baseline.cu (F3: Searchlight-style baseline)
cudaError_t baseline_sat_launch(const float* tf, int rows, int cols, double* racc, double* sat, cudaStream_t st);
cudaError_t baseline_cand_launch(const double* sat, int rows, int cols, const int* sizes, int n_sizes,
                                 const float* noise_floor, double p10, double conv, uint32_t* bits, cudaStream_t st);

} // namespace ssb
