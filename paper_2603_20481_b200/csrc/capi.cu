// capi.cu -- the extern "C" boundary (include/specsense_b200.h): context,
// device workspace, argument validation with the reference's error
// semantics, and the fused batch pipelines that chain K1..K6 on one stream.
#include "specsense_b200.h"
#include "internal.h"
#include "baseline_host.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
int ilog2(int n) {
    int m = 0;
    while ((1 << m) < n) ++m;
    return m;
}

} // namespace

struct ss_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    bool fma_variant = true;
    std::string err;
    std::map<int, double2*> tw;                       // per log2(n_fft)
    std::map<std::pair<int, int>, double*> sg;        // per (window, order)
    std::map<std::pair<int, int>, double*> win;       // STFT window per (n_fft, kind)
    std::map<std::string, DevBuf> ws;                 // grow-only workspace
    // host-input pipeline: copy stream + per-staging-buffer events
    cudaStream_t copy = nullptr;
    cudaEvent_t in_ready[2] = {};
    cudaEvent_t buf_free[2] = {};
    int* pinned = nullptr;                             // pinned host word: CCL pool-overflow flag
    // streaming engine contexts: size the CCL run pool for the worst case so
    // detect never synchronises the host to check for a pool overflow
    bool exact_pool = false;
    int64_t launches = 0;
    // optional per-stage timing (CUDA events on the context stream)
    // asynchronous batches (ss_set_async): device-side check flags
    // {pool overflow seen, largest box count above capacity}, read by ss_wait
    bool async = false;
    int* async_flags = nullptr;
    bool timing = false;
    cudaEvent_t ev[2 * 8] = {};
    bool ev_used[8] = {};
    double stage_ms[8] = {};
};

namespace {

// host-input staging chunk (two buffers): large enough that per-chunk launch
// overhead is noise next to the PCIe copy, small enough that pipeline fill is short
constexpr size_t kStageChunkBytes = size_t(256) << 20;
// fused-PSD K1 needs this fraction of its last wave of plot slots filled
constexpr double kFusedPsdMinFill = 0.85;

ss_status fail(ss_ctx* c, ss_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

ss_status cuda_fail(ss_ctx* c, cudaError_t e, const char* where) {
    return fail(c, SS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define SS_CK(ctx, expr)                                           \
    do {                                                           \
        cudaError_t e_ = (expr);                                   \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #expr); \
    } while (0)

template <typename T>
T* wsbuf(ss_ctx* c, const char* name, size_t count, ss_status* st) {
    DevBuf& b = c->ws[name];
    const size_t need = sizeof(T) * (count ? count : 1);
    if (b.bytes < need) {
        if (b.p) {
            cudaStreamSynchronize(c->stream);
            cudaFree(b.p);
            b.p = nullptr;
            b.bytes = 0;
        }
        const size_t alloc = need + need / 8;
        if (cudaMalloc(&b.p, alloc) != cudaSuccess) {
            cudaGetLastError();
            *st = fail(c, SS_ENOMEM, std::string("device allocation failed: ") + name);
            return nullptr;
        }
        b.bytes = alloc;
    }
    return static_cast<T*>(b.p);
}

#define SS_WS(var, T, name, count)                    \
    T* var = nullptr;                                 \
    do {                                              \
        ss_status st_ = SS_OK;                        \
        var = wsbuf<T>(ctx, name, (count), &st_);     \
        if (!var) return st_;                         \
    } while (0)

// stage ids for ss_stage_times: 0 K1 fft_mag(+PSD), 1 K2 psd_cols, 2 K3 floor,
// 3 K4 binarize, 4 K5 consolidate, 5 K6 ccl, 6 H2D, 7 D2H
void tmark(ss_ctx* ctx, int stage, int end) {
    if (!ctx->timing) return;
    cudaEvent_t& e = ctx->ev[2 * stage + end];
    if (!e) cudaEventCreate(&e);
    // under stream capture (the engine's per-bank graphs) a plain record only
    // orders the capture; an external record becomes a timed event node
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &cap);
    if (cap == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, ctx->stream, cudaEventRecordExternal);
    else cudaEventRecord(e, ctx->stream);
    if (end) ctx->ev_used[stage] = true;
}

// call after the stream is synchronised
void tcollect(ss_ctx* ctx) {
    if (!ctx->timing) return;
    for (int i = 0; i < 8; ++i) {
        if (!ctx->ev_used[i]) continue;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ctx->ev[2 * i], ctx->ev[2 * i + 1]) == cudaSuccess) ctx->stage_ms[i] += ms;
        ctx->ev_used[i] = false;
    }
}

ss_status twiddles(ss_ctx* ctx, int n_fft, const double2** out) {
    const int lg = ilog2(n_fft);
    auto it = ctx->tw.find(lg);
    if (it == ctx->tw.end()) {
        std::vector<double2> host;
        if (lg <= 13) ssb::fft_twiddles(lg, host);
        else ssb::fft_large_w1(lg, host);  // large N: the compact per-pass w1 table
        double2* d = nullptr;
        SS_CK(ctx, cudaMalloc(&d, sizeof(double2) * host.size()));
        SS_CK(ctx, cudaMemcpy(d, host.data(), sizeof(double2) * host.size(), cudaMemcpyHostToDevice));
        it = ctx->tw.emplace(lg, d).first;
    }
    *out = it->second;
    return SS_OK;
}

// K1 for n_fft <= 8192; above, the global-memory pass chain (no fused PSD)
ss_status frontend_launch(ss_ctx* ctx, const ssb::FftLaunch& L);

ss_status window_table(ss_ctx* ctx, int n_fft, int kind, const double** out) {
    auto key = std::make_pair(n_fft, kind);
    auto it = ctx->win.find(key);
    if (it == ctx->win.end()) {
        std::vector<double> w;
        ssb::fft_window(n_fft, kind, w);
        double* d = nullptr;
        SS_CK(ctx, cudaMalloc(&d, sizeof(double) * w.size()));
        SS_CK(ctx, cudaMemcpy(d, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
        it = ctx->win.emplace(key, d).first;
    }
    *out = it->second;
    return SS_OK;
}

// frame geometry of the STFT extension: hop in [1, n_fft], 16-byte aligned
// frame starts for the TMA stage loads
ss_status check_stft(ss_ctx* ctx, int n_fft, int hop, int window, ss_fmt fmt) {
    if (window != SS_WIN_RECT && window != SS_WIN_HANN) return fail(ctx, SS_EVALIDATION, "unknown window");
    if (hop < 1 || hop > n_fft) return fail(ctx, SS_EVALIDATION, "hop must be in [1, n_fft]");
    const int align = fmt == SS_FMT_F32 ? 2 : 4;
    if (hop % align != 0) return fail(ctx, SS_EUNSUPPORTED, "hop must keep frames 16-byte aligned (multiple of 2 f32 / 4 i16 samples)");
    return SS_OK;
}

ss_status check_savgol(ss_ctx* ctx, int window, int order) {
    // detector.cpp:144-149
    if (window < 5 || window % 2 == 0) return fail(ctx, SS_EVALIDATION, "savgol window must be odd and >= 5");
    if (order < 1 || order >= window) return fail(ctx, SS_EVALIDATION, "savgol order must be in [1, window)");
    return SS_OK;
}

ss_status weights(ss_ctx* ctx, int window, int order, const double** out) {
    ss_status s = check_savgol(ctx, window, order);
    if (s != SS_OK) return s;
    auto key = std::make_pair(window, order);
    auto it = ctx->sg.find(key);
    if (it == ctx->sg.end()) {
        std::vector<double> w;
        if (!ssb::savgol_weights_host(window, order, w))
            return fail(ctx, SS_EVALIDATION, "savgol normal equations are singular");
        double* d = nullptr;
        SS_CK(ctx, cudaMalloc(&d, sizeof(double) * w.size()));
        SS_CK(ctx, cudaMemcpy(d, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
        it = ctx->sg.emplace(key, d).first;
    }
    *out = it->second;
    return SS_OK;
}

// DetectorConfig::validate (detector.cpp:153-159)
ss_status check_cfg(ss_ctx* ctx, const ss_detector_cfg& c, int n_cols) {
    ss_status s = check_savgol(ctx, c.savgol_window, c.savgol_order);
    if (s != SS_OK) return s;
    if (c.savgol_window > n_cols)
        return fail(ctx, SS_EVALIDATION, "savgol window exceeds the number of frequency bins");
    if (c.psd_margin_db < 0.0) return fail(ctx, SS_EVALIDATION, "psd_margin_db must be non-negative");
    if (c.min_component_area < 1) return fail(ctx, SS_EVALIDATION, "min_component_area must be >= 1");
    return SS_OK;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// async-mode checks, on the device: OR a CCL pool-overflow flag in; record
// the largest box count above the capacity
__global__ void note_overflow_kernel(const int* of, int* flags) {
    if (*of) flags[0] = 1;
}
__global__ void note_capacity_kernel(const int* n_boxes, int n, int cap, int* flags) {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (n_boxes[i] > cap) atomicMax(flags + 1, n_boxes[i]);
}

ss_status async_flags(ss_ctx* ctx, int** out) {
    if (!ctx->async_flags) {
        SS_CK(ctx, cudaMalloc(&ctx->async_flags, 2 * sizeof(int)));
        SS_CK(ctx, cudaMemsetAsync(ctx->async_flags, 0, 2 * sizeof(int), ctx->stream));
    }
    *out = ctx->async_flags;
    return SS_OK;
}

// CCL over n_plots bit masks with a pool of pool_cap runs; fills the workspace
// pointers and launches.
ss_status run_ccl(ss_ctx* ctx, const uint32_t* bits, int n_plots, int rows, int cols, int min_area,
                  long long pool_cap, int* n_comp, long long cap, long long* extents, int* bin_boxes,
                  double* boxes, const unsigned long long* start_seq, double fs, int32_t* labels,
                  int* overflow_host, int time_bins = 0, int* overflow_acc = nullptr) {
    ssb::CclLaunch L;
    L.time_bins = time_bins;
    L.bits = bits;
    L.n_plots = n_plots;
    L.rows = rows;
    L.cols = cols;
    L.min_area = min_area;
    L.n_comp = n_comp;
    L.cap = cap;
    L.extents = extents;
    L.bin_boxes = bin_boxes;
    L.boxes = boxes;
    L.start_seq = start_seq;
    L.fs = fs;
    L.labels = labels;
    ssb::CclWorkspace& w = L.ws;
    SS_WS(rr, int, "ccl.row_runs", static_cast<size_t>(n_plots) * rows);
    SS_WS(so, int2, "ccl.seg_off", static_cast<size_t>(n_plots) * rows * ssb::kCclSeg);
    SS_WS(ro, int, "ccl.row_off", static_cast<size_t>(n_plots) * (rows + 1));
    SS_WS(pb, long long, "ccl.plot_base", n_plots);
    SS_WS(pok, int, "ccl.plot_ok", n_plots);
    SS_WS(of, int, "ccl.overflow", 1);
    SS_WS(rb, int, "ccl.run_begin", pool_cap);
    SS_WS(re, int, "ccl.run_end", pool_cap);
    SS_WS(rw, int, "ccl.run_row", pool_cap);
    SS_WS(pa, int, "ccl.parent", pool_cap);
    SS_WS(ar, unsigned long long, "ccl.area", pool_cap);
    SS_WS(mnf, int, "ccl.min_f", pool_cap);
    SS_WS(mxf, int, "ccl.max_f", pool_cap);
    SS_WS(mxt, int, "ccl.max_t", pool_cap);
    SS_WS(dn, int, "ccl.dense", pool_cap);
    w.row_runs = rr;
    w.seg_off = so;
    w.row_off = ro;
    w.plot_base = pb;
    w.plot_ok = pok;
    w.overflow = of;
    w.run_begin = rb;
    w.run_end = re;
    w.run_row = rw;
    w.parent = pa;
    w.area = ar;
    w.min_f = mnf;
    w.max_f = mxf;
    w.max_t = mxt;
    w.dense = dn;
    w.pool_cap = pool_cap;
    SS_CK(ctx, ssb::ccl_launch(L, ctx->stream));
    // count, scan, plot_base, emit, union_block, [union_boundary], flatten, compact, [labels]
    ctx->launches += 7 + (rows > 16 ? 1 : 0) + (labels ? 1 : 0);
    if (overflow_host) SS_CK(ctx, cudaMemcpyAsync(overflow_host, of, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (overflow_acc) {
        note_overflow_kernel<<<1, 1, 0, ctx->stream>>>(of, overflow_acc);
        SS_CK(ctx, cudaGetLastError());
        ctx->launches += 1;
    }
    return SS_OK;
}

long long default_pool(int n_plots, int rows, int cols) {
    const long long per_row = std::min<long long>((cols + 1) / 2, 32);
    return static_cast<long long>(n_plots) * rows * per_row + 1024;
}

long long worst_pool(int rows, int cols) { return static_cast<long long>(rows) * ((cols + 1) / 2) + 16; }

// Stages 2..6 on TF plots resident in device memory.  psd_ready: raw PSD
// already in psd (fused into K1); else computed here.
ss_status detect_device(ss_ctx* ctx, const float* tf, int n_plots, int rows, int cols,
                        const unsigned long long* seq_dev, double fs, const ss_detector_cfg& cfg,
                        float* psd, bool psd_ready, const ss_batch_out& out_dev, int time_bins = 0,
                        const float* col_lo = nullptr, const float* col_hi = nullptr) {
    const int W = (cols + 31) / 32;
    const double* wts = nullptr;
    ss_status s = weights(ctx, cfg.savgol_window, cfg.savgol_order, &wts);
    if (s != SS_OK) return s;
    if (!psd_ready) {
        tmark(ctx, 1, 0);
        SS_CK(ctx, ssb::psd_cols_launch(tf, n_plots, rows, cols, 0, cols, psd, ctx->stream));
        tmark(ctx, 1, 1);
        ctx->launches += 1;
    }
    SS_WS(sm, float, "det.smoothed", static_cast<size_t>(n_plots) * cols);
    SS_WS(ft, float, "det.floor_thr", static_cast<size_t>(n_plots) * 2);
    SS_WS(act, int, "det.active", static_cast<size_t>(n_plots) * cols);
    SS_WS(nact, int, "det.n_active", n_plots);
    SS_WS(abits, uint32_t, "det.active_bits", static_cast<size_t>(n_plots) * W);
    SS_WS(m0, uint32_t, "det.mask0", static_cast<size_t>(n_plots) * ssb::mask_rs(rows) * W);
    SS_WS(m1, uint32_t, "det.mask1", static_cast<size_t>(n_plots) * ssb::mask_rs(rows) * W);
    ssb::FloorLaunch F;
    F.raw = psd;
    F.n_plots = n_plots;
    F.n = cols;
    F.window = cfg.savgol_window;
    F.weights = wts;
    F.pow10_margin = std::pow(10.0, cfg.psd_margin_db / 10.0);  // detector.cpp:247 (host libm)
    F.fma_variant = ctx->fma_variant;
    F.smoothed = out_dev.psd_smoothed ? out_dev.psd_smoothed : sm;
    F.floor_thr = out_dev.floor_thr ? out_dev.floor_thr : ft;
    F.active = out_dev.active ? out_dev.active : act;
    F.n_active = out_dev.n_active ? out_dev.n_active : nact;
    F.active_bits = abits;
    const bool persistent = ssb::binarize_tile_persistent(rows, cols);
    int* glist = nullptr;
    int* gcount = nullptr;
    if (persistent) {  // K4's work list of active column groups, built by K3
        SS_WS(gl, int, "det.group_list", static_cast<size_t>(n_plots) * ((cols + 7) / 8));
        SS_WS(gc, int, "det.group_count", 1);
        SS_CK(ctx, cudaMemsetAsync(gc, 0, sizeof(int), ctx->stream));
        glist = F.group_list = gl;
        gcount = F.group_count = gc;
    }
    if (ssb::floor_needs_scratch(F.n, F.window)) {
        SS_WS(fscr, float, "floor.scratch", 2 * static_cast<size_t>(F.n_plots) * F.n);
        F.scratch = fscr;
    }
    tmark(ctx, 2, 0);
    SS_CK(ctx, ssb::floor_launch(F, ctx->stream));
    tmark(ctx, 2, 1);
    ssb::BinarizeLaunch B;
    B.tf = tf;
    B.n_plots = n_plots;
    B.rows = rows;
    B.cols = cols;
    B.active_bits = abits;
    const bool tile = ssb::binarize_tile_ok(rows, cols);
    if (tile) {
        B.col_lo = col_lo;  // column extremes from the fused K1, when it made them
        B.col_hi = col_hi;
        B.group_list = glist;
        B.group_count = gcount;
        B.mask_bytes = reinterpret_cast<uint8_t*>(m0);  // the bit mask, written bytewise
        B.skip_empty = true;  // empty column groups stay unwritten; K5 reads them as background
    } else {
        B.mask_bits = m0;
    }
    tmark(ctx, 3, 0);
    SS_CK(ctx, ssb::binarize_launch(B, ctx->stream));
    tmark(ctx, 3, 1);
    tmark(ctx, 4, 0);
    SS_CK(ctx, ssb::consolidate_bits_launch(m0, n_plots, rows, cols, cfg.one_d_opening_along_time != 0, m1, ctx->stream,
                                            tile ? abits : nullptr));
    tmark(ctx, 4, 1);
    ctx->launches += 3;
    const long long cap = out_dev.box_capacity > 0 ? out_dev.box_capacity : 0;
    SS_WS(ncomp, int, "det.n_comp", n_plots);
    if (ctx->exact_pool) {
        tmark(ctx, 5, 0);
        s = run_ccl(ctx, m1, n_plots, rows, cols, cfg.min_component_area, worst_pool(rows, cols) * n_plots,
                    out_dev.n_boxes ? out_dev.n_boxes : ncomp, cap, nullptr, reinterpret_cast<int*>(out_dev.bin_boxes),
                    reinterpret_cast<double*>(out_dev.boxes), seq_dev, fs, nullptr, nullptr, time_bins);
        tmark(ctx, 5, 1);
        return s;
    }
    if (ctx->async) {  // no host round trip: the overflow check goes to ss_wait
        int* flags = nullptr;
        s = async_flags(ctx, &flags);
        if (s != SS_OK) return s;
        tmark(ctx, 5, 0);
        s = run_ccl(ctx, m1, n_plots, rows, cols, cfg.min_component_area, default_pool(n_plots, rows, cols),
                    out_dev.n_boxes ? out_dev.n_boxes : ncomp, cap, nullptr,
                    reinterpret_cast<int*>(out_dev.bin_boxes), reinterpret_cast<double*>(out_dev.boxes), seq_dev, fs,
                    nullptr, nullptr, time_bins, flags);
        tmark(ctx, 5, 1);
        return s;
    }
    int* overflow_h = ctx->pinned;
    tmark(ctx, 5, 0);
    s = run_ccl(ctx, m1, n_plots, rows, cols, cfg.min_component_area, default_pool(n_plots, rows, cols),
                out_dev.n_boxes ? out_dev.n_boxes : ncomp, cap, nullptr,
                reinterpret_cast<int*>(out_dev.bin_boxes), reinterpret_cast<double*>(out_dev.boxes), seq_dev, fs,
                nullptr, overflow_h, time_bins);
    if (s != SS_OK) return s;
    tmark(ctx, 5, 1);
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    tcollect(ctx);
    const int overflow = *overflow_h;
    if (overflow) {
        // rare: some plot had more runs than the shared pool; redo every plot
        // alone with its exact worst-case pool
        int* nb = out_dev.n_boxes ? out_dev.n_boxes : ncomp;
        for (int p = 0; p < n_plots; ++p) {
            const size_t mo = static_cast<size_t>(p) * ssb::mask_rs(rows) * W;
            s = run_ccl(ctx, m1 + mo, 1, rows, cols, cfg.min_component_area, worst_pool(rows, cols), nb + p, cap,
                        nullptr, out_dev.bin_boxes ? reinterpret_cast<int*>(out_dev.bin_boxes) + 4 * cap * p : nullptr,
                        out_dev.boxes ? reinterpret_cast<double*>(out_dev.boxes) + 4 * cap * p : nullptr,
                        seq_dev ? seq_dev + p : nullptr, fs, nullptr, nullptr, time_bins);
            if (s != SS_OK) return s;
        }
        SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return SS_OK;
}

ss_status frontend_launch(ss_ctx* ctx, const ssb::FftLaunch& L) {
    if (L.logn <= 13) {
        SS_CK(ctx, ssb::fft_mag_launch(L, ctx->stream));
        ctx->launches += 1;
        return SS_OK;
    }
    if (L.psd) return fail(ctx, SS_EUNSUPPORTED, "fused PSD needs n_fft <= 8192");
    const long long n = 1LL << L.logn;
    const long long chunk = std::max(1LL, std::min(L.total_rows, (1LL << 26) / n));  // <= 1 GiB per scratch
    SS_WS(a, double2, "large.a", static_cast<size_t>(chunk * n));
    SS_WS(b, double2, "large.b", static_cast<size_t>(chunk * n));
    int nl = 0;
    SS_CK(ctx, ssb::fft_large_launch(L, L.tw, a, b, chunk, ctx->stream, &nl));
    ctx->launches += nl;
    return SS_OK;
}

} // namespace

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

void ss_default_detector_cfg(ss_detector_cfg* cfg) {
    if (!cfg) return;
    cfg->savgol_window = 31;
    cfg->savgol_order = 3;
    cfg->psd_margin_db = 3.0;
    cfg->min_component_area = 4;
    cfg->one_d_opening_along_time = 0;
}

ss_status ss_open(int device, ss_ctx** out) {
    if (!out) return SS_EVALIDATION;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
        cudaGetLastError();
        return SS_ECUDA;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) return SS_EUNSUPPORTED;
    if (cudaSetDevice(device) != cudaSuccess) return SS_ECUDA;
    ss_ctx* c = new ss_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->fma_variant = ssb::host_has_fma_avx2();
    if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return SS_ECUDA;
    }
    c->stream = c->own;
    if (cudaMallocHost(&c->pinned, 16 * sizeof(int)) != cudaSuccess) {
        cudaStreamDestroy(c->own);
        delete c;
        return SS_ECUDA;
    }
    *out = c;
    return SS_OK;
}

void ss_close(ss_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->tw) cudaFree(kv.second);
    for (auto& kv : ctx->sg) cudaFree(kv.second);
    for (auto& kv : ctx->win) cudaFree(kv.second);
    for (auto& kv : ctx->ws) cudaFree(kv.second.p);
    if (ctx->async_flags) cudaFree(ctx->async_flags);
    for (cudaEvent_t e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (int b = 0; b < 2; ++b) {
        if (ctx->in_ready[b]) cudaEventDestroy(ctx->in_ready[b]);
        if (ctx->buf_free[b]) cudaEventDestroy(ctx->buf_free[b]);
    }
    if (ctx->copy) {
        cudaStreamSynchronize(ctx->copy);
        cudaStreamDestroy(ctx->copy);
    }
    cudaStreamDestroy(ctx->own);
    cudaFreeHost(ctx->pinned);
    delete ctx;
}

const char* ss_last_error(const ss_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

ss_status ss_set_stream(ss_ctx* ctx, void* stream) {
    if (!ctx) return SS_EVALIDATION;
    ctx->stream = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream
    return SS_OK;
}

ss_status ss_synchronize(ss_ctx* ctx) {
    if (!ctx) return SS_EVALIDATION;
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return SS_OK;
}

ss_status ss_set_async(ss_ctx* ctx, int on) {
    if (!ctx) return SS_EVALIDATION;
    ctx->async = on != 0;
    return SS_OK;
}

ss_status ss_wait(ss_ctx* ctx) {
    if (!ctx) return SS_EVALIDATION;
    int* h = ctx->pinned + 8;  // pinned words 8, 9
    h[0] = h[1] = 0;
    if (ctx->async_flags) {
        SS_CK(ctx, cudaMemcpyAsync(h, ctx->async_flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        SS_CK(ctx, cudaMemsetAsync(ctx->async_flags, 0, 2 * sizeof(int), ctx->stream));
    }
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    tcollect(ctx);
    if (h[0]) return fail(ctx, SS_ECAPACITY, "CCL run pool overflow in an asynchronous batch: re-run it with async off");
    if (h[1]) return fail(ctx, SS_ECAPACITY, "box capacity too small: " + std::to_string(h[1]));
    return SS_OK;
}

int64_t ss_launch_count(const ss_ctx* ctx) { return ctx ? ctx->launches : 0; }

ss_status ss_enable_stage_timing(ss_ctx* ctx, int on) {
    if (!ctx) return SS_EVALIDATION;
    ctx->timing = on != 0;
    for (double& v : ctx->stage_ms) v = 0.0;
    return SS_OK;
}

ss_status ss_stage_times(const ss_ctx* ctx, double* ms8) {
    if (!ctx || !ms8) return SS_EVALIDATION;
    for (int i = 0; i < 8; ++i) ms8[i] = ctx->stage_ms[i];
    return SS_OK;
}

ss_status ss_tf_plots(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int rows, int n_plots, float* tf) {
    if (!ctx) return SS_EVALIDATION;
    if (n_fft < 8 || !is_pow2(n_fft))
        return fail(ctx, SS_EVALIDATION, "FFT size must be a power of two >= 8, got " + std::to_string(n_fft));
    if (n_fft > (1 << ssb::kLargeLogNMax)) return fail(ctx, SS_EUNSUPPORTED, "device FFT supports n_fft <= 1048576");
    if (rows < 0 || n_plots < 0) return fail(ctx, SS_EVALIDATION, "negative plot geometry");
    if (fmt != SS_FMT_F32 && fmt != SS_FMT_I16) return fail(ctx, SS_EVALIDATION, "unknown sample format");
    if (static_cast<long long>(rows) * n_plots == 0) return SS_OK;
    if (reinterpret_cast<uintptr_t>(iq) % 16 != 0) return fail(ctx, SS_EVALIDATION, "IQ buffer must be 16-byte aligned");
    const double2* tw = nullptr;
    ss_status s = twiddles(ctx, n_fft, &tw);
    if (s != SS_OK) return s;
    ssb::FftLaunch L;
    L.logn = ilog2(n_fft);
    L.fmt = fmt;
    L.psd = false;
    L.iq = iq;
    L.tf = tf;
    L.tw = tw;
    L.total_rows = static_cast<long long>(rows) * n_plots;
    L.rows_per_plot = rows;
    L.n_plots = n_plots;
    L.num_sms = ctx->num_sms;
    return frontend_launch(ctx, L);
}

ss_status ss_stft_plots(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                        int n_plots, float* tf) {
    if (!ctx) return SS_EVALIDATION;
    if (n_fft < 8 || !is_pow2(n_fft))
        return fail(ctx, SS_EVALIDATION, "FFT size must be a power of two >= 8, got " + std::to_string(n_fft));
    if (n_fft > (1 << ssb::kLargeLogNMax)) return fail(ctx, SS_EUNSUPPORTED, "device FFT supports n_fft <= 1048576");
    if (rows < 0 || n_plots < 0) return fail(ctx, SS_EVALIDATION, "negative plot geometry");
    ss_status s = check_stft(ctx, n_fft, hop, window, fmt);
    if (s != SS_OK) return s;
    if (static_cast<long long>(rows) * n_plots == 0) return SS_OK;
    if (reinterpret_cast<uintptr_t>(iq) % 16 != 0) return fail(ctx, SS_EVALIDATION, "IQ buffer must be 16-byte aligned");
    const double2* tw = nullptr;
    s = twiddles(ctx, n_fft, &tw);
    if (s != SS_OK) return s;
    const double* w = nullptr;
    s = window_table(ctx, n_fft, window, &w);
    if (s != SS_OK) return s;
    ssb::FftLaunch L;
    L.logn = ilog2(n_fft);
    L.fmt = fmt;
    L.iq = iq;
    L.tf = tf;
    L.tw = tw;
    L.total_rows = static_cast<long long>(rows) * n_plots;
    L.rows_per_plot = rows;
    L.n_plots = n_plots;
    L.num_sms = ctx->num_sms;
    L.hop = hop;
    L.win = w;
    return frontend_launch(ctx, L);
}

ss_status ss_psd_cols(ss_ctx* ctx, const float* tf, int rows, int cols, int c0, int c1, float* out) {
    if (!ctx) return SS_EVALIDATION;
    if (rows < 1 || cols < 1) return fail(ctx, SS_EVALIDATION, "empty TF plot");
    if (c0 < 0 || c1 > cols || c0 >= c1) return fail(ctx, SS_EVALIDATION, "PSD column range out of bounds");
    SS_CK(ctx, ssb::psd_cols_launch(tf, 1, rows, cols, c0, c1, out, ctx->stream));
    ctx->launches += 1;
    return SS_OK;
}

ss_status ss_savgol_smooth(ss_ctx* ctx, const float* values, int n, int window, int order, float* out) {
    if (!ctx) return SS_EVALIDATION;
    const double* w = nullptr;
    ss_status s = check_savgol(ctx, window, order);
    if (s != SS_OK) return s;
    if (n < window) return fail(ctx, SS_EVALIDATION, "savgol window exceeds the input length");
    s = weights(ctx, window, order, &w);
    if (s != SS_OK) return s;
    SS_CK(ctx, ssb::savgol_launch(values, n, window, w, out, ctx->stream));
    ctx->launches += 1;
    return SS_OK;
}

ss_status ss_floor(ss_ctx* ctx, const float* raw, int n, const ss_detector_cfg* cfg, float* smoothed,
                   float* floor_thr, int32_t* active, int32_t* n_active) {
    if (!ctx || !cfg) return SS_EVALIDATION;
    ss_status s = check_savgol(ctx, cfg->savgol_window, cfg->savgol_order);
    if (s != SS_OK) return s;
    if (n < cfg->savgol_window) return fail(ctx, SS_EVALIDATION, "savgol window exceeds the input length");
    const double* w = nullptr;
    s = weights(ctx, cfg->savgol_window, cfg->savgol_order, &w);
    if (s != SS_OK) return s;
    SS_WS(nact, int, "floor.n_active", 1);
    ssb::FloorLaunch F;
    F.raw = raw;
    F.n_plots = 1;
    F.n = n;
    F.window = cfg->savgol_window;
    F.weights = w;
    F.pow10_margin = std::pow(10.0, cfg->psd_margin_db / 10.0);
    F.fma_variant = ctx->fma_variant;
    F.smoothed = smoothed;
    F.floor_thr = floor_thr;
    F.active = active;
    F.n_active = nact;
    if (ssb::floor_needs_scratch(F.n, F.window)) {
        SS_WS(fscr, float, "floor.scratch", 2 * static_cast<size_t>(F.n));
        F.scratch = fscr;
    }
    SS_CK(ctx, ssb::floor_launch(F, ctx->stream));
    ctx->launches += 1;
    int h = 0;
    SS_CK(ctx, cudaMemcpyAsync(&h, nact, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (n_active) *n_active = h;
    return SS_OK;
}

ss_status ss_prune(ss_ctx* ctx, const float* raw, int n, float threshold, int32_t* active, int32_t* n_active) {
    if (!ctx) return SS_EVALIDATION;
    if (n < 0) return fail(ctx, SS_EVALIDATION, "negative PSD length");
    if (n == 0) {
        if (n_active) *n_active = 0;
        return SS_OK;
    }
    SS_WS(nact, int, "prune.n_active", 1);
    SS_CK(ctx, ssb::prune_launch(raw, n, threshold, active, nact, ctx->stream));
    ctx->launches += 1;
    int h = 0;
    SS_CK(ctx, cudaMemcpyAsync(&h, nact, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (n_active) *n_active = h;
    return SS_OK;
}

ss_status ss_otsu(ss_ctx* ctx, const float* values, int n, int32_t* valid, float* threshold) {
    if (!ctx) return SS_EVALIDATION;
    if (n < 1) return fail(ctx, SS_EVALIDATION, "otsu on an empty column");
    SS_WS(bits, uint32_t, "otsu.bits", 1);
    SS_WS(thr, float, "otsu.thr", 1);
    SS_WS(val, int, "otsu.valid", 1);
    const uint32_t one = 1u;
    SS_CK(ctx, cudaMemcpyAsync(bits, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    ssb::BinarizeLaunch B;
    B.tf = values;
    B.n_plots = 1;
    B.rows = n;
    B.cols = 1;
    B.active_bits = bits;
    B.col_thr = thr;
    B.col_valid = val;
    SS_CK(ctx, ssb::binarize_launch(B, ctx->stream));
    ctx->launches += 1;
    float t = 0.0f;
    int v = 0;
    SS_CK(ctx, cudaMemcpyAsync(&t, thr, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaMemcpyAsync(&v, val, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (valid) *valid = v;
    if (threshold) *threshold = v ? t : 0.0f;
    return SS_OK;
}

ss_status ss_binarize_cols(ss_ctx* ctx, const float* tf, int rows, int cols, const int32_t* active_host,
                           int n_active, int c0, int c1, uint8_t* mask) {
    if (!ctx) return SS_EVALIDATION;
    if (rows < 0 || cols < 0) return fail(ctx, SS_EVALIDATION, "binarize output mask shape mismatch");
    if (c0 < 0 || c1 > cols || c0 > c1) return fail(ctx, SS_EVALIDATION, "binarize column range out of bounds");
    if (c1 == c0) return SS_OK;
    const int W = (cols + 31) / 32;
    std::vector<uint32_t> bits(static_cast<size_t>(W), 0u);
    for (int i = 0; i < n_active; ++i) {
        const int k = active_host[i];
        if (k < 0 || k >= cols) return fail(ctx, SS_EVALIDATION, "active column index out of range");
        bits[static_cast<size_t>(k >> 5)] |= 1u << (k & 31);
    }
    if (rows == 0) return SS_OK;
    SS_WS(dbits, uint32_t, "bin.bits", W);
    SS_CK(ctx, cudaMemcpyAsync(dbits, bits.data(), sizeof(uint32_t) * W, cudaMemcpyHostToDevice, ctx->stream));
    ssb::BinarizeLaunch B;
    B.tf = tf;
    B.n_plots = 1;
    B.rows = rows;
    B.cols = cols;
    B.active_bits = dbits;
    B.mask_u8 = mask;
    B.c0 = c0;
    B.c1 = c1;
    SS_CK(ctx, ssb::binarize_launch(B, ctx->stream));
    ctx->launches += 1;
    // the bit vector lives on the host stack: finish before returning
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return SS_OK;
}

ss_status ss_morph_cols(ss_ctx* ctx, const uint8_t* src, int rows, int cols, ss_morph_op op, int se_rows,
                        int se_cols, int c0, int c1, uint8_t* dst) {
    if (!ctx) return SS_EVALIDATION;
    // check_se (detector.cpp:345-349), morphology_cols range checks (:443-447)
    if (se_rows < 1 || se_cols < 1 || se_rows % 2 == 0 || se_cols % 2 == 0)
        return fail(ctx, SS_EVALIDATION, "structuring element dimensions must be odd and >= 1");
    if (rows < 1 || cols < 1) return fail(ctx, SS_EVALIDATION, "empty mask");
    if (c0 < 0 || c1 > cols || c0 > c1) return fail(ctx, SS_EVALIDATION, "morphology column range out of bounds");
    if (op < SS_ERODE || op > SS_CLOSE) return fail(ctx, SS_EVALIDATION, "unknown morphology op");
    if (src == dst) return fail(ctx, SS_EVALIDATION, "morphology dst must not alias src");
    SS_WS(tmp, uint8_t, "morph.tmp", static_cast<size_t>(rows) * cols);
    SS_CK(ctx, ssb::morph_u8_launch(src, rows, cols, op, se_rows, se_cols, c0, c1, tmp, dst, ctx->stream));
    ctx->launches += (op >= SS_OPEN) ? 2 : 1;
    return SS_OK;
}

ss_status ss_consolidate(ss_ctx* ctx, const uint8_t* src, int rows, int cols, int along_time, uint8_t* dst) {
    if (!ctx) return SS_EVALIDATION;
    if (rows < 1 || cols < 1) return fail(ctx, SS_EVALIDATION, "empty mask");
    const int W = (cols + 31) / 32;
    SS_WS(a, uint32_t, "cons.a", static_cast<size_t>(ssb::mask_rs(rows)) * W);
    SS_WS(b, uint32_t, "cons.b", static_cast<size_t>(ssb::mask_rs(rows)) * W);
    SS_CK(ctx, ssb::pack_u8_launch(src, 1, rows, cols, a, ctx->stream));
    SS_CK(ctx, ssb::consolidate_bits_launch(a, 1, rows, cols, along_time != 0, b, ctx->stream));
    SS_CK(ctx, ssb::unpack_launch(b, 1, rows, cols, dst, ctx->stream));
    ctx->launches += 3;
    return SS_OK;
}

ss_status ss_components(ss_ctx* ctx, const uint8_t* mask, int rows, int cols, int min_area, int32_t* labels,
                        ss_extent* extents_host, int64_t cap, int64_t* n_out) {
    if (!ctx) return SS_EVALIDATION;
    if (min_area < 1) return fail(ctx, SS_EVALIDATION, "min_component_area must be >= 1");
    if (rows < 1 || cols < 1) {
        if (n_out) *n_out = 0;
        return SS_OK;
    }
    const int W = (cols + 31) / 32;
    SS_WS(bits, uint32_t, "comp.bits", static_cast<size_t>(ssb::mask_rs(rows)) * W);
    SS_WS(ncomp, int, "comp.n", 1);
    const long long dcap = cap > 0 ? cap : 1;
    SS_WS(ext, long long, "comp.ext", static_cast<size_t>(5 * dcap));
    SS_CK(ctx, ssb::pack_u8_launch(mask, 1, rows, cols, bits, ctx->stream));
    ctx->launches += 1;
    ss_status s = run_ccl(ctx, bits, 1, rows, cols, min_area, worst_pool(rows, cols), ncomp, dcap, ext, nullptr,
                          nullptr, nullptr, 1.0, labels, nullptr);
    if (s != SS_OK) return s;
    int n = 0;
    SS_CK(ctx, cudaMemcpyAsync(&n, ncomp, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (n_out) *n_out = n;
    if (n > cap) return fail(ctx, SS_ECAPACITY, "component capacity too small: " + std::to_string(n));
    if (n > 0 && extents_host)
        SS_CK(ctx, cudaMemcpy(extents_host, ext, sizeof(ss_extent) * static_cast<size_t>(n), cudaMemcpyDeviceToHost));
    return SS_OK;
}

ss_status ss_detect_batch(ss_ctx* ctx, const float* tf, int n_plots, int rows, int cols, const uint64_t* start_seq,
                          double sample_rate_hz, const ss_detector_cfg* cfg, const ss_batch_out* out) {
    if (!ctx || !cfg || !out) return SS_EVALIDATION;
    ss_status s = check_cfg(ctx, *cfg, cols);
    if (s != SS_OK) return s;
    if (rows < 1 || cols < 1 || n_plots < 0) return fail(ctx, SS_EVALIDATION, "empty TF plot");
    if (!(sample_rate_hz > 0.0)) return fail(ctx, SS_EVALIDATION, "sample_rate_hz must be positive");
    if (n_plots == 0) return SS_OK;
    SS_WS(psd, float, "det.psd", static_cast<size_t>(n_plots) * cols);
    SS_WS(seq, unsigned long long, "det.seq", n_plots);
    std::vector<unsigned long long> hseq(static_cast<size_t>(n_plots), 0ull);
    if (start_seq)
        for (int p = 0; p < n_plots; ++p) hseq[p] = start_seq[p];
    SS_CK(ctx, cudaMemcpyAsync(seq, hseq.data(), sizeof(unsigned long long) * n_plots, cudaMemcpyHostToDevice,
                               ctx->stream));
    float* praw = out->psd_raw ? out->psd_raw : psd;
    s = detect_device(ctx, tf, n_plots, rows, cols, seq, sample_rate_hz, *cfg, praw, false, *out);
    if (s != SS_OK) return s;
    if (out->n_boxes && out->box_capacity >= 0 && ctx->async) {
        int* flags = nullptr;
        s = async_flags(ctx, &flags);
        if (s != SS_OK) return s;
        note_capacity_kernel<<<1, 256, 0, ctx->stream>>>(out->n_boxes, n_plots, out->box_capacity, flags);
        SS_CK(ctx, cudaGetLastError());
        ctx->launches += 1;
        return SS_OK;
    }
    if (out->n_boxes && out->box_capacity >= 0) {
        std::vector<int> nb(static_cast<size_t>(n_plots));
        SS_CK(ctx, cudaMemcpy(nb.data(), out->n_boxes, sizeof(int) * n_plots, cudaMemcpyDeviceToHost));
        for (int v : nb)
            if (v > out->box_capacity) return fail(ctx, SS_ECAPACITY, "box capacity too small: " + std::to_string(v));
    }
    return SS_OK;
}

static ss_status sense_impl(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                            int n_plots, uint64_t first_seq, double sample_rate_hz, const ss_detector_cfg* cfg,
                            float* tf_out, const ss_batch_out* out);

ss_status ss_sense_batch(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int rows, int n_plots, uint64_t first_seq,
                         double sample_rate_hz, const ss_detector_cfg* cfg, float* tf_out, const ss_batch_out* out) {
    return sense_impl(ctx, iq, fmt, n_fft, n_fft, SS_WIN_RECT, rows, n_plots, first_seq, sample_rate_hz, cfg, tf_out,
                      out);
}

ss_status ss_stft_sense_batch(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                              int n_plots, uint64_t first_frame, double sample_rate_hz, const ss_detector_cfg* cfg,
                              float* tf_out, const ss_batch_out* out) {
    return sense_impl(ctx, iq, fmt, n_fft, hop, window, rows, n_plots, first_frame, sample_rate_hz, cfg, tf_out, out);
}

__global__ void seq_fill_kernel(unsigned long long* seq, int n, unsigned long long first, int rows) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) seq[p] = first + static_cast<unsigned long long>(p) * rows;
}

// K1 (+PSD) and the detector chain on device-resident IQ; `tf` and every
// non-null pointer in `dev` are device memory.  No host synchronisation.
// seq_dev: per-plot start sequence numbers already on the device (the
// engine's graph-captured path), else they are filled from first_seq.
static ss_status sense_device(ss_ctx* ctx, const void* diq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                              int n_plots, uint64_t first_seq, double sample_rate_hz, const ss_detector_cfg& cfg,
                              float* tf, const ss_batch_out& dev, const unsigned long long* seq_dev = nullptr) {
    const bool stft = hop != n_fft || window != SS_WIN_RECT;
    const int cols = n_fft;
    SS_WS(psd, float, "det.psd", static_cast<size_t>(n_plots) * cols);
    float* praw = dev.psd_raw ? dev.psd_raw : psd;
    const double2* tw = nullptr;
    ss_status s = twiddles(ctx, n_fft, &tw);
    if (s != SS_OK) return s;
    // Fused PSD (K1 accumulates each plot's column sums in row order, one plot
    // per row group) only when the batch fills whole waves of plot slots;
    // otherwise K1 spreads all rows over every SM and K2 sums the columns.
    const int slots = ssb::fft_psd_slots_per_sm(ilog2(n_fft), fmt, stft) * ctx->num_sms;
    bool fused = false;
    if (slots > 0) {
        const long long waves = (n_plots + slots - 1) / slots;
        fused = static_cast<double>(n_plots) >= kFusedPsdMinFill * static_cast<double>(waves * slots);
    }
    ssb::FftLaunch L;
    L.logn = ilog2(n_fft);
    L.fmt = fmt;
    L.psd = fused;
    L.iq = diq;
    L.tf = tf;
    L.psd_out = praw;
    float* col_lo = nullptr;
    float* col_hi = nullptr;
    if (fused && ssb::fft_psd_extremes(ilog2(n_fft)) && ssb::binarize_tile_ok(rows, cols) &&
        ssb::binarize_wants_extremes(rows)) {
        SS_WS(clo, float, "det.col_lo", static_cast<size_t>(n_plots) * cols);
        SS_WS(chi, float, "det.col_hi", static_cast<size_t>(n_plots) * cols);
        col_lo = L.col_lo = clo;
        col_hi = L.col_hi = chi;
    }
    L.tw = tw;
    L.total_rows = static_cast<long long>(rows) * n_plots;
    L.rows_per_plot = rows;
    L.n_plots = n_plots;
    L.num_sms = ctx->num_sms;
    if (stft) {
        const double* w = nullptr;
        s = window_table(ctx, n_fft, window, &w);
        if (s != SS_OK) return s;
        L.hop = hop;
        L.win = w;
    }
    tmark(ctx, 0, 0);
    s = frontend_launch(ctx, L);
    if (s != SS_OK) return s;
    tmark(ctx, 0, 1);
    if (!fused) {
        tmark(ctx, 1, 0);
        SS_CK(ctx, ssb::psd_cols_launch(tf, n_plots, rows, cols, 0, cols, praw, ctx->stream));
        tmark(ctx, 1, 1);
        ctx->launches += 1;
    }
    const unsigned long long* seq = seq_dev;
    if (!seq) {
        SS_WS(sq, unsigned long long, "det.seq", n_plots);
        seq_fill_kernel<<<(n_plots + 255) / 256, 256, 0, ctx->stream>>>(sq, n_plots, first_seq, rows);
        SS_CK(ctx, cudaGetLastError());
        ctx->launches += 1;
        seq = sq;
    }
    return detect_device(ctx, tf, n_plots, rows, cols, seq, sample_rate_hz, cfg, praw, true, dev, hop, col_lo, col_hi);
}

// outputs of plots [p0, p0 + n) inside a batch-out block of box capacity K
static ss_batch_out out_slice(const ss_batch_out& o, int p0, int cols, long long K) {
    ss_batch_out r = o;
    const size_t p = static_cast<size_t>(p0);
    if (r.psd_raw) r.psd_raw += p * cols;
    if (r.psd_smoothed) r.psd_smoothed += p * cols;
    if (r.floor_thr) r.floor_thr += p * 2;
    if (r.active) r.active += p * cols;
    if (r.n_active) r.n_active += p;
    if (r.boxes) r.boxes += p * static_cast<size_t>(K);
    if (r.bin_boxes) r.bin_boxes += p * static_cast<size_t>(K);
    if (r.n_boxes) r.n_boxes += p;
    return r;
}

// Host (or unaligned) IQ: chunks of plots are copied into two staging buffers
// on a private copy stream while the previous chunk computes on ctx->stream,
// so the PCIe transfer (the e2e bound) overlaps K1..K6.
static ss_status ensure_copy_stream(ss_ctx* ctx) {
    if (ctx->copy) return SS_OK;
    SS_CK(ctx, cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        SS_CK(ctx, cudaEventCreateWithFlags(&ctx->in_ready[b], cudaEventDisableTiming));
        SS_CK(ctx, cudaEventCreateWithFlags(&ctx->buf_free[b], cudaEventDisableTiming));
    }
    return SS_OK;
}

static ss_status sense_impl(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                            int n_plots, uint64_t first_seq, double sample_rate_hz, const ss_detector_cfg* cfg,
                            float* tf_out, const ss_batch_out* out) {
    if (!ctx || !cfg || !out) return SS_EVALIDATION;
    if (n_fft < 8 || !is_pow2(n_fft))
        return fail(ctx, SS_EVALIDATION, "FFT size must be a power of two >= 8, got " + std::to_string(n_fft));
    if (n_fft > (1 << ssb::kLargeLogNMax)) return fail(ctx, SS_EUNSUPPORTED, "device FFT supports n_fft <= 1048576");
    if (rows < 1) return fail(ctx, SS_EVALIDATION, "plot_rows must be >= 1");
    if (!(sample_rate_hz > 0.0)) return fail(ctx, SS_EVALIDATION, "sample_rate_hz must be positive");
    if (fmt != SS_FMT_F32 && fmt != SS_FMT_I16) return fail(ctx, SS_EVALIDATION, "unknown sample format");
    ss_status s = check_cfg(ctx, *cfg, n_fft);
    if (s != SS_OK) return s;
    s = check_stft(ctx, n_fft, hop, window, fmt);
    if (s != SS_OK) return s;
    if (n_plots <= 0) return SS_OK;
    const int cols = n_fft;
    const size_t sbytes = fmt == SS_FMT_F32 ? 8 : 4;
    const size_t plot_stride = static_cast<size_t>(rows) * hop;      // samples between plot starts
    const size_t ntf = static_cast<size_t>(n_plots) * rows * cols;
    float* tf = tf_out;
    if (!tf) {
        SS_WS(t, float, "sense.tf", ntf);
        tf = t;
    }
    // outputs: device pointers used directly, host pointers staged
    ss_batch_out dev = *out;
    const bool host_out = (out->psd_raw && !is_device_ptr(out->psd_raw)) || (out->boxes && !is_device_ptr(out->boxes)) ||
                          (out->n_boxes && !is_device_ptr(out->n_boxes)) ||
                          (out->bin_boxes && !is_device_ptr(out->bin_boxes)) ||
                          (out->floor_thr && !is_device_ptr(out->floor_thr)) ||
                          (out->psd_smoothed && !is_device_ptr(out->psd_smoothed)) ||
                          (out->active && !is_device_ptr(out->active)) ||
                          (out->n_active && !is_device_ptr(out->n_active));
    const long long K = out->box_capacity > 0 ? out->box_capacity : 0;
    if (host_out) {
        SS_WS(a1, float, "sense.o.raw", static_cast<size_t>(n_plots) * cols);
        SS_WS(a2, float, "sense.o.sm", static_cast<size_t>(n_plots) * cols);
        SS_WS(a3, float, "sense.o.ft", static_cast<size_t>(n_plots) * 2);
        SS_WS(a4, int32_t, "sense.o.act", static_cast<size_t>(n_plots) * cols);
        SS_WS(a5, int32_t, "sense.o.nact", n_plots);
        SS_WS(a6, ss_box, "sense.o.box", static_cast<size_t>(n_plots) * (K ? K : 1));
        SS_WS(a7, ss_bin_box, "sense.o.bbox", static_cast<size_t>(n_plots) * (K ? K : 1));
        SS_WS(a8, int32_t, "sense.o.nbox", n_plots);
        dev.psd_raw = a1;
        dev.psd_smoothed = a2;
        dev.floor_thr = a3;
        dev.active = a4;
        dev.n_active = a5;
        dev.boxes = a6;
        dev.bin_boxes = a7;
        dev.n_boxes = a8;
    }
    if (is_device_ptr(iq) && reinterpret_cast<uintptr_t>(iq) % 16 == 0) {
        s = sense_device(ctx, iq, fmt, n_fft, hop, window, rows, n_plots, first_seq, sample_rate_hz, *cfg, tf, dev);
        if (s != SS_OK) return s;
    } else {
        s = ensure_copy_stream(ctx);
        if (s != SS_OK) return s;
        const size_t plot_bytes = plot_stride * sbytes;
        const int cp = static_cast<int>(std::max<size_t>(1, std::min<size_t>(n_plots, kStageChunkBytes / plot_bytes)));
        const size_t chunk_span = (static_cast<size_t>(cp) * rows - 1) * hop + n_fft;
        unsigned char* stage[2];
        {
            SS_WS(s0, unsigned char, "sense.iq0", chunk_span * sbytes);
            stage[0] = s0;
        }
        if (cp < n_plots) {
            SS_WS(s1, unsigned char, "sense.iq1", chunk_span * sbytes);
            stage[1] = s1;
        } else {
            stage[1] = stage[0];
        }
        const int nchunks = (n_plots + cp - 1) / cp;
        // chunk c -> staging buffer c & 1; the copy of chunk c + 1 is queued
        // before chunk c computes, so the copy engine never idles on the
        // host's per-chunk synchronisation inside detect_device
        auto issue_copy = [&](int c) -> ss_status {
            const int b = c & 1;
            const int p0 = c * cp;
            const int np = std::min(cp, n_plots - p0);
            const size_t span = (static_cast<size_t>(np) * rows - 1) * hop + n_fft;
            const unsigned char* src = static_cast<const unsigned char*>(iq) + p0 * plot_stride * sbytes;
            SS_CK(ctx, cudaStreamWaitEvent(ctx->copy, ctx->buf_free[b], 0));
            SS_CK(ctx, cudaMemcpyAsync(stage[b], src, span * sbytes, cudaMemcpyDefault, ctx->copy));
            SS_CK(ctx, cudaEventRecord(ctx->in_ready[b], ctx->copy));
            return SS_OK;
        };
        s = issue_copy(0);
        if (s != SS_OK) return s;
        for (int c = 0; c < nchunks; ++c) {
            const int b = c & 1;
            const int p0 = c * cp;
            const int np = std::min(cp, n_plots - p0);
            if (c + 1 < nchunks) {
                s = issue_copy(c + 1);
                if (s != SS_OK) return s;
            }
            SS_CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->in_ready[b], 0));
            s = sense_device(ctx, stage[b], fmt, n_fft, hop, window, rows, np, first_seq + p0 * static_cast<uint64_t>(rows),
                             sample_rate_hz, *cfg, tf + static_cast<size_t>(p0) * rows * cols,
                             out_slice(dev, p0, cols, K));
            if (s != SS_OK) return s;
            SS_CK(ctx, cudaEventRecord(ctx->buf_free[b], ctx->stream));
        }
    }
    if (host_out) {
        tmark(ctx, 7, 0);
        auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
            if (!dst) return cudaSuccess;
            return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream);
        };
        SS_CK(ctx, cp(out->psd_raw, dev.psd_raw, sizeof(float) * n_plots * cols));
        SS_CK(ctx, cp(out->psd_smoothed, dev.psd_smoothed, sizeof(float) * n_plots * cols));
        SS_CK(ctx, cp(out->floor_thr, dev.floor_thr, sizeof(float) * n_plots * 2));
        SS_CK(ctx, cp(out->active, dev.active, sizeof(int32_t) * n_plots * cols));
        SS_CK(ctx, cp(out->n_active, dev.n_active, sizeof(int32_t) * n_plots));
        SS_CK(ctx, cp(out->boxes, dev.boxes, sizeof(ss_box) * n_plots * K));
        SS_CK(ctx, cp(out->bin_boxes, dev.bin_boxes, sizeof(ss_bin_box) * n_plots * K));
        SS_CK(ctx, cp(out->n_boxes, dev.n_boxes, sizeof(int32_t) * n_plots));
        tmark(ctx, 7, 1);
    }
    if (ctx->async) {  // the capacity check goes to ss_wait as well
        if (out->n_boxes) {
            int* flags = nullptr;
            s = async_flags(ctx, &flags);
            if (s != SS_OK) return s;
            note_capacity_kernel<<<1, 256, 0, ctx->stream>>>(dev.n_boxes, n_plots, K, flags);
            SS_CK(ctx, cudaGetLastError());
            ctx->launches += 1;
        }
        return SS_OK;
    }
    if (out->n_boxes) {
        std::vector<int> nb(static_cast<size_t>(n_plots));
        SS_CK(ctx, cudaMemcpyAsync(nb.data(), dev.n_boxes, sizeof(int) * n_plots, cudaMemcpyDeviceToHost, ctx->stream));
        SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
        tcollect(ctx);
        for (int v : nb)
            if (v > K) return fail(ctx, SS_ECAPACITY, "box capacity too small: " + std::to_string(v));
    } else if (host_out) {
        SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
        tcollect(ctx);
    }
    return SS_OK;
}

void ss_default_baseline_cfg(ss_baseline_cfg* cfg) {
    if (!cfg) return;
    cfg->conv_threshold = 2.0;
    cfg->rate_change_threshold = 0.5;
    cfg->noise_offset_db = 3.0;
    cfg->max_kernel_rows = 0;
    cfg->max_kernel_cols = 0;
}

static const char* baseline_cfg_error(const ss_baseline_cfg& c) {
    if (!(c.conv_threshold > 0.0)) return "conv_threshold must be > 0";
    if (!(c.rate_change_threshold > 0.0)) return "rate_change_threshold must be > 0";
    if (c.max_kernel_rows < 0 || c.max_kernel_cols < 0) return "kernel caps must be >= 0";
    return nullptr;
}

static std::vector<int32_t> baseline_sizes(int rows, int cols, const ss_baseline_cfg& c) {
    const int rcap = c.max_kernel_rows > 0 ? std::min(c.max_kernel_rows, rows) : rows;
    const int ccap = c.max_kernel_cols > 0 ? std::min(c.max_kernel_cols, cols) : cols;
    std::vector<int32_t> v;
    for (int kr = 1; kr <= rcap; kr *= 2)
        for (int kc = 1; kc <= ccap; kc *= 2) {
            v.push_back(kr);
            v.push_back(kc);
        }
    return v;
}

int ss_baseline_kernel_sizes(int rows, int cols, const ss_baseline_cfg* cfg, int32_t* sizes, int cap) {
    if (!cfg || baseline_cfg_error(*cfg) || rows < 1 || cols < 1) return -1;
    const std::vector<int32_t> v = baseline_sizes(rows, cols, *cfg);
    const int n = static_cast<int>(v.size() / 2);
    if (n > cap) return -2;
    if (sizes) std::memcpy(sizes, v.data(), sizeof(int32_t) * v.size());
    return n;
}

ss_status ss_baseline_detect(ss_ctx* ctx, const float* tf, int rows, int cols, uint64_t start_seq,
                             double sample_rate_hz, const ss_baseline_cfg* cfg, ss_box* boxes, ss_bin_box* bin_boxes,
                             int cap, int* n_boxes) {
    if (!ctx || !tf || !cfg || !n_boxes) return SS_EVALIDATION;
    if (const char* m = baseline_cfg_error(*cfg)) return fail(ctx, SS_EVALIDATION, m);
    if (rows < 1 || cols < 1) return fail(ctx, SS_EVALIDATION, "plot must be non-empty");
    if (!(sample_rate_hz > 0.0)) return fail(ctx, SS_EVALIDATION, "sample_rate_hz must be positive");
    ss_detector_cfg dc;
    ss_default_detector_cfg(&dc);  // the baseline's floor uses the default DetectorConfig (baseline.cpp:110-115)
    ss_status s = check_cfg(ctx, dc, cols);
    if (s != SS_OK) return s;
    const size_t cells = static_cast<size_t>(rows) * cols;
    const float* dtf = tf;
    if (!is_device_ptr(tf)) {
        SS_WS(st, float, "bl.tf", cells);
        SS_CK(ctx, cudaMemcpyAsync(st, tf, sizeof(float) * cells, cudaMemcpyHostToDevice, ctx->stream));
        dtf = st;
    }
    // PSD + smooth_and_floor (noise floor), as detect's stages
    SS_WS(psd, float, "bl.psd", cols);
    SS_CK(ctx, ssb::psd_cols_launch(dtf, 1, rows, cols, 0, cols, psd, ctx->stream));
    const double* wts = nullptr;
    s = weights(ctx, dc.savgol_window, dc.savgol_order, &wts);
    if (s != SS_OK) return s;
    const int W = (cols + 31) / 32;
    SS_WS(sm, float, "bl.sm", cols);
    SS_WS(ft, float, "bl.ft", 2);
    SS_WS(act, int, "bl.act", cols);
    SS_WS(nact, int, "bl.nact", 1);
    SS_WS(abits, uint32_t, "bl.abits", W);
    ssb::FloorLaunch F;
    F.raw = psd;
    F.n_plots = 1;
    F.n = cols;
    F.window = dc.savgol_window;
    F.weights = wts;
    F.pow10_margin = std::pow(10.0, dc.psd_margin_db / 10.0);
    F.fma_variant = ctx->fma_variant;
    F.smoothed = sm;
    F.floor_thr = ft;
    F.active = act;
    F.n_active = nact;
    F.active_bits = abits;
    if (ssb::floor_needs_scratch(F.n, F.window)) {
        SS_WS(fscr, float, "floor.scratch", 2 * static_cast<size_t>(F.n_plots) * F.n);
        F.scratch = fscr;
    }
    SS_CK(ctx, ssb::floor_launch(F, ctx->stream));
    // summed-area table and the kernel bank's candidate bitmaps
    SS_WS(racc, double, "bl.racc", cells);
    SS_WS(sat, double, "bl.sat", static_cast<size_t>(rows + 1) * (cols + 1));
    SS_CK(ctx, ssb::baseline_sat_launch(dtf, rows, cols, racc, sat, ctx->stream));
    const std::vector<int32_t> sizes = baseline_sizes(rows, cols, *cfg);
    const int K = static_cast<int>(sizes.size() / 2);
    SS_WS(dsizes, int32_t, "bl.sizes", sizes.size());
    SS_CK(ctx, cudaMemcpyAsync(dsizes, sizes.data(), sizeof(int32_t) * sizes.size(), cudaMemcpyHostToDevice, ctx->stream));
    const size_t nbits = static_cast<size_t>(K) * rows * W;
    SS_WS(cand, uint32_t, "bl.cand", nbits);
    const double p10 = std::pow(10.0, cfg->noise_offset_db / 10.0);  // baseline.cpp:117 (host libm, config only)
    SS_CK(ctx, ssb::baseline_cand_launch(sat, rows, cols, dsizes, K, ft, p10, cfg->conv_threshold, cand, ctx->stream));
    ctx->launches += 6;
    std::vector<double> hsat(static_cast<size_t>(rows + 1) * (cols + 1));
    std::vector<uint32_t> hcand(nbits);
    SS_CK(ctx, cudaMemcpyAsync(hsat.data(), sat, sizeof(double) * hsat.size(), cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaMemcpyAsync(hcand.data(), cand, sizeof(uint32_t) * nbits, cudaMemcpyDeviceToHost, ctx->stream));
    SS_CK(ctx, cudaStreamSynchronize(ctx->stream));
    const std::vector<ssb::BaselineRect> rects =
        ssb::baseline_greedy(hsat.data(), hcand.data(), sizes.data(), K, rows, cols, cfg->rate_change_threshold);
    *n_boxes = static_cast<int>(rects.size());
    const double dt = static_cast<double>(cols) / sample_rate_hz;  // TFPlotView::dt_s / df_hz
    const double df = sample_rate_hz / static_cast<double>(cols);
    const int keep = std::min(static_cast<int>(rects.size()), std::max(cap, 0));
    for (int i = 0; i < keep; ++i) {
        const ssb::BaselineRect& r = rects[static_cast<size_t>(i)];
        if (bin_boxes) bin_boxes[i] = ss_bin_box{r.t0, r.t1, r.f0, r.f1};
        if (boxes) {
            ss_box& b = boxes[i];
            b.t0_s = (static_cast<double>(start_seq) + r.t0) * dt;
            b.t1_s = (static_cast<double>(start_seq) + r.t1) * dt;
            b.f0_hz = (r.f0 - cols / 2) * df;
            b.f1_hz = (r.f1 - cols / 2) * df;
        }
    }
    if (static_cast<int>(rects.size()) > cap) return fail(ctx, SS_ECAPACITY, "box capacity too small: " + std::to_string(rects.size()));
    return SS_OK;
}

ss_status ss_test_libm(ss_ctx* ctx, const float* x, int64_t n, int which, int variant, float* out) {
    if (!ctx) return SS_EVALIDATION;
    const bool fma = variant < 0 ? ctx->fma_variant : variant != 0;
    SS_CK(ctx, ssb::libm_test_launch(x, n, which, fma, out, ctx->stream));
    ctx->launches += 1;
    return SS_OK;
}

int64_t ss_fft_twiddle_count(int n_fft) {
    if (n_fft < 8 || !is_pow2(n_fft) || n_fft > 8192) return -1;
    std::vector<double2> t;
    ssb::fft_twiddles(ilog2(n_fft), t);
    return static_cast<int64_t>(t.size());
}

ss_status ss_fft_twiddles(int n_fft, double* out_re_im) {
    if (n_fft < 8 || !is_pow2(n_fft) || n_fft > 8192) return SS_EVALIDATION;
    std::vector<double2> t;
    ssb::fft_twiddles(ilog2(n_fft), t);
    std::memcpy(out_re_im, t.data(), sizeof(double2) * t.size());
    return SS_OK;
}

} // extern "C"

// ---- hooks for the streaming engine (engine.cpp), not part of the C ABI
namespace ssb {

ss_status engine_ctx_open(int device, ss_ctx** out) {
    const ss_status s = ss_open(device, out);
    if (s == SS_OK) (*out)->exact_pool = true;
    return s;
}

cudaStream_t engine_ctx_stream(ss_ctx* ctx) { return ctx->stream; }

ss_status engine_check(ss_ctx* ctx, int n_fft, int rows, ss_fmt fmt, double fs, const ss_detector_cfg& cfg) {
    if (n_fft < 8 || !is_pow2(n_fft))
        return fail(ctx, SS_EVALIDATION, "FFT size must be a power of two >= 8, got " + std::to_string(n_fft));
    if (n_fft > (1 << ssb::kLargeLogNMax)) return fail(ctx, SS_EUNSUPPORTED, "device FFT supports n_fft <= 1048576");
    if (rows < 1) return fail(ctx, SS_EVALIDATION, "plot_rows must be >= 1");
    if (!(fs > 0.0)) return fail(ctx, SS_EVALIDATION, "sample_rate_hz must be positive");
    if (fmt != SS_FMT_F32 && fmt != SS_FMT_I16) return fail(ctx, SS_EVALIDATION, "unknown sample format");
    return check_cfg(ctx, cfg, n_fft);
}

// one window, device-resident IQ -> device outputs, on the context stream, no
// host sync; seq_dev (device, 1 value) replaces start_seq when non-null so
// the launch sequence can be captured once into a CUDA graph per bank
ss_status engine_sense(ss_ctx* ctx, const void* diq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                       uint64_t start_seq, double fs, const ss_detector_cfg& cfg, float* tf, const ss_batch_out& dev,
                       const unsigned long long* seq_dev) {
    return sense_device(ctx, diq, fmt, n_fft, hop, window, rows, 1, start_seq, fs, cfg, tf, dev, seq_dev);
}

ss_status engine_check_stft(ss_ctx* ctx, int n_fft, int hop, int window, ss_fmt fmt) {
    return check_stft(ctx, n_fft, hop, window, fmt);
}

void engine_add_launches(ss_ctx* ctx, int64_t n) { ctx->launches += n; }

// Stage events for one graph capture: with ev16 non-null the context's stage
// marks (tmark) record into the caller's 16 events, so a captured window chain
// carries its own per-stage event nodes; used8 returns which stages recorded.
// With ev16 null, stage timing is off again and the context forgets the events.
void engine_stage_events(ss_ctx* ctx, cudaEvent_t* ev16, bool* used8) {
    if (ev16) {
        for (int i = 0; i < 16; ++i) ctx->ev[i] = ev16[i];
        for (bool& u : ctx->ev_used) u = false;
        ctx->timing = true;
        return;
    }
    if (used8)
        for (int i = 0; i < 8; ++i) used8[i] = ctx->ev_used[i];
    for (cudaEvent_t& e : ctx->ev) e = nullptr;
    for (bool& u : ctx->ev_used) u = false;
    ctx->timing = false;
}

} // namespace ssb
