// dropin.cpp -- the reference's C++ stage API (include/specsense/*.hpp)
// implemented over the C ABI, so reference callers (runtime, baseline, CLI,
// acceptance) relink against libspecsense_b200.so unchanged.
//
// Host spans are staged through a persistent per-thread workspace (device
// buffers that only grow + a pinned staging buffer, one stream synchronize per
// call); every computation runs on the GPU.  Status codes map back onto the reference's exception types
// (proj/include/specsense/types.hpp:43-70).
#include "specsense/detector.hpp"
#include "specsense/frontend.hpp"
#include "specsense_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

namespace specsense {
namespace {

// Per-host-thread context: one ss_ctx on a private non-blocking stream, a set
// of device buffers that only grow (no cudaMalloc / cudaFree per call once
// warm), and a pinned staging buffer through which small host spans travel
// (memcpy + async copy instead of a pageable cudaMemcpy per span).
struct Ctx {
    ss_ctx* h = nullptr;
    cudaStream_t s = nullptr;
    struct Slot {
        void* p = nullptr;
        std::size_t bytes = 0;
    };
    Slot slots[16];
    unsigned char* pin = nullptr;
    std::size_t pin_cap = 0, pin_used = 0, pin_want = 0;
    struct Pending {
        void* dst;
        const void* src;
        std::size_t n;
    };
    std::vector<Pending> pend;

    Ctx() {
        const char* dev = std::getenv("SPECSENSE_DEVICE");
        const ss_status st = ss_open(dev ? std::atoi(dev) : 0, &h);
        if (st != SS_OK) throw Error("specsense-b200: no usable sm_100 device (ss_open status " + std::to_string(st) + ")");
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) throw Error("cudaStreamCreate failed");
        ss_set_stream(h, s);
    }
    ~Ctx() {
        cudaStreamSynchronize(s);
        for (Slot& b : slots) cudaFree(b.p);
        cudaFreeHost(pin);
        ss_close(h);
        cudaStreamDestroy(s);
    }
};

constexpr std::size_t kPinnedMax = std::size_t(64) << 20;  // larger spans copy from pageable memory directly

Ctx& ctx_obj() {
    thread_local Ctx c;
    return c;
}

ss_ctx* ctx() { return ctx_obj().h; }

void check(ss_status s) {
    if (s == SS_OK) return;
    const std::string m = ss_last_error(ctx());
    if (s == SS_EVALIDATION) throw ValidationError(m);
    if (s == SS_EFORMAT) throw FormatError(m);
    throw Error(m);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// One drop-in call: device slots handed out in order, host inputs staged in,
// host outputs collected at finish() (one stream synchronize per call).
class Call {
  public:
    Call() : c_(ctx_obj()) {
        c_.pend.clear();
        if (c_.pin_want > c_.pin_cap) {  // grow the pinned stage between calls, never during one
            cudaFreeHost(c_.pin);
            c_.pin = nullptr;
            c_.pin_cap = 0;
            const std::size_t want = std::min(kPinnedMax, c_.pin_want + c_.pin_want / 4);
            if (cudaMallocHost(&c_.pin, want) == cudaSuccess) c_.pin_cap = want;
            else cudaGetLastError();
        }
        c_.pin_used = 0;
        c_.pin_want = 0;
    }
    Call(const Call&) = delete;
    Call& operator=(const Call&) = delete;

    template <typename T>
    T* dev(std::size_t count) {
        if (next_ >= 16) throw Error("drop-in: too many device buffers in one call");
        Ctx::Slot& b = c_.slots[next_++];
        const std::size_t need = sizeof(T) * (count ? count : 1);
        if (b.bytes < need) {
            cuda_check(cudaStreamSynchronize(c_.s), "stream sync");
            cudaFree(b.p);
            b.p = nullptr;
            b.bytes = 0;
            const std::size_t alloc = need + need / 4;
            cuda_check(cudaMalloc(&b.p, alloc), "cudaMalloc");
            b.bytes = alloc;
        }
        return static_cast<T*>(b.p);
    }
    template <typename T>
    T* in(const T* host, std::size_t count) {
        T* d = dev<T>(count);
        put(d, host, count);
        return d;
    }
    template <typename T>
    void put(T* d, const T* host, std::size_t count) {
        const std::size_t n = sizeof(T) * count;
        if (!n) return;
        if (unsigned char* st = stage(n)) {
            std::memcpy(st, host, n);
            cuda_check(cudaMemcpyAsync(d, st, n, cudaMemcpyHostToDevice, c_.s), "H2D");
        } else {
            cuda_check(cudaMemcpyAsync(d, host, n, cudaMemcpyHostToDevice, c_.s), "H2D");
        }
    }
    template <typename T>
    void get(T* host, const T* d, std::size_t count) {
        const std::size_t n = sizeof(T) * count;
        if (!n) return;
        if (unsigned char* st = stage(n)) {
            cuda_check(cudaMemcpyAsync(st, d, n, cudaMemcpyDeviceToHost, c_.s), "D2H");
            c_.pend.push_back({host, st, n});
        } else {
            cuda_check(cudaMemcpyAsync(host, d, n, cudaMemcpyDeviceToHost, c_.s), "D2H");
        }
    }
    void finish() {
        cuda_check(cudaStreamSynchronize(c_.s), "stream sync");
        for (const auto& p : c_.pend) std::memcpy(p.dst, p.src, p.n);
        c_.pend.clear();
    }
    void rewind() { next_ = 0; }

  private:
    unsigned char* stage(std::size_t n) {
        const std::size_t off = (c_.pin_used + 255) & ~std::size_t(255);
        c_.pin_want = std::max(c_.pin_want, off + n);
        if (off + n > c_.pin_cap) return nullptr;
        c_.pin_used = off + n;
        return c_.pin + off;
    }
    Ctx& c_;
    int next_ = 0;
};

ss_detector_cfg to_c(const detector::DetectorConfig& c) {
    ss_detector_cfg o;
    o.savgol_window = c.savgol_window;
    o.savgol_order = c.savgol_order;
    o.psd_margin_db = c.psd_margin_db;
    o.min_component_area = c.min_component_area;
    o.one_d_opening_along_time = c.one_d_opening_along_time ? 1 : 0;
    return o;
}

bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

} // namespace

// ============================================================ frontend

namespace frontend {

void FrontendConfig::validate() const {
    if (!(sample_rate_hz > 0.0)) throw ValidationError("sample_rate_hz must be positive");
    if (n_fft < 8 || !pow2(n_fft))
        throw ValidationError("FFT size must be a power of two >= 8, got " + std::to_string(n_fft));
    if (plot_rows < 1) throw ValidationError("plot_rows must be >= 1");
}

Resolution resolution(double sample_rate_hz, int n_fft) {
    FrontendConfig c;
    c.sample_rate_hz = sample_rate_hz;
    c.n_fft = n_fft;
    c.validate();
    return {n_fft / sample_rate_hz, sample_rate_hz / n_fft};
}

double stream_bit_rate_bps(double sample_rate_hz, int bits_per_component) {
    if (!(sample_rate_hz > 0.0)) throw ValidationError("sample_rate_hz must be positive");
    if (bits_per_component <= 0) throw ValidationError("bits_per_component must be positive");
    return sample_rate_hz * 2.0 * bits_per_component;
}

static std::vector<float> tf_device(const void* host, std::size_t bytes, ss_fmt fmt, int n_fft, int rows,
                                    int n_plots) {
    const std::size_t n = static_cast<std::size_t>(rows) * n_fft * n_plots;
    std::vector<float> out(n);
    if (n == 0) return out;
    Call c;
    const unsigned char* iq = c.in(static_cast<const unsigned char*>(host), bytes);
    float* tf = c.dev<float>(n);
    check(ss_tf_plots(ctx(), iq, fmt, n_fft, rows, n_plots, tf));
    c.get(out.data(), tf, n);
    c.finish();
    return out;
}

void fft_row(std::span<const cfloat> chunk, std::span<float> out) {
    const int n = static_cast<int>(chunk.size());
    if (n < 8 || !pow2(n)) throw ValidationError("FFT size must be a power of two >= 8, got " + std::to_string(n));
    if (out.size() != chunk.size()) throw ValidationError("fft_row output size must match the chunk size");
    const auto row = tf_device(chunk.data(), chunk.size_bytes(), SS_FMT_F32, n, 1, 1);
    std::copy(row.begin(), row.end(), out.begin());
}

std::vector<float> fft_row(std::span<const cfloat> chunk) {
    std::vector<float> out(chunk.size());
    fft_row(chunk, out);
    return out;
}

TFPlot make_plot(std::span<const cfloat> samples, double sample_rate_hz, int n_fft, std::uint64_t start_seq) {
    if (n_fft < 8 || !pow2(n_fft))
        throw ValidationError("FFT size must be a power of two >= 8, got " + std::to_string(n_fft));
    if (!(sample_rate_hz > 0.0)) throw ValidationError("sample_rate_hz must be positive");
    TFPlot p;
    p.rows = static_cast<int>(samples.size() / static_cast<std::size_t>(n_fft));
    p.cols = n_fft;
    p.start_seq = start_seq;
    p.sample_rate_hz = sample_rate_hz;
    p.data = tf_device(samples.data(), static_cast<std::size_t>(p.rows) * n_fft * sizeof(cfloat), SS_FMT_F32, n_fft,
                       p.rows, 1);
    return p;
}

static std::vector<TFPlot> split(std::vector<float>&& all, const FrontendConfig& c, int n_plots) {
    std::vector<TFPlot> plots(static_cast<std::size_t>(n_plots));
    const std::size_t per = static_cast<std::size_t>(c.plot_rows) * c.n_fft;
    for (int p = 0; p < n_plots; ++p) {
        TFPlot& t = plots[static_cast<std::size_t>(p)];
        t.rows = c.plot_rows;
        t.cols = c.n_fft;
        t.start_seq = static_cast<std::uint64_t>(p) * c.plot_rows;
        t.sample_rate_hz = c.sample_rate_hz;
        t.data.assign(all.begin() + static_cast<std::ptrdiff_t>(p * per),
                      all.begin() + static_cast<std::ptrdiff_t>((p + 1) * per));
    }
    return plots;
}

std::vector<TFPlot> make_plots(std::span<const cfloat> samples, const FrontendConfig& config) {
    config.validate();
    const std::size_t per = static_cast<std::size_t>(config.plot_rows) * config.n_fft;
    const int n_plots = static_cast<int>(samples.size() / per);
    return split(tf_device(samples.data(), n_plots * per * sizeof(cfloat), SS_FMT_F32, config.n_fft,
                           config.plot_rows, n_plots),
                 config, n_plots);
}

std::vector<TFPlot> make_plots_i16(std::span<const std::int16_t> iq, const FrontendConfig& config) {
    config.validate();
    const std::size_t per = static_cast<std::size_t>(config.plot_rows) * config.n_fft;
    const int n_plots = static_cast<int>(iq.size() / 2 / per);
    return split(tf_device(iq.data(), n_plots * per * 2 * sizeof(std::int16_t), SS_FMT_I16, config.n_fft,
                           config.plot_rows, n_plots),
                 config, n_plots);
}

} // namespace frontend

// ============================================================ detector

namespace detector {

void DetectorConfig::validate(int n_cols) const {
    if (savgol_window < 5 || savgol_window % 2 == 0) throw ValidationError("savgol window must be odd and >= 5");
    if (savgol_order < 1 || savgol_order >= savgol_window) throw ValidationError("savgol order must be in [1, window)");
    if (savgol_window > n_cols) throw ValidationError("savgol window exceeds the number of frequency bins");
    if (psd_margin_db < 0.0) throw ValidationError("psd_margin_db must be non-negative");
    if (min_component_area < 1) throw ValidationError("min_component_area must be >= 1");
}

StageTimes& StageTimes::operator+=(const StageTimes& o) {
    psd += o.psd;
    floor_prune += o.floor_prune;
    binarize += o.binarize;
    morphology += o.morphology;
    label += o.label;
    return *this;
}

static std::size_t cells(const frontend::TFPlotView& p) { return static_cast<std::size_t>(p.rows) * p.cols; }

void estimate_psd_into(const frontend::TFPlotView& plot, int col_begin, int col_end, float* out) {
    if (plot.rows < 1 || plot.cols < 1) throw ValidationError("empty TF plot");
    if (col_begin < 0 || col_end > plot.cols || col_begin >= col_end)
        throw ValidationError("PSD column range out of bounds");
    Call c;
    const float* tf = c.in(plot.data, cells(plot));
    float* o = c.dev<float>(static_cast<std::size_t>(col_end - col_begin));
    check(ss_psd_cols(ctx(), tf, plot.rows, plot.cols, col_begin, col_end, o));
    c.get(out, o, static_cast<std::size_t>(col_end - col_begin));
    c.finish();
}

std::vector<float> estimate_psd(const frontend::TFPlotView& plot) {
    std::vector<float> psd(static_cast<std::size_t>(plot.cols));
    estimate_psd_into(plot, 0, plot.cols, psd.data());
    return psd;
}

std::vector<float> savgol_smooth(std::span<const float> values, int window, int order) {
    const std::size_t n = values.size();
    Call c;
    const float* v = c.in(values.data(), n);
    float* o = c.dev<float>(n);
    check(ss_savgol_smooth(ctx(), v, static_cast<int>(n), window, order, o));
    std::vector<float> out(n);
    c.get(out.data(), o, n);
    c.finish();
    return out;
}

static std::vector<int> floor_prune(PsdProfile& profile, const DetectorConfig& config) {
    const std::size_t n = profile.raw.size();
    const ss_detector_cfg c = to_c(config);
    Call k;
    const float* raw = k.in(profile.raw.data(), n);
    float* sm = k.dev<float>(n);
    float* ft = k.dev<float>(2);
    std::int32_t* act = k.dev<std::int32_t>(n);
    std::int32_t na = 0;
    check(ss_floor(ctx(), raw, static_cast<int>(n), &c, sm, ft, act, &na));  // returns after the count is on the host
    profile.smoothed.resize(n);
    k.get(profile.smoothed.data(), sm, n);
    float f[2];
    k.get(f, ft, 2);
    std::vector<int> active(static_cast<std::size_t>(na));
    k.get(active.data(), act, active.size());
    k.finish();
    profile.noise_floor = f[0];
    profile.threshold = f[1];
    return active;
}

void smooth_and_floor(PsdProfile& profile, const DetectorConfig& config) { floor_prune(profile, config); }

std::vector<int> prune_columns(const PsdProfile& profile) {
    const std::size_t n = profile.raw.size();
    Call k;
    const float* raw = k.in(profile.raw.data(), n);
    std::int32_t* act = k.dev<std::int32_t>(n);
    std::int32_t na = 0;
    check(ss_prune(ctx(), raw, static_cast<int>(n), profile.threshold, act, &na));
    std::vector<int> active(static_cast<std::size_t>(na));
    k.get(active.data(), act, active.size());
    k.finish();
    return active;
}

OtsuResult otsu_threshold(std::span<const float> values) {
    if (values.empty()) throw ValidationError("otsu on an empty column");
    Call k;
    const float* v = k.in(values.data(), values.size());
    std::int32_t valid = 0;
    float thr = 0.0f;
    check(ss_otsu(ctx(), v, static_cast<int>(values.size()), &valid, &thr));  // synchronous
    return {valid != 0, thr};
}

void binarize_columns(const frontend::TFPlotView& plot, std::span<const int> active_columns, int col_begin,
                      int col_end, Mask& out) {
    if (out.rows != plot.rows || out.cols != plot.cols) throw ValidationError("binarize output mask shape mismatch");
    Call k;
    const float* tf = k.in(plot.data, cells(plot));
    std::uint8_t* m = k.in(out.v.data(), out.v.size());
    check(ss_binarize_cols(ctx(), tf, plot.rows, plot.cols, active_columns.data(),
                           static_cast<int>(active_columns.size()), col_begin, col_end, m));
    k.get(out.v.data(), m, out.v.size());
    k.finish();
}

Mask binarize(const frontend::TFPlotView& plot, std::span<const int> active_columns) {
    Mask mask(plot.rows, plot.cols);
    binarize_columns(plot, active_columns, 0, plot.cols, mask);
    return mask;
}

void morphology_cols(const Mask& src, Mask& dst, MorphOp op, StructuringElement se, int col_begin, int col_end,
                     MorphScratch&) {
    if (dst.rows != src.rows || dst.cols != src.cols) throw ValidationError("morphology output mask shape mismatch");
    Call k;
    const std::uint8_t* s = k.in(src.v.data(), src.v.size());
    std::uint8_t* d = k.in(dst.v.data(), dst.v.size());
    check(ss_morph_cols(ctx(), s, src.rows, src.cols, static_cast<ss_morph_op>(op), se.rows, se.cols, col_begin,
                        col_end, d));
    k.get(dst.v.data(), d, dst.v.size());
    k.finish();
}

Mask morphology(const Mask& mask, MorphOp op, StructuringElement se) {
    Mask out(mask.rows, mask.cols);
    MorphScratch scratch;
    morphology_cols(mask, out, op, se, 0, mask.cols, scratch);
    return out;
}

Mask consolidate(const Mask& mask, bool one_d_opening_along_time) {
    Mask out(mask.rows, mask.cols);
    Call k;
    const std::uint8_t* s = k.in(mask.v.data(), mask.v.size());
    std::uint8_t* d = k.dev<std::uint8_t>(mask.v.size());
    check(ss_consolidate(ctx(), s, mask.rows, mask.cols, one_d_opening_along_time ? 1 : 0, d));
    k.get(out.v.data(), d, out.v.size());
    k.finish();
    return out;
}

static LabeledComponents components(const Mask& mask, int min_area, bool with_labels) {
    if (min_area < 1) throw ValidationError("min_component_area must be >= 1");
    LabeledComponents lc;
    lc.rows = mask.rows;
    lc.cols = mask.cols;
    const std::size_t n = mask.v.size();
    Call k;
    const std::uint8_t* m = k.in(mask.v.data(), n);
    std::int32_t* labels = k.dev<std::int32_t>(with_labels ? n : 1);
    std::int64_t cap = 1024, count = 0;
    std::vector<ss_extent> ext;
    for (;;) {
        ext.resize(static_cast<std::size_t>(cap));
        const ss_status s = ss_components(ctx(), m, mask.rows, mask.cols, min_area, with_labels ? labels : nullptr,
                                          ext.data(), cap, &count);
        if (s == SS_ECAPACITY && count > cap) {
            cap = count;
            continue;
        }
        check(s);
        break;
    }
    lc.extents.reserve(static_cast<std::size_t>(count));
    for (std::int64_t i = 0; i < count; ++i) {
        const ss_extent& e = ext[static_cast<std::size_t>(i)];
        lc.extents.push_back({static_cast<int>(e.min_t), static_cast<int>(e.max_t), static_cast<int>(e.min_f),
                              static_cast<int>(e.max_f), static_cast<long long>(e.area)});
    }
    if (with_labels) {
        lc.labels.resize(n);
        k.get(lc.labels.data(), labels, n);
        k.finish();
    }
    return lc;
}

LabeledComponents label_components(const Mask& mask, int min_component_area) {
    return components(mask, min_component_area, true);
}

std::vector<ComponentExtent> component_extents(const Mask& mask, int min_component_area) {
    return components(mask, min_component_area, false).extents;
}

BinBox extent_to_bin_box(const ComponentExtent& e) { return {e.min_t, e.max_t + 1, e.min_f, e.max_f + 1}; }

BoundingBox bin_box_to_physical(const BinBox& b, const frontend::TFPlotView& plot) {
    BoundingBox out;
    const double dt = plot.dt_s();
    const double df = plot.df_hz();
    out.t0_s = (static_cast<double>(plot.start_seq) + b.t0) * dt;
    out.t1_s = (static_cast<double>(plot.start_seq) + b.t1) * dt;
    out.f0_hz = (b.f0 - plot.cols / 2) * df;
    out.f1_hz = (b.f1 - plot.cols / 2) * df;
    return out;
}

// Device outputs of one batch call and their host copies.
struct BatchBufs {
    float *raw, *sm, *ft;
    std::int32_t *act, *nact, *nbox;
    ss_box* bx;
    ss_bin_box* bb;
};

// Runs one batch call with a growing box capacity; the inputs occupy the
// call's first `keep` device slots and survive a retry.
template <class Call_>
static std::vector<Detections> run_batch(Call& k, int keep, int P, int F, Call_&& call) {
    const std::size_t PF = static_cast<std::size_t>(P) * F;
    int K = 256;
    for (;;) {
        k.rewind();
        for (int i = 0; i < keep; ++i) k.dev<unsigned char>(0);  // skip the input slots (never shrink)
        BatchBufs d{k.dev<float>(PF), k.dev<float>(PF), k.dev<float>(2 * static_cast<std::size_t>(P)),
                    k.dev<std::int32_t>(PF), k.dev<std::int32_t>(static_cast<std::size_t>(P)),
                    k.dev<std::int32_t>(static_cast<std::size_t>(P)), k.dev<ss_box>(PF ? static_cast<std::size_t>(P) * K : 1),
                    k.dev<ss_bin_box>(static_cast<std::size_t>(P) * K)};
        ss_batch_out o{d.raw, d.sm, d.ft, d.act, d.nact, d.bx, d.bb, d.nbox, K};
        const ss_status s = call(o);
        std::vector<std::int32_t> nb(static_cast<std::size_t>(P));
        if (s == SS_ECAPACITY) {
            k.get(nb.data(), d.nbox, nb.size());
            k.finish();
            int mx = K;
            for (int v : nb) mx = v > mx ? v : mx;
            K = mx + 1;
            continue;
        }
        check(s);
        std::vector<float> hraw(PF), hsm(PF), hft(static_cast<std::size_t>(P) * 2);
        std::vector<std::int32_t> hact(PF), hnact(static_cast<std::size_t>(P));
        std::vector<ss_box> hbx(static_cast<std::size_t>(P) * K);
        std::vector<ss_bin_box> hbb(hbx.size());
        k.get(nb.data(), d.nbox, nb.size());
        k.get(hraw.data(), d.raw, PF);
        k.get(hsm.data(), d.sm, PF);
        k.get(hft.data(), d.ft, hft.size());
        k.get(hact.data(), d.act, PF);
        k.get(hnact.data(), d.nact, hnact.size());
        k.get(hbx.data(), d.bx, hbx.size());
        k.get(hbb.data(), d.bb, hbb.size());
        k.finish();
        std::vector<Detections> out(static_cast<std::size_t>(P));
        for (int p = 0; p < P; ++p) {
            Detections& r = out[static_cast<std::size_t>(p)];
            const std::size_t o0 = static_cast<std::size_t>(p) * F;
            const auto at = [o0](auto& v, std::size_t i) { return v.begin() + static_cast<std::ptrdiff_t>(o0 + i); };
            r.psd.raw.assign(at(hraw, 0), at(hraw, F));
            r.psd.smoothed.assign(at(hsm, 0), at(hsm, F));
            r.psd.noise_floor = hft[2 * static_cast<std::size_t>(p)];
            r.psd.threshold = hft[2 * static_cast<std::size_t>(p) + 1];
            r.active_columns.assign(at(hact, 0), at(hact, static_cast<std::size_t>(hnact[static_cast<std::size_t>(p)])));
            for (int i = 0; i < nb[static_cast<std::size_t>(p)]; ++i) {
                const ss_box& b = hbx[static_cast<std::size_t>(p) * K + i];
                const ss_bin_box& q = hbb[static_cast<std::size_t>(p) * K + i];
                r.boxes.push_back({b.f0_hz, b.f1_hz, b.t0_s, b.t1_s});
                r.bin_boxes.push_back({q.t0, q.t1, q.f0, q.f1});
            }
        }
        return out;
    }
}

std::vector<Detections> detect_batch(std::span<const frontend::TFPlotView> plots, const DetectorConfig& config) {
    if (plots.empty()) return {};
    const int P = static_cast<int>(plots.size());
    const int T = plots[0].rows, F = plots[0].cols;
    config.validate(F);
    for (const auto& v : plots)
        if (v.rows != T || v.cols != F || v.sample_rate_hz != plots[0].sample_rate_hz)
            throw ValidationError("detect_batch: plots must share rows, cols and sample rate");
    const std::size_t per = static_cast<std::size_t>(T) * F;
    Call k;
    float* tf = k.dev<float>(per * static_cast<std::size_t>(P));
    std::vector<std::uint64_t> seq(static_cast<std::size_t>(P));
    for (int p = 0; p < P; ++p) {
        k.put(tf + per * static_cast<std::size_t>(p), plots[static_cast<std::size_t>(p)].data, per);
        seq[static_cast<std::size_t>(p)] = plots[static_cast<std::size_t>(p)].start_seq;
    }
    const ss_detector_cfg c = to_c(config);
    return run_batch(k, 1, P, F, [&](const ss_batch_out& o) {
        return ss_detect_batch(ctx(), tf, P, T, F, seq.data(), plots[0].sample_rate_hz, &c, &o);
    });
}

Detections detect(const frontend::TFPlotView& plot, const DetectorConfig& config, StageTimes* times) {
    if (times) ss_enable_stage_timing(ctx(), 1);
    auto d = detect_batch(std::span<const frontend::TFPlotView>(&plot, 1), config);
    if (times) {
        double ms[8];
        ss_stage_times(ctx(), ms);
        ss_enable_stage_timing(ctx(), 0);
        times->psd += ms[1] * 1e-3;
        times->floor_prune += ms[2] * 1e-3;
        times->binarize += ms[3] * 1e-3;
        times->morphology += ms[4] * 1e-3;
        times->label += ms[5] * 1e-3;
    }
    return std::move(d[0]);
}

std::vector<Detections> sense(std::span<const cfloat> samples, const frontend::FrontendConfig& fc,
                              const DetectorConfig& config) {
    fc.validate();
    config.validate(fc.n_fft);
    const std::size_t per = static_cast<std::size_t>(fc.plot_rows) * fc.n_fft;
    const int P = static_cast<int>(samples.size() / per);
    if (P == 0) return {};
    Call k;
    const cfloat* iq = k.in(samples.data(), per * static_cast<std::size_t>(P));
    const ss_detector_cfg c = to_c(config);
    return run_batch(k, 1, P, fc.n_fft, [&](const ss_batch_out& o) {
        return ss_sense_batch(ctx(), iq, SS_FMT_F32, fc.n_fft, fc.plot_rows, P, 0, fc.sample_rate_hz, &c, nullptr, &o);
    });
}

} // namespace detector
} // namespace specsense
