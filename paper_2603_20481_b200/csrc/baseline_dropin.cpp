// baseline_dropin.cpp -- specsense::baseline and specsense::metrics
// (include/specsense/{baseline,metrics}.hpp) over the C ABI.  baseline_detect
// runs ss_baseline_detect (GPU SAT + kernel bank, host greedy); the metrics
// are host arithmetic with the reference's definitions
// (proj/src/metrics.cpp:7-79); compare() times detect and baseline_detect
// per plot on the GPU (proj/src/baseline.cpp:207-232).
#include "specsense/baseline.hpp"
#include "specsense_b200.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>

namespace specsense {
namespace metrics {

double iou(const BoundingBox& a, const BoundingBox& b) {
    const double aa = a.area(), ab = b.area();
    if (aa <= 0.0 || ab <= 0.0) return 0.0;
    const double fi = std::max(0.0, std::min(a.f1_hz, b.f1_hz) - std::max(a.f0_hz, b.f0_hz));
    const double ti = std::max(0.0, std::min(a.t1_s, b.t1_s) - std::max(a.t0_s, b.t0_s));
    const double inter = fi * ti;
    return inter / (aa + ab - inter);
}

double IoUMatrix::row_max(int gt) const {
    double m = 0.0;
    for (int d = 0; d < n_det; ++d) m = std::max(m, at(gt, d));
    return m;
}

double IoUMatrix::col_max(int det) const {
    double m = 0.0;
    for (int g = 0; g < n_gt; ++g) m = std::max(m, at(g, det));
    return m;
}

IoUMatrix iou_matrix(std::span<const BoundingBox> gt, std::span<const BoundingBox> det) {
    IoUMatrix m;
    m.n_gt = static_cast<int>(gt.size());
    m.n_det = static_cast<int>(det.size());
    m.v.resize(gt.size() * det.size());
    for (std::size_t g = 0; g < gt.size(); ++g)
        for (std::size_t d = 0; d < det.size(); ++d) m.v[g * det.size() + d] = iou(gt[g], det[d]);
    return m;
}

MatchCounts count_matches(const IoUMatrix& m, double theta) {
    MatchCounts c;
    for (int g = 0; g < m.n_gt; ++g) c.n_true += m.row_max(g) > theta ? 1 : 0;
    for (int d = 0; d < m.n_det; ++d) c.n_false += m.col_max(d) < theta ? 1 : 0;
    return c;
}

EvalResult evaluate(const IoUMatrix& m, double theta) {
    const MatchCounts c = count_matches(m, theta);
    EvalResult r;
    r.theta = theta;
    r.n_gt = m.n_gt;
    r.n_det = m.n_det;
    r.n_true = c.n_true;
    r.n_false = c.n_false;
    r.p_d = m.n_gt > 0 ? static_cast<double>(c.n_true) / m.n_gt : 0.0;
    r.p_fa = m.n_det > 0 ? static_cast<double>(c.n_false) / m.n_det : 0.0;
    double s = 0.0;
    for (int g = 0; g < m.n_gt; ++g) s += m.row_max(g);
    r.mean_iou = m.n_gt > 0 ? s / m.n_gt : 0.0;
    return r;
}

EvalResult evaluate(std::span<const BoundingBox> gt, std::span<const BoundingBox> det, double theta) {
    return evaluate(iou_matrix(gt, det), theta);
}

std::vector<EvalResult> sweep(std::span<const BoundingBox> gt, std::span<const BoundingBox> det,
                              std::span<const double> thetas) {
    const IoUMatrix m = iou_matrix(gt, det);
    std::vector<EvalResult> out;
    for (double t : thetas) out.push_back(evaluate(m, t));
    return out;
}

} // namespace metrics

namespace baseline {
namespace {

ss_baseline_cfg to_c(const BaselineConfig& c) {
    return ss_baseline_cfg{c.conv_threshold, c.rate_change_threshold, c.noise_offset_db, c.max_kernel_rows,
                           c.max_kernel_cols};
}

struct Ctx {
    ss_ctx* h = nullptr;
    Ctx() {
        const char* dev = std::getenv("SPECSENSE_DEVICE");
        if (ss_open(dev ? std::atoi(dev) : 0, &h) != SS_OK) throw Error("specsense-b200: no usable sm_100 device");
        ss_set_stream(h, nullptr);
    }
    ~Ctx() { ss_close(h); }
};

ss_ctx* ctx() {
    thread_local Ctx c;
    return c.h;
}

} // namespace

void BaselineConfig::validate() const {
    if (!(conv_threshold > 0.0)) throw ValidationError("conv_threshold must be > 0");
    if (!(rate_change_threshold > 0.0)) throw ValidationError("rate_change_threshold must be > 0");
    if (max_kernel_rows < 0 || max_kernel_cols < 0) throw ValidationError("kernel caps must be >= 0");
}

std::vector<std::pair<int, int>> kernel_sizes(int rows, int cols, const BaselineConfig& config) {
    config.validate();
    if (rows < 1 || cols < 1) throw ValidationError("plot must be non-empty");
    const ss_baseline_cfg c = to_c(config);
    const int n = ss_baseline_kernel_sizes(rows, cols, &c, nullptr, 1 << 20);
    std::vector<int32_t> v(static_cast<std::size_t>(2 * std::max(n, 0)));
    ss_baseline_kernel_sizes(rows, cols, &c, v.data(), n);
    std::vector<std::pair<int, int>> out;
    for (int i = 0; i < n; ++i) out.emplace_back(v[2 * i], v[2 * i + 1]);
    return out;
}

std::vector<BoundingBox> baseline_detect(const frontend::TFPlotView& plot, const BaselineConfig& config) {
    config.validate();
    const ss_baseline_cfg c = to_c(config);
    int cap = 4096;
    for (;;) {
        std::vector<ss_box> b(static_cast<std::size_t>(cap));
        int n = 0;
        const ss_status s = ss_baseline_detect(ctx(), plot.data, plot.rows, plot.cols, plot.start_seq,
                                               plot.sample_rate_hz, &c, b.data(), nullptr, cap, &n);
        if (s == SS_ECAPACITY) {
            cap = n;
            continue;
        }
        if (s == SS_EVALIDATION) throw ValidationError(ss_last_error(ctx()));
        if (s != SS_OK) throw Error(ss_last_error(ctx()));
        std::vector<BoundingBox> out(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) out[i] = BoundingBox{b[i].f0_hz, b[i].f1_hz, b[i].t0_s, b[i].t1_s};
        return out;
    }
}

CompareRow make_compare_row(const std::string& name, std::span<const std::vector<BoundingBox>> dets,
                            std::span<const std::vector<BoundingBox>> truth, double theta, double mean_latency_s) {
    if (dets.size() != truth.size()) throw ValidationError("detections/truth plot counts differ");
    long long n_gt = 0, n_det = 0, n_true = 0, n_false = 0;
    double iou_sum = 0.0;
    for (std::size_t p = 0; p < truth.size(); ++p) {
        const metrics::IoUMatrix m = metrics::iou_matrix(truth[p], dets[p]);
        const metrics::MatchCounts c = metrics::count_matches(m, theta);
        n_gt += m.n_gt;
        n_det += m.n_det;
        n_true += c.n_true;
        n_false += c.n_false;
        for (int g = 0; g < m.n_gt; ++g) iou_sum += m.row_max(g);
    }
    CompareRow r;
    r.detector = name;
    r.mean_latency_s = mean_latency_s;
    r.p_d = n_gt > 0 ? static_cast<double>(n_true) / static_cast<double>(n_gt) : 0.0;
    r.p_fa = n_det > 0 ? static_cast<double>(n_false) / static_cast<double>(n_det) : 0.0;
    r.mean_iou = n_gt > 0 ? iou_sum / static_cast<double>(n_gt) : 0.0;
    return r;
}

Comparison compare(std::span<const frontend::TFPlotView> plots, std::span<const std::vector<BoundingBox>> truth,
                   const detector::DetectorConfig& dc, const BaselineConfig& bc, double theta) {
    if (plots.size() != truth.size()) throw ValidationError("plots/truth counts differ");
    if (plots.empty()) throw ValidationError("compare needs at least one plot");
    using Clock = std::chrono::steady_clock;
    std::vector<std::vector<BoundingBox>> pipe(plots.size()), base(plots.size());
    double pipe_s = 0.0, base_s = 0.0;
    for (std::size_t p = 0; p < plots.size(); ++p) {
        auto t0 = Clock::now();
        pipe[p] = detector::detect(plots[p], dc).boxes;
        pipe_s += std::chrono::duration<double>(Clock::now() - t0).count();
        t0 = Clock::now();
        base[p] = baseline_detect(plots[p], bc);
        base_s += std::chrono::duration<double>(Clock::now() - t0).count();
    }
    const double n = static_cast<double>(plots.size());
    Comparison c;
    c.rows.push_back(make_compare_row("pipeline", pipe, truth, theta, pipe_s / n));
    c.rows.push_back(make_compare_row("baseline", base, truth, theta, base_s / n));
    c.speedup = pipe_s > 0.0 ? base_s / pipe_s : 0.0;
    return c;
}

} // namespace baseline
} // namespace specsense
