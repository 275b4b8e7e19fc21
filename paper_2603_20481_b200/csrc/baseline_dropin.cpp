// baseline_dropin.cpp -- specsense::baseline's detector half
// (include/specsense/baseline.hpp: BaselineConfig::validate, kernel_sizes,
// baseline_detect; proj/src/baseline.cpp:15-178) over the C ABI.
// baseline_detect runs ss_baseline_detect (GPU SAT + kernel bank, host greedy).
// The evaluation helpers (make_compare_row / compare, baseline.cpp:180-232, and
// all of metrics.cpp) are out of scope: a caller links the
// reference's own objects for them (oracle/Makefile, `suite` recipe).
#include "specsense/baseline.hpp"
#include "specsense_b200.h"

#include <algorithm>
#include <cstdlib>

namespace specsense {

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

} // namespace baseline
} // namespace specsense
