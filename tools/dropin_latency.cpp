// dropin_latency.cpp -- per-call latency of the C++ drop-in's stage API on the
// B200 (persistent per-thread workspace): frontend::fft_row on one 1024-point
// row (the reference calls it row by row: signals.cpp:249), detector::detect on
// one (500, 1024) plot and otsu_threshold on one 500-value column.  Prints one
// JSON line (median microseconds over 2000 / 200 / 2000 calls after warm-up).
#include "specsense/detector.hpp"
#include "specsense/frontend.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

using namespace specsense;
using Clock = std::chrono::steady_clock;

template <class F>
static double median_us(int reps, F&& fn) {
    for (int i = 0; i < 20; ++i) fn();
    std::vector<double> t;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = Clock::now();
        fn();
        t.push_back(std::chrono::duration<double, std::micro>(Clock::now() - t0).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    std::mt19937 rng(7);
    std::normal_distribution<float> g(0.f, 1.f);
    std::vector<cfloat> row(1024);
    for (auto& s : row) s = {g(rng), g(rng)};
    std::vector<float> mags(1024);
    const double fft_us = median_us(2000, [&] { frontend::fft_row(row, mags); });

    std::vector<float> plot(500 * 1024);
    for (auto& v : plot) v = std::abs(g(rng));
    const frontend::TFPlotView view{plot.data(), 500, 1024, 0, 100e6};
    const double det_us = median_us(200, [&] { (void)detector::detect(view, detector::DetectorConfig{}); });
    std::vector<float> col(plot.begin(), plot.begin() + 500);
    const double otsu_us = median_us(2000, [&] { (void)detector::otsu_threshold(col); });
    std::printf("{\"fft_row_1024_us\": %.1f, \"detect_500x1024_us\": %.1f, \"otsu_500_us\": %.1f}\n", fft_us, det_us,
                otsu_us);
    return 0;
}
