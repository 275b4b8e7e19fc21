// baseline_demo.cpp -- a reference-style caller of specsense::baseline and
// specsense::metrics (include/specsense/{baseline,metrics}.hpp) linked
// against libspecsense_b200.so.  Reads one rows x cols f32 TF plot and a
// ground-truth box list, writes kernel sizes, baseline boxes and the
// compare() table to a binary file for tests/test_gpu_dropin.py.
//
//   baseline_demo <tf.f32> <rows> <cols> <fs> <start_seq> <truth.f64> <out.bin>
#include "specsense/baseline.hpp"

#include <fstream>
#include <iostream>
#include <vector>

using namespace specsense;

int main(int argc, char** argv) {
    if (argc != 8) {
        std::cerr << "usage: baseline_demo <tf.f32> <rows> <cols> <fs> <start_seq> <truth.f64> <out.bin>\n";
        return 2;
    }
    try {
        const int rows = std::stoi(argv[2]), cols = std::stoi(argv[3]);
        std::vector<float> tf(static_cast<std::size_t>(rows) * cols);
        std::ifstream(argv[1], std::ios::binary).read(reinterpret_cast<char*>(tf.data()),
                                                     static_cast<std::streamsize>(tf.size() * sizeof(float)));
        std::ifstream tfile(argv[6], std::ios::binary | std::ios::ate);
        const auto tbytes = static_cast<std::size_t>(tfile.tellg());
        std::vector<BoundingBox> truth(tbytes / sizeof(BoundingBox));
        tfile.seekg(0);
        tfile.read(reinterpret_cast<char*>(truth.data()), static_cast<std::streamsize>(tbytes));
        frontend::TFPlotView view{tf.data(), rows, cols, std::stoull(argv[5]), std::stod(argv[4])};
        std::ofstream out(argv[7], std::ios::binary);
        auto put = [&](const void* p, std::size_t n) { out.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };

        const auto ks = baseline::kernel_sizes(rows, cols);
        const int nk = static_cast<int>(ks.size());
        put(&nk, sizeof(nk));
        for (const auto& [a, b] : ks) {
            const int v[2] = {a, b};
            put(v, sizeof(v));
        }
        const auto boxes = baseline::baseline_detect(view);
        const int nb = static_cast<int>(boxes.size());
        put(&nb, sizeof(nb));
        put(boxes.data(), sizeof(BoundingBox) * boxes.size());
        const std::vector<std::vector<BoundingBox>> tp{truth};
        const frontend::TFPlotView views[1] = {view};
        const auto cmp = baseline::compare(views, tp, detector::DetectorConfig{}, baseline::BaselineConfig{}, 0.5);
        for (const auto& r : cmp.rows) {
            const double v[4] = {r.mean_latency_s, r.p_d, r.p_fa, r.mean_iou};
            put(v, sizeof(v));
        }
        put(&cmp.speedup, sizeof(double));
        // metrics spot values: evaluate(truth, baseline boxes, 0.3)
        const auto ev = metrics::evaluate(truth, boxes, 0.3);
        const double e[4] = {static_cast<double>(ev.n_true), static_cast<double>(ev.n_false), ev.p_fa, ev.mean_iou};
        put(e, sizeof(e));
        try {
            baseline::BaselineConfig bad;
            bad.conv_threshold = 0.0;
            baseline::kernel_sizes(rows, cols, bad);
            const int flag = 0;
            put(&flag, sizeof(flag));
        } catch (const ValidationError&) {
            const int flag = 1;
            put(&flag, sizeof(flag));
        }
        return 0;
    } catch (const Error& e) {
        std::cerr << "specsense error: " << e.what() << "\n";
        return 1;
    }
}
