// baseline_demo.cpp -- a reference-style caller of specsense::baseline
// (include/specsense/baseline.hpp) linked against libspecsense_b200.so.
// Reads one rows x cols f32 TF plot, writes kernel sizes and baseline boxes to
// a binary file for tests/test_gpu_dropin.py.  (compare() and the metrics are
// the reference's own evaluation code: the reference's test_baseline.cpp runs
// them over this library, oracle/Makefile `suite`.)
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
