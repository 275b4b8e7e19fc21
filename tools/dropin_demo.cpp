// dropin_demo.cpp -- a reference-style caller of the C++ drop-in API
// (include/specsense/*.hpp), linked against libspecsense_b200.so exactly as a
// reference user would relink.  Reads raw f32 IQ, runs make_plots + detect
// and a chain of stage functions, and dumps everything to a binary file that
// tests/test_gpu_dropin.py compares against the reference oracle.
//
//   dropin_demo <iq.f32> <fs> <n_fft> <rows> <out.bin>
#include "specsense/detector.hpp"
#include "specsense/frontend.hpp"

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <vector>

using namespace specsense;

namespace {
std::ofstream out;
template <class T>
void put(const T* p, std::size_t n) {
    out.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(sizeof(T) * n));
}
template <class T>
void put1(T v) {
    put(&v, 1);
}
} // namespace

int main(int argc, char** argv) {
    if (argc != 6) {
        std::cerr << "usage: dropin_demo <iq.f32> <fs> <n_fft> <rows> <out.bin>\n";
        return 2;
    }
    try {
        std::ifstream f(argv[1], std::ios::binary | std::ios::ate);
        const auto bytes = static_cast<std::size_t>(f.tellg());
        std::vector<cfloat> samples(bytes / sizeof(cfloat));
        f.seekg(0);
        f.read(reinterpret_cast<char*>(samples.data()), static_cast<std::streamsize>(bytes));
        frontend::FrontendConfig fc;
        fc.sample_rate_hz = std::atof(argv[2]);
        fc.n_fft = std::atoi(argv[3]);
        fc.plot_rows = std::atoi(argv[4]);
        out.open(argv[5], std::ios::binary);

        const auto plots = frontend::make_plots(samples, fc);
        put1<std::int32_t>(static_cast<std::int32_t>(plots.size()));
        detector::DetectorConfig cfg;
        for (const auto& p : plots) {
            detector::StageTimes st;
            const auto det = detector::detect(p.view(), cfg, &st);
            put(p.data.data(), p.data.size());
            put(det.psd.raw.data(), det.psd.raw.size());
            put(det.psd.smoothed.data(), det.psd.smoothed.size());
            put1(det.psd.noise_floor);
            put1(det.psd.threshold);
            put1<std::int32_t>(static_cast<std::int32_t>(det.active_columns.size()));
            put(det.active_columns.data(), det.active_columns.size());
            put1<std::int32_t>(static_cast<std::int32_t>(det.boxes.size()));
            for (std::size_t i = 0; i < det.boxes.size(); ++i) {
                const double b[4] = {det.boxes[i].f0_hz, det.boxes[i].f1_hz, det.boxes[i].t0_s, det.boxes[i].t1_s};
                const std::int32_t q[4] = {det.bin_boxes[i].t0, det.bin_boxes[i].t1, det.bin_boxes[i].f0,
                                           det.bin_boxes[i].f1};
                put(b, 4);
                put(q, 4);
            }
            put1(st.total());
        }
        // stage chain on plot 0: fft_row, estimate_psd, smooth_and_floor,
        // prune_columns, binarize, consolidate, label_components
        const auto row = frontend::fft_row(std::span<const cfloat>(samples.data(), static_cast<std::size_t>(fc.n_fft)));
        put(row.data(), row.size());
        const auto v = plots.at(0).view();
        detector::PsdProfile prof;
        prof.raw = detector::estimate_psd(v);
        detector::smooth_and_floor(prof, cfg);
        const auto act = detector::prune_columns(prof);
        const auto mask = detector::binarize(v, act);
        const auto cons = detector::consolidate(mask);
        const auto lc = detector::label_components(cons, cfg.min_component_area);
        put(prof.raw.data(), prof.raw.size());
        put1(prof.threshold);
        put1<std::int32_t>(static_cast<std::int32_t>(act.size()));
        put(act.data(), act.size());
        put(mask.v.data(), mask.v.size());
        put(cons.v.data(), cons.v.size());
        put(lc.labels.data(), lc.labels.size());
        put1<std::int32_t>(static_cast<std::int32_t>(lc.extents.size()));
        try {
            frontend::fft_row(std::vector<cfloat>(100));
            put1<std::int32_t>(0);
        } catch (const ValidationError&) {
            put1<std::int32_t>(1);  // the reference's exception type crosses the ABI
        }
        out.close();
    } catch (const Error& e) {
        std::cerr << "specsense error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
