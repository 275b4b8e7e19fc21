// runtime_demo.cpp -- a reference-style caller of specsense::runtime::run
// (include/specsense/runtime.hpp) linked against libspecsense_b200.so: an
// in-memory ChunkSource cycles raw f32 IQ as F-sample chunks, run() streams
// them through the GPU engine, and every window's boxes plus the report go
// to a binary file for tests/test_gpu_dropin.py.
//
//   runtime_demo <iq.f32> <fs> <n_fft> <rows> <n_windows> <paced 0|1> <out.bin>
#include "specsense/runtime.hpp"

#include <chrono>
#include <fstream>
#include <iostream>
#include <thread>
#include <vector>

using namespace specsense;

namespace {

class CyclingSource final : public frontend::ChunkSource {
  public:
    CyclingSource(std::vector<cfloat> s, int n_fft, std::uint64_t total, bool pace, double fs)
        : s_(std::move(s)), f_(n_fft), total_(total), pace_(pace), fs_(fs), t0_(std::chrono::steady_clock::now()) {}
    bool next(frontend::IQChunk& out) override {
        if (seq_ >= total_) return false;
        const std::size_t n = s_.size() / static_cast<std::size_t>(f_);
        const std::size_t at = static_cast<std::size_t>(seq_ % n) * static_cast<std::size_t>(f_);
        if (pace_) {
            // the stream starts when the engine first asks for a chunk (engine
            // set-up time is not part of the paced stream)
            if (seq_ == 0) t0_ = std::chrono::steady_clock::now();
            const auto due = t0_ + std::chrono::duration<double>(static_cast<double>(seq_ + 1) * f_ / fs_);
            std::this_thread::sleep_until(due);
        }
        out.seq = seq_++;
        out.samples.assign(s_.begin() + static_cast<std::ptrdiff_t>(at), s_.begin() + static_cast<std::ptrdiff_t>(at + f_));
        return true;
    }
    bool paced() const override { return pace_; }

  private:
    std::vector<cfloat> s_;
    int f_;
    std::uint64_t total_, seq_ = 0;
    bool pace_;
    double fs_;
    std::chrono::steady_clock::time_point t0_;
};

} // namespace

int main(int argc, char** argv) {
    if (argc != 8) {
        std::cerr << "usage: runtime_demo <iq.f32> <fs> <n_fft> <rows> <n_windows> <paced 0|1> <out.bin>\n";
        return 2;
    }
    try {
        std::ifstream f(argv[1], std::ios::binary | std::ios::ate);
        const auto bytes = static_cast<std::size_t>(f.tellg());
        std::vector<cfloat> samples(bytes / sizeof(cfloat));
        f.seekg(0);
        f.read(reinterpret_cast<char*>(samples.data()), static_cast<std::streamsize>(bytes));
        frontend::FrontendConfig fc;
        fc.sample_rate_hz = std::stod(argv[2]);
        fc.n_fft = std::stoi(argv[3]);
        fc.plot_rows = std::stoi(argv[4]);
        const std::uint64_t windows = std::stoull(argv[5]);
        const bool paced = std::stoi(argv[6]) != 0;
        CyclingSource src(std::move(samples), fc.n_fft, windows * static_cast<std::uint64_t>(fc.plot_rows), paced,
                          fc.sample_rate_hz);
        std::ofstream out(argv[7], std::ios::binary);
        auto put = [&](const void* p, std::size_t n) { out.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };
        runtime::RuntimeConfig rc;
        const runtime::RunReport rep =
            runtime::run(src, fc, detector::DetectorConfig{}, rc,
                         [&](const runtime::PlotRecord& r, std::span<const BoundingBox> b) {
                             const std::uint64_t head[2] = {r.plot_index, b.size()};
                             put(head, sizeof(head));
                             put(b.data(), sizeof(BoundingBox) * b.size());
                         });
        const std::uint64_t end[2] = {~0ull, rep.plots};
        put(end, sizeof(end));
        const double stats[8] = {static_cast<double>(rep.overruns), rep.p50_s, rep.p90_s, rep.p99_s,
                                 rep.max_s, rep.fraction_met, rep.wall_time_s, rep.fft_time_s};
        put(stats, sizeof(stats));
        const auto cc = rep.ccdf();
        const std::uint64_t ncc = cc.size();
        put(&ncc, sizeof(ncc));
        for (const auto& [l, fr] : cc) {
            put(&l, sizeof(l));
            put(&fr, sizeof(fr));
        }
        // partition / nearest_rank spot values for the host-logic test
        const auto sl = runtime::partition(1024, 3, 4);
        for (const auto& s : sl) {
            const int v[4] = {s.core_begin, s.core_end, s.ext_begin, s.ext_end};
            put(v, sizeof(v));
        }
        return 0;
    } catch (const Error& e) {
        std::cerr << "specsense error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
