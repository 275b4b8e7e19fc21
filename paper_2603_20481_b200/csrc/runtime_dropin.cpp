// runtime_dropin.cpp -- specsense::runtime (include/specsense/runtime.hpp)
// over the streaming engine (ss_engine_*, csrc/engine.cpp).
//
// run(): an ingest thread pulls chunks from the caller's ChunkSource, packs
// runs of consecutive chunks into a host batch and pushes them into the
// engine's HBM banks (gaps in the sequence -> ss_engine_mark_lost, as the
// reference's ingest marks lost ranges, proj/src/runtime.cpp:289-303); the
// calling thread polls finished windows in order, converts them to
// PlotRecord + BoundingBox spans for the handler, and summarises.  Report
// arithmetic follows proj/src/runtime.cpp:170-214.
#include "specsense/runtime.hpp"
#include "specsense_b200.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>

namespace specsense::runtime {
namespace {

using Clock = std::chrono::steady_clock;

void throw_status(ss_status s, const std::string& m) {
    if (s == SS_EVALIDATION) throw ValidationError(m);
    if (s == SS_EFORMAT) throw FormatError(m);
    throw Error(m);
}

struct Engine {
    ss_engine* h = nullptr;
    ~Engine() { ss_engine_close(h); }
    void check(ss_status s) const {
        if (s != SS_OK) throw_status(s, ss_engine_last_error(h));
    }
};

} // namespace

void RuntimeConfig::validate() const {
    if (n_compute_workers < 1) throw ValidationError("n_compute_workers must be >= 1");
    if (n_sensing_workers < 1) throw ValidationError("n_sensing_workers must be >= 1");
    if (halo_bins < 3) throw ValidationError("halo_bins must be >= 3");
    if (chunk_queue_capacity < 0) throw ValidationError("chunk_queue_capacity must be >= 0");
    if (deadline_s < 0.0) throw ValidationError("deadline_s must be >= 0");
}

std::vector<Slab> partition(int n_cols, int n_slabs, int halo) {
    if (n_slabs < 1 || n_slabs > n_cols) throw ValidationError("n_slabs must be in [1, n_cols]");
    if (halo < 3) throw ValidationError("halo must be >= 3");
    std::vector<Slab> out(static_cast<std::size_t>(n_slabs));
    // the first n_cols % n_slabs cores are one column wider
    const int q = n_cols / n_slabs, extra = n_cols % n_slabs;
    for (int i = 0, at = 0; i < n_slabs; ++i) {
        Slab& s = out[static_cast<std::size_t>(i)];
        s.core_begin = at;
        at += q + (i < extra ? 1 : 0);
        s.core_end = at;
        s.ext_begin = std::max(0, s.core_begin - halo);
        s.ext_end = std::min(n_cols, s.core_end + halo);
    }
    return out;
}

detector::Mask consolidate_sliced(const detector::Mask& mask, int n_slabs, int halo, bool one_d_opening_along_time) {
    (void)partition(mask.cols, n_slabs, halo);  // same argument checks as the reference
    // the slab-parallel form is bit-identical to the whole-image one for any
    // slab count (the reference's contract); the device runs it whole
    return detector::consolidate(mask, one_d_opening_along_time);
}

double nearest_rank(std::span<const double> sorted, double q) {
    if (sorted.empty()) return 0.0;
    const long long n = static_cast<long long>(sorted.size());
    const long long k = std::clamp(static_cast<long long>(std::ceil(q * static_cast<double>(n))), 1LL, n);
    return sorted[static_cast<std::size_t>(k - 1)];
}

RunReport summarize(std::vector<PlotRecord> records, std::uint64_t overruns, double deadline_s) {
    RunReport r;
    std::sort(records.begin(), records.end(),
              [](const PlotRecord& a, const PlotRecord& b) { return a.plot_index < b.plot_index; });
    r.records = std::move(records);
    r.plots = r.records.size();
    r.overruns = overruns;
    r.deadline_s = deadline_s;
    if (!r.records.empty()) {
        std::vector<double> lat;
        lat.reserve(r.records.size());
        std::uint64_t met = 0;
        for (const PlotRecord& p : r.records) {
            lat.push_back(p.latency_s);
            met += p.met ? 1 : 0;
        }
        std::sort(lat.begin(), lat.end());
        r.fraction_met = static_cast<double>(met) / static_cast<double>(lat.size());
        r.p50_s = nearest_rank(lat, 0.50);
        r.p90_s = nearest_rank(lat, 0.90);
        r.p99_s = nearest_rank(lat, 0.99);
        r.max_s = lat.back();
        r.percentiles_valid = lat.size() >= 100;
    }
    r.realtime_met = r.fraction_met >= 0.99;
    return r;
}

std::vector<std::pair<double, double>> RunReport::ccdf() const {
    std::vector<double> lat;
    lat.reserve(records.size());
    for (const PlotRecord& p : records) lat.push_back(p.latency_s);
    std::sort(lat.begin(), lat.end());
    std::vector<std::pair<double, double>> pts;
    const double n = static_cast<double>(lat.size());
    for (std::size_t i = 0; i < lat.size(); ++i) {
        const bool last_of_value = i + 1 == lat.size() || lat[i + 1] != lat[i];
        if (last_of_value) pts.emplace_back(lat[i], static_cast<double>(lat.size() - i - 1) / n);
    }
    return pts;
}

RunReport run(frontend::ChunkSource& source, const frontend::FrontendConfig& fc,
              const detector::DetectorConfig& dc, const RuntimeConfig& rc, const DetectionHandler& on_detections) {
    fc.validate();
    dc.validate(fc.n_fft);
    rc.validate();
    const int F = fc.n_fft, T = fc.plot_rows;
    const double deadline = rc.deadline_s > 0.0 ? rc.deadline_s : fc.plot_span_s();
    constexpr int kCap = 16384;  // boxes kept per window

    ss_engine_cfg ec{};
    ec.n_fft = F;
    ec.plot_rows = T;
    ec.fmt = SS_FMT_F32;
    ec.sample_rate_hz = fc.sample_rate_hz;
    ec.n_banks = 2;
    ec.paced = source.paced() ? 1 : 0;
    ec.deadline_s = deadline;
    ec.box_capacity = kCap;
    ec.stage_timing = 1;  // RunReport::stage_totals / fft_time_s, as the reference reports them
    ss_detector_cfg c{};
    c.savgol_window = dc.savgol_window;
    c.savgol_order = dc.savgol_order;
    c.psd_margin_db = dc.psd_margin_db;
    c.min_component_area = dc.min_component_area;
    c.one_d_opening_along_time = dc.one_d_opening_along_time ? 1 : 0;
    Engine eng;
    const ss_status st = ss_engine_open(0, &ec, &c, &eng.h);
    if (st != SS_OK) {
        const std::string m = eng.h ? ss_engine_last_error(eng.h) : "no usable sm_100 device";
        throw_status(st, "specsense-b200 engine: " + m);
    }

    const auto wall0 = Clock::now();
    std::mutex err_mu;
    std::string err;
    std::atomic<bool> failed{false};
    auto capture = [&](const char* where, const std::exception& e) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (!failed.exchange(true)) err = std::string(where) + ": " + e.what();
    };

    // ingest: every chunk goes straight to the engine, which stages it in the
    // bank's pinned buffer and sends runs of 64 chunks per H2D (no batch copy)
    std::thread ingest([&] {
        try {
            std::uint64_t expected = 0;
            frontend::IQChunk chunk;
            while (!failed.load() && source.next(chunk)) {
                if (chunk.samples.size() != static_cast<std::size_t>(F))
                    throw ValidationError("chunk size " + std::to_string(chunk.samples.size()) + " != n_fft");
                // as runtime.cpp:283-285: a gap is lost, expected follows the chunk
                // (stale chunks go on to the engine, which retires them)
                if (chunk.seq > expected) eng.check(ss_engine_mark_lost(eng.h, expected, chunk.seq));
                eng.check(ss_engine_push(eng.h, chunk.samples.data(), 1, chunk.seq));
                expected = chunk.seq + 1;
            }
        } catch (const std::exception& e) {
            capture("ingest", e);
        }
        ss_engine_finish(eng.h);
    });

    std::vector<PlotRecord> records;
    double fft_total = 0.0;
    detector::StageTimes stages;
    std::vector<ss_box> raw(kCap);
    std::vector<BoundingBox> boxes;
    try {
        for (;;) {
            ss_plot_record r{};
            int got = 0;
            const ss_status s = ss_engine_poll(eng.h, -1, &r, raw.data(), nullptr, kCap, &got);
            if (!got) {
                eng.check(s);
                break;
            }
            eng.check(s);
            PlotRecord rec;
            rec.plot_index = r.plot_index;
            rec.start_seq = r.start_seq;
            rec.latency_s = r.latency_s;
            rec.deadline_s = r.deadline_s;
            rec.met = r.met != 0;
            rec.n_boxes = r.n_boxes;
            // per-stage device time of the window's graph (CUDA event nodes):
            // K1 is the reference's compute-worker FFT, K2..K6 its sensing stages
            fft_total += r.stage_s[0];
            stages.psd += r.stage_s[1];
            stages.floor_prune += r.stage_s[2];
            stages.binarize += r.stage_s[3];
            stages.morphology += r.stage_s[4];
            stages.label += r.stage_s[5];
            boxes.resize(static_cast<std::size_t>(std::min(r.n_boxes, kCap)));
            for (std::size_t i = 0; i < boxes.size(); ++i)
                boxes[i] = BoundingBox{raw[i].f0_hz, raw[i].f1_hz, raw[i].t0_s, raw[i].t1_s};
            records.push_back(rec);
            if (on_detections) on_detections(rec, boxes);
        }
    } catch (const std::exception& e) {
        capture("manager", e);
        // drain: releases banks a blocked unpaced push may be waiting on; the
        // ingest thread sees the failure, finishes the stream, poll runs dry
        for (;;) {
            int got = 0;
            ss_engine_poll(eng.h, -1, nullptr, nullptr, nullptr, 0, &got);
            if (!got) break;
        }
    }
    ingest.join();
    if (failed.load()) throw Error("engine aborted, " + err);
    uint64_t overruns = 0;
    eng.check(ss_engine_stats(eng.h, nullptr, &overruns, nullptr, nullptr));
    RunReport rep = summarize(std::move(records), overruns, deadline);
    rep.fft_time_s = fft_total;
    rep.stage_totals = stages;
    rep.wall_time_s = std::chrono::duration<double>(Clock::now() - wall0).count();
    return rep;
}

} // namespace specsense::runtime
