// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat extern "C" face over the UNMODIFIED reference library (the
// /root/reference/proj/src/*.cpp sources compiled by oracle/Makefile into
// oracle/_ref/libspecsense_ref.so together with oracle/fftw_shim.c), so the
// Python tests, smoke() and bench.py's CPU leg can call the reference itself
// through ctypes.  No reference source is copied: this file only includes the
// reference headers in place and forwards.  Every exception is caught and
// turned into a negative return code plus a message (ref_last_error).
//
// Return codes: >= 0 success (often a count), -1 ValidationError,
// -2 FormatError, -3 SchemaError, -4 IoError, -5 other specsense::Error,
// -6 std::exception, -7 capacity too small.

#include "specsense/baseline.hpp"
#include "specsense/detector.hpp"
#include "specsense/frontend.hpp"
#include "specsense/metrics.hpp"
#include "specsense/runtime.hpp"
#include "specsense/signals.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace specsense;

namespace {

thread_local std::string g_err;

template <class F>
long long guard(F&& f) {
    try {
        return f();
    } catch (const ValidationError& e) {
        g_err = e.what();
        return -1;
    } catch (const FormatError& e) {
        g_err = e.what();
        return -2;
    } catch (const SchemaError& e) {
        g_err = e.what();
        return -3;
    } catch (const IoError& e) {
        g_err = e.what();
        return -4;
    } catch (const Error& e) {
        g_err = e.what();
        return -5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -6;
    }
}

frontend::TFPlotView view_of(const float* tf, int rows, int cols, unsigned long long start_seq,
                             double fs) {
    frontend::TFPlotView v;
    v.data = tf;
    v.rows = rows;
    v.cols = cols;
    v.start_seq = start_seq;
    v.sample_rate_hz = fs;
    return v;
}

detector::Mask mask_of(const unsigned char* m, int rows, int cols) {
    detector::Mask out(rows, cols);
    std::memcpy(out.v.data(), m, static_cast<std::size_t>(rows) * cols);
    return out;
}

detector::DetectorConfig dcfg(int window, int order, double margin_db, int min_area,
                              int along_time) {
    detector::DetectorConfig c;
    c.savgol_window = window;
    c.savgol_order = order;
    c.psd_margin_db = margin_db;
    c.min_component_area = min_area;
    c.one_d_opening_along_time = along_time != 0;
    return c;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// frontend::fft_row (proj/src/frontend.cpp:127-149)
long long ref_fft_row(const float* iq, int n, float* out) {
    return guard([&]() -> long long {
        std::span<const cfloat> in(reinterpret_cast<const cfloat*>(iq), static_cast<std::size_t>(n));
        frontend::fft_row(in, std::span<float>(out, static_cast<std::size_t>(n)));
        return 0;
    });
}

// frontend::make_plots (proj/src/frontend.cpp:173-183). Writes n_plots*rows*n_fft
// floats; returns the plot count.
long long ref_make_plots(const float* iq, long long n_samples, double fs, int n_fft, int rows,
                         float* out, long long out_capacity_floats) {
    return guard([&]() -> long long {
        frontend::FrontendConfig fc;
        fc.sample_rate_hz = fs;
        fc.n_fft = n_fft;
        fc.plot_rows = rows;
        std::span<const cfloat> in(reinterpret_cast<const cfloat*>(iq),
                                   static_cast<std::size_t>(n_samples));
        const auto plots = frontend::make_plots(in, fc);
        const long long per = static_cast<long long>(rows) * n_fft;
        if (static_cast<long long>(plots.size()) * per > out_capacity_floats) return -7;
        for (std::size_t p = 0; p < plots.size(); ++p)
            std::memcpy(out + p * per, plots[p].data.data(), sizeof(float) * per);
        return static_cast<long long>(plots.size());
    });
}

// detector::estimate_psd_into (proj/src/detector.cpp:170-184)
long long ref_estimate_psd_into(const float* tf, int rows, int cols, int c0, int c1, float* out) {
    return guard([&]() -> long long {
        detector::estimate_psd_into(view_of(tf, rows, cols, 0, 1.0), c0, c1, out);
        return 0;
    });
}

// detector::savgol_smooth (proj/src/detector.cpp:192-208)
long long ref_savgol_smooth(const float* v, int n, int window, int order, float* out) {
    return guard([&]() -> long long {
        const auto r = detector::savgol_smooth(std::span<const float>(v, static_cast<std::size_t>(n)),
                                               window, order);
        std::memcpy(out, r.data(), sizeof(float) * r.size());
        return 0;
    });
}

// detector::smooth_and_floor + prune_columns (proj/src/detector.cpp:210-255)
long long ref_floor_prune(const float* raw, int n, int window, int order, double margin_db,
                          float* smoothed, float* floor_thr, int* active) {
    return guard([&]() -> long long {
        detector::PsdProfile p;
        p.raw.assign(raw, raw + n);
        detector::smooth_and_floor(p, dcfg(window, order, margin_db, 4, 0));
        std::memcpy(smoothed, p.smoothed.data(), sizeof(float) * n);
        floor_thr[0] = p.noise_floor;
        floor_thr[1] = p.threshold;
        const auto act = detector::prune_columns(p);
        std::copy(act.begin(), act.end(), active);
        return static_cast<long long>(act.size());
    });
}

// detector::otsu_threshold (proj/src/detector.cpp:257-271); returns valid.
long long ref_otsu_threshold(const float* v, int n, float* thr) {
    return guard([&]() -> long long {
        const auto r = detector::otsu_threshold(std::span<const float>(v, static_cast<std::size_t>(n)));
        *thr = r.threshold;
        return r.valid ? 1 : 0;
    });
}

// detector::binarize_columns (proj/src/detector.cpp:273-335) into a caller mask.
long long ref_binarize_columns(const float* tf, int rows, int cols, const int* active, int n_active,
                               int c0, int c1, unsigned char* mask_inout) {
    return guard([&]() -> long long {
        detector::Mask m = mask_of(mask_inout, rows, cols);
        detector::binarize_columns(view_of(tf, rows, cols, 0, 1.0),
                                   std::span<const int>(active, static_cast<std::size_t>(n_active)),
                                   c0, c1, m);
        std::memcpy(mask_inout, m.v.data(), m.v.size());
        return 0;
    });
}

// detector::morphology_cols (proj/src/detector.cpp:441-472). op: 0 erode,
// 1 dilate, 2 open, 3 close.
long long ref_morphology_cols(const unsigned char* src, int rows, int cols, int op, int se_rows,
                              int se_cols, int c0, int c1, unsigned char* dst_inout) {
    return guard([&]() -> long long {
        const detector::Mask s = mask_of(src, rows, cols);
        detector::Mask d = mask_of(dst_inout, rows, cols);
        detector::MorphScratch scratch;
        detector::morphology_cols(s, d, static_cast<detector::MorphOp>(op), {se_rows, se_cols}, c0, c1,
                                  scratch);
        std::memcpy(dst_inout, d.v.data(), d.v.size());
        return 0;
    });
}

// detector::consolidate (proj/src/detector.cpp:482-492)
long long ref_consolidate(const unsigned char* src, int rows, int cols, int along_time,
                          unsigned char* dst) {
    return guard([&]() -> long long {
        const auto r = detector::consolidate(mask_of(src, rows, cols), along_time != 0);
        std::memcpy(dst, r.v.data(), r.v.size());
        return 0;
    });
}

// runtime::consolidate_sliced (proj/src/runtime.cpp:147-168)
long long ref_consolidate_sliced(const unsigned char* src, int rows, int cols, int n_slabs, int halo,
                                 int along_time, unsigned char* dst) {
    return guard([&]() -> long long {
        const auto r = runtime::consolidate_sliced(mask_of(src, rows, cols), n_slabs, halo,
                                                   along_time != 0);
        std::memcpy(dst, r.v.data(), r.v.size());
        return 0;
    });
}

// detector::label_components (proj/src/detector.cpp:604-620). extents: 5
// int64 per component (min_t, max_t, min_f, max_f, area). labels may be null.
long long ref_label_components(const unsigned char* m, int rows, int cols, int min_area,
                               int* labels, long long* extents, long long cap) {
    return guard([&]() -> long long {
        const auto lc = detector::label_components(mask_of(m, rows, cols), min_area);
        if (static_cast<long long>(lc.extents.size()) > cap) return -7;
        if (labels) std::memcpy(labels, lc.labels.data(), sizeof(int) * lc.labels.size());
        for (std::size_t i = 0; i < lc.extents.size(); ++i) {
            const auto& e = lc.extents[i];
            long long* o = extents + 5 * i;
            o[0] = e.min_t;
            o[1] = e.max_t;
            o[2] = e.min_f;
            o[3] = e.max_f;
            o[4] = e.area;
        }
        return static_cast<long long>(lc.extents.size());
    });
}

// detector::detect (proj/src/detector.cpp:637-670). Outputs: psd4 =
// raw/smoothed (n each) then floor, threshold; active indices; boxes as 4
// doubles (f0,f1,t0,t1) and bin boxes as 4 ints (t0,t1,f0,f1). Returns the box
// count; *n_active receives the active-column count.
long long ref_detect(const float* tf, int rows, int cols, unsigned long long start_seq, double fs,
                     int window, int order, double margin_db, int min_area, int along_time,
                     float* raw, float* smoothed, float* floor_thr, int* active, int* n_active,
                     double* boxes, int* bin_boxes, long long cap) {
    return guard([&]() -> long long {
        const auto det = detector::detect(view_of(tf, rows, cols, start_seq, fs),
                                          dcfg(window, order, margin_db, min_area, along_time));
        if (static_cast<long long>(det.boxes.size()) > cap) return -7;
        if (raw) std::memcpy(raw, det.psd.raw.data(), sizeof(float) * cols);
        if (smoothed) std::memcpy(smoothed, det.psd.smoothed.data(), sizeof(float) * cols);
        if (floor_thr) {
            floor_thr[0] = det.psd.noise_floor;
            floor_thr[1] = det.psd.threshold;
        }
        if (active) std::copy(det.active_columns.begin(), det.active_columns.end(), active);
        if (n_active) *n_active = static_cast<int>(det.active_columns.size());
        for (std::size_t i = 0; i < det.boxes.size(); ++i) {
            boxes[4 * i + 0] = det.boxes[i].f0_hz;
            boxes[4 * i + 1] = det.boxes[i].f1_hz;
            boxes[4 * i + 2] = det.boxes[i].t0_s;
            boxes[4 * i + 3] = det.boxes[i].t1_s;
            bin_boxes[4 * i + 0] = det.bin_boxes[i].t0;
            bin_boxes[4 * i + 1] = det.bin_boxes[i].t1;
            bin_boxes[4 * i + 2] = det.bin_boxes[i].f0;
            bin_boxes[4 * i + 3] = det.bin_boxes[i].f1;
        }
        return static_cast<long long>(det.boxes.size());
    });
}

// signals::scenario_from_json + synthesize (proj/src/signals.cpp:149-226,
// 415-470). Writes interleaved float32 IQ and truth boxes (f0,f1,t0,t1,kind).
long long ref_synthesize(const char* scenario_json, float* iq, long long cap_samples,
                         double* truth, long long cap_truth, long long* n_truth) {
    return guard([&]() -> long long {
        const auto sc = signals::scenario_from_json(scenario_json);
        const auto syn = signals::synthesize(sc);
        if (static_cast<long long>(syn.samples.size()) > cap_samples) return -7;
        if (static_cast<long long>(syn.truth.boxes.size()) > cap_truth) return -7;
        if (iq) std::memcpy(iq, syn.samples.data(), sizeof(cfloat) * syn.samples.size());
        for (std::size_t i = 0; i < syn.truth.boxes.size(); ++i) {
            const auto& b = syn.truth.boxes[i];
            truth[5 * i + 0] = b.box.f0_hz;
            truth[5 * i + 1] = b.box.f1_hz;
            truth[5 * i + 2] = b.box.t0_s;
            truth[5 * i + 3] = b.box.t1_s;
            truth[5 * i + 4] = static_cast<double>(static_cast<int>(b.kind));
        }
        *n_truth = static_cast<long long>(syn.truth.boxes.size());
        return static_cast<long long>(syn.samples.size());
    });
}

// Sample count a scenario renders to (for buffer sizing).
long long ref_scenario_samples(const char* scenario_json) {
    return guard([&]() -> long long {
        const auto sc = signals::scenario_from_json(scenario_json);
        return std::llround(sc.duration_s * sc.sample_rate_hz);
    });
}

// metrics::iou (proj/src/metrics.cpp:7-15)
double ref_iou(const double* a, const double* b) {
    BoundingBox x{a[0], a[1], a[2], a[3]};
    BoundingBox y{b[0], b[1], b[2], b[3]};
    return metrics::iou(x, y);
}

// CPU baseline: make_plot + detect over `n_plots` plots of `samples` (plot p
// uses the p-th window, cycling), spread over n_threads std::threads, each
// plot handled end to end by one thread -- the reference's stage functions
// are pure and safe concurrently on disjoint data.  Returns the
// number of boxes found; *seconds receives the wall time.
long long ref_bench_detect(const float* iq, long long n_samples, double fs, int n_fft, int rows,
                           long long n_plots, int n_threads, double* seconds) {
    return guard([&]() -> long long {
        const long long per = static_cast<long long>(rows) * n_fft;
        const long long windows = n_samples / per;
        if (windows < 1) throw ValidationError("not one full plot of samples");
        std::atomic<long long> next{0}, boxes{0};
        const auto t0 = std::chrono::steady_clock::now();
        auto work = [&]() {
            long long local = 0;
            for (;;) {
                const long long p = next.fetch_add(1);
                if (p >= n_plots) break;
                const long long w = p % windows;
                std::span<const cfloat> in(reinterpret_cast<const cfloat*>(iq) + w * per,
                                           static_cast<std::size_t>(per));
                const auto plot = frontend::make_plot(in, fs, n_fft,
                                                      static_cast<std::uint64_t>(w) * rows);
                const auto det = detector::detect(plot.view(), detector::DetectorConfig{});
                local += static_cast<long long>(det.boxes.size());
            }
            boxes += local;
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < std::max(1, n_threads); ++t) pool.emplace_back(work);
        for (auto& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return boxes.load();
    });
}

// CPU baseline through the reference's own streaming engine runtime::run
// (proj/src/runtime.cpp:221-487) with an unpaced MemorySource cycling the
// samples for n_plots windows.  stats: plots, overruns, wall_s, p50, p99,
// fraction_met, fft_time_s.
long long ref_run_engine(const float* iq, long long n_samples, double fs, int n_fft, int rows,
                         long long n_plots, int n_compute, int n_sensing, double* stats) {
    return guard([&]() -> long long {
        frontend::FrontendConfig fc;
        fc.sample_rate_hz = fs;
        fc.n_fft = n_fft;
        fc.plot_rows = rows;
        runtime::RuntimeConfig rc;
        rc.n_compute_workers = n_compute;
        rc.n_sensing_workers = n_sensing;
        std::vector<cfloat> samples(reinterpret_cast<const cfloat*>(iq),
                                    reinterpret_cast<const cfloat*>(iq) + n_samples);
        frontend::MemorySource src(std::move(samples), n_fft,
                                   static_cast<std::uint64_t>(n_plots) * rows);
        std::atomic<long long> boxes{0};
        const auto rep = runtime::run(src, fc, detector::DetectorConfig{}, rc,
                                      [&](const runtime::PlotRecord&, std::span<const BoundingBox> b) {
                                          boxes += static_cast<long long>(b.size());
                                      });
        stats[0] = static_cast<double>(rep.plots);
        stats[1] = static_cast<double>(rep.overruns);
        stats[2] = rep.wall_time_s;
        stats[3] = rep.p50_s;
        stats[4] = rep.p99_s;
        stats[5] = rep.fraction_met;
        stats[6] = rep.fft_time_s;
        return boxes.load();
    });
}


// runtime::summarize (runtime.cpp:166-199) on scripted records: stats =
// {plots, overruns, deadline, fraction_met, realtime_met, p50, p90, p99, max,
// percentiles_valid}; ccdf points (latency, fraction) into ccdf[2*i..]
// (capacity cap points).  Returns the ccdf point count.
long long ref_summarize(long long n, const unsigned long long* plot_index, const double* latency, const int* met,
                        unsigned long long overruns, double deadline, double* stats, double* ccdf, long long cap) {
    return guard([&]() -> long long {
        std::vector<runtime::PlotRecord> recs(static_cast<std::size_t>(n));
        for (long long i = 0; i < n; ++i) {
            recs[i].plot_index = plot_index[i];
            recs[i].latency_s = latency[i];
            recs[i].met = met[i] != 0;
            recs[i].deadline_s = deadline;
        }
        const auto rep = runtime::summarize(std::move(recs), overruns, deadline);
        stats[0] = static_cast<double>(rep.plots);
        stats[1] = static_cast<double>(rep.overruns);
        stats[2] = rep.deadline_s;
        stats[3] = rep.fraction_met;
        stats[4] = rep.realtime_met ? 1.0 : 0.0;
        stats[5] = rep.p50_s;
        stats[6] = rep.p90_s;
        stats[7] = rep.p99_s;
        stats[8] = rep.max_s;
        stats[9] = rep.percentiles_valid ? 1.0 : 0.0;
        const auto pts = rep.ccdf();
        if (static_cast<long long>(pts.size()) > cap) return -7;
        for (std::size_t i = 0; i < pts.size(); ++i) {
            ccdf[2 * i] = pts[i].first;
            ccdf[2 * i + 1] = pts[i].second;
        }
        return static_cast<long long>(pts.size());
    });
}

// runtime::run over an unpaced MemorySource of n_plots windows (cycling the
// samples), collecting every window's boxes: out_plot[i] = plot_index of box
// i, out_boxes[4*i..] = (f0, f1, t0, t1).  Returns the box count.
long long ref_run_engine_boxes(const float* iq, long long n_samples, double fs, int n_fft, int rows, long long n_plots,
                               int n_compute, int n_sensing, unsigned long long* out_plot, double* out_boxes,
                               long long cap, unsigned long long* plots_seen) {
    return guard([&]() -> long long {
        frontend::FrontendConfig fc;
        fc.sample_rate_hz = fs;
        fc.n_fft = n_fft;
        fc.plot_rows = rows;
        runtime::RuntimeConfig rc;
        rc.n_compute_workers = n_compute;
        rc.n_sensing_workers = n_sensing;
        std::vector<cfloat> samples(reinterpret_cast<const cfloat*>(iq),
                                    reinterpret_cast<const cfloat*>(iq) + n_samples);
        frontend::MemorySource src(std::move(samples), n_fft, static_cast<std::uint64_t>(n_plots) * rows);
        long long nb = 0;
        bool overflow = false;
        const auto rep = runtime::run(src, fc, detector::DetectorConfig{}, rc,
                                      [&](const runtime::PlotRecord& r, std::span<const BoundingBox> b) {
                                          for (const BoundingBox& x : b) {
                                              if (nb >= cap) {
                                                  overflow = true;
                                                  return;
                                              }
                                              out_plot[nb] = r.plot_index;
                                              out_boxes[4 * nb] = x.f0_hz;
                                              out_boxes[4 * nb + 1] = x.f1_hz;
                                              out_boxes[4 * nb + 2] = x.t0_s;
                                              out_boxes[4 * nb + 3] = x.t1_s;
                                              ++nb;
                                          }
                                      });
        *plots_seen = rep.plots;
        return overflow ? -7 : nb;
    });
}


static baseline::BaselineConfig bl_cfg(double conv, double rate, double offset, int mkr, int mkc) {
    baseline::BaselineConfig c;
    c.conv_threshold = conv;
    c.rate_change_threshold = rate;
    c.noise_offset_db = offset;
    c.max_kernel_rows = mkr;
    c.max_kernel_cols = mkc;
    return c;
}

// baseline::kernel_sizes -> (kr, kc) pairs; returns the count.
long long ref_kernel_sizes(int rows, int cols, double conv, double rate, double offset, int mkr, int mkc, int* out,
                           long long cap) {
    return guard([&]() -> long long {
        const auto v = baseline::kernel_sizes(rows, cols, bl_cfg(conv, rate, offset, mkr, mkc));
        if (static_cast<long long>(v.size()) > cap) return -7;
        for (std::size_t i = 0; i < v.size(); ++i) {
            out[2 * i] = v[i].first;
            out[2 * i + 1] = v[i].second;
        }
        return static_cast<long long>(v.size());
    });
}

// baseline::baseline_detect on one plot -> boxes (f0, f1, t0, t1); returns the count.
long long ref_baseline_detect(const float* tf, int rows, int cols, unsigned long long start_seq, double fs, double conv,
                              double rate, double offset, int mkr, int mkc, double* boxes, long long cap) {
    return guard([&]() -> long long {
        frontend::TFPlotView v{tf, rows, cols, start_seq, fs};
        const auto b = baseline::baseline_detect(v, bl_cfg(conv, rate, offset, mkr, mkc));
        if (static_cast<long long>(b.size()) > cap) return -7;
        for (std::size_t i = 0; i < b.size(); ++i) {
            boxes[4 * i] = b[i].f0_hz;
            boxes[4 * i + 1] = b[i].f1_hz;
            boxes[4 * i + 2] = b[i].t0_s;
            boxes[4 * i + 3] = b[i].t1_s;
        }
        return static_cast<long long>(b.size());
    });
}

} // extern "C"
