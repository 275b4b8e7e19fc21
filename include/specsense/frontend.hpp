// specsense/frontend.hpp -- drop-in TF-plot front end on the B200.
//
// Same declarations as the hot-path part of proj/include/specsense/
// frontend.hpp (fft_row :47-48, TFPlotView / TFPlot :52-76, make_plot(s)
// :79-84, FrontendConfig :12-24, resolution / stream_bit_rate_bps :32-38);
// every call runs on the GPU through the C ABI (include/specsense_b200.h).
// The ChunkSource interface (:137-144) is declared so runtime::run
// (specsense/runtime.hpp) accepts the reference's sources; the concrete
// file / memory / UDP sources stay in the reference's I/O code.
#pragma once

#include "specsense/types.hpp"

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

namespace specsense::frontend {

// Capture geometry: fs, F (power of two >= 8; <= 2^20 on the device), T.
struct FrontendConfig {
    double sample_rate_hz = 0.0;
    int n_fft = 1024;
    int plot_rows = 2000;

    void validate() const;  // ValidationError on a bad fs / F / T

    double dt_s() const { return n_fft / sample_rate_hz; }
    double df_hz() const { return sample_rate_hz / n_fft; }
    double plot_span_s() const { return plot_rows * dt_s(); }
};

struct Resolution {
    double dt_s;
    double df_hz;
};

Resolution resolution(double sample_rate_hz, int n_fft);
double stream_bit_rate_bps(double sample_rate_hz, int bits_per_component);

struct IQChunk {
    std::uint64_t seq = 0;
    std::vector<cfloat> samples;
};

enum class SampleFormat { F32, I16 };

// Pull-style chunk producer: next() fills one F-sample chunk, false at end of
// stream; paced() sources deliver in real time and are shed, not blocked.
class ChunkSource {
  public:
    virtual ~ChunkSource() = default;
    virtual bool next(IQChunk& out) = 0;
    virtual bool paced() const { return false; }
};

// out[k] = |DFT(chunk)[(k + F/2) mod F]|, F = chunk.size().
void fft_row(std::span<const cfloat> chunk, std::span<float> out);
std::vector<float> fft_row(std::span<const cfloat> chunk);

// Non-owning row-major T x F plot; row t is chunk start_seq + t.
struct TFPlotView {
    const float* data = nullptr;
    int rows = 0;
    int cols = 0;
    std::uint64_t start_seq = 0;
    double sample_rate_hz = 0.0;

    const float* row(int t) const { return data + static_cast<std::size_t>(t) * cols; }
    float at(int t, int f) const { return row(t)[f]; }
    double dt_s() const { return cols / sample_rate_hz; }
    double df_hz() const { return sample_rate_hz / cols; }
    double row_start_time_s(int t) const { return (start_seq + t) * dt_s(); }
    double col_center_freq_hz(int k) const { return (k - cols / 2) * df_hz(); }
};

struct TFPlot {
    std::vector<float> data;
    int rows = 0;
    int cols = 0;
    std::uint64_t start_seq = 0;
    double sample_rate_hz = 0.0;

    float* row(int t) { return data.data() + static_cast<std::size_t>(t) * cols; }
    TFPlotView view() const { return {data.data(), rows, cols, start_seq, sample_rate_hz}; }
};

TFPlot make_plot(std::span<const cfloat> samples, double sample_rate_hz, int n_fft,
                 std::uint64_t start_seq = 0);

// Consecutive full windows of config.plot_rows rows; a partial tail is dropped.
std::vector<TFPlot> make_plots(std::span<const cfloat> samples, const FrontendConfig& config);

// B200 extension: interleaved int16 IQ (frontend.cpp:376-385 scaling) -> plots.
std::vector<TFPlot> make_plots_i16(std::span<const std::int16_t> iq_interleaved,
                                   const FrontendConfig& config);

} // namespace specsense::frontend
