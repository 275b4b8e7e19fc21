/*
 * specsense_b200.h -- the C-ABI drop-in boundary of the B200 spectrum-sensing
 * hot path (plain pointers and sizes; no C++ or torch types cross it).
 *
 * The reference exposes the path as C++ free functions in the static library
 * `specsense` (proj/src/CMakeLists.txt:1-13); there is no FFI.  Each entry
 * point below replaces one of those functions (file:line cited); the C++
 * drop-in library (include/specsense/*.hpp, implemented over this ABI in
 * paper_2603_20481_b200/csrc/dropin.cpp) keeps the reference's signatures and
 * exception types, so callers relink instead of rewriting.
 *
 * Memory: unless stated otherwise every array argument is DEVICE memory on the
 * context's GPU, owned by the caller.  ss_sense_batch also accepts HOST
 * buffers (pinned or pageable) and stages them itself.  Work is enqueued on
 * the context's stream (ss_set_stream); functions that return counts or
 * validate data-dependent results synchronise that stream.
 *
 * Errors: functions return an ss_status; ss_last_error(ctx) holds the
 * message.  Status codes map one-to-one onto the reference's exception types
 * (proj/include/specsense/types.hpp:43-70): SS_EVALIDATION -> ValidationError,
 * SS_EFORMAT -> FormatError; SS_ECUDA / SS_ENOMEM / SS_EUNSUPPORTED /
 * SS_ECAPACITY -> specsense::Error.  There is no CPU fallback: without a
 * usable sm_100 device ss_open fails with SS_ECUDA.
 */
#ifndef SPECSENSE_B200_H
#define SPECSENSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 1

typedef enum {
    SS_OK = 0,
    SS_EVALIDATION = 1, /* bad sizes / config / ranges (ValidationError) */
    SS_EFORMAT = 2,     /* malformed payloads (FormatError) */
    SS_ECUDA = 3,       /* CUDA runtime failure or no device */
    SS_ENOMEM = 4,      /* device allocation failed */
    SS_EUNSUPPORTED = 5,/* valid for the reference, not supported on device (e.g. n_fft > 2^20) */
    SS_ECAPACITY = 6    /* caller-provided output capacity too small */
} ss_status;

typedef enum { SS_FMT_F32 = 0, SS_FMT_I16 = 1 } ss_fmt; /* frontend.hpp:134 SampleFormat */

typedef enum { SS_ERODE = 0, SS_DILATE = 1, SS_OPEN = 2, SS_CLOSE = 3 } ss_morph_op; /* detector.hpp:54 */

/* STFT extension windows (BASELINE config 5 as written; no reference oracle):
   rectangular, or periodic Hann w[n] = 0.5*(1 - cos(2*pi*n/N)). */
typedef enum { SS_WIN_RECT = 0, SS_WIN_HANN = 1 } ss_window;

typedef struct ss_ctx ss_ctx;

/* DetectorConfig (proj/include/specsense/detector.hpp:11-23), same defaults. */
typedef struct {
    int savgol_window;            /* 31 */
    int savgol_order;             /* 3 */
    double psd_margin_db;         /* 3.0 */
    int min_component_area;       /* 4 */
    int one_d_opening_along_time; /* 0 */
} ss_detector_cfg;

/* BoundingBox (types.hpp:17-26): half-open [t0,t1) x [f0,f1), seconds x Hz. */
typedef struct {
    double f0_hz, f1_hz, t0_s, t1_s;
} ss_box;

/* BinBox (types.hpp:30-39): half-open bin ranges. */
typedef struct {
    int32_t t0, t1, f0, f1;
} ss_bin_box;

/* ComponentExtent (detector.hpp:118-122): inclusive extents + pixel area. */
typedef struct {
    int64_t min_t, max_t, min_f, max_f, area;
} ss_extent;

/* Per-plot outputs of the fused pipeline (Detections, detector.hpp:159-164).
   Arrays are caller-owned; any pointer may be NULL to skip that output.
   Shapes for a batch of P plots with F columns and box capacity K:
     psd_raw, psd_smoothed : P x F floats       floor_thr : P x 2 (floor, threshold)
     active                : P x F ints (first n_active[p] valid)   n_active : P
     boxes                 : P x K ss_box       bin_boxes : P x K ss_bin_box
     n_boxes               : P (true count; > K means the record arrays overflowed)
   Memory kind follows the batch call: device for ss_detect_batch; host or
   device (auto-detected per pointer) for ss_sense_batch. */
typedef struct {
    float* psd_raw;
    float* psd_smoothed;
    float* floor_thr;
    int32_t* active;
    int32_t* n_active;
    ss_box* boxes;
    ss_bin_box* bin_boxes;
    int32_t* n_boxes;
    int32_t box_capacity; /* K */
} ss_batch_out;

/* ---- context ---------------------------------------------------------- */
ss_status ss_open(int device, ss_ctx** out);
void ss_close(ss_ctx* ctx);
const char* ss_last_error(const ss_ctx* ctx);
int ss_abi_version(void);
void ss_default_detector_cfg(ss_detector_cfg* cfg);
/* Enqueue subsequent work on `stream` (a cudaStream_t; NULL = CUDA's legacy
   default stream).  A new context uses its own non-blocking stream. */
ss_status ss_set_stream(ss_ctx* ctx, void* stream);
ss_status ss_synchronize(ss_ctx* ctx);
/* Asynchronous batches.  With on != 0, ss_sense_batch, ss_stft_sense_batch and
   ss_detect_batch return as soon as their work is queued on the context
   stream -- no host synchronisation, so back-to-back batches overlap (outputs
   in pinned host memory or on the device; a pageable host output makes its
   copy, and so the call, synchronous).  The checks a synchronous call makes
   before returning (box capacity, CCL run-pool overflow) run on the device and
   are reported by ss_wait for every batch since the previous ss_wait:
   SS_ECAPACITY if a plot had more boxes than box_capacity or more runs than
   the shared pool (its results are then incomplete: re-run those batches with
   async off, which sizes the pool exactly).  on = 0 restores synchronous calls. */
ss_status ss_set_async(ss_ctx* ctx, int on);
/* Wait for all queued work of the context; SS_ECAPACITY as described above. */
ss_status ss_wait(ss_ctx* ctx);
/* Device kernel launches issued by this context so far (instrumentation). */
int64_t ss_launch_count(const ss_ctx* ctx);
/* Per-stage CUDA-event timing of the batch pipelines (on the context stream):
   ss_enable_stage_timing resets the accumulators; ss_stage_times returns the
   accumulated milliseconds of [K1 fft_mag, K2 psd, K3 floor, K4 binarize,
   K5 consolidate, K6 ccl, H2D staging, D2H results] in ms8[0..7]. */
ss_status ss_enable_stage_timing(ss_ctx* ctx, int on);
ss_status ss_stage_times(const ss_ctx* ctx, double* ms8);

/* ---- frontend --------------------------------------------------------- */
/* frontend::make_plot / make_plots (frontend.cpp:157-183) over n_plots
   consecutive plots of `rows` rows: iq holds n_plots*rows*n_fft samples
   (interleaved I,Q; 16-byte aligned), tf receives n_plots*rows*n_fft floats,
   row r column k = |X_r[(k + n_fft/2) mod n_fft]| (frontend.cpp:127-149).
   n_fft: power of two, 8 <= n_fft <= 2^20 on device (reference: any power of
   two >= 8, frontend.cpp:37-42; larger sizes -> SS_EUNSUPPORTED).  Up to
   8192 one CTA transforms a row in shared memory (K1); above, the same
   SSFFT-2 passes run as a chain of global-memory kernels. */
ss_status ss_tf_plots(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int rows, int n_plots,
                      float* tf);

/* STFT extension of ss_tf_plots (the reference is
   rectangular with hop = n_fft): frame f covers samples
   [f*hop, f*hop + n_fft), each sample multiplied by the window in double
   before the same SSFFT-2 transform.  iq holds (n_plots*rows - 1)*hop +
   n_fft samples.  hop = n_fft with SS_WIN_RECT reproduces ss_tf_plots. */
ss_status ss_stft_plots(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                        int n_plots, float* tf);

/* ---- detector stages (one plot unless noted) --------------------------- */
/* estimate_psd_into (detector.cpp:170-184): out[k - c0] for k in [c0, c1). */
ss_status ss_psd_cols(ss_ctx* ctx, const float* tf, int rows, int cols, int c0, int c1, float* out);
/* savgol_smooth (detector.cpp:192-208). */
ss_status ss_savgol_smooth(ss_ctx* ctx, const float* values, int n, int window, int order,
                           float* out);
/* smooth_and_floor + prune_columns (detector.cpp:210-255) for one PSD row:
   smoothed[n], floor_thr[2] = {noise_floor, threshold}, active[<= n],
   *n_active (HOST int). */
ss_status ss_floor(ss_ctx* ctx, const float* raw, int n, const ss_detector_cfg* cfg,
                   float* smoothed, float* floor_thr, int32_t* active, int32_t* n_active);
/* prune_columns (detector.cpp:250-255): active = {k : raw[k] >= threshold}
   ascending; *n_active (HOST). */
ss_status ss_prune(ss_ctx* ctx, const float* raw, int n, float threshold, int32_t* active,
                   int32_t* n_active);
/* otsu_threshold (detector.cpp:257-271); *valid, *threshold are HOST. */
ss_status ss_otsu(ss_ctx* ctx, const float* values, int n, int32_t* valid, float* threshold);
/* binarize_columns (detector.cpp:273-335): writes columns [c0, c1) of the
   rows x cols byte mask; active_host is a HOST array of plot-wide indices. */
ss_status ss_binarize_cols(ss_ctx* ctx, const float* tf, int rows, int cols,
                           const int32_t* active_host, int n_active, int c0, int c1,
                           uint8_t* mask);
/* morphology_cols (detector.cpp:441-472) on byte masks; dst must not alias src. */
ss_status ss_morph_cols(ss_ctx* ctx, const uint8_t* src, int rows, int cols, ss_morph_op op,
                        int se_rows, int se_cols, int c0, int c1, uint8_t* dst);
/* consolidate (detector.cpp:482-492) on byte masks. */
ss_status ss_consolidate(ss_ctx* ctx, const uint8_t* src, int rows, int cols, int along_time,
                         uint8_t* dst);
/* label_components / component_extents (detector.cpp:598-620): extents
   (HOST, capacity cap) in first-pixel order; labels (DEVICE rows x cols int32,
   0 = background) may be NULL; *n_out (HOST) = component count. */
ss_status ss_components(ss_ctx* ctx, const uint8_t* mask, int rows, int cols, int min_area,
                        int32_t* labels, ss_extent* extents_host, int64_t cap, int64_t* n_out);

/* ---- fused batch pipelines -------------------------------------------- */
/* detect (detector.cpp:637-670) on n_plots plot-major TF plots already in
   device memory; plot p's start_seq = start_seq[p] (HOST array, may be NULL
   = all 0).  Outputs in DEVICE memory. */
ss_status ss_detect_batch(ss_ctx* ctx, const float* tf, int n_plots, int rows, int cols,
                          const uint64_t* start_seq, double sample_rate_hz,
                          const ss_detector_cfg* cfg, const ss_batch_out* out);

/* IQ -> boxes for n_plots consecutive windows (make_plots + detect per
   window, i.e. the runtime's per-plot work, runtime.cpp:324-445): plot p
   covers samples [p*rows*n_fft, (p+1)*rows*n_fft) with start_seq =
   first_seq + p*rows.  iq may be host or device memory; tf_out (DEVICE,
   n_plots*rows*n_fft floats) may be NULL when the TF plots are not wanted
   (they are still produced in the context's workspace). */
ss_status ss_sense_batch(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int rows, int n_plots,
                         uint64_t first_seq, double sample_rate_hz, const ss_detector_cfg* cfg,
                         float* tf_out, const ss_batch_out* out);

/* STFT-extension form of ss_sense_batch: frames as in ss_stft_plots, plot p's
   first frame = first_frame + p*rows, box times use the frame step hop/fs. */
ss_status ss_stft_sense_batch(ss_ctx* ctx, const void* iq, ss_fmt fmt, int n_fft, int hop, int window, int rows,
                              int n_plots, uint64_t first_frame, double sample_rate_hz,
                              const ss_detector_cfg* cfg, float* tf_out, const ss_batch_out* out);

/* ---- streaming engine ---------------------------------------------------
   GPU form of the reference's real-time engine (runtime::run,
   proj/src/runtime.cpp:221-487, with frontend::PingPongBuffer,
   proj/include/specsense/frontend.hpp:86-135): F-sample chunks with a
   sequence number stream into HBM banks; window w (T frames: samples
   [w*T*hop, w*T*hop + (T-1)*hop + F), i.e. chunks w*T .. w*T+T-1 for the
   reference's hop = F) fills bank w % n_banks (a chunk straddling two
   overlapping STFT windows goes to both); when its samples are in, the
   whole window runs K1..K6 on the
   engine's stream and its boxes land in pinned host memory.  A bank stays
   held until its record is polled (the reference releases after the
   detection handler).  Rows for a window whose bank is still held are
   dropped and the window is counted as one overrun (paced) or the push
   blocks until the bank is released (unpaced: back-pressure, no loss).
   Latency = host time from the push that delivered the window's last row
   to the moment its boxes are in host memory (the reference: bank complete
   -> boxes emitted, runtime.cpp:441).  Thread model: one pushing thread,
   one polling thread. */
typedef struct ss_engine ss_engine;

typedef struct {
    int n_fft;             /* F: power of two, 8..2^20 */
    int plot_rows;         /* T */
    ss_fmt fmt;            /* chunk sample format */
    double sample_rate_hz;
    int n_banks;           /* >= 2; 2 = the reference's ping-pong */
    int paced;             /* 1: shed windows (overruns); 0: push blocks */
    double deadline_s;     /* <= 0: the plot span T*hop/fs */
    int box_capacity;      /* boxes kept per plot */
    int hop;               /* STFT extension: frame step in samples (0: n_fft, the reference's frames) */
    int window;            /* STFT extension: an ss_window value, 0 = rectangular */
    int shard_count;       /* multi-GPU: windows are dealt round-robin over shard_count engines */
    int shard_index;       /* ... this engine senses windows w with w % shard_count == shard_index
                              (0 / 0: every window); others are skipped, not counted as lost */
    int stage_timing;      /* 1: per-stage device times in ss_plot_record.stage_s (event-record nodes
                              in each window's graph: about 0.12 ms of device time per P window);
                              0: only gpu_s, the window's whole device time */
} ss_engine_cfg;

/* runtime::PlotRecord (proj/include/specsense/runtime.hpp:62-69) + extras */
typedef struct {
    uint64_t plot_index;   /* window id */
    uint64_t start_seq;
    double latency_s;      /* bank complete -> boxes on the host */
    double deadline_s;
    int32_t met;           /* latency_s <= deadline_s */
    int32_t n_boxes;       /* true count (> capacity: only the first capacity returned) */
    int32_t n_active;
    float noise_floor;
    float threshold;
    double complete_s;     /* engine clock: window complete */
    double done_s;         /* engine clock: boxes on the host */
    double gpu_s;          /* device time from the window's first kernel to its boxes' D2H end */
    double stage_s[8];     /* device time per stage, ss_stage_times ids (0 K1 FFT, 1 K2 PSD, 2 K3 floor
                              + prune, 3 K4 binarize, 4 K5 consolidate, 5 K6 label + boxes; 6, 7 unused) */
} ss_plot_record;

ss_status ss_engine_open(int device, const ss_engine_cfg* cfg, const ss_detector_cfg* det, ss_engine** out);
void ss_engine_close(ss_engine* eng);
const char* ss_engine_last_error(const ss_engine* eng);
/* n_chunks chunks of n_fft samples (host or device memory, contiguous),
   sequence numbers first_seq, first_seq + 1, ...  Synchronous for the caller's
   buffer, like frontend::PingPongBuffer writers: when push returns, the samples
   have been copied out of `samples` (staged or DMA'd) and it may be reused. */
ss_status ss_engine_push(ss_engine* eng, const void* samples, int64_t n_chunks, uint64_t first_seq);
/* As ss_engine_push, but a DMA straight from a pinned / device `samples` is only
   queued: the caller keeps the buffer unchanged until ss_engine_push_fence
   returns (or the engine is finished / closed), and back-to-back pushes'
   copies overlap (an immutable source such as the runtime's MemorySource). */
ss_status ss_engine_push_async(ss_engine* eng, const void* samples, int64_t n_chunks, uint64_t first_seq);
/* Every copy out of the caller's buffers queued by ss_engine_push_async has
   finished. */
ss_status ss_engine_push_fence(ss_engine* eng);
/* Chunks [first_seq, last_seq) were lost upstream: their windows drop
   (frontend::PingPongBuffer::mark_lost_range). */
ss_status ss_engine_mark_lost(ss_engine* eng, uint64_t first_seq, uint64_t last_seq);
/* End of stream: an incomplete last window is discarded. */
ss_status ss_engine_finish(ss_engine* eng);
/* Next completed window in completion (= window) order.  wait_ms < 0 waits
   until a record is ready or the stream is finished and drained; *got = 1
   when rec/boxes/bin_boxes (each may be NULL, capacity cap) were filled.
   SS_ECUDA with *got = 1: that window's sensing faulted on the device; its
   record is consumed but rec/boxes hold no result (ss_engine_last_error). */
ss_status ss_engine_poll(ss_engine* eng, int wait_ms, ss_plot_record* rec, ss_box* boxes, ss_bin_box* bin_boxes,
                         int cap, int* got);
/* windows completed (handed to the GPU), windows dropped (overruns), rows
   retired (used + dropped + lost), windows in flight or awaiting poll */
ss_status ss_engine_stats(ss_engine* eng, uint64_t* completed, uint64_t* overruns, uint64_t* rows_retired,
                          uint64_t* pending);

/* ---- baseline detector -------------------------------------------------
   The reference's Searchlight-style comparison detector (baseline::
   baseline_detect, proj/src/baseline.cpp:103-176): dyadic
   mean-filter bank over the summed-area table of |x|^2, seeds where a kernel
   mean exceeds conv_threshold x floor x 10^(offset/10), greedy box growth,
   merge of overlapping boxes.  SAT and the kernel bank run on the GPU, the
   sequential greedy walk on the host; results are bit-identical. */
typedef struct {
    double conv_threshold;          /* 2.0 */
    double rate_change_threshold;   /* 0.5 */
    double noise_offset_db;         /* 3.0 */
    int max_kernel_rows;            /* 0 = plot height */
    int max_kernel_cols;            /* 0 = plot width */
} ss_baseline_cfg;

void ss_default_baseline_cfg(ss_baseline_cfg* cfg);
/* baseline::kernel_sizes (baseline.cpp:96-101): (kr, kc) pairs into sizes
   (2*cap ints).  Returns the count; -1 invalid input, -2 cap too small.
   Host only. */
int ss_baseline_kernel_sizes(int rows, int cols, const ss_baseline_cfg* cfg, int32_t* sizes, int cap);
/* baseline::baseline_detect on one rows x cols TF plot (host or device
   memory); boxes / bin_boxes (HOST, may be NULL) sorted by (t0, f0, t1, f1),
   at most cap kept, *n_boxes = true count. */
ss_status ss_baseline_detect(ss_ctx* ctx, const float* tf, int rows, int cols, uint64_t start_seq,
                             double sample_rate_hz, const ss_baseline_cfg* cfg, ss_box* boxes, ss_bin_box* bin_boxes,
                             int cap, int* n_boxes);

/* ---- test hooks -------------------------------------------------------- */
/* Device ports of glibc log10f (which=0) / powf(10, x) (which=1) over n
   DEVICE floats; variant: 1 FMA build, 0 SSE2 build, -1 host-matched. */
ss_status ss_test_libm(ss_ctx* ctx, const float* x, int64_t n, int which, int variant, float* out);
/* SSFFT-1 per-pass twiddle table for n_fft (HOST out, ss_fft_twiddle_count doubles2). */
int64_t ss_fft_twiddle_count(int n_fft);
ss_status ss_fft_twiddles(int n_fft, double* out_re_im);

#ifdef __cplusplus
}
#endif
#endif /* SPECSENSE_B200_H */
