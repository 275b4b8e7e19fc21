/*
 * oracle/restate.h -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's hot path (proj/src/frontend.cpp:127-183, proj/src/detector.cpp),
 * used by tests/, smoke() and bench.py's cpu_baseline leg as the checker.  The
 * product never links it.  Each function cites the reference lines it follows;
 * tests/test_oracle_restate.py pins it bit-for-bit against the reference
 * itself (oracle/_ref/libspecsense_ref.so) and the golden fixtures.
 */
#ifndef ORACLE_RESTATE_H
#define ORACLE_RESTATE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* frontend::fft_row / make_plot (frontend.cpp:127-171). fmt 0 = f32 IQ, 1 = i16. */
int oracle_tf_plot(const void* iq, int fmt, int n_fft, int rows, float* out);

/* STFT extension: window (0 rect, 1 periodic Hann) and frame step `hop`. */
int oracle_stft_plot(const void* iq, int fmt, int n_fft, int hop, int window, int rows, float* out);

/* detector::estimate_psd_into (detector.cpp:170-184). */
int oracle_psd(const float* tf, int rows, int cols, int c0, int c1, float* out);

/* detector.cpp:84-142 (solve_e0 + savgol_weights), FMA at :105,:106,:112. */
int oracle_savgol_weights(int window, int order, double* w);

/* detector::savgol_smooth (detector.cpp:192-208). */
int oracle_savgol_smooth(const float* v, int n, int window, int order, float* out);

/* detector::smooth_and_floor + prune_columns (detector.cpp:210-255).
   Returns the active-column count. */
int oracle_floor_prune(const float* raw, int n, int window, int order, double margin_db,
                       float* smoothed, float* floor_out, float* thr_out, int* active);

/* detector::otsu_threshold (detector.cpp:257-271). Returns valid. */
int oracle_otsu(const float* v, int n, float* thr);

/* detector::binarize_columns (detector.cpp:273-335). mask is uint8 rows x cols. */
int oracle_binarize_columns(const float* tf, int rows, int cols, const int* active, int n_active,
                            int c0, int c1, uint8_t* mask);

/* detector::morphology (detector.cpp:345-480) by direct definition:
   out-of-image = background for erode and dilate. op 0 erode, 1 dilate,
   2 open, 3 close. */
int oracle_morphology(const uint8_t* src, int rows, int cols, int op, int se_rows, int se_cols,
                      uint8_t* dst);

/* detector::consolidate (detector.cpp:482-492). */
int oracle_consolidate(const uint8_t* src, int rows, int cols, int along_time, uint8_t* dst);

/* detector::label_components (detector.cpp:505-620): 4-connected, area filter
   before numbering, ids dense in first-pixel order.  extents: 5 int64 per
   component (min_t, max_t, min_f, max_f, area).  labels (int32 rows*cols) may
   be NULL.  Returns the component count, or -7 when cap is too small. */
long long oracle_components(const uint8_t* mask, int rows, int cols, int min_area, int32_t* labels,
                            long long* extents, long long cap);

/* detector::detect (detector.cpp:637-670).  boxes: 4 doubles per box
   (f0, f1, t0, t1); bin_boxes: 4 ints (t0, t1, f0, f1). */
long long oracle_detect(const float* tf, int rows, int cols, uint64_t start_seq, double fs,
                        int window, int order, double margin_db, int min_area, int along_time,
                        float* raw, float* smoothed, float* floor_thr, int* active, int* n_active,
                        double* boxes, int* bin_boxes, long long cap);

#ifdef __cplusplus
}
#endif
#endif
