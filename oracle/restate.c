/*
 * oracle/restate.c -- TEST INFRASTRUCTURE ONLY (see restate.h).  Plain C,
 * compiled with -ffp-contract=off: the only fused multiply-adds are the
 * explicit fma() calls at the sites GCC contracts in the reference build
 * (-O3 -march=x86-64-v3/native; objdump -l of detector.o / frontend.o):
 * frontend.cpp:147, detector.cpp:105, 106, 112 (and :70, :179 where fusion
 * is provably bit-neutral).
 */
#include "restate.h"

#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_EVALIDATION (-1)
#define ORACLE_ECAPACITY (-7)

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* frontend.cpp:127-149 (fft_row) and 157-171 (make_plot), decode per
   frontend.cpp:376-385 (i16 * (1.0f/32768)). */
int oracle_tf_plot(const void* iq, int fmt, int n_fft, int rows, float* out) {
    if (n_fft < 8 || !is_pow2(n_fft) || rows < 0) return ORACLE_EVALIDATION;
    fftw_complex* in = fftw_alloc_complex((size_t)n_fft);
    fftw_complex* spec = fftw_alloc_complex((size_t)n_fft);
    fftw_plan plan = fftw_plan_dft_1d(n_fft, in, in, FFTW_FORWARD, FFTW_ESTIMATE);
    const int half = n_fft / 2;
    for (int r = 0; r < rows; ++r) {
        const size_t base = (size_t)r * (size_t)n_fft;
        if (fmt == 0) {
            const float* f = (const float*)iq + 2 * base;
            for (int i = 0; i < n_fft; ++i) {
                in[i][0] = (double)f[2 * i];
                in[i][1] = (double)f[2 * i + 1];
            }
        } else {
            const int16_t* s = (const int16_t*)iq + 2 * base;
            const float scale = 1.0f / 32768.0f;
            for (int i = 0; i < n_fft; ++i) {
                in[i][0] = (double)((float)s[2 * i] * scale);
                in[i][1] = (double)((float)s[2 * i + 1] * scale);
            }
        }
        fftw_execute_dft(plan, in, spec);
        float* o = out + base;
        for (int k = 0; k < n_fft; ++k) {
            const int src = k < half ? k + half : k - half;
            const double re = spec[src][0];
            const double im = spec[src][1];
            o[k] = (float)sqrt(fma(re, re, im * im));
        }
    }
    fftw_destroy_plan(plan);
    fftw_free(in);
    fftw_free(spec);
    return 0;
}

/* STFT extension (no reference oracle): frontend.cpp:127-171
   with a window multiply (double) before the transform and frames every `hop`
   samples.  window 0 = rectangular, 1 = periodic Hann 0.5*(1 - cos(2 pi n / N)). */
int oracle_stft_plot(const void* iq, int fmt, int n_fft, int hop, int window, int rows, float* out) {
    if (n_fft < 8 || !is_pow2(n_fft) || rows < 0 || hop < 1) return ORACLE_EVALIDATION;
    double* w = (double*)malloc(sizeof(double) * (size_t)n_fft);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int n = 0; n < n_fft; ++n)
        w[n] = window == 1 ? 0.5 * (1.0 - cos((two_pi * (double)n) / (double)n_fft)) : 1.0;
    fftw_complex* in = fftw_alloc_complex((size_t)n_fft);
    fftw_complex* spec = fftw_alloc_complex((size_t)n_fft);
    fftw_plan plan = fftw_plan_dft_1d(n_fft, in, in, FFTW_FORWARD, FFTW_ESTIMATE);
    const int half = n_fft / 2;
    for (int r = 0; r < rows; ++r) {
        const size_t base = (size_t)r * (size_t)hop;
        for (int i = 0; i < n_fft; ++i) {
            double re, im;
            if (fmt == 0) {
                const float* f = (const float*)iq + 2 * (base + (size_t)i);
                re = (double)f[0];
                im = (double)f[1];
            } else {
                const int16_t* q = (const int16_t*)iq + 2 * (base + (size_t)i);
                re = (double)((float)q[0] * (1.0f / 32768.0f));
                im = (double)((float)q[1] * (1.0f / 32768.0f));
            }
            in[i][0] = re * w[i];
            in[i][1] = im * w[i];
        }
        fftw_execute_dft(plan, in, spec);
        float* o = out + (size_t)r * (size_t)n_fft;
        for (int k = 0; k < n_fft; ++k) {
            const int src = k < half ? k + half : k - half;
            o[k] = (float)sqrt(fma(spec[src][0], spec[src][0], spec[src][1] * spec[src][1]));
        }
    }
    fftw_destroy_plan(plan);
    fftw_free(in);
    fftw_free(spec);
    free(w);
    return 0;
}

/* detector.cpp:170-184 */
int oracle_psd(const float* tf, int rows, int cols, int c0, int c1, float* out) {
    if (rows < 1 || cols < 1) return ORACLE_EVALIDATION;
    if (c0 < 0 || c1 > cols || c0 >= c1) return ORACLE_EVALIDATION;
    const double inv = 1.0 / rows;
    for (int k = c0; k < c1; ++k) {
        double acc = 0.0;
        for (int r = 0; r < rows; ++r) {
            const double v = (double)tf[(size_t)r * cols + k];
            acc = fma(v, v, acc); /* v*v is exact: fusion is bit-neutral */
        }
        out[k - c0] = (float)(acc * inv);
    }
    return 0;
}

static int check_savgol(int window, int order) {
    if (window < 5 || window % 2 == 0) return ORACLE_EVALIDATION;
    if (order < 1 || order >= window) return ORACLE_EVALIDATION;
    return 0;
}

/* detector.cpp:84-116 (solve_e0) + 120-142 (savgol_weights) */
int oracle_savgol_weights(int window, int order, double* w) {
    if (check_savgol(window, order)) return ORACLE_EVALIDATION;
    const int h = (window - 1) / 2;
    const int n = order + 1;
    double* g = (double*)calloc((size_t)n * n, sizeof(double));
    double* x = (double*)calloc((size_t)n, sizeof(double));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            double acc = 0.0;
            for (int j = -h; j <= h; ++j) acc += pow((double)j, (double)(a + b));
            g[a * n + b] = acc;
        }
    x[0] = 1.0;
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (fabs(g[r * n + col]) > fabs(g[piv * n + col])) piv = r;
        if (piv != col) {
            for (int c = 0; c < n; ++c) {
                const double t = g[col * n + c];
                g[col * n + c] = g[piv * n + c];
                g[piv * n + c] = t;
            }
            const double t = x[col];
            x[col] = x[piv];
            x[piv] = t;
        }
        const double d = g[col * n + col];
        if (d == 0.0) {
            free(g);
            free(x);
            return ORACLE_EVALIDATION;
        }
        for (int r = col + 1; r < n; ++r) {
            const double f = g[r * n + col] / d;
            if (f == 0.0) continue;
            for (int c = col; c < n; ++c) g[r * n + c] = fma(-f, g[col * n + c], g[r * n + c]);
            x[r] = fma(-f, x[col], x[r]);
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        double acc = x[r];
        for (int c = r + 1; c < n; ++c) acc = fma(-g[r * n + c], x[c], acc);
        x[r] = acc / g[r * n + r];
    }
    for (int j = -h; j <= h; ++j) {
        double c = 0.0, jp = 1.0;
        for (int a = 0; a < n; ++a) {
            c = c + x[a] * jp;
            jp = jp * j;
        }
        w[j + h] = c;
    }
    free(g);
    free(x);
    return 0;
}

static int mirror_index(int i, int n) {
    if (i < 0) return -i;
    if (i >= n) return 2 * (n - 1) - i;
    return i;
}

/* detector.cpp:192-208 */
int oracle_savgol_smooth(const float* v, int n, int window, int order, float* out) {
    if (check_savgol(window, order)) return ORACLE_EVALIDATION;
    if (n < window) return ORACLE_EVALIDATION;
    double* w = (double*)malloc(sizeof(double) * (size_t)window);
    oracle_savgol_weights(window, order, w);
    const int h = (window - 1) / 2;
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int j = -h; j <= h; ++j) acc = acc + w[j + h] * (double)v[mirror_index(i + j, n)];
        out[i] = (float)acc;
    }
    free(w);
    return 0;
}

/* detector.cpp:210-255 */
int oracle_floor_prune(const float* raw, int n, int window, int order, double margin_db,
                       float* smoothed, float* floor_out, float* thr_out, int* active) {
    float* db = (float*)malloc(sizeof(float) * (size_t)n);
    float* sdb = (float*)malloc(sizeof(float) * (size_t)n);
    for (int k = 0; k < n; ++k) db[k] = raw[k] > 0.0f ? 10.0f * log10f(raw[k]) : -3000.0f;
    int rc = oracle_savgol_smooth(db, n, window, order, sdb);
    if (rc) {
        free(db);
        free(sdb);
        return rc;
    }
    for (int k = 0; k < n; ++k) smoothed[k] = powf(10.0f, sdb[k] / 10.0f);
    const float* s = smoothed;
    int found = 0;
    float fl = INFINITY;
    int i = 1;
    while (i < n - 1) {
        int j = i;
        while (j + 1 < n && s[j + 1] == s[i]) ++j;
        const int left_up = s[i - 1] > s[i];
        const int right_up = j + 1 < n && s[j + 1] > s[i];
        if (left_up && right_up && s[i] < fl) {
            fl = s[i];
            found = 1;
        }
        i = j + 1;
    }
    if (!found) {
        fl = s[0];
        for (int k = 1; k < n; ++k)
            if (s[k] < fl) fl = s[k];
    }
    *floor_out = fl;
    const float thr = (float)((double)fl * pow(10.0, margin_db / 10.0));
    *thr_out = thr;
    int na = 0;
    for (int k = 0; k < n; ++k)
        if (raw[k] >= thr) active[na++] = k;
    free(db);
    free(sdb);
    return na;
}

/* detector.cpp:28-73: BinScale / bin_of / otsu_split / otsu_edge_value */
typedef struct {
    float lo, scale;
    int valid;
} bin_scale;

static bin_scale make_bin_scale(float lo, float hi) {
    bin_scale s;
    s.lo = lo;
    s.scale = 256.0f / (hi - lo);
    s.valid = hi > lo && isfinite(s.scale);
    return s;
}

static int bin_of(float v, bin_scale s) {
    const int b = (int)((v - s.lo) * s.scale);
    return b > 255 ? 255 : b;
}

static int otsu_split(const uint32_t* hist, uint64_t total) {
    double sum_all = 0.0;
    for (int i = 0; i < 256; ++i) sum_all += (double)i * hist[i];
    int best = 0;
    double best_var = -1.0;
    uint64_t w0 = 0;
    double sum0 = 0.0;
    for (int i = 0; i < 256; ++i) {
        w0 += hist[i];
        sum0 += (double)i * hist[i];
        const uint64_t w1 = total - w0;
        double var = 0.0;
        if (w0 > 0 && w1 > 0) {
            const double mu0 = sum0 / (double)w0;
            const double mu1 = (sum_all - sum0) / (double)w1;
            var = (double)w0 * (double)w1 * (mu0 - mu1) * (mu0 - mu1);
        }
        if (var > best_var) {
            best_var = var;
            best = i;
        }
    }
    return best;
}

static float otsu_edge_value(bin_scale s, float hi, int split) {
    return (float)((double)s.lo + ((double)split + 1.0) * ((double)hi - s.lo) / 256.0);
}

/* detector.cpp:257-271 */
int oracle_otsu(const float* v, int n, float* thr) {
    if (n < 1) return ORACLE_EVALIDATION;
    float lo = v[0], hi = v[0];
    for (int i = 0; i < n; ++i) {
        lo = (v[i] < lo) ? v[i] : lo;
        hi = (hi < v[i]) ? v[i] : hi;
    }
    const bin_scale s = make_bin_scale(lo, hi);
    if (!s.valid) {
        *thr = 0.0f;
        return 0;
    }
    uint32_t hist[256] = {0};
    for (int i = 0; i < n; ++i) ++hist[bin_of(v[i], s)];
    *thr = otsu_edge_value(s, hi, otsu_split(hist, (uint64_t)n));
    return 1;
}

/* detector.cpp:273-335 */
int oracle_binarize_columns(const float* tf, int rows, int cols, const int* active, int n_active,
                            int c0, int c1, uint8_t* mask) {
    if (c0 < 0 || c1 > cols || c0 > c1) return ORACLE_EVALIDATION;
    const int w = c1 - c0;
    if (w == 0) return 0;
    float* lo = (float*)malloc(sizeof(float) * (size_t)w);
    float* hi = (float*)malloc(sizeof(float) * (size_t)w);
    float* thr = (float*)malloc(sizeof(float) * (size_t)w);
    for (int k = 0; k < w; ++k) {
        lo[k] = INFINITY;
        hi[k] = -INFINITY;
        thr[k] = INFINITY;
    }
    for (int r = 0; r < rows; ++r) {
        const float* row = tf + (size_t)r * cols + c0;
        for (int k = 0; k < w; ++k) {
            lo[k] = (row[k] < lo[k]) ? row[k] : lo[k];
            hi[k] = (hi[k] < row[k]) ? row[k] : hi[k];
        }
    }
    uint32_t* hist = (uint32_t*)malloc(sizeof(uint32_t) * 256);
    for (int a = 0; a < n_active; ++a) {
        const int k = active[a];
        if (k < 0 || k >= cols) {
            free(lo); free(hi); free(thr); free(hist);
            return ORACLE_EVALIDATION;
        }
        if (k < c0 || k >= c1) continue;
        const bin_scale s = make_bin_scale(lo[k - c0], hi[k - c0]);
        if (!s.valid) continue;
        memset(hist, 0, sizeof(uint32_t) * 256);
        for (int r = 0; r < rows; ++r) ++hist[bin_of(tf[(size_t)r * cols + k], s)];
        thr[k - c0] = otsu_edge_value(s, hi[k - c0], otsu_split(hist, (uint64_t)rows));
    }
    for (int r = 0; r < rows; ++r) {
        const float* row = tf + (size_t)r * cols + c0;
        uint8_t* m = mask + (size_t)r * cols + c0;
        for (int k = 0; k < w; ++k) m[k] = row[k] > thr[k] ? 1 : 0;
    }
    free(lo);
    free(hi);
    free(thr);
    free(hist);
    return 0;
}

static void morph_basic(const uint8_t* src, int rows, int cols, int erode, int se_rows, int se_cols,
                        uint8_t* dst) {
    const int hr = se_rows / 2, hc = se_cols / 2;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            int acc = erode;
            for (int dr = -hr; dr <= hr; ++dr)
                for (int dc = -hc; dc <= hc; ++dc) {
                    const int rr = r + dr, cc = c + dc;
                    const int v = rr >= 0 && rr < rows && cc >= 0 && cc < cols &&
                                  src[(size_t)rr * cols + cc] != 0;
                    acc = erode ? (acc && v) : (acc || v);
                }
            dst[(size_t)r * cols + c] = acc ? 1 : 0;
        }
}

/* detector.cpp:345-480, by the direct definition (outside = background) */
int oracle_morphology(const uint8_t* src, int rows, int cols, int op, int se_rows, int se_cols,
                      uint8_t* dst) {
    if (se_rows < 1 || se_cols < 1 || se_rows % 2 == 0 || se_cols % 2 == 0) return ORACLE_EVALIDATION;
    if (rows < 1 || cols < 1) return ORACLE_EVALIDATION;
    if (op == 0 || op == 1) {
        morph_basic(src, rows, cols, op == 0, se_rows, se_cols, dst);
        return 0;
    }
    uint8_t* tmp = (uint8_t*)malloc((size_t)rows * cols);
    const int first_erodes = op == 2;
    morph_basic(src, rows, cols, first_erodes, se_rows, se_cols, tmp);
    morph_basic(tmp, rows, cols, !first_erodes, se_rows, se_cols, dst);
    free(tmp);
    return 0;
}

/* detector.cpp:482-492 */
int oracle_consolidate(const uint8_t* src, int rows, int cols, int along_time, uint8_t* dst) {
    uint8_t* a = (uint8_t*)malloc((size_t)rows * cols);
    int rc = oracle_morphology(src, rows, cols, 3, 3, 3, dst);
    if (!rc) rc = oracle_morphology(dst, rows, cols, 2, 3, 3, a);
    if (!rc) rc = oracle_morphology(a, rows, cols, 2, along_time ? 3 : 1, along_time ? 1 : 3, dst);
    free(a);
    return rc;
}

/* detector.cpp:505-620, restated as a row-major BFS flood fill
   (same contract as proj/tests/oracles.cpp:135-183). */
long long oracle_components(const uint8_t* mask, int rows, int cols, int min_area, int32_t* labels,
                            long long* extents, long long cap) {
    if (min_area < 1) return ORACLE_EVALIDATION;
    const size_t npx = (size_t)rows * cols;
    uint8_t* seen = (uint8_t*)calloc(npx ? npx : 1, 1);
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (npx ? npx : 1));
    if (labels) memset(labels, 0, sizeof(int32_t) * npx);
    long long count = 0;
    for (size_t p0 = 0; p0 < npx; ++p0) {
        if (!mask[p0] || seen[p0]) continue;
        size_t head = 0, tail = 0;
        queue[tail++] = (int32_t)p0;
        seen[p0] = 1;
        long long min_t = (long long)(p0 / cols), max_t = min_t;
        long long min_f = (long long)(p0 % cols), max_f = min_f;
        while (head < tail) {
            const int32_t p = queue[head++];
            const int r = p / cols, c = p % cols;
            if (r < min_t) min_t = r;
            if (r > max_t) max_t = r;
            if (c < min_f) min_f = c;
            if (c > max_f) max_f = c;
            const int nr[4] = {r - 1, r + 1, r, r};
            const int nc[4] = {c, c, c - 1, c + 1};
            for (int i = 0; i < 4; ++i) {
                if (nr[i] < 0 || nr[i] >= rows || nc[i] < 0 || nc[i] >= cols) continue;
                const size_t q = (size_t)nr[i] * cols + nc[i];
                if (!mask[q] || seen[q]) continue;
                seen[q] = 1;
                queue[tail++] = (int32_t)q;
            }
        }
        if ((long long)tail < min_area) continue;
        if (count >= cap) {
            free(seen);
            free(queue);
            return ORACLE_ECAPACITY;
        }
        long long* e = extents + 5 * count;
        e[0] = min_t;
        e[1] = max_t;
        e[2] = min_f;
        e[3] = max_f;
        e[4] = (long long)tail;
        ++count;
        if (labels)
            for (size_t i = 0; i < tail; ++i) labels[queue[i]] = (int32_t)count;
    }
    free(seen);
    free(queue);
    return count;
}

/* detector.cpp:637-670 (+ 622-635 box conversion) */
long long oracle_detect(const float* tf, int rows, int cols, uint64_t start_seq, double fs,
                        int window, int order, double margin_db, int min_area, int along_time,
                        float* raw, float* smoothed, float* floor_thr, int* active, int* n_active,
                        double* boxes, int* bin_boxes, long long cap) {
    if (check_savgol(window, order) || window > cols || margin_db < 0.0 || min_area < 1)
        return ORACLE_EVALIDATION;
    if (rows < 1 || cols < 1) return ORACLE_EVALIDATION;
    int rc = oracle_psd(tf, rows, cols, 0, cols, raw);
    if (rc) return rc;
    const int na = oracle_floor_prune(raw, cols, window, order, margin_db, smoothed, &floor_thr[0],
                                      &floor_thr[1], active);
    if (na < 0) return na;
    *n_active = na;
    const size_t npx = (size_t)rows * cols;
    uint8_t* m = (uint8_t*)calloc(npx, 1);
    uint8_t* c = (uint8_t*)malloc(npx);
    oracle_binarize_columns(tf, rows, cols, active, na, 0, cols, m);
    oracle_consolidate(m, rows, cols, along_time, c);
    long long* ext = (long long*)malloc(sizeof(long long) * 5 * (size_t)(cap > 0 ? cap : 1));
    const long long n = oracle_components(c, rows, cols, min_area, NULL, ext, cap);
    if (n >= 0) {
        const double dt = (double)cols / fs;
        const double df = fs / (double)cols;
        for (long long i = 0; i < n; ++i) {
            const int t0 = (int)ext[5 * i + 0], t1 = (int)ext[5 * i + 1] + 1;
            const int f0 = (int)ext[5 * i + 2], f1 = (int)ext[5 * i + 3] + 1;
            bin_boxes[4 * i + 0] = t0;
            bin_boxes[4 * i + 1] = t1;
            bin_boxes[4 * i + 2] = f0;
            bin_boxes[4 * i + 3] = f1;
            boxes[4 * i + 0] = (double)(f0 - cols / 2) * df;
            boxes[4 * i + 1] = (double)(f1 - cols / 2) * df;
            boxes[4 * i + 2] = ((double)start_seq + t0) * dt;
            boxes[4 * i + 3] = ((double)start_seq + t1) * dt;
        }
    }
    free(m);
    free(c);
    free(ext);
    return n;
}
