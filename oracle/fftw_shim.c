/*
 * oracle/fftw_shim.c -- TEST INFRASTRUCTURE ONLY.  This is the CPU FFT the
 * oracle (the unmodified reference sources built under oracle/_ref, and the C
 * restatement oracle/restate.c) links in place of FFTW3, which is absent from
 * this image.  Nothing in the product imports or links it; tests, smoke() and
 * bench.py's cpu_baseline / --impl reference leg are its only users.
 *
 * Forward power-of-two transforms (the only kind the hot path issues:
 * proj/src/frontend.cpp:54-60 plans FFTW_FORWARD, n = 2^m >= 8, and executes at
 * :139) follow the "SSFFT-2" arithmetic specification written out in DESIGN.md
 * section 3.1 -- the same specification the device kernel
 * paper_2603_20481_b200/csrc/fft_mag.cu implements independently -- so TF
 * plots are bit-identical by construction:
 *
 *   * Stockham DIT autosort, passes of radix 16, then one pass of radix
 *     2^(m mod 4) when m mod 4 != 0 (N=8: a single radix-8 pass);
 *   * pass (Ns, R): butterfly j reads src[j + r*N/R], multiplies v[r] (r >= 1)
 *     by w_r unless Ns == 1, runs DFT_R, and writes
 *     dst[(j - j mod Ns)*R + j mod Ns + r*Ns]; w_1 = tw[(j mod Ns)*N/(Ns*R)]
 *     and w_2..w_15 come from a fixed product tree (w2 = w1 w1, w3 = w2 w1,
 *     w4 = w2 w2, w5..7 = w4 w1..3, w8 = w4 w4, w9..15 = w8 w1..7);
 *   * tw[e] = (cos(t), -sin(t)), t = (2*pi * e) / N, glibc double cos/sin;
 *   * cmul(a, w) = (fma(a.re, w.re, -(a.im*w.im)), fma(a.re, w.im, a.im*w.re));
 *   * DFT4 / DFT8 (even-odd of two DFT4) / DFT16 (4x4 with internal twiddles)
 *     exactly as coded below; this file is compiled with -ffp-contract=off so
 *     only the explicit fma() calls fuse.
 *
 * Everything else (backward transforms, non-power-of-two lengths) is only used
 * by signals::synthesize (proj/src/signals.cpp:83-95) to render seeded test
 * inputs: backward power-of-two = conj(FFT(conj x)); other lengths =
 * Bluestein over the power-of-two FFT.  FFT bit parity is not pinned by the
 * reference (its tests pin only a 1e-5 naive-DFT tolerance and Parseval 1e-6:
 * proj/tests/test_frontend.cpp:114-135), tests/test_oracle_fft.py pins this
 * shim against both and against numpy's pocketfft.
 */
#define _POSIX_C_SOURCE 200112L
#include "fftw3.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double re, im;
} cd;

#define SS_R2 0x1.6a09e667f3bcdp-1 /* sqrt(2)/2 */
#define SS_C1 0x1.d906bcf328d46p-1 /* cos(pi/8) */
#define SS_S1 0x1.87de2a6aea963p-2 /* sin(pi/8) */

static inline cd c_add(cd a, cd b) { cd r = {a.re + b.re, a.im + b.im}; return r; }
static inline cd c_sub(cd a, cd b) { cd r = {a.re - b.re, a.im - b.im}; return r; }
static inline cd c_mul(cd a, cd w) {
    const double t1 = a.im * w.im;
    const double t2 = a.im * w.re;
    cd r = {fma(a.re, w.re, -t1), fma(a.re, w.im, t2)};
    return r;
}
/* a * (-i) */
static inline cd c_mi(cd a) { cd r = {a.im, -a.re}; return r; }
/* a * W8 = a * (1 - i)/sqrt2 */
static inline cd c_w8(cd a) { cd r = {(a.re + a.im) * SS_R2, (a.im - a.re) * SS_R2}; return r; }
/* a * W8^3 = a * (-1 - i)/sqrt2 */
static inline cd c_w83(cd a) { cd r = {(a.im - a.re) * SS_R2, -((a.re + a.im) * SS_R2)}; return r; }

static void dft2(cd* v) {
    const cd a = v[0], b = v[1];
    v[0] = c_add(a, b);
    v[1] = c_sub(a, b);
}

/* in-place DFT4 of v[0], v[s], v[2s], v[3s] */
static void dft4s(cd* v, int s) {
    const cd t0 = c_add(v[0], v[2 * s]);
    const cd t1 = c_sub(v[0], v[2 * s]);
    const cd t2 = c_add(v[s], v[3 * s]);
    const cd t3 = c_sub(v[s], v[3 * s]);
    v[0] = c_add(t0, t2);
    v[2 * s] = c_sub(t0, t2);
    v[s].re = t1.re + t3.im;
    v[s].im = t1.im - t3.re;
    v[3 * s].re = t1.re - t3.im;
    v[3 * s].im = t1.im + t3.re;
}

static void dft8(cd* v) {
    cd e[4] = {v[0], v[2], v[4], v[6]};
    cd o[4] = {v[1], v[3], v[5], v[7]};
    dft4s(e, 1);
    dft4s(o, 1);
    o[1] = c_w8(o[1]);
    o[2] = c_mi(o[2]);
    o[3] = c_w83(o[3]);
    for (int k = 0; k < 4; ++k) {
        v[k] = c_add(e[k], o[k]);
        v[k + 4] = c_sub(e[k], o[k]);
    }
}

/* 4x4: DFT4 over n2 (stride 4) for each n1, twiddle W16^(n1*k2), DFT4 over n1. */
static void dft16(cd* v) {
    cd y[16]; /* y[n1*4 + k2] */
    for (int n1 = 0; n1 < 4; ++n1) {
        cd t[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
        dft4s(t, 1);
        for (int k2 = 0; k2 < 4; ++k2) y[n1 * 4 + k2] = t[k2];
    }
    const cd w1 = {SS_C1, -SS_S1};  /* W16^1 */
    const cd w3 = {SS_S1, -SS_C1};  /* W16^3 */
    const cd w9 = {-SS_C1, SS_S1};  /* W16^9 */
    /* n1 = 1: k2 = 1,2,3 -> W^1, W^2, W^3 */
    y[1 * 4 + 1] = c_mul(y[1 * 4 + 1], w1);
    y[1 * 4 + 2] = c_w8(y[1 * 4 + 2]);
    y[1 * 4 + 3] = c_mul(y[1 * 4 + 3], w3);
    /* n1 = 2: W^2, W^4, W^6 */
    y[2 * 4 + 1] = c_w8(y[2 * 4 + 1]);
    y[2 * 4 + 2] = c_mi(y[2 * 4 + 2]);
    y[2 * 4 + 3] = c_w83(y[2 * 4 + 3]);
    /* n1 = 3: W^3, W^6, W^9 */
    y[3 * 4 + 1] = c_mul(y[3 * 4 + 1], w3);
    y[3 * 4 + 2] = c_w83(y[3 * 4 + 2]);
    y[3 * 4 + 3] = c_mul(y[3 * 4 + 3], w9);
    for (int k2 = 0; k2 < 4; ++k2) {
        cd t[4] = {y[0 * 4 + k2], y[1 * 4 + k2], y[2 * 4 + k2], y[3 * 4 + k2]};
        dft4s(t, 1);
        for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = t[k1];
    }
}

static void dft_r(cd* v, int r) {
    switch (r) {
    case 2: dft2(v); break;
    case 4: dft4s(v, 1); break;
    case 8: dft8(v); break;
    case 16: dft16(v); break;
    default: abort();
    }
}

static int ilog2(int n) {
    int m = 0;
    while ((1 << m) < n) ++m;
    return m;
}

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* SSFFT-1 twiddle table: tw[e] = (cos t, -sin t), t = (2 pi e) / N. */
static cd* make_table(int n) {
    cd* tw = (cd*)malloc(sizeof(cd) * (size_t)n);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int e = 0; e < n; ++e) {
        const double t = (two_pi * (double)e) / (double)n;
        tw[e].re = cos(t);
        tw[e].im = -sin(t);
    }
    return tw;
}

#if defined(__AVX2__) && defined(__FMA__)
/* AVX2 form of the radix-16 pass: four butterflies per iteration, one per
   vector lane, every operation the scalar code's (IEEE per lane, the same
   explicit fma in cmul, no contraction), so the bits are identical; only the
   CPU baseline gets faster.  Lanes hold butterflies j, j+2, j+1, j+3 (the
   order unpacklo/hi produce from interleaved complex pairs). */
#include <immintrin.h>
typedef struct {
    __m256d re, im;
} cv;
static inline cv cv_add(cv a, cv b) { cv r = {_mm256_add_pd(a.re, b.re), _mm256_add_pd(a.im, b.im)}; return r; }
static inline cv cv_sub(cv a, cv b) { cv r = {_mm256_sub_pd(a.re, b.re), _mm256_sub_pd(a.im, b.im)}; return r; }
static inline cv cv_mul(cv a, cv w) {
    const __m256d t1 = _mm256_mul_pd(a.im, w.im);
    const __m256d t2 = _mm256_mul_pd(a.im, w.re);
    cv r = {_mm256_fmadd_pd(a.re, w.re, _mm256_sub_pd(_mm256_setzero_pd(), t1)), _mm256_fmadd_pd(a.re, w.im, t2)};
    return r;
}
static inline cv cv_mi(cv a) { cv r = {a.im, _mm256_sub_pd(_mm256_setzero_pd(), a.re)}; return r; }
static inline cv cv_w8(cv a) {
    const __m256d k = _mm256_set1_pd(SS_R2);
    cv r = {_mm256_mul_pd(_mm256_add_pd(a.re, a.im), k), _mm256_mul_pd(_mm256_sub_pd(a.im, a.re), k)};
    return r;
}
static inline cv cv_w83(cv a) {
    const __m256d k = _mm256_set1_pd(SS_R2);
    cv r = {_mm256_mul_pd(_mm256_sub_pd(a.im, a.re), k),
            _mm256_sub_pd(_mm256_setzero_pd(), _mm256_mul_pd(_mm256_add_pd(a.re, a.im), k))};
    return r;
}
static inline cv cv_set1(cd w) { cv r = {_mm256_set1_pd(w.re), _mm256_set1_pd(w.im)}; return r; }
static inline void dft4v(cv* t) {
    const cv t0 = cv_add(t[0], t[2]), t1 = cv_sub(t[0], t[2]);
    const cv t2 = cv_add(t[1], t[3]), t3 = cv_sub(t[1], t[3]);
    t[0] = cv_add(t0, t2);
    t[2] = cv_sub(t0, t2);
    t[1].re = _mm256_add_pd(t1.re, t3.im);
    t[1].im = _mm256_sub_pd(t1.im, t3.re);
    t[3].re = _mm256_sub_pd(t1.re, t3.im);
    t[3].im = _mm256_add_pd(t1.im, t3.re);
}
static void dft16v(cv* v) {
    cv y[16];
    for (int n1 = 0; n1 < 4; ++n1) {
        cv t[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
        dft4v(t);
        for (int k2 = 0; k2 < 4; ++k2) y[n1 * 4 + k2] = t[k2];
    }
    const cd w1 = {SS_C1, -SS_S1}, w3 = {SS_S1, -SS_C1}, w9 = {-SS_C1, SS_S1};
    y[5] = cv_mul(y[5], cv_set1(w1));
    y[6] = cv_w8(y[6]);
    y[7] = cv_mul(y[7], cv_set1(w3));
    y[9] = cv_w8(y[9]);
    y[10] = cv_mi(y[10]);
    y[11] = cv_w83(y[11]);
    y[13] = cv_mul(y[13], cv_set1(w3));
    y[14] = cv_w83(y[14]);
    y[15] = cv_mul(y[15], cv_set1(w9));
    for (int k2 = 0; k2 < 4; ++k2) {
        cv t[4] = {y[k2], y[4 + k2], y[8 + k2], y[12 + k2]};
        dft4v(t);
        for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = t[k1];
    }
}
/* one radix-16 Stockham pass (n/16 butterflies, a multiple of 4) */
static void pass16_avx(const cd* src, cd* dst, int n, int ns, const cd* tw, int step) {
    const int nr = n / 16;
    for (int j = 0; j < nr; j += 4) {
        cv v[16];
        for (int q = 0; q < 16; ++q) {
            const double* a = (const double*)(src + j + q * nr);
            const __m256d lo = _mm256_loadu_pd(a), hi = _mm256_loadu_pd(a + 4);
            v[q].re = _mm256_unpacklo_pd(lo, hi);  /* butterflies j, j+2, j+1, j+3 */
            v[q].im = _mm256_unpackhi_pd(lo, hi);
        }
        const int k = j % ns;
        if (ns > 1) {
            /* ns >= 16 here: the four butterflies share a block, k .. k+3 */
            const cd a0 = tw[(k + 0) * step], a1 = tw[(k + 1) * step], a2 = tw[(k + 2) * step], a3 = tw[(k + 3) * step];
            cv w[16];
            w[1].re = _mm256_set_pd(a3.re, a1.re, a2.re, a0.re);
            w[1].im = _mm256_set_pd(a3.im, a1.im, a2.im, a0.im);
            w[2] = cv_mul(w[1], w[1]);
            w[3] = cv_mul(w[2], w[1]);
            w[4] = cv_mul(w[2], w[2]);
            w[5] = cv_mul(w[4], w[1]);
            w[6] = cv_mul(w[4], w[2]);
            w[7] = cv_mul(w[4], w[3]);
            w[8] = cv_mul(w[4], w[4]);
            for (int q = 9; q < 16; ++q) w[q] = cv_mul(w[8], w[q - 8]);
            for (int q = 1; q < 16; ++q) v[q] = cv_mul(v[q], w[q]);
        }
        dft16v(v);
        if (ns > 1) {
            const int base = (j - k) * 16 + k;  /* four consecutive outputs per q */
            for (int q = 0; q < 16; ++q) {
                double* o = (double*)(dst + base + q * ns);
                _mm256_storeu_pd(o, _mm256_unpacklo_pd(v[q].re, v[q].im));
                _mm256_storeu_pd(o + 4, _mm256_unpackhi_pd(v[q].re, v[q].im));
            }
        } else {
            for (int q = 0; q < 16; ++q) {
                double re[4], im[4];
                _mm256_storeu_pd(re, v[q].re);
                _mm256_storeu_pd(im, v[q].im);
                static const int lane_of[4] = {0, 2, 1, 3};  /* butterfly j+i sits in lane lane_of[i] */
                for (int i = 0; i < 4; ++i) {
                    dst[(j + i) * 16 + q].re = re[lane_of[i]];
                    dst[(j + i) * 16 + q].im = im[lane_of[i]];
                }
            }
        }
    }
}
#define SSFFT_HAVE_AVX2 1
#endif

/* Forward power-of-two SSFFT-1; in and out may alias. */
static void ssfft_forward(int n, const cd* tw, const cd* in, cd* out, cd* scratch) {
    const int m = ilog2(n);
    int radices[8];
    int np = 0;
    if (n == 8) {
        radices[np++] = 8;
    } else {
        for (int i = 0; i < m / 4; ++i) radices[np++] = 16;
        if (m % 4) radices[np++] = 1 << (m % 4);
    }
    /* ping-pong between scratch buffers; the final pass lands in out */
    cd* bufa = scratch;
    cd* bufb = scratch + n;
    memcpy(bufa, in, sizeof(cd) * (size_t)n);
    cd* src = bufa;
    cd* dst = bufb;
    int ns = 1;
    for (int p = 0; p < np; ++p) {
        const int r = radices[p];
        const int nr = n / r;
        const int step = n / (ns * r);
#ifdef SSFFT_HAVE_AVX2
        if (r == 16 && nr % 4 == 0 && (ns == 1 || ns >= 16)) {
            pass16_avx(src, dst, n, ns, tw, step);
            ns *= r;
            cd* t = src;
            src = dst;
            dst = t;
            continue;
        }
#endif
        for (int j = 0; j < nr; ++j) {
            const int k = j % ns;
            cd v[16];
            for (int q = 0; q < r; ++q) v[q] = src[j + q * nr];
            if (ns > 1) {
                /* SSFFT-2: w1 = tw[k*step]; higher powers by a fixed product tree */
                cd w[16];
                w[1] = tw[k * step];
                if (r > 2) w[2] = c_mul(w[1], w[1]);
                if (r > 3) w[3] = c_mul(w[2], w[1]);
                if (r > 4) {
                    w[4] = c_mul(w[2], w[2]);
                    w[5] = c_mul(w[4], w[1]);
                    w[6] = c_mul(w[4], w[2]);
                    w[7] = c_mul(w[4], w[3]);
                }
                if (r > 8) {
                    w[8] = c_mul(w[4], w[4]);
                    for (int q = 9; q < 16; ++q) w[q] = c_mul(w[8], w[q - 8]);
                }
                for (int q = 1; q < r; ++q) v[q] = c_mul(v[q], w[q]);
            }
            dft_r(v, r);
            const int base = (j - k) * r + k;
            for (int q = 0; q < r; ++q) dst[base + q * ns] = v[q];
        }
        ns *= r;
        cd* t = src;
        src = dst;
        dst = t;
    }
    memcpy(out, src, sizeof(cd) * (size_t)n);
}

struct oracle_fftw_plan_s {
    int n;
    int sign;
    fftw_complex* in;
    fftw_complex* out;
    /* power-of-two state */
    int pow2;
    cd* tw;
    /* Bluestein state (non power of two) */
    int m;     /* convolution length */
    cd* mtw;   /* table for m */
    cd* chirp; /* c[k] = exp(sign * i * pi * k^2 / n) */
    cd* bfft;  /* FFT of the conjugate-chirp kernel */
};

fftw_complex* fftw_alloc_complex(size_t n) {
    void* p = NULL;
    if (posix_memalign(&p, 64, sizeof(fftw_complex) * (n ? n : 1)) != 0) return NULL;
    return (fftw_complex*)p;
}

void fftw_free(void* p) { free(p); }

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
    (void)flags;
    if (n < 1) return NULL;
    struct oracle_fftw_plan_s* p = (struct oracle_fftw_plan_s*)calloc(1, sizeof(*p));
    p->n = n;
    p->sign = sign;
    p->in = in;
    p->out = out;
    p->pow2 = is_pow2(n) && n >= 2;
    if (p->pow2) {
        if (n >= 8) {
            p->tw = make_table(n);
        }
        return p;
    }
    if (n == 1) return p;
    int m = 1;
    while (m < 2 * n - 1) m <<= 1;
    if (m < 8) m = 8;
    p->m = m;
    p->mtw = make_table(m);
    p->chirp = (cd*)malloc(sizeof(cd) * (size_t)n);
    const double pi = 3.14159265358979323846;
    const uint64_t two_n = 2u * (uint64_t)n;
    for (int k = 0; k < n; ++k) {
        const uint64_t kk = ((uint64_t)k * (uint64_t)k) % two_n;
        const double t = pi * (double)kk / (double)n;
        /* forward (sign -1): exp(-i pi k^2/n); backward: conjugate */
        p->chirp[k].re = cos(t);
        p->chirp[k].im = sign < 0 ? -sin(t) : sin(t);
    }
    cd* b = (cd*)calloc((size_t)m, sizeof(cd));
    for (int k = 0; k < n; ++k) {
        cd c = {p->chirp[k].re, -p->chirp[k].im};
        b[k] = c;
        if (k) b[m - k] = c;
    }
    p->bfft = (cd*)malloc(sizeof(cd) * (size_t)m);
    cd* scratch = (cd*)malloc(sizeof(cd) * 2 * (size_t)m);
    ssfft_forward(m, p->mtw, b, p->bfft, scratch);
    free(scratch);
    free(b);
    return p;
}

static void small_pow2(int n, int sign, const cd* in, cd* out) {
    /* n in {2, 4}: direct definitions, used only by synthesis */
    cd v[4];
    for (int i = 0; i < n; ++i) v[i] = in[i];
    if (sign > 0)
        for (int i = 0; i < n; ++i) v[i].im = -v[i].im;
    if (n == 2) dft2(v);
    else dft4s(v, 1);
    if (sign > 0)
        for (int i = 0; i < n; ++i) v[i].im = -v[i].im;
    for (int i = 0; i < n; ++i) out[i] = v[i];
}

/* per-thread scratch (2n complex), grown on demand: the reference calls
   fftw_execute_dft once per row, and a fresh 2n-element malloc per call is an
   mmap + page faults for n >= 4096 */
static _Thread_local cd* tls_scratch = NULL;
static _Thread_local size_t tls_cap = 0;
static cd* scratch_for(size_t count) {
    if (count > tls_cap) {
        free(tls_scratch);
        tls_scratch = (cd*)malloc(sizeof(cd) * count);
        tls_cap = tls_scratch ? count : 0;
    }
    return tls_scratch;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in_, fftw_complex* out_) {
    const int n = p->n;
    cd* in = (cd*)in_;
    cd* out = (cd*)out_;
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    if (p->pow2) {
        if (n < 8) {
            small_pow2(n, p->sign, in, out);
            return;
        }
        cd* scratch = scratch_for(2 * (size_t)n);
        if (p->sign < 0) {
            ssfft_forward(n, p->tw, in, out, scratch);
        } else {
            cd* tmp = (cd*)malloc(sizeof(cd) * (size_t)n);
            for (int i = 0; i < n; ++i) {
                tmp[i].re = in[i].re;
                tmp[i].im = -in[i].im;
            }
            ssfft_forward(n, p->tw, tmp, out, scratch);
            for (int i = 0; i < n; ++i) out[i].im = -out[i].im;
            free(tmp);
        }
        return;
    }
    /* Bluestein */
    const int m = p->m;
    cd* a = (cd*)calloc((size_t)m, sizeof(cd));
    cd* scratch = (cd*)malloc(sizeof(cd) * 2 * (size_t)m);
    for (int k = 0; k < n; ++k) a[k] = c_mul(in[k], p->chirp[k]);
    ssfft_forward(m, p->mtw, a, a, scratch);
    for (int k = 0; k < m; ++k) {
        cd t = c_mul(a[k], p->bfft[k]);
        a[k].re = t.re;
        a[k].im = -t.im; /* conj for inverse via forward */
    }
    ssfft_forward(m, p->mtw, a, a, scratch);
    const double inv_m = 1.0 / (double)m;
    for (int k = 0; k < n; ++k) {
        cd c = {a[k].re * inv_m, -a[k].im * inv_m};
        out[k] = c_mul(c, p->chirp[k]);
    }
    free(scratch);
    free(a);
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    free(p->tw);
    free(p->mtw);
    free(p->chirp);
    free(p->bfft);
    free(p);
}

/* Test hook: the SSFFT-1 twiddle table, so tests can check the device table
   the product builds is the same array of doubles. */
void oracle_ssfft_table(int n, double* out_re_im) {
    cd* tw = make_table(n);
    memcpy(out_re_im, tw, sizeof(cd) * (size_t)n);
    free(tw);
}
