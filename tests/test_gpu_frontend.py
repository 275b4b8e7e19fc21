"""GPU parity: K1 FFT-magnitude TF plots vs the reference's make_plots / fft_row
(proj/src/frontend.cpp:127-183) built as the oracle.  Bit-exact (== on fp32)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand_iq(rng, n, scale=1.0):
    return ((rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)) * scale).astype(np.complex64)


@pytest.mark.parametrize("n_fft", [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192])
def test_tf_plot_bit_exact_all_sizes(ss, ref, n_fft):
    rng = np.random.default_rng(n_fft)
    rows = max(3, min(97, (1 << 18) // n_fft))
    x = _rand_iq(rng, rows * n_fft * 2 + 5)   # two plots + a partial tail (dropped)
    got = ss.make_plots(x, 1e6, n_fft, rows)
    exp = ref.make_plots(x, 1e6, n_fft, rows)
    assert got.shape == exp.shape == (2, rows, n_fft)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("n_fft", [1024, 4096])
def test_tf_plot_int16_bit_exact(ss, ref, n_fft):
    """I16 decode: raw * (1/32768) (frontend.cpp:376-385), then the same FFT."""
    rng = np.random.default_rng(7 + n_fft)
    rows = 40
    raw = rng.integers(-32768, 32768, size=2 * rows * n_fft, dtype=np.int16)
    got = ss.make_plots(raw, 1e6, n_fft, rows, fmt=1)
    as_f32 = (raw.astype(np.float32) * np.float32(1.0 / 32768.0)).view(np.complex64)
    exp = ref.make_plots(as_f32, 1e6, n_fft, rows)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_tf_plot_dynamic_range(ss, ref):
    """Huge / tiny / zero inputs exercise the exact sqrt fallback paths."""
    rng = np.random.default_rng(3)
    n_fft, rows = 1024, 16
    x = _rand_iq(rng, rows * n_fft)
    x[: n_fft] = 0                       # all-zero row
    x[n_fft: 2 * n_fft] = 0.5 - 0.5j      # constant row (energy in the DC bin)
    x[2 * n_fft: 3 * n_fft] *= np.float32(1e30)
    x[3 * n_fft: 4 * n_fft] *= np.float32(1e-30)
    x[4 * n_fft: 5 * n_fft] = 0
    x[4 * n_fft + 17] = 1e-38 + 0j        # subnormal-range magnitudes
    got = ss.make_plots(x, 1e6, n_fft, rows)
    exp = ref.make_plots(x, 1e6, n_fft, rows)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    assert np.all(got[0, 0] == 0)


def test_fft_row_contracts(ss, ref):
    """proj/tests/test_frontend.cpp:97-144: zero, constant, naive DFT 1e-5, Parseval 1e-6."""
    z = ss.fft_row(np.zeros(64, np.complex64))
    assert np.all(z == 0)
    c = ss.fft_row(np.full(64, 0.5 - 0.5j, np.complex64))
    assert c[32] == pytest.approx(64 * abs(0.5 - 0.5j), rel=1e-6)
    rng = np.random.default_rng(42)
    x = _rand_iq(rng, 128)
    row = ss.fft_row(x)
    naive = np.abs(np.fft.fftshift(np.fft.fft(x.astype(np.complex128))))
    assert np.allclose(row, naive, rtol=1e-5)
    for n in (256, 1024):
        x = _rand_iq(rng, n)
        row = ss.fft_row(x).astype(np.float64)
        e = n * np.sum(np.abs(x.astype(np.complex128)) ** 2)
        assert abs(np.sum(row * row) - e) / e < 1e-6
    with pytest.raises(ss.ValidationError):
        ss.fft_row(np.zeros(100, np.complex64))


def test_make_plots_start_seq_and_tail(ss, ref):
    """12 full chunks + partial tail -> 2 plots of 5 rows (test_frontend.cpp:146-179)."""
    rng = np.random.default_rng(11)
    x = _rand_iq(rng, 12 * 32 + 17)
    got = ss.make_plots(x, 1e6, 32, 5)
    assert got.shape == (2, 5, 32)
    for p in range(2):
        for r in range(5):
            at = (p * 5 + r) * 32
            assert np.array_equal(got[p, r], ref.fft_row(x[at: at + 32]))


def test_validation(ss):
    with pytest.raises(ss.ValidationError):
        ss.make_plots(np.zeros(100, np.complex64), 1e6, 1000, 5)
    with pytest.raises(ss.ValidationError):
        ss.make_plots(np.zeros(100, np.complex64), 0.0, 16, 5)
    with pytest.raises(ss.ValidationError):
        ss.make_plots(np.zeros(100, np.complex64), 1e6, 16, 0)


@pytest.mark.parametrize("n_fft,hop,window", [(1024, 512, 1), (4096, 2048, 1), (256, 64, 1), (1024, 1024, 1),
                                              (512, 256, 0), (8192, 4096, 1)])
def test_stft_extension_bit_exact(ss, ora, n_fft, hop, window):
    """STFT extension (config 5 as written: Hann, 50 % overlap) vs the oracle's
    restatement (frontend path + window multiply + hop); no reference oracle."""
    rng = np.random.default_rng(n_fft + hop)
    rows = max(3, min(90, (1 << 18) // n_fft))
    n = (2 * rows - 1) * hop + n_fft + 7
    x = _rand_iq(rng, n)
    got = ss.stft_plots(x, 1e6, n_fft, hop, window, rows)
    assert got.shape == (2, rows, n_fft)
    exp = ora.stft_plot(x, n_fft, hop, window, 2 * rows).reshape(2, rows, n_fft)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_stft_rect_equals_make_plots(ss, ref):
    rng = np.random.default_rng(9)
    x = _rand_iq(rng, 40 * 1024)
    assert np.array_equal(ss.stft_plots(x, 1e6, 1024, 1024, 0, 20), ref.make_plots(x, 1e6, 1024, 20))


def test_stft_int16(ss, ora):
    rng = np.random.default_rng(10)
    raw = rng.integers(-32768, 32768, size=2 * (39 * 512 + 1024), dtype=np.int16)
    got = ss.stft_plots(raw, 1e6, 1024, 512, 1, 20, fmt=1)
    exp = ora.stft_plot(raw, 1024, 512, 1, 40).reshape(2, 20, 1024)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("n_fft,rows", [(16384, 6), (32768, 3), (65536, 2), (262144, 1)])
def test_large_fft_bit_exact(ss, ref, n_fft, rows):
    """n_fft beyond one CTA's shared memory: the global-memory SSFFT-2 pass chain
    (fft_mag.cu, large N) against the reference's make_plots."""
    rng = np.random.default_rng(n_fft)
    x = _rand_iq(rng, 2 * rows * n_fft + 3)
    got = ss.make_plots(x, 1e6, n_fft, rows)
    exp = ref.make_plots(x, 1e6, n_fft, rows)
    assert got.shape == exp.shape == (2, rows, n_fft)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_large_fft_int16_and_stft(ss, ref, ora):
    rng = np.random.default_rng(5)
    n_fft = 16384
    raw = rng.integers(-32768, 32768, size=2 * 4 * n_fft, dtype=np.int16)
    got = ss.make_plots(raw, 1e6, n_fft, 2, fmt=1)
    as_f32 = (raw.astype(np.float32) * np.float32(1 / 32768)).view(np.complex64)
    assert np.array_equal(got.view(np.uint32), ref.make_plots(as_f32, 1e6, n_fft, 2).view(np.uint32))
    x = _rand_iq(rng, 9 * 8192 + n_fft)
    got = ss.stft_plots(x, 1e6, n_fft, 8192, 1, 5)
    exp = ora.stft_plot(x, n_fft, 8192, 1, 10).reshape(2, 5, n_fft)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def _midpoint_cases(seed=11, n_mid=3000, span=13200):
    """Float pairs (a, b) whose magnitude sqrt(a^2 + b^2) lies within `span`
    double ulps of a float rounding midpoint, on both sides: a = the float half
    an ulp below the midpoint m, b scanned ulp by ulp around sqrt(m^2 - a^2)
    (one float ulp of b moves the magnitude by ~45 double ulps)."""
    rng = np.random.default_rng(seed)
    mant = rng.integers(1 << 23, 1 << 24, n_mid).astype(np.float64)
    expo = rng.choice(np.array([-60, -20, -3, 0, 1, 7, 30, 60]), n_mid).astype(np.float64)
    hu = np.ldexp(0.5, (expo - 23).astype(np.int64))           # half a float ulp
    m = np.ldexp(mant, (expo - 23).astype(np.int64)) + hu       # midpoint (25 significant bits)
    a = (m - hu).astype(np.float32)
    b0 = np.sqrt(hu * (2.0 * m - hu)).astype(np.float32)
    k = np.arange(-320, 321, dtype=np.int32)
    bb = (b0.view(np.int32)[:, None] + k[None, :]).view(np.float32)   # b0 +- k float ulps
    aa = np.broadcast_to(a[:, None], bb.shape)
    a64, b64 = aa.astype(np.float64), bb.astype(np.float64)
    q = a64 * a64 + b64 * b64                 # both squares exact: one rounding, = fma(re, re, im*im)
    s = np.sqrt(q)
    dist = (s.view(np.uint64) & np.uint64(0x1FFFFFFF)).astype(np.int64) - (1 << 28)
    keep = np.abs(dist) <= span
    return aa[keep], bb[keep], s[keep].astype(np.float32), dist[keep]


def test_magnitudes_around_float_midpoints(ss, ref):
    """K1's magnitude rounds a one-step Newton square root to float and redoes,
    with the IEEE square root, the points whose estimate lies in [-12288, +4]
    double ulps of a float rounding midpoint (fft_mag.cu: mags).  An impulse
    x[0] = a + ib transforms to X[k] = a + ib in every bin (n_fft = 8), so
    |X| = sqrt(a^2 + b^2) for chosen floats: ~1.7M magnitudes within 13,200 ulps
    of a midpoint, both sides, window edges included, against numpy's correctly
    rounded sqrt and against the reference.  (A build with a 1,024-ulp window
    fails this test; the proven 12,288-ulp window passes.)"""
    a, b, want, dist = _midpoint_cases()
    assert a.size > 500_000
    # the sample brackets the window: inside, at its edges, and just outside
    for lo, hi in [(-12288, 4), (-12400, -12200), (-13200, -12300), (-8, 16), (100, 13200)]:
        assert np.count_nonzero((dist >= lo) & (dist <= hi)) > 500, (lo, hi)
    n = a.size
    x = np.zeros((n, 8), np.complex64)
    x[:, 0] = a + 1j * b
    got = ss.make_plots(x.reshape(-1), 1e6, 8, n)[0]
    assert np.array_equal(got.view(np.uint32), np.broadcast_to(want.view(np.uint32)[:, None], got.shape))
    exp = ref.make_plots(x.reshape(-1), 1e6, 8, n)[0]
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
