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
