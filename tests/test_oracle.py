"""CPU tests of the oracle itself (no GPU): the C restatement (oracle/restate.c)
against the reference built from its own sources (oracle/_ref), the FFTW-API
shim against independent FFTs and the reference's FFT contracts, and both
against the committed golden fixtures."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from _masks import burst_plot, random_blob_mask, random_mask, random_plot
from paper_2603_20481_b200 import signals

GOLD = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- FFT shim

@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192])
def test_shim_fft_matches_numpy_fp32(ref, n):
    """Any fp64-accurate FFT rounds to the same fp32 magnitudes."""
    rng = np.random.default_rng(n)
    bad = 0
    for _ in range(8):
        x = (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(np.complex64)
        exp = np.abs(np.fft.fftshift(np.fft.fft(x.astype(np.complex128)))).astype(np.float32)
        bad += int(np.sum(ref.fft_row(x) != exp))
    assert bad == 0


@pytest.mark.parametrize("capture", [0, 1])
def test_shim_full_c5r_plot_matches_numpy_fp64(ref, capture):
    """Independent pin of the FFT arithmetic on a whole bench-sized plot: one
    100 ms config-5 capture rendered by the reference's signals::synthesize,
    made into its 2441 x 4096 TF plot by the reference's make_plots (the SSFFT-2
    shim, which K1 matches bit for bit), against numpy's pocketfft in fp64
    rounded to fp32: 0 mismatches over 9,998,336 magnitudes."""
    iq, _ = ref.synthesize(signals.scenario_json(signals.c5_scenario(capture)))
    tf = ref.make_plots(iq, 100e6, 4096, 2441)[0]
    x = iq[: 2441 * 4096].reshape(2441, 4096).astype(np.complex128)
    exp = np.abs(np.fft.fftshift(np.fft.fft(x, axis=1), axes=1)).astype(np.float32)
    assert int(np.sum(exp != tf)) == 0


def test_shim_fft_contracts(ref):
    """proj/tests/test_frontend.cpp:97-135: zero, constant, naive DFT 1e-5, Parseval 1e-6."""
    assert np.all(ref.fft_row(np.zeros(64, np.complex64)) == 0)
    c = ref.fft_row(np.full(64, 0.5 - 0.5j, np.complex64))
    assert c[32] == pytest.approx(64 * abs(0.5 - 0.5j), rel=1e-6)
    assert np.all(np.delete(c, 32) < c[32] * 1e-5)
    rng = np.random.default_rng(42)
    x = (rng.uniform(-1, 1, 128) + 1j * rng.uniform(-1, 1, 128)).astype(np.complex64)
    n = np.arange(128)
    naive = np.abs(np.exp(-2j * np.pi * np.outer(n, n) / 128) @ x.astype(np.complex128))
    assert np.allclose(ref.fft_row(x), np.fft.fftshift(naive), rtol=1e-5)
    for size in (256, 1024):
        x = (rng.uniform(-1, 1, size) + 1j * rng.uniform(-1, 1, size)).astype(np.complex64)
        row = ref.fft_row(x).astype(np.float64)
        e = size * np.sum(np.abs(x.astype(np.complex128)) ** 2)
        assert abs(np.sum(row * row) - e) / e < 1e-6


def test_restated_tf_plot_equals_reference(ref, ora):
    rng = np.random.default_rng(5)
    for n_fft, rows in [(8, 11), (256, 40), (1024, 20), (4096, 6)]:
        x = (rng.normal(size=rows * n_fft) + 1j * rng.normal(size=rows * n_fft)).astype(np.complex64)
        assert np.array_equal(ora.tf_plot(x, n_fft, rows), ref.make_plots(x, 1e6, n_fft, rows)[0])
    raw = rng.integers(-32768, 32768, size=2 * 16 * 1024, dtype=np.int16)
    as_f = (raw.astype(np.float32) * np.float32(1 / 32768)).view(np.complex64)
    assert np.array_equal(ora.tf_plot(raw, 1024, 16), ref.make_plots(as_f, 1e6, 1024, 16)[0])


def test_shim_twiddle_table(ora):
    t = ora.ssfft_table(4096)
    e = np.arange(4096)
    th = 2 * np.pi * e / 4096
    assert np.allclose(t[:, 0], np.cos(th), atol=1e-15) and np.allclose(t[:, 1], -np.sin(th), atol=1e-15)


# ---------------------------------------------------------------- detector stages

def test_restated_psd(ref, ora):
    rng = np.random.default_rng(17)
    for rows, cols in [(64, 128), (2441, 40), (1, 7)]:
        tf = random_plot(rng, rows, cols)
        assert np.array_equal(ora.psd(tf), ref.estimate_psd(tf))
    tf = random_plot(rng, 32, 40)
    assert np.array_equal(ora.psd(tf, 7, 18), ref.estimate_psd(tf, 7, 18))


@pytest.mark.parametrize("window,order", [(5, 2), (7, 3), (9, 4), (31, 3), (5, 1), (21, 6), (51, 4)])
def test_restated_savgol(ref, ora, window, order):
    rng = np.random.default_rng(23 + window)
    v = rng.uniform(-10, 10, 300).astype(np.float32)
    assert np.array_equal(ora.savgol_smooth(v, window, order), ref.savgol_smooth(v, window, order))


def test_savgol_polynomial_and_least_squares(ora):
    """test_detector.cpp:122-166: matches a per-window least-squares fit; polynomials pass."""
    v = np.array([3.0, 1.5, 4.0, 1.0, 5.0, 9.0, 2.0, 6.0, 5.5], np.float32)
    got = ora.savgol_smooth(v, 5, 2)
    idx = lambda i: -i if i < 0 else (2 * 8 - i if i > 8 else i)  # noqa: E731
    exp = []
    for i in range(9):
        xs = np.arange(-2, 3)
        ys = np.array([v[idx(i + k)] for k in xs], np.float64)
        exp.append(np.polyval(np.polyfit(xs, ys, 2), 0.0))
    assert np.allclose(got, exp, rtol=1e-5)
    x = np.arange(32) * 0.25
    poly = (1.0 + 0.5 * x - 0.125 * x * x).astype(np.float32)
    assert np.allclose(ora.savgol_smooth(poly, 7, 2)[3:-3], poly[3:-3], rtol=1e-5)


def test_restated_floor_prune(ref, ora):
    rng = np.random.default_rng(31)
    cases = [np.full(32, 2.0, np.float32), np.zeros(64, np.float32),
             np.array([1 + abs(i - 16) * 0.5 for i in range(33)], np.float32),
             (rng.exponential(1.0, 4096) * 4096).astype(np.float32)]
    for raw in cases:
        for margin in (3.0, 0.0, 6.0):
            w, o = (31, 3) if len(raw) >= 31 else (5, 2)
            a = ora.floor_prune(raw, w, o, margin)
            b = ref.floor_prune(raw, w, o, margin)
            assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]
            assert np.array_equal(a[3], b[3])


def test_prune_margin_monotone(ref):
    """test_detector.cpp:236-247: raising the margin never adds active columns."""
    rng = np.random.default_rng(31)
    for _ in range(20):
        raw = rng.uniform(0.5, 4, 64).astype(np.float32)
        low = ref.floor_prune(raw, 7, 2, 1.0)[3]
        high = ref.floor_prune(raw, 7, 2, 4.0)[3]
        assert set(high) <= set(low)


def test_restated_otsu(ref, ora):
    rng = np.random.default_rng(41)
    for trial in range(300):
        if trial % 3 == 0:
            v = rng.random(200)
        elif trial % 3 == 1:
            v = np.abs(rng.normal(2.0, 0.7, 200))
        else:
            v = np.where(np.arange(200) % 4 == 0, 5 + rng.random(200), rng.random(200))
        v = v.astype(np.float32)
        assert ora.otsu(v) == ref.otsu_threshold(v)
    assert ref.otsu_threshold(np.full(100, 3.0, np.float32))[0] is False


def test_restated_binarize(ref, ora):
    rng = np.random.default_rng(47)
    for rows, cols in [(40, 24), (300, 96), (7, 1)]:
        tf = random_plot(rng, rows, cols)
        tf[:, min(5, cols - 1)] = 1.5
        act = np.sort(rng.choice(cols, size=max(1, cols // 2), replace=False)).astype(np.int32)
        assert np.array_equal(ora.binarize_columns(tf, act), ref.binarize_columns(tf, act))


def test_restated_morphology(ref, ora):
    rng = np.random.default_rng(61)
    for trial in range(30):
        m = random_mask(rng, 14, 18, 0.4) if trial % 2 else random_blob_mask(rng, 20, 20)
        for se in [(3, 3), (1, 3), (3, 1), (5, 3)]:
            for op in range(4):
                assert np.array_equal(ora.morphology(m, op, se), ref.morphology_cols(m, op, se))


def test_morphology_algebra(ref):
    """test_detector.cpp:370-394: idempotence and erode/dilate duality."""
    rng = np.random.default_rng(67)
    for _ in range(30):
        m = random_blob_mask(rng, 20, 20)
        for op in (2, 3):
            once = ref.morphology_cols(m, op, (3, 3))
            assert np.array_equal(ref.morphology_cols(once, op, (3, 3)), once)
        m = random_mask(rng, 12, 16, 0.35)
        pad = np.pad(m, 2)
        dual = 1 - ref.morphology_cols(1 - pad, 0, (3, 3))
        assert np.array_equal(dual[2:-2, 2:-2], ref.morphology_cols(m, 1, (3, 3)))


@pytest.mark.parametrize("along_time", [False, True])
def test_restated_consolidate(ref, ora, along_time):
    rng = np.random.default_rng(79)
    for _ in range(30):
        m = random_blob_mask(rng, 22, 26)
        assert np.array_equal(ora.consolidate(m, along_time), ref.consolidate(m, along_time))


def test_consolidate_sliced_invariance(ref):
    """runtime::consolidate_sliced equals consolidate for any slab count
    (proj/tests/test_runtime.cpp:150-162) -- the slab contract our single-pass
    fused morphology replaces."""
    rng = np.random.default_rng(19)
    m = random_blob_mask(rng, 64, 200)
    whole = ref.consolidate(m)
    for slabs in (1, 2, 3, 7, 16):
        assert np.array_equal(ref.consolidate_sliced(m, slabs), whole)


def test_restated_components(ref, ora):
    rng = np.random.default_rng(83)
    for trial in range(60):
        m = random_mask(rng, 18, 22, 0.45) if trial % 2 == 0 else random_blob_mask(rng, 18, 22)
        area = trial % 3 + 1
        e1, l1 = ora.components(m, area)
        e2, l2 = ref.label_components(m, area)
        assert np.array_equal(e1, e2) and np.array_equal(l1, l2)


def test_restated_detect(ref, ora):
    rng = np.random.default_rng(2024)
    for rows, cols in [(128, 256), (300, 512)]:
        tf = burst_plot(rng, rows, cols)
        a = ora.detect(tf, start_seq=3, fs=2e6)
        b = ref.detect(tf, start_seq=3, fs=2e6)
        for k in a:
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


# ---------------------------------------------------------------- golden fixtures

def test_golden_fft_rows(ref, ora):
    g = np.load(GOLD / "fft_rows.npz")
    for n in [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]:
        x, y = g[f"x{n}"], g[f"y{n}"]
        assert np.array_equal(ref.fft_row(x), y)
        assert np.array_equal(ora.tf_plot(x, n, 1)[0], y)


def test_golden_masks(ref, ora):
    g = np.load(GOLD / "masks.npz")
    for i in range(6):
        m = g[f"m{i}"]
        assert np.array_equal(ref.consolidate(m, False), g[f"cons{i}"])
        assert np.array_equal(ora.consolidate(m, True), g[f"consT{i}"])
        e, l = ora.components(m, 1 + i % 3)
        assert np.array_equal(e, g[f"ext{i}"]) and np.array_equal(l, g[f"lab{i}"])


@pytest.mark.parametrize("case", ["single_burst_128x256", "mixed_kinds_128x512", "paper_T500x1024"])
def test_golden_detect_cases(ref, ora, case):
    cases = {c["name"]: c for c in json.loads((GOLD / "detect_cases.json").read_text())}
    c = cases[case]
    iq, truth = ref.synthesize(signals.scenario_json(c["scenario"]))
    assert sha(iq) == c["iq_sha256"]
    fs = c["scenario"]["sample_rate_hz"]
    tf = ref.make_plots(iq, fs, c["n_fft"], c["rows"])
    for p, gp in enumerate(c["plots"]):
        assert sha(tf[p]) == gp["tf_sha256"]
        assert sha(ora.tf_plot(iq[p * c["rows"] * c["n_fft"]:], c["n_fft"], c["rows"])) == gp["tf_sha256"]
        d = ora.detect(tf[p], start_seq=p * c["rows"], fs=fs)
        assert d["raw"].view(np.uint32).tolist() == gp["raw"]
        assert sha(d["smoothed"]) == gp["smoothed_sha256"]
        assert int(np.float32(d["threshold"]).view(np.uint32)) == gp["threshold_bits"]
        assert d["active"].tolist() == gp["active"]
        assert d["bin_boxes"].tolist() == gp["bin_boxes"]
        assert d["boxes"].view(np.uint64).tolist() == gp["boxes_bits"]


def test_single_burst_iou_reference(ref):
    """test_detector.cpp:608-650 on the oracle: one box, IoU >= 0.6."""
    c = {c["name"]: c for c in json.loads((GOLD / "detect_cases.json").read_text())}["single_burst_128x256"]
    assert len(c["plots"][0]["bin_boxes"]) == 1
    box = np.array(c["plots"][0]["boxes_bits"], np.uint64).view(np.float64)[0]
    assert ref.iou(box, np.array(c["truth"][0][:4])) >= 0.6


def test_stft_restatement_rect_is_tf_plot(ora):
    rng = np.random.default_rng(12)
    x = (rng.normal(size=30 * 512) + 1j * rng.normal(size=30 * 512)).astype(np.complex64)
    assert np.array_equal(ora.stft_plot(x, 512, 512, 0, 30), ora.tf_plot(x, 512, 30))
    h = ora.stft_plot(x, 512, 256, 1, 50)
    assert h.shape == (50, 512) and np.all(np.isfinite(h))


@pytest.mark.parametrize("n_fft,hop", [(1024, 512), (4096, 2048), (256, 64)])
def test_stft_restatement_matches_numpy(ora, n_fft, hop):
    """The STFT extension has no reference oracle: pin the restatement against an
    independent fp64 FFT (numpy) of the Hann-windowed frames at the fp32 level
    (the same criterion the FFT shim meets for the reference's frontend)."""
    rng = np.random.default_rng(n_fft + hop)
    rows = 24
    x = (rng.normal(size=(rows - 1) * hop + n_fft) + 1j * rng.normal(size=(rows - 1) * hop + n_fft)).astype(np.complex64)
    got = ora.stft_plot(x, n_fft, hop, 1, rows)
    n = np.arange(n_fft)
    w = 0.5 * (1.0 - np.cos(2 * np.pi * n / n_fft))
    frames = np.stack([x[r * hop: r * hop + n_fft].astype(np.complex128) * w for r in range(rows)])
    exp = np.abs(np.fft.fftshift(np.fft.fft(frames, axis=1), axes=1)).astype(np.float32)
    assert np.sum(got != exp) == 0
