"""GPU parity through the C++ drop-in: tools/dropin_demo (a reference-style C++
caller linked against libspecsense_b200.so) vs the reference oracle."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2603_20481_b200 import signals

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
DEMO = ROOT / "paper_2603_20481_b200" / "_lib" / "dropin_demo"


class Reader:
    def __init__(self, b):
        self.b, self.o = b, 0

    def take(self, dtype, n):
        a = np.frombuffer(self.b, dtype, n, self.o)
        self.o += a.nbytes
        return a

    def one(self, dtype):
        return self.take(dtype, 1)[0]


def test_dropin_demo_matches_reference(ref, tmp_path):
    assert DEMO.exists(), "build() links tools/dropin_demo.cpp"
    sc = signals.paper_scenario(rows=1000)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    f = tmp_path / "iq.f32"
    iq.astype(np.complex64).tofile(f)
    out = tmp_path / "out.bin"
    fs, n_fft, rows = 100e6, 1024, 500
    subprocess.run([str(DEMO), str(f), str(fs), str(n_fft), str(rows), str(out)], check=True)
    r = Reader(out.read_bytes())
    exp_tf = ref.make_plots(iq, fs, n_fft, rows)
    n = r.one(np.int32)
    assert n == len(exp_tf) == 2
    for p in range(n):
        exp = ref.detect(exp_tf[p], start_seq=p * rows, fs=fs)
        assert np.array_equal(r.take(np.float32, rows * n_fft), exp_tf[p].reshape(-1))
        assert np.array_equal(r.take(np.float32, n_fft), exp["raw"])
        assert np.array_equal(r.take(np.float32, n_fft), exp["smoothed"])
        assert r.one(np.float32) == np.float32(exp["noise_floor"])
        assert r.one(np.float32) == np.float32(exp["threshold"])
        na = r.one(np.int32)
        assert np.array_equal(r.take(np.int32, na), exp["active"])
        nb = r.one(np.int32)
        assert nb == len(exp["boxes"]) > 0
        for i in range(nb):
            assert np.array_equal(r.take(np.float64, 4), exp["boxes"][i])
            assert np.array_equal(r.take(np.int32, 4), exp["bin_boxes"][i])
        assert r.one(np.float64) > 0  # StageTimes from device events
    assert np.array_equal(r.take(np.float32, n_fft), ref.fft_row(iq[:n_fft]))
    raw = r.take(np.float32, n_fft)
    assert np.array_equal(raw, ref.estimate_psd(exp_tf[0]))
    sm, fl, thr, act = ref.floor_prune(raw)
    assert r.one(np.float32) == np.float32(thr)
    na = r.one(np.int32)
    assert np.array_equal(r.take(np.int32, na), act)
    mask = r.take(np.uint8, rows * n_fft).reshape(rows, n_fft)
    assert np.array_equal(mask, ref.binarize_columns(exp_tf[0], act))
    cons = r.take(np.uint8, rows * n_fft).reshape(rows, n_fft)
    assert np.array_equal(cons, ref.consolidate(mask))
    lab = r.take(np.int32, rows * n_fft).reshape(rows, n_fft)
    eext, elab = ref.label_components(cons, 4)
    assert np.array_equal(lab, elab)
    assert r.one(np.int32) == len(eext)
    assert r.one(np.int32) == 1


RT_DEMO = ROOT / "paper_2603_20481_b200" / "_lib" / "runtime_demo"


def _run_rt_demo(tmp_path, iq, fs, n_fft, rows, windows, paced):
    f = tmp_path / "rt_iq.f32"
    iq.astype(np.complex64).tofile(f)
    out = tmp_path / "rt.bin"
    subprocess.run([str(RT_DEMO), str(f), str(fs), str(n_fft), str(rows), str(windows), str(int(paced)), str(out)],
                   check=True, timeout=120)
    r = Reader(out.read_bytes())
    per = {}
    while True:
        idx, nb = r.take(np.uint64, 2)
        if idx == np.uint64(~np.uint64(0)):
            plots = int(nb)
            break
        per[int(idx)] = r.take(np.float64, 4 * int(nb)).reshape(-1, 4)
    stats = r.take(np.float64, 8)
    ncc = int(r.one(np.uint64))
    ccdf = r.take(np.float64, 2 * ncc).reshape(-1, 2)
    slabs = r.take(np.int32, 12).reshape(3, 4)
    return per, plots, stats, ccdf, slabs


def test_runtime_dropin_matches_reference_engine(ref, tmp_path):
    """specsense::runtime::run (C++ drop-in over the GPU engine) vs the reference's
    own runtime::run on the same cycling source: every window's boxes identical."""
    assert RT_DEMO.exists(), "build() links tools/runtime_demo.cpp"
    fs, n_fft, rows = 100e6, 1024, 500
    sc = signals.paper_scenario(rows=3 * rows)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    iq = np.ascontiguousarray(iq[: 3 * rows * n_fft])
    per, plots, stats, ccdf, slabs = _run_rt_demo(tmp_path, iq, fs, n_fft, rows, 7, False)
    exp, seen = ref.run_engine_boxes(iq, fs, n_fft, rows, 7)
    assert plots == seen == 7 and sorted(per) == list(range(7))
    for w in range(7):
        e = np.asarray(exp.get(w, np.zeros((0, 4))), np.float64).reshape(-1, 4)
        assert np.array_equal(per[w].view(np.uint64), e.view(np.uint64)), w
    overruns, p50, p90, p99, mx, frac, wall, gpu = stats
    assert overruns == 0 and 0 < p50 <= p90 <= p99 <= mx and frac == 1.0 and gpu > 0
    assert ccdf[-1, 1] == 0.0 and np.all(np.diff(ccdf[:, 0]) > 0)
    # partition(1024, 3, 4): widths 342/341/341, halo clamped at the edges
    assert slabs.tolist() == [[0, 342, 0, 346], [342, 683, 338, 687], [683, 1024, 679, 1024]]


def test_runtime_dropin_paced(ref, tmp_path):
    """A paced source at 100 MS/s: every window sensed well inside its 5.12 ms span."""
    fs, n_fft, rows = 100e6, 1024, 500
    sc = signals.paper_scenario(rows=2 * rows)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    per, plots, stats, ccdf, _ = _run_rt_demo(tmp_path, np.ascontiguousarray(iq[: 2 * rows * n_fft]), fs, n_fft,
                                              rows, 20, True)
    assert plots == 20 and stats[0] == 0 and stats[5] == 1.0


BL_DEMO = ROOT / "paper_2603_20481_b200" / "_lib" / "baseline_demo"


def test_baseline_dropin_matches_reference(ref, tmp_path):
    """specsense::baseline through the C++ drop-in vs the reference."""
    assert BL_DEMO.exists(), "build() links tools/baseline_demo.cpp"
    sc = signals.paper_scenario(rows=500)
    iq, truth = ref.synthesize(signals.scenario_json(sc))
    fs, rows, cols = 100e6, 500, 1024
    tf = ref.make_plots(iq, fs, cols, rows)[0]
    (tmp_path / "tf.f32").write_bytes(tf.astype(np.float32).tobytes())
    span = rows * cols / fs
    gt = np.array([[b[0], b[1], max(b[2], 0.0), min(b[3], span)] for b in truth if b[2] < span], np.float64)
    (tmp_path / "gt.f64").write_bytes(gt.tobytes())
    out = tmp_path / "bl.bin"
    subprocess.run([str(BL_DEMO), str(tmp_path / "tf.f32"), str(rows), str(cols), str(fs), "0",
                    str(tmp_path / "gt.f64"), str(out)], check=True, timeout=120)
    r = Reader(out.read_bytes())
    nk = r.one(np.int32)
    assert np.array_equal(r.take(np.int32, 2 * nk).reshape(-1, 2), ref.kernel_sizes(rows, cols))
    nb = r.one(np.int32)
    got = r.take(np.float64, 4 * nb).reshape(-1, 4)
    exp = ref.baseline_detect(tf, 0, fs)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    assert r.one(np.int32) == 1
