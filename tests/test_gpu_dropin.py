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
