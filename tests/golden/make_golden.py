"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

The reference repo ships no golden vectors (every fixture in proj/tests is
regenerated from a seed), so these are produced by running the UNMODIFIED
reference sources (oracle/_ref/libspecsense_ref.so: reference + FFTW-API
shim) on seeded inputs.  Run in the build container (needs oracle/_ref):

    python tests/golden/make_golden.py

Outputs are small: IQ is regenerated from the recorded scenario by the
reference's own signals::synthesize and pinned by SHA-256; TF plots are pinned
by SHA-256; PSD / active sets / masks / boxes are stored verbatim.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from _masks import random_blob_mask, random_mask  # noqa: E402
from _oracle import ref  # noqa: E402
from paper_2603_20481_b200 import signals  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def detect_case(R, sc, n_fft, rows, name):
    iq, truth = R.synthesize(signals.scenario_json(sc))
    fs = sc["sample_rate_hz"]
    tf = R.make_plots(iq, fs, n_fft, rows)
    plots = []
    for p in range(len(tf)):
        d = R.detect(tf[p], start_seq=p * rows, fs=fs)
        plots.append(dict(tf_sha256=sha(tf[p]), raw=d["raw"].view(np.uint32).tolist(),
                          smoothed_sha256=sha(d["smoothed"]),
                          noise_floor_bits=int(np.float32(d["noise_floor"]).view(np.uint32)),
                          threshold_bits=int(np.float32(d["threshold"]).view(np.uint32)),
                          active=d["active"].tolist(), bin_boxes=d["bin_boxes"].tolist(),
                          boxes_bits=d["boxes"].view(np.uint64).tolist()))
    return dict(name=name, scenario=sc, n_fft=n_fft, rows=rows, iq_sha256=sha(iq),
                truth=truth.tolist(), plots=plots)


def main():
    R = ref()
    cases = []
    fs = 1e6
    single = dict(sample_rate_hz=fs, duration_s=0.0328, noise_power=1.0, seed=77,
                  signals=[dict(kind="ofdm-like", center_freq_hz=120e3, bandwidth_hz=100e3, t_start_s=0.008,
                                duration_s=0.016, power=10 ** 2.0 * (1.0 / fs) * 100e3)])
    cases.append(detect_case(R, single, 256, 128, "single_burst_128x256"))
    mixed = dict(sample_rate_hz=fs, duration_s=0.131, noise_power=1.0, seed=4242,
                 signals=[dict(kind="tone-burst", center_freq_hz=-200e3, bandwidth_hz=20e3, t_start_s=0.01,
                               duration_s=0.05, power=0.2),
                          dict(kind="noise-like", center_freq_hz=250e3, bandwidth_hz=80e3, t_start_s=0.04,
                               duration_s=0.06, power=2.0),
                          dict(kind="ofdm-like", center_freq_hz=0.0, bandwidth_hz=150e3, t_start_s=0.07,
                               duration_s=0.05, power=3.0)])
    cases.append(detect_case(R, mixed, 512, 128, "mixed_kinds_128x512"))
    cases.append(detect_case(R, signals.paper_scenario(rows=1000), 1024, 500, "paper_T500x1024"))
    cases.append(detect_case(R, signals.c5_scenario(0), 4096, 2441, "c5r_capture0_2441x4096"))
    (HERE / "detect_cases.json").write_text(json.dumps(cases))

    # FFT rows: seeded uniform chunks, every supported size
    rng = np.random.default_rng(20260320)
    fft = {}
    for n in [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]:
        x = (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(np.complex64)
        fft[f"x{n}"] = x
        fft[f"y{n}"] = R.fft_row(x)
    np.savez_compressed(HERE / "fft_rows.npz", **fft)

    # morphology / CCL on seeded masks
    rng = np.random.default_rng(99)
    st = {}
    for i in range(6):
        m = random_mask(rng, 23, 41, 0.45) if i % 2 else random_blob_mask(rng, 30, 57)
        st[f"m{i}"] = m
        st[f"cons{i}"] = R.consolidate(m, False)
        st[f"consT{i}"] = R.consolidate(m, True)
        ext, lab = R.label_components(m, 1 + i % 3)
        st[f"ext{i}"] = ext
        st[f"lab{i}"] = lab
    np.savez_compressed(HERE / "masks.npz", **st)
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
