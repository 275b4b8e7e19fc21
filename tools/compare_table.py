"""Acceptance criterion 4 (pipeline vs Searchlight-style baseline: speed and
detection quality) on the paper scenario at (T, F) = (2000, 1024): both
detectors on the GPU through this framework, and the reference's own CPU
implementations (oracle/_ref) on the same plots.  Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from _oracle import ref as _ref  # noqa: E402

from paper_2603_20481_b200 import baseline as bl, signals, specsense as ss  # noqa: E402

R = _ref()
fs, F, T, P = 100e6, 1024, 2000, 4
sc = signals.paper_scenario(rows=P * T)
iq, truth = R.synthesize(signals.scenario_json(sc))
tf = R.make_plots(iq, fs, F, T)
gt = []
for p in range(P):
    t0, t1 = p * T * F / fs, (p + 1) * T * F / fs
    gt.append([[b[0], b[1], max(b[2], t0), min(b[3], t1)] for b in truth if b[2] < t1 and b[3] > t0])

gpu_rows, gpu_speedup = bl.compare(list(tf), gt, fs, theta=0.5, start_seqs=[p * T for p in range(P)])
gpu_rows, gpu_speedup = bl.compare(list(tf), gt, fs, theta=0.5, start_seqs=[p * T for p in range(P)])  # warm

cpu_pipe, cpu_base = [], []
tp = tb = 0.0
for p in range(P):
    t0 = time.perf_counter()
    cpu_pipe.append(R.detect(tf[p], start_seq=p * T, fs=fs)["boxes"])
    tp += time.perf_counter() - t0
    t0 = time.perf_counter()
    cpu_base.append(R.baseline_detect(tf[p], p * T, fs))
    tb += time.perf_counter() - t0
cpu_rows = [bl.make_compare_row("pipeline", cpu_pipe, gt, 0.5, tp / P),
            bl.make_compare_row("baseline", cpu_base, gt, 0.5, tb / P)]
same = all(np.array_equal(ss.detect(tf[p], sample_rate_hz=fs, start_seq=p * T).boxes, cpu_pipe[p]) and
           np.array_equal(bl.baseline_detect(tf[p], fs, p * T)[0], cpu_base[p]) for p in range(P))
out = {"config": f"paper scenario, {P} plots of (T, F) = ({T}, {F}) @ 100 MS/s, theta 0.5",
       "gpu": {"rows": [r.__dict__ for r in gpu_rows], "speedup_baseline_over_pipeline": gpu_speedup},
       "reference_cpu_1_thread": {"rows": [r.__dict__ for r in cpu_rows], "speedup_baseline_over_pipeline": tb / tp},
       "boxes_bit_identical_gpu_vs_reference": same}
print(json.dumps(out, indent=1))
