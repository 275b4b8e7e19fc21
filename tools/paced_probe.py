"""Paced-engine latency outliers vs GPU clock / P-state samples.  Diagnostic only."""
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2603_20481_b200 import runtime as rt  # noqa: E402

iq = bench._p_samples()
fc = rt.FrontendConfig(bench.FS, bench.P_F, bench.P_T)
rt.run(rt.MemorySource(iq, bench.P_F, total_chunks=3 * bench.P_T, block=256), fc)
mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
if mode == "after_unpaced":
    rt.run(rt.MemorySource(iq, bench.P_F, total_chunks=1000 * bench.P_T, block=256), fc)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,pstate,clocks.sm,clocks.mem,power.draw,utilization.gpu",
                        "--format=csv,noheader", "-lms", "20"], stdout=subprocess.PIPE, text=True)
t0 = time.time()
reps = []
for _ in range(2):
  reps.append(rt.run(rt.MemorySource(iq, bench.P_F, total_chunks=150 * bench.P_T, pace=True, sample_rate_hz=bench.FS,
                             block=64), fc))
smi.terminate()
out = smi.communicate()[0].splitlines()
print("wall t0", t0)
for rep in reps:
    print("slowest", [(r.plot_index, round(1e3 * r.latency_s, 2), round(1e3 * r.gpu_s, 3), round(r.complete_s, 3)) for r in
                      sorted(rep.records, key=lambda r: -r.latency_s)[:5]], "overruns", rep.overruns)
prev = None
for l in out:
    f = [x.strip() for x in l.split(",")]
    key = tuple(f[1:4])
    if key != prev:
        print(l)
        prev = key
