"""Where does the streaming engine spend its time at config P?  Diagnostic only."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2603_20481_b200 import runtime as rt, specsense as ss  # noqa: E402

F, T, FS = bench.P_F, bench.P_T, bench.FS
iq = bench._p_samples()
fc = rt.FrontendConfig(FS, F, T)
src = rt.MemorySource(iq, F, pinned=True)
buf = src._buf

# (a) device-resident batch pipeline, 1 window
d = torch.from_numpy(iq.view(np.float32)).cuda()
ctx = ss._ctx()
for B in (1, 4):
    ss.sense(iq[: B * T * F], FS, F, T)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        ss.sense(iq[: B * T * F], FS, F, T)
    torch.cuda.synchronize()
    print(f"ss.sense host numpy B={B}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms/call")

for nb in (2, 4, 8):
    for block in (T, 256, 64):
        eng = rt.Engine(fc, runtime_config=rt.RuntimeConfig(n_banks=nb))
        W = 40
        import threading
        pushed = []

        def writer():
            t0 = time.perf_counter()
            for w in range(W):
                pos = (w % 5) * T
                for b0 in range(0, T, block):
                    k = min(block, T - b0)
                    eng.push(buf[(pos + b0) * F:(pos + b0 + k) * F], w * T + b0)
            pushed.append(time.perf_counter() - t0)
            eng.finish()

        t0 = time.perf_counter()
        th = threading.Thread(target=writer)
        th.start()
        lat = []
        while (g := eng.poll(-1)) is not None:
            lat.append(g[0].latency_s)
        th.join()
        wall = time.perf_counter() - t0
        lat.sort()
        print(f"banks={nb} block={block:4d}: {W / wall:7.1f} plots/s  push-loop {pushed[0] * 1e3:6.1f} ms  "
              f"lat p50 {lat[len(lat) // 2] * 1e3:.3f} ms max {lat[-1] * 1e3:.3f} ms  "
              f"H2D {W * T * F * 8 / wall / 1e9:.1f} GB/s")
        eng.close()
