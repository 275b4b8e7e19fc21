"""C++ drop-in runtime::run (tools/runtime_demo) on the paper configuration P,
unpaced: windows/s without Python in the ingest loop.  Prints one JSON line."""
import json
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

iq = bench._p_samples()
with tempfile.TemporaryDirectory() as d:
    f = Path(d) / "iq.f32"
    iq.astype(np.complex64).tofile(f)
    out = Path(d) / "out.bin"
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    subprocess.run([str(ROOT / "paper_2603_20481_b200/_lib/runtime_demo"), str(f), "100e6", "1024", "2000", str(n),
                    "0", str(out)], check=True)
    b = out.read_bytes()
    # skip per-window records: find the end marker
    o = 0
    while True:
        idx, nb = np.frombuffer(b, np.uint64, 2, o)
        o += 16
        if idx == np.uint64(~np.uint64(0)):
            break
        o += 32 * int(nb)
    stats = np.frombuffer(b, np.float64, 8, o)
    print(json.dumps({"windows": int(nb), "overruns": stats[0], "p50_ms": 1e3 * stats[1], "p99_ms": 1e3 * stats[3],
                      "wall_s": stats[6], "windows_per_s": int(nb) / stats[6], "gpu_s": stats[7]}))
