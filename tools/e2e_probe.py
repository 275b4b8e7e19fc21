"""Where does the host-buffer (e2e) sense call spend its time?  Times a raw
pinned H2D copy, and ss_sense_batch with host input at several batch sizes,
against the device-resident call.  Diagnostic only."""
import ctypes as C
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2603_20481_b200 import _native as NAT, signals, specsense as ss  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5r"]
ctx = ss.Context.get(0)
lib = ctx.lib
K = 2048
cfg = ss.DetectorConfig().c()
Bmax = 64
cap = signals.synthesize_torch(signals.c5_scenario(1), device="cuda")[:wl.stride]
dev_iq = torch.zeros(wl.samples(Bmax), dtype=torch.complex64, device="cuda")
for b in range(Bmax):
    dev_iq[b * wl.stride:(b + 1) * wl.stride] = cap
host_iq = torch.empty_like(dev_iq, device="cpu").pin_memory()
host_iq.copy_(dev_iq)


def outs(B, pinned):
    shapes = [((B, 4096), torch.float32), ((B, 4096), torch.float32), ((B, 2), torch.float32),
              ((B, 4096), torch.int32), ((B,), torch.int32), ((B, K, 4), torch.float64),
              ((B, K, 4), torch.int32), ((B,), torch.int32)]
    if pinned:
        t = [torch.empty(s, dtype=d, pin_memory=True) for s, d in shapes]
    else:
        t = [torch.empty(s, dtype=d, device="cuda") for s, d in shapes]
    return t, NAT.BatchOut(*(C.c_void_p(v.data_ptr()) for v in t), K)


def sense(src, B, bo):
    if wl.name == "c5r":
        r = lib.ss_sense_batch(ctx.h, C.c_void_p(src), NAT.SS_FMT_F32, 4096, wl.rows, B, C.c_uint64(0),
                               C.c_double(100e6), C.byref(cfg), None, C.byref(bo))
    else:
        r = lib.ss_stft_sense_batch(ctx.h, C.c_void_p(src), NAT.SS_FMT_F32, 4096, wl.hop, wl.window, wl.rows, B,
                                    C.c_uint64(0), C.c_double(100e6), C.byref(cfg), None, C.byref(bo))
    ctx.check(r)


def timeit(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


nbytes = wl.samples(Bmax) * 8
dst = torch.empty_like(dev_iq)
t = timeit(lambda: dst.copy_(host_iq, non_blocking=True))
print(f"raw pinned H2D {nbytes / 1e9:.2f} GB: {t * 1e3:.1f} ms = {nbytes / t / 1e9:.1f} GB/s")
for B in (1, 3, 6, 16, 64):
    to, bo = outs(B, True)
    th = timeit(lambda: sense(host_iq.data_ptr(), B, bo))
    td_, bd = outs(B, False)
    td = timeit(lambda: sense(dev_iq.data_ptr(), B, bd))
    lib.ss_enable_stage_timing(ctx.h, 1)
    sense(dev_iq.data_ptr(), B, bd)
    torch.cuda.synchronize()
    st = (C.c_double * 8)()
    lib.ss_stage_times(ctx.h, st)
    lib.ss_enable_stage_timing(ctx.h, 0)
    print("   stages ms:", [round(v, 3) for v in st])
    print(f"B={B:3d} host {th * 1e3:8.1f} ms ({B / th:7.1f} f/s, H2D-equiv {wl.samples(B) * 8 / th / 1e9:5.1f} GB/s)"
          f"  device {td * 1e3:7.2f} ms")
