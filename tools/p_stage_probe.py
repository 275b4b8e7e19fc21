import ctypes as C, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2603_20481_b200 import _native as NAT, specsense as ss
F, T = 1024, 2000
iq = bench._p_samples()
d = torch.from_numpy(iq.view(np.float32).copy()).cuda()
ctx = ss.Context.get(0); ctx.set_stream(torch.cuda.current_stream().cuda_stream)
lib = ctx.lib
cfg = ss.DetectorConfig().c()
K = 1024
for B in [int(x) for x in (sys.argv[1:] or ["1", "2", "5"])]:
    outs = [torch.empty(s, dtype=dt, device="cuda") for s, dt in [((B, F), torch.float32), ((B, F), torch.float32), ((B, 2), torch.float32), ((B, F), torch.int32), ((B,), torch.int32), ((B, K, 4), torch.float64), ((B, K, 4), torch.int32), ((B,), torch.int32)]]
    bo = NAT.BatchOut(*(C.c_void_p(t.data_ptr()) for t in outs), K)
    tf = torch.empty(B * T * F, device="cuda")
    def go():
        ctx.check(lib.ss_sense_batch(ctx.h, C.c_void_p(d.data_ptr()), 0, F, T, B, C.c_uint64(0), C.c_double(100e6), C.byref(cfg), C.c_void_p(tf.data_ptr()), C.byref(bo)))
    go(); torch.cuda.synchronize()
    lib.ss_enable_stage_timing(ctx.h, 1)
    t0 = time.perf_counter()
    for _ in range(20): go()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    st = (C.c_double * 8)(); lib.ss_stage_times(ctx.h, st); lib.ss_enable_stage_timing(ctx.h, 0)
    print(f"B={B}: {dt*1e3:.3f} ms/call wall;", "stages ms/call:", [round(v / 20, 4) for v in st])
