#!/usr/bin/env python
"""Benchmark: spectrum-occupancy frames/s on B200 (and the reference CPU arm).

Workload (BASELINE.json config 5, reference-parity mode "C5r"):
one frame = one 100 ms capture of complex fp32 IQ at 100 MS/s -> a rectangular,
hop-4096, F = 4096 TF plot (T = 2441 rows, 1,664 tail samples dropped exactly as
proj/src/frontend.cpp:177) -> PSD / SG floor / prune -> per-column Otsu ->
close3x3/open3x3/open1x3 -> 4-connected components -> boxes.  A step is one
batch of `--batch` captures through ss_sense_batch (the fused C-ABI call).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--mode c5r|hann]

--mode hann runs config 5 as BASELINE.json writes it (periodic Hann, hop 2048,
T = 4881 frames per 100 ms plot of a continuous stream) through the STFT
extension entry point ss_stft_sense_batch; its CPU arm is the oracle port.

Under torchrun each rank processes its own captures (weak scaling); boxes
are gathered to every rank with one NCCL all_gather per step (the path's only
exchange); time = max over ranks of CUDA-event time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FS = 100e6
N_FFT = 4096
CAPTURE_S = 0.1
FP64_PEAK_TFLOPS = 33.9                        # measured DFMA peak, tools/fp64_peak.cu (profiles/fp64_peak.txt)


class Workload:
    """One plot = `rows` frames of `n_fft` samples every `hop` samples of a
    continuous 100 MS/s stream.  c5r: hop = n_fft, rect (the reference's own
    frontend, frontend.cpp:127-183) -> plots are back-to-back 100 ms captures.
    hann: config 5 as written (periodic Hann, 50 % overlap, STFT extension)."""

    def __init__(self, name, hop, window, desc, i16=False):
        self.name, self.hop, self.window, self.desc = name, hop, window, desc
        self.i16 = i16
        self.sb = 4 if i16 else 8                                      # bytes per complex sample
        self.rows = (int(CAPTURE_S * FS) - N_FFT) // hop + 1          # 2441 | 4881
        self.stride = self.rows * hop                                  # new samples per plot
        self.tail = N_FFT - hop                                        # extra samples after the last plot
        # K1 algorithmic bytes per plot: read its new IQ once + write the TF plot
        self.alg_bytes = self.stride * self.sb + self.rows * N_FFT * 4
        self.alg_flop64 = self.rows * 5 * N_FFT * 12                   # conventional 5 N log2 N per row
        # FP64 warp-instructions K1 executes per row and warp (ncu source view of
        # fft_mag_kernel<12,0,1,0,0>: 809.5 = DADD 408 + DFMA
        # 204.8 + DMUL 196.7): the SSFFT-2 work itself, counted for the default
        # (rect, fp32) kernel only
        self.k1_fp64_instr = 810 if (name == "c5r" and window == 0) else None

    def samples(self, plots):
        return plots * self.stride + self.tail


WORKLOADS = {
    "c5r": Workload("c5r", N_FFT, 0, "C5r: 100 ms fp32 IQ @ 100 MS/s, F=4096 rect hop 4096 (T=2441), "
                                      "default DetectorConfig"),
    "hann": Workload("hann", N_FFT // 2, 1, "C5h: 100 ms fp32 IQ @ 100 MS/s, F=4096 periodic Hann hop 2048 "
                                            "(T=4881, STFT extension), default DetectorConfig"),
    "c5r16": Workload("c5r16", N_FFT, 0, "C5r with int16 IQ (the reference's quantiser, gain 2^-6; decoded "
                                         "exactly as frontend.cpp:376-385), F=4096 rect hop 4096 (T=2441)", i16=True),
}
METRIC = "spectrum-occupancy frames/s (config 5: 100 ms fp32 IQ capture @ 100 MS/s -> 2441x4096 TF plot -> boxes)"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _caps_host(wl, D, rank=0):
    """The D distinct seeded captures of a step (identical bytes on both arms:
    the same seeds through the same renderer), as numpy arrays of one plot's
    samples each (complex64, or int16 interleaved for c5r16)."""
    import torch

    from paper_2603_20481_b200 import signals
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    caps = [signals.synthesize_torch(signals.c5_scenario(1000 * rank + i), device=dev)[:wl.stride] for i in range(D)]
    if wl.i16:
        caps = [signals.quantize_i16(c)[0] for c in caps]
    return [c.cpu().numpy() for c in caps]


def _as_c64(x):
    """int16 interleaved -> the complex64 the reference decodes it to (raw * 2^-15, exact)."""
    import numpy as np
    if x.dtype == np.int16:
        f = x.astype(np.float32) * np.float32(1.0 / 32768.0)
        return (f[0::2] + 1j * f[1::2]).astype(np.complex64)
    return x


def _plot_input(caps, b, wl, B):
    """Samples of plot b of a batch of B tiled from caps (its stride, plus the
    next capture's first `tail` samples for overlapping STFT plots; zeros after
    the last plot)."""
    import numpy as np
    D = len(caps)
    x = _as_c64(caps[b % D])
    if wl.tail:
        nxt = _as_c64(caps[(b + 1) % D])[:wl.tail] if b + 1 < B else np.zeros(wl.tail, np.complex64)
        x = np.concatenate([x, nxt])
    return x


def cpu_reference(wl, threads: int, seconds_budget: float, D: int):
    """The reference's CPU path on host cores, `threads` threads, over the same
    D distinct captures the GPU arm tiles.

    c5r / c5r16: oracle/_ref (the unmodified reference sources + the FFTW-API
    shim): make_plot + detect per capture, one capture per std::thread at a time
    (kind "reference").  hann: the reference has no windowed/overlapped
    frontend, so the oracle restatement (oracle_stft_plot + oracle_detect,
    ctypes calls release the GIL) runs one plot per thread (kind "port")."""
    sys.path.insert(0, str(ROOT / "tests"))
    import numpy as np

    from _oracle import ora, ref

    caps = _caps_host(wl, D)
    if wl.hop == N_FFT and wl.window == 0:  # the reference's own frontend (int16 decodes exactly to these floats)
        R = ref()
        iq = np.concatenate([_as_c64(c) for c in caps])
        t0 = time.perf_counter()
        R.bench_detect(iq, FS, N_FFT, wl.rows, threads, threads)       # calibrate: one capture per thread
        one_round = time.perf_counter() - t0
        n = max(1, int(seconds_budget / max(one_round, 1e-3))) * threads
        _, secs = R.bench_detect(iq, FS, N_FFT, wl.rows, n, threads)
        return n / secs, n, secs, "reference"
    from concurrent.futures import ThreadPoolExecutor
    O = ora()

    def one(i):
        tf = O.stft_plot(_plot_input(caps, i % D, wl, D + 1), N_FFT, wl.hop, wl.window, wl.rows)
        O.detect(tf, start_seq=0, fs=FS)

    with ThreadPoolExecutor(threads) as pool:
        t0 = time.perf_counter()
        list(pool.map(one, range(threads)))
        one_round = time.perf_counter() - t0
        n = max(1, int(seconds_budget / max(one_round, 1e-3))) * threads
        t0 = time.perf_counter()
        list(pool.map(one, range(n)))
        secs = time.perf_counter() - t0
    return n / secs, n, secs, "port"


def cpu_verify(wl, caps, got, threads, B):
    """Checker for the timed batch (runs in the CPU leg, after timing): the
    reference (c5r / c5r16: oracle/_ref) or the oracle port (hann) on the same
    bytes as the first D plots of the batch; every output compared bit for bit.
    got: dict of host arrays for plots 0..D-1 (tf, psd_raw, psd_smoothed,
    floor_thr, active, n_active, boxes, bin_boxes, n_boxes)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    from _oracle import ora, ref

    D = len(caps)
    rect = wl.hop == N_FFT and wl.window == 0
    R = ref() if rect else ora()

    def one(b):
        x = _plot_input(caps, b, wl, B)
        if rect:
            tf = R.make_plots(x, FS, N_FFT, wl.rows)[0]
        else:
            tf = R.stft_plot(x, N_FFT, wl.hop, wl.window, wl.rows)
        e = R.detect(tf, start_seq=b * wl.rows, fs=FS)
        bad = []
        if not np.array_equal(got["tf"][b].view(np.uint32), tf.view(np.uint32)):
            bad.append("tf")
        if not np.array_equal(got["psd_raw"][b].view(np.uint32), e["raw"].view(np.uint32)):
            bad.append("psd_raw")
        if not np.array_equal(got["psd_smoothed"][b].view(np.uint32), e["smoothed"].view(np.uint32)):
            bad.append("psd_smoothed")
        if not (np.float32(got["floor_thr"][b][0]) == np.float32(e["noise_floor"])
                and np.float32(got["floor_thr"][b][1]) == np.float32(e["threshold"])):
            bad.append("floor")
        na = int(got["n_active"][b])
        if not np.array_equal(got["active"][b][:na], e["active"]):
            bad.append("active")
        nb = int(got["n_boxes"][b])
        if nb != len(e["bin_boxes"]) or not np.array_equal(got["bin_boxes"][b][:nb], e["bin_boxes"]):
            bad.append("bin_boxes")
        else:
            bx = got["boxes"][b][:nb]
            if rect:
                ok = np.array_equal(bx.view(np.uint64), e["boxes"].view(np.uint64))
            else:  # STFT extension: times on the hop/fs frame grid
                bb = e["bin_boxes"].astype(np.float64)
                dt, df = wl.hop / FS, FS / N_FFT
                ok = (np.array_equal(bx[:, 0], (bb[:, 2] - N_FFT // 2) * df)
                      and np.array_equal(bx[:, 2], (b * wl.rows + bb[:, 0]) * dt)
                      and np.array_equal(bx[:, 3], (b * wl.rows + bb[:, 1]) * dt))
            if not ok:
                bad.append("boxes")
        return bad

    with ThreadPoolExecutor(max(1, min(threads, D))) as pool:
        res = list(pool.map(one, range(D)))
    mism = [b for b, r in enumerate(res) if r]
    return {"plots": D, "mismatches": len(mism), "checker": "oracle/_ref (reference sources)" if rect else
            "oracle restatement (STFT extension)", "compared": "tf bits, psd raw/smoothed, floor/threshold, "
            "active set, bin boxes, boxes", "failed": {str(b): res[b] for b in mism}}


def _cpu_sample(wl, n, secs):
    if wl.hop == N_FFT and wl.window == 0:
        return (f"{n} C5r captures (make_plot + detect each, one capture per thread) in {secs:.1f} s; "
                "reference sources + builder FFTW-API shim (FFTW absent)")
    return (f"{n} C5h plots (oracle_stft_plot + oracle_detect each, one plot per thread) in {secs:.1f} s; "
            "oracle restatement (the reference has no Hann/overlap frontend)")


def _config(wl, B, D, ws):
    """The workload description printed identically by both arms."""
    return {"workload": wl.desc, "captures_per_step_per_gpu": B, "distinct_captures": D,
            "l2": f"inputs > L2 ({wl.samples(B) * wl.sb / 1e9:.1f} GB IQ per step per GPU, no flush needed)",
            "parallelism": f"capture-sharded x{ws}"}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    wl = WORKLOADS[args.mode]
    threads = os.cpu_count() or 1
    D = min(args.distinct, args.batch)
    total_caps, total_s, kind = 0, 0.0, "reference"
    for i in range(args.warmup + args.steps):
        v, n, secs, kind = cpu_reference(wl, threads, args.ref_step_seconds, D)
        if i >= args.warmup:
            total_caps += n
            total_s += secs
    value = total_caps / total_s
    line = {
        "impl": "reference", "metric": _metric(wl), "value": value, "unit": "frames/s", "n_gpus": max(ws, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": _config(wl, args.batch, D, max(ws, args.gpus)),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": kind,
                         "sample": f"over {args.steps} steps: " + _cpu_sample(wl, total_caps, total_s)},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


DATA = "synthetic: seeded config-5 captures (16 rectangular bursts, 5-40 MHz, 0.1-5 ms, 0-20 dB) on unit AWGN"


def _metric(wl):
    if wl.name == "c5r":
        return METRIC
    if wl.name == "c5r16":
        return METRIC.replace("fp32 IQ", "int16 IQ")
    return ("spectrum-occupancy frames/s (config 5 as written: 100 ms fp32 IQ @ 100 MS/s -> "
            "4881x4096 Hann/50% TF plot -> boxes)")


def _quality(dets_per_capture, truth_per_capture, span_plot):
    """Detection quality the way the reference's acceptance gate pools it
    (acceptance.cpp:84-102): truth clipped to each plot's window, IoU matrix,
    strict-theta matches at 0.4 / 0.5, mean best-match IoU; plus p_fa."""
    from paper_2603_20481_b200 import metrics
    n_gt = n_det = t04 = t05 = n_false = 0
    iou_sum = 0.0
    nplots = 0
    for dets, truth in zip(dets_per_capture, truth_per_capture):
        for p, d in enumerate(dets):
            w0, w1 = p * span_plot, (p + 1) * span_plot
            gt = [[t[0], t[1], max(t[2], w0), min(t[3], w1)] for t in truth if min(t[3], w1) > max(t[2], w0)]
            m = metrics.iou_matrix(gt, d)
            t04 += metrics.count_matches(m, 0.4)[0]
            tr, fa = metrics.count_matches(m, 0.5)
            t05 += tr
            n_false += fa
            n_gt += len(gt)
            n_det += len(d)
            iou_sum += sum(m.row_max(g) for g in range(m.n_gt))
            nplots += 1
    return {"plots": nplots, "n_gt": n_gt, "mean_iou": iou_sum / max(n_gt, 1), "p_d_0.4": t04 / max(n_gt, 1),
            "p_d_0.5": t05 / max(n_gt, 1), "p_fa_0.5": n_false / max(n_det, 1),
            "boxes_per_plot": n_det / max(nplots, 1)}


def measure(args, wl, B, D, steps, warmup, e2e_batch, with_gather=True):
    """One workload on this rank: timed device-resident steps (value), the
    e2e leg through host buffers, and the outputs of plots 0..D-1 for checking."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_20481_b200 import _native as NAT, parallel, specsense as ss

    ws, rank, local = _dist()
    ctx = ss.Context.get(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    K = args.box_capacity

    # ---- inputs: D distinct seeded captures, tiled to B captures, resident in HBM
    caps = _caps_host(wl, D, rank)
    if wl.i16:
        iq = torch.zeros(2 * wl.samples(B), dtype=torch.int16, device="cuda")
        for b in range(B):
            iq[2 * b * wl.stride:2 * (b + 1) * wl.stride] = torch.from_numpy(caps[b % D])
    else:
        iq = torch.zeros(wl.samples(B), dtype=torch.complex64, device="cuda")
        dcaps = [torch.from_numpy(c).cuda() for c in caps]
        for b in range(B):
            iq[b * wl.stride:(b + 1) * wl.stride] = dcaps[b % D]
        del dcaps
    fmt = NAT.SS_FMT_I16 if wl.i16 else NAT.SS_FMT_F32
    tf = torch.empty(B * wl.rows * N_FFT, dtype=torch.float32, device="cuda")
    outs = dict(
        psd_raw=torch.empty((B, N_FFT), dtype=torch.float32, device="cuda"),
        psd_smoothed=torch.empty((B, N_FFT), dtype=torch.float32, device="cuda"),
        floor_thr=torch.empty((B, 2), dtype=torch.float32, device="cuda"),
        active=torch.empty((B, N_FFT), dtype=torch.int32, device="cuda"),
        n_active=torch.empty(B, dtype=torch.int32, device="cuda"),
        boxes=torch.empty((B, K, 4), dtype=torch.float64, device="cuda"),
        bin_boxes=torch.empty((B, K, 4), dtype=torch.int32, device="cuda"),
        n_boxes=torch.empty(B, dtype=torch.int32, device="cuda"),
    )
    bout = NAT.BatchOut(*(C.c_void_p(v.data_ptr()) for v in outs.values()), K)
    cfg = ss.DetectorConfig().c()
    gathered = [None]

    def sense(src_ptr, nb, tf_ptr, out):
        if wl.hop == N_FFT and wl.window == 0:    # the reference-parity entry point
            return lib.ss_sense_batch(ctx.h, C.c_void_p(src_ptr), fmt, N_FFT, wl.rows, nb,
                                      C.c_uint64(0), C.c_double(FS), C.byref(cfg), tf_ptr, C.byref(out))
        return lib.ss_stft_sense_batch(ctx.h, C.c_void_p(src_ptr), fmt, N_FFT, wl.hop, wl.window,
                                       wl.rows, nb, C.c_uint64(0), C.c_double(FS), C.byref(cfg), tf_ptr,
                                       C.byref(out))

    def step(src_ptr, out):
        ctx.check(sense(src_ptr, B, C.c_void_p(tf.data_ptr()), out))
        if ws > 1 and with_gather:  # the path's one exchange: detections to rank 0, sized by the box counts
            gathered[0] = parallel.gather_detections(outs["n_boxes"], outs["boxes"])

    for _ in range(warmup):
        step(iq.data_ptr(), bout)
    torch.cuda.synchronize()

    # ---- timed: device-resident inputs (value)
    lib.ss_enable_stage_timing(ctx.h, 1)
    l0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(steps):
            step(iq.data_ptr(), bout)
        ev1.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    launches = ctx.launches() - l0
    st = (C.c_double * 8)()
    lib.ss_stage_times(ctx.h, st)
    lib.ss_enable_stage_timing(ctx.h, 0)
    if ws > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    sec_per_step = elapsed / steps
    stage_names = ["k1_fft_mag_psd", "k2_psd", "k3_floor", "k4_binarize", "k5_consolidate", "k6_ccl", "h2d", "d2h"]
    stage_ms = {n: st[i] / steps for i, n in enumerate(stage_names) if st[i] > 0}
    k1_ms = stage_ms.get("k1_fft_mag_psd", float("nan"))
    hbm_peak, peak_kind = _peaks()
    achieved = B * wl.alg_bytes / (k1_ms / 1e3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "k1_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(wl.name, {}).get("bytes_per_capture")
        traffic = traffic * B if traffic else None
    # whole-step algorithmic bytes (read IQ once, write the API-visible TF plot once) per step time
    pipeline = {"achieved": B * wl.alg_bytes / sec_per_step / 1e9, "unit": "GB/s",
                "frac": B * wl.alg_bytes / sec_per_step / 1e9 / hbm_peak}
    got = {k: v[:D].cpu().numpy() for k, v in outs.items()}
    got["tf"] = tf[: D * wl.rows * N_FFT].view(D, wl.rows, N_FFT).cpu().numpy()
    n_gathered = None
    if ws > 1 and with_gather and rank == 0 and gathered[0] is not None:
        n_gathered = int(sum(int(c.sum()) for c, _ in gathered[0]))

    # ---- e2e: host (pinned) IQ in, host boxes out, through the same C-ABI call
    Be = 0 if args.no_e2e else max(1, min(B, e2e_batch))
    e2e = None
    if Be:
        per = 2 if wl.i16 else 1
        while True:  # N ranks pin N buffers on one host: shrink the e2e batch rather than fail
            try:
                host_iq = torch.empty(per * wl.samples(Be), dtype=iq.dtype, pin_memory=True)
                break
            except RuntimeError:
                if Be == 1:
                    raise
                Be = max(1, Be // 2)
        host_iq.copy_(iq[: per * wl.samples(Be)])
        host_out = {k: torch.empty((Be,) + tuple(v.shape[1:]), dtype=v.dtype, pin_memory=True)
                    for k, v in outs.items()}
        hout = NAT.BatchOut(*(C.c_void_p(v.data_ptr()) for v in host_out.values()), K)

        def e2e_step():
            ctx.check(sense(host_iq.data_ptr(), Be, None, hout))

        for _ in range(max(1, warmup // 2)):
            e2e_step()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # asynchronous batches (ss_set_async): step i+1's host->device copies
        # queue behind step i without a host round trip; ss_wait checks them all
        ctx.check(lib.ss_set_async(ctx.h, 1))
        e0.record(stream)
        for _ in range(steps):
            e2e_step()
        e1.record(stream)
        ctx.check(lib.ss_wait(ctx.h))
        ctx.check(lib.ss_set_async(ctx.h, 0))
        torch.cuda.synchronize()
        e2e_el = e0.elapsed_time(e1) / 1e3
        if ws > 1:
            t = torch.tensor([e2e_el], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_el = float(t.item())
        d2h = sum(v.numel() * v.element_size() for v in host_out.values())
        # the host-buffer path computes the same detections as the device-resident one
        nchk = min(Be, D)
        hn = host_out["n_boxes"][:nchk].numpy()
        same = bool(np.array_equal(hn, got["n_boxes"][:nchk])
                    and np.array_equal(host_out["psd_raw"][:nchk].numpy(), got["psd_raw"][:nchk])
                    and all(np.array_equal(host_out["bin_boxes"][b, :min(int(hn[b]), K)].numpy(),
                                           got["bin_boxes"][b, :min(int(hn[b]), K)]) for b in range(nchk)))
        e2e = {"value": ws * Be / (e2e_el / steps), "unit": "frames/s",
               "h2d_bytes_per_step": wl.samples(Be) * wl.sb, "d2h_bytes_per_step": d2h, "captures_per_step": Be,
               "same_as_device_path": bool(same)}
        del host_iq, host_out
    res = {"value": ws * B / sec_per_step, "ms_per_step": 1e3 * sec_per_step, "stage_ms_per_step": stage_ms,
           "launches": launches, "clocks": clk.summary(), "caps": caps, "got": got, "e2e": e2e,
           "gathered_boxes": n_gathered,
           "roofline": {"bound": "hbm", "kernel": "k1_fft_mag_psd", "achieved": achieved, "peak": hbm_peak,
                        "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                        "alg_bytes_per_capture": wl.alg_bytes,
                        "fp64_tflops": B * wl.alg_flop64 / (k1_ms / 1e3) / 1e12,
                        "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                        "fp64_frac": B * wl.alg_flop64 / (k1_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                        "pipeline": pipeline,
                        "fp64_executed": _fp64_executed(wl, k1_ms / B),
                        "note": "K1 is bounded by FP64 pipe + issue slots as much as by HBM (DESIGN.md §4): "
                                "both fractions are given, against measured peaks; `pipeline` = the same "
                                "algorithmic bytes over the whole step"}}
    del iq, tf, outs
    torch.cuda.empty_cache()
    return res


def _fp64_executed(wl, k1_ms_per_capture):
    """K1 against the FP64 pipe executing the instructions it actually issues:
    rows x N/16 threads x the per-thread FP64 instruction count, at the measured
    DFMA lane rate (FP64_PEAK_TFLOPS / 2 flops).  `frac` = that floor over the
    measured K1 time; `hbm_frac_cap` = the HBM fraction K1 would reach at it."""
    if wl.k1_fp64_instr is None:
        return None
    lane_ops = wl.rows * (N_FFT // 16) * wl.k1_fp64_instr
    floor_us = lane_ops / (FP64_PEAK_TFLOPS * 1e12 / 2) * 1e6
    meas_us = k1_ms_per_capture * 1e3
    hbm_us = wl.alg_bytes / (_peaks()[0] * 1e9) * 1e6
    return {"warp_instr_per_row_warp": wl.k1_fp64_instr, "floor_us_per_capture": floor_us,
            "measured_us_per_capture": meas_us, "frac": floor_us / meas_us, "hbm_frac_cap": hbm_us / floor_us}


def quality_at(wl, caps, rows, K=4096):
    """Config-5 detection quality of the device pipeline on the D distinct
    captures cut into plots of `rows` frames (evaluation only, untimed)."""
    import numpy as np

    from paper_2603_20481_b200 import signals, specsense as ss
    dets, truth = [], []
    for i, c in enumerate(caps):
        x = _as_c64(c)
        if wl.tail:  # the capture alone, zero-padded for its last overlapping frame
            x = np.concatenate([x, np.zeros(wl.tail, np.complex64)])
        dd = ss.sense(x, FS, N_FFT, rows, box_capacity=K, hop=wl.hop, window=wl.window)
        dets.append([d.boxes for d in dd])
        truth.append(signals.truth_boxes(signals.c5_scenario(i)).tolist())
    return _quality(dets, truth, rows * wl.hop / FS)


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    wl = WORKLOADS[args.mode]
    B = args.batch
    D = min(args.distinct, B)
    threads = os.cpu_count() or 1
    m = measure(args, wl, B, D, args.steps, args.warmup, args.e2e_batch)

    # config 5 as written (Hann, 50 % overlap, T = 4881) in the same run, on the STFT entry point
    hann = None
    if args.mode == "c5r" and not args.no_hann:
        hw = WORKLOADS["hann"]
        hann = measure(args, hw, B, D, max(2, args.steps // 2), max(1, args.warmup // 2), args.e2e_batch // 2,
                       with_gather=False)

    line = None
    if rank == 0:
        # ---- CPU leg (rank 0): the checker on the timed batch, then (N = 1) the reference's timing
        parity = None if args.no_verify else cpu_verify(wl, m["caps"], m["got"], threads, B)
        cpu = None
        if ws == 1 and not args.no_cpu:
            v, n, secs, kind = cpu_reference(wl, threads, args.cpu_seconds, D)
            cpu = {"value": v, "unit": "frames/s", "cores": threads, "kind": kind, "sample": _cpu_sample(wl, n, secs)}
        quality = {f"T{wl.rows}": quality_at(wl, m["caps"], wl.rows)}
        if wl.name != "hann":
            quality["T500"] = quality_at(wl, m["caps"], 500)
        line = {
            "metric": _metric(wl), "value": m["value"], "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": _config(wl, B, D, ws),
            "iq_gbps": m["value"] * wl.stride * 32 / 1e9,
            "stage_ms_per_step": m["stage_ms_per_step"],
            "roofline": m["roofline"],
            "e2e": m["e2e"],
            "gpu_launches": m["launches"],
            "clocks": m["clocks"],
            "parity": parity,
            "detection": {"theta": [0.4, 0.5], "note": "reference semantics at F=4096 (dense false alarms at "
                          "T=2441 are the reference's own behaviour, bit-identical)", **quality},
            "cpu_baseline": cpu,
        }
        if ws > 1:
            line["gathered_boxes_rank0"] = m["gathered_boxes"]
        if hann is not None:
            hp = None if args.no_verify else cpu_verify(WORKLOADS["hann"], hann["caps"], hann["got"], threads, B)
            hcpu = None
            if ws == 1 and not args.no_cpu:
                v, n, secs, kind = cpu_reference(WORKLOADS["hann"], threads, args.cpu_seconds / 2, D)
                hcpu = {"value": v, "unit": "frames/s", "cores": threads, "kind": kind,
                        "sample": _cpu_sample(WORKLOADS["hann"], n, secs)}
            line["config5_as_written"] = {
                "metric": _metric(WORKLOADS["hann"]), "value": hann["value"], "unit": "frames/s",
                "ms_per_step": hann["ms_per_step"], "config": _config(WORKLOADS["hann"], B, D, ws),
                "stage_ms_per_step": hann["stage_ms_per_step"], "roofline": hann["roofline"],
                "e2e": hann["e2e"], "gpu_launches": hann["launches"], "parity": hp,
                "detection": {"T4881": quality_at(WORKLOADS["hann"], hann["caps"], WORKLOADS["hann"].rows)},
                "cpu_baseline": hcpu}
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line))
        bad = (line["parity"] or {}).get("mismatches", 0) + \
            ((line.get("config5_as_written") or {}).get("parity") or {}).get("mismatches", 0)
        if bad:
            sys.exit(f"parity FAILED on the timed batch: {line['parity']}")


# ---------------------------------------------------------------- stream mode
# the real-time engine at the paper's configuration P
# (fs = 100 MS/s, F = 1024, T = 2000: one window per 20.48 ms), fed from
# pinned host memory through ss_engine_* (ingest thread -> HBM banks -> GPU).
P_F, P_T = 1024, 2000


def _p_samples(n_windows=5):
    sys.path.insert(0, str(ROOT / "tests"))
    from paper_2603_20481_b200 import signals
    from _oracle import ref

    sc = signals.paper_scenario(rows=n_windows * P_T)
    iq, _ = ref().synthesize(signals.scenario_json(sc))
    return iq[: n_windows * P_T * P_F]


def run_stream(args):
    import numpy as np  # noqa: F401
    import torch

    from paper_2603_20481_b200 import runtime as rt

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    iq = _p_samples()
    fc = rt.FrontendConfig(FS, P_F, P_T)
    windows = max(args.steps, 1) * args.stream_windows
    # warm-up pass (allocations, pinned copies, clocks)
    rt.run(rt.MemorySource(iq, P_F, total_chunks=args.warmup * P_T, block=args.stream_block), fc)
    src = rt.MemorySource(iq, P_F, total_chunks=windows * P_T, block=args.stream_block)
    with Clocks(local) as clk:
        rep = rt.run(src, fc)
        wall = rep.wall_time_s  # first push -> last record (the engine's setup is not in it)
    # paced at the real sample rate: latency against the 20.48 ms deadline
    paced_windows = max(20, int(args.stream_paced_s / fc.plot_span_s()))
    prep = rt.run(rt.MemorySource(iq, P_F, total_chunks=paced_windows * P_T, pace=True, sample_rate_hz=FS,
                                  block=64), fc)
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = _stream_reference(iq, args.cpu_seconds)
    if rank == 0:
        line = {
            "metric": "streaming-engine plots/s (config P: 100 MS/s fp32, F=1024, T=2000 windows, host-fed)",
            "value": rep.plots / wall, "unit": "plots/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic: the acceptance-style paper scenario, cycled",
            "config": {"workload": "P stream: MemorySource (pinned) -> ss_engine (2 HBM banks) -> boxes",
                       "windows_per_step": args.stream_windows, "parallelism": "replicas" if ws > 1 else "single"},
            "stream": {"unpaced": {"plots": rep.plots, "overruns": rep.overruns, "wall_s": wall,
                                   "p50_ms": 1e3 * rep.p50_s, "p99_ms": 1e3 * rep.p99_s,
                                   "iq_gbps": rep.plots * P_T * P_F * 32 / wall / 1e9,
                                   "h2d_gbps": rep.plots * P_T * P_F * 8 / wall / 1e9},
                       "paced": {"plots": prep.plots, "overruns": prep.overruns, "p50_ms": 1e3 * prep.p50_s,
                                 "p90_ms": 1e3 * prep.p90_s, "p99_ms": 1e3 * prep.p99_s, "max_ms": 1e3 * prep.max_s,
                                 "deadline_ms": 1e3 * prep.deadline_s, "fraction_met": prep.fraction_met,
                                 "realtime_met": prep.realtime_met, "percentiles_valid": prep.percentiles_valid,
                                 "slowest": [[r.plot_index, round(1e3 * r.latency_s, 3), round(1e3 * r.gpu_s, 3), round(r.complete_s, 4)]
                                             for r in sorted(prep.records, key=lambda r: -r.latency_s)[:6]]}},
            "e2e": {"value": rep.plots / wall, "unit": "plots/s", "h2d_bytes_per_step": args.stream_windows * P_T * P_F * 8,
                    "d2h_bytes_per_step": args.stream_windows * 1024 * 64},
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))


def run_stream5(args):
    """Config 5 as written, streaming: 100 MS/s fp32 chunks of 4096 samples into
    the engine with the STFT extension (periodic Hann, hop 2048, T = 4881
    frames = 99.96 ms windows overlapping by 2048 samples).  Unpaced windows/s
    from pinned host memory, and latency at the real sample rate."""
    import numpy as np
    import torch

    from paper_2603_20481_b200 import runtime as rt, signals

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    wl = WORKLOADS["hann"]
    caps = [signals.synthesize_torch(signals.c5_scenario(i), device="cuda").cpu().numpy() for i in range(3)]
    iq = np.concatenate(caps)
    fc = rt.FrontendConfig(FS, N_FFT, wl.rows)
    kw = dict(hop=wl.hop, window=wl.window)
    per_win = wl.stride // N_FFT + 1
    rt.run(rt.MemorySource(iq, N_FFT, total_chunks=2 * per_win, block=256), fc, **kw)
    windows = max(args.steps, 1) * args.stream_windows5
    src = rt.MemorySource(iq, N_FFT, total_chunks=windows * wl.stride // N_FFT + 1, block=256)
    with Clocks(local) as clk:
        rep = rt.run(src, fc, **kw)
        wall = rep.wall_time_s
    paced_w = max(5, int(args.stream_paced_s / (wl.stride / FS)))
    prep = rt.run(rt.MemorySource(iq, N_FFT, total_chunks=paced_w * wl.stride // N_FFT + 1, pace=True,
                                  sample_rate_hz=FS, block=64), fc, **kw)
    if rank == 0:
        print(json.dumps({
            "metric": "streaming-engine windows/s (config 5 as written: 100 MS/s fp32, 4096-pt Hann, 50% overlap, "
                      "100 ms windows, host-fed)",
            "value": rep.plots / wall, "unit": "windows/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic: seeded config-5 captures, cycled",
            "config": {"workload": "C5h stream: MemorySource (pinned) -> ss_engine (STFT hop 2048, Hann) -> boxes"},
            "stream": {"unpaced": {"windows": rep.plots, "overruns": rep.overruns, "wall_s": wall,
                                   "h2d_gbps": rep.plots * wl.stride * 8 / wall / 1e9, "p50_ms": 1e3 * rep.p50_s},
                       "paced": {"windows": prep.plots, "overruns": prep.overruns, "p50_ms": 1e3 * prep.p50_s,
                                 "p99_ms": 1e3 * prep.p99_s, "max_ms": 1e3 * prep.max_s,
                                 "deadline_ms": 1e3 * prep.deadline_s, "fraction_met": prep.fraction_met}},
            "e2e": {"value": rep.plots / wall, "unit": "windows/s",
                    "h2d_bytes_per_step": args.stream_windows5 * wl.stride * 8, "d2h_bytes_per_step": 0},
            "clocks": clk.summary(), "cpu_baseline": None}))


def _stream_reference(iq, seconds):
    """The reference engine (runtime::run over an unpaced MemorySource, the
    acceptance split: 16 sensing + 4 compute workers on >= 16 cores, else 4 + 2)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import ref

    R = ref()
    cores = os.cpu_count() or 1
    n_sense, n_comp = (16, 4) if cores >= 16 else (4, 2)
    _, st = R.run_engine(iq, FS, P_F, P_T, 4, n_comp, n_sense)
    per = st["wall_s"] / max(st["plots"], 1)
    n = max(8, int(seconds / max(per, 1e-3)))
    _, st = R.run_engine(iq, FS, P_F, P_T, n, n_comp, n_sense)
    return {"value": st["plots"] / st["wall_s"], "unit": "plots/s", "cores": n_sense + n_comp, "kind": "reference",
            "sample": f"{int(st['plots'])} P windows through runtime::run ({n_comp} compute + {n_sense} sensing "
                      f"workers, unpaced MemorySource) in {st['wall_s']:.1f} s",
            "p50_ms": 1e3 * st["p50_s"], "p99_ms": 1e3 * st["p99_s"], "fraction_met": st["fraction_met"]}


def run_stream_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    iq = _p_samples()
    vals = []
    for i in range(args.warmup + args.steps):
        c = _stream_reference(iq, args.ref_step_seconds)
        if i >= args.warmup:
            vals.append(c)
    v = sum(c["value"] for c in vals) / len(vals)
    line = {"impl": "reference",
            "metric": "streaming-engine plots/s (config P: 100 MS/s fp32, F=1024, T=2000 windows, host-fed)",
            "value": v, "unit": "plots/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the acceptance-style paper scenario, cycled",
            "config": {"workload": "P stream: MemorySource -> runtime::run (CPU)"},
            "cpu_baseline": dict(vals[-1], value=v),
            "e2e": {"value": v, "unit": "plots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _maybe_spawn(args):
    """`--gpus N` outside torchrun: re-launch this command as N ranks (one
    process per GPU) through torch.distributed.run on 127.0.0.1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execvp(cmd[0], cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--mode", default="c5r", choices=sorted(WORKLOADS) + ["stream", "stream5"],
                    help="c5r: reference-parity rect/hop-N frontend (default); hann: config 5 as written; "
                         "stream: the real-time engine at config P (latency + plots/s)")
    ap.add_argument("--stream-windows", type=int, default=200, help="stream mode: windows per timed step")
    ap.add_argument("--stream-windows5", type=int, default=20, help="stream5 mode: windows per timed step")
    ap.add_argument("--stream-block", type=int, default=1000,
                    help="stream mode: chunks per MemorySource block (one engine push each) in the unpaced run")
    ap.add_argument("--stream-paced-s", type=float, default=3.0, help="stream mode: seconds of paced real-time input")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=296, help="captures per step per GPU")
    ap.add_argument("--distinct", type=int, default=8)
    ap.add_argument("--e2e-batch", type=int, default=64)
    ap.add_argument("--box-capacity", type=int, default=2048)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (kernel experiments only)")
    ap.add_argument("--no-hann", action="store_true", help="skip the config-5-as-written (Hann) line")
    ap.add_argument("--no-verify", action="store_true", help="skip the CPU check of the timed batch")
    args = ap.parse_args()
    _maybe_spawn(args)
    if args.mode == "stream":
        (run_stream_reference if args.impl == "reference" else run_stream)(args)
    elif args.mode == "stream5":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the reference has no Hann/overlap frontend"}))
        else:
            run_stream5(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
