"""Python mirror of the reference's real-time engine API (specsense::runtime,
proj/include/specsense/runtime.hpp:11-110) over the GPU streaming engine
(ss_engine_*, paper_2603_20481_b200/csrc/engine.cpp).

``run(source, frontend_config, detector_config, runtime_config, on_detections)``
pulls chunk blocks from a source on an ingest thread, streams them into HBM
banks, and collects one ``PlotRecord`` per sensed window; ``summarize`` /
``nearest_rank`` / ``RunReport.ccdf`` restate the reference's report
arithmetic (runtime.cpp:166-214) in host code.  Python sources yield BLOCKS
of consecutive chunks (``(first_seq, samples[k*F])``): a per-chunk Python
loop cannot keep up with 100 MS/s.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .specsense import DetectorConfig, Error, FormatError, ValidationError


# ---- configuration / records (runtime.hpp:13-90)
@dataclass
class FrontendConfig:
    sample_rate_hz: float
    n_fft: int = 1024
    plot_rows: int = 2000

    def plot_span_s(self) -> float:
        return self.plot_rows * self.n_fft / self.sample_rate_hz


@dataclass
class RuntimeConfig:
    """runtime.hpp:13-24.  The CPU worker counts and halo are validated like
    the reference and otherwise unused (the GPU runs every window whole);
    ``n_banks`` is the HBM bank count (2 = the reference's ping-pong);
    ``stage_timing`` makes the engine time every stage of every window on the
    device (ss_plot_record.stage_s: event-record nodes in each window's graph,
    about 0.12 ms of device time per P window; the C++ drop-in's
    runtime::run always sets it for RunReport::stage_totals)."""
    n_compute_workers: int = 1
    n_sensing_workers: int = 1
    halo_bins: int = 4
    chunk_queue_capacity: int = 0
    deadline_s: float = 0.0
    n_banks: int = 2
    box_capacity: int = 16384
    stage_timing: bool = False

    def validate(self):
        if self.n_compute_workers < 1 or self.n_sensing_workers < 1:
            raise ValidationError("worker counts must be positive")
        if self.halo_bins < 3:
            raise ValidationError("halo_bins must be >= 3")
        if self.chunk_queue_capacity < 0:
            raise ValidationError("chunk_queue_capacity must be >= 0")
        if self.deadline_s < 0:
            raise ValidationError("deadline_s must be >= 0")


@dataclass
class PlotRecord:
    plot_index: int
    start_seq: int
    latency_s: float
    deadline_s: float
    met: bool
    n_boxes: int
    n_active: int = 0
    noise_floor: float = 0.0
    threshold: float = 0.0
    complete_s: float = 0.0
    done_s: float = 0.0
    gpu_s: float = 0.0


@dataclass
class RunReport:
    records: list = field(default_factory=list)
    plots: int = 0
    overruns: int = 0
    deadline_s: float = 0.0
    fraction_met: float = 0.0
    realtime_met: bool = False
    p50_s: float = 0.0
    p90_s: float = 0.0
    p99_s: float = 0.0
    max_s: float = 0.0
    percentiles_valid: bool = False
    wall_time_s: float = 0.0

    def ccdf(self) -> list[tuple[float, float]]:
        """(latency, fraction strictly greater), one point per distinct latency (runtime.cpp:201-214)."""
        lat = sorted(r.latency_s for r in self.records)
        n = len(lat)
        pts = []
        for i, v in enumerate(lat):
            if i + 1 < n and lat[i + 1] == v:
                continue
            pts.append((v, (n - (i + 1)) / n))
        return pts


def nearest_rank(sorted_values, q: float) -> float:
    """Element at 1-based index ceil(q*n), clamped to [1, n] (runtime.hpp:92-94)."""
    n = len(sorted_values)
    if n == 0:
        return 0.0
    k = math.ceil(q * n)
    k = min(max(k, 1), n)
    return sorted_values[k - 1]


def summarize(records, overruns: int, deadline_s: float) -> RunReport:
    """runtime.cpp:166-199: sort by plot index, fraction met, nearest-rank p50/p90/p99."""
    rep = RunReport()
    rep.records = sorted(records, key=lambda r: r.plot_index)
    rep.plots = len(rep.records)
    rep.overruns = int(overruns)
    rep.deadline_s = deadline_s
    if rep.records:
        lat = sorted(r.latency_s for r in rep.records)
        rep.fraction_met = sum(1 for r in rep.records if r.met) / len(lat)
        rep.p50_s = nearest_rank(lat, 0.50)
        rep.p90_s = nearest_rank(lat, 0.90)
        rep.p99_s = nearest_rank(lat, 0.99)
        rep.max_s = lat[-1]
        rep.percentiles_valid = len(lat) >= 100
    rep.realtime_met = rep.fraction_met >= 0.99
    return rep


# ---- sources (frontend.hpp:137-200): blocks of consecutive chunks
class MemorySource:
    """Cycles an in-memory sample buffer as F-sample chunks until total_chunks
    were emitted (0 = one pass), `block` chunks per yield; pace=True releases
    them no faster than sample_rate_hz (frontend.cpp:443-462)."""

    def __init__(self, samples: np.ndarray, n_fft: int, total_chunks: int = 0, pace: bool = False,
                 sample_rate_hz: float = 0.0, block: int = 256, pinned: bool = True):
        if pace and not sample_rate_hz > 0:
            raise ValidationError("paced source needs a sample rate")
        self.n_fft = n_fft
        self.fmt = N.SS_FMT_I16 if samples.dtype == np.int16 else N.SS_FMT_F32
        n = len(samples) // (n_fft * (2 if self.fmt == N.SS_FMT_I16 else 1))
        if n == 0:
            raise ValidationError("source shorter than one chunk")
        flat = np.ascontiguousarray(samples[: n * n_fft * (2 if self.fmt == N.SS_FMT_I16 else 1)])
        self._buf, self._pin = _pinned_copy(flat) if pinned else (flat, None)
        self.chunks = n
        self.total = total_chunks or n
        self.pace = pace
        self.fs = sample_rate_hz
        self.block = block

    def paced(self) -> bool:
        return self.pace

    # the yielded views point into one private buffer that is never written
    # again: the engine may DMA out of them asynchronously (Engine.push stable)
    stable = True

    def blocks(self):
        """Yields (first_seq, ndarray view of k chunks); views never wrap the buffer end."""
        seq = 0
        per = self.n_fft * (2 if self.fmt == N.SS_FMT_I16 else 1)
        t0 = time.perf_counter()
        while seq < self.total:
            pos = seq % self.chunks
            k = min(self.block, self.total - seq, self.chunks - pos)
            if self.pace:
                due = t0 + (seq + k) * self.n_fft / self.fs
                while True:
                    now = time.perf_counter()
                    if now >= due:
                        break
                    time.sleep(min(due - now, 0.001))
            yield seq, self._buf[pos * per:(pos + k) * per]
            seq += k


def _pinned_copy(a: np.ndarray):
    """(page-locked copy of a, owning torch tensor): H2D from it is async DMA."""
    import torch

    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    out = t.numpy().view(a.dtype).reshape(a.shape)
    out[...] = a
    return out, t


# ---- the engine
class Engine:
    """ss_engine_*: push chunk blocks, poll per-window records + boxes."""

    def __init__(self, frontend_config: FrontendConfig, detector_config: DetectorConfig | None = None,
                 runtime_config: RuntimeConfig | None = None, fmt: int = N.SS_FMT_F32, paced: bool = False,
                 device: int = 0, hop: int = 0, window: int = 0, shard: tuple[int, int] = (0, 1)):
        """hop / window: the STFT extension (frames every hop samples, 1 = periodic
        Hann); the defaults are the reference's back-to-back rectangular frames.
        shard = (index, count): this engine senses windows w % count == index
        (multi-GPU: one engine per device, every chunk pushed to all)."""
        import torch

        if not torch.cuda.is_available():
            raise Error("specsense-b200 needs a CUDA device (no CPU fallback)")
        rc = runtime_config or RuntimeConfig()
        rc.validate()
        self.lib = N.load()
        self.F = frontend_config.n_fft
        self.T = frontend_config.plot_rows
        self.fs = frontend_config.sample_rate_hz
        self.fmt = fmt
        self.cap = rc.box_capacity
        cfg = N.EngineCfg(self.F, self.T, fmt, self.fs, rc.n_banks, int(paced), rc.deadline_s, rc.box_capacity,
                          hop, window, shard[1], shard[0], int(rc.stage_timing))
        det = (detector_config or DetectorConfig()).c()
        h = C.c_void_p()
        st = self.lib.ss_engine_open(device, C.byref(cfg), C.byref(det), C.byref(h))
        self.h = h
        if st != N.SS_OK:
            msg = self.lib.ss_engine_last_error(h).decode() if h else f"ss_engine_open status {st}"
            self.close()
            raise (ValidationError if st == N.SS_EVALIDATION else Error)(msg)
        self._finished = False
        self._boxes = (N.Box * self.cap)()
        self._bins = (N.BinBox * self.cap)()

    def _check(self, st):
        if st == N.SS_OK:
            return
        msg = self.lib.ss_engine_last_error(self.h).decode()
        if st == N.SS_EVALIDATION:
            raise ValidationError(msg)
        if st == N.SS_EFORMAT:
            raise FormatError(msg)
        raise Error(f"status {st}: {msg}")

    def push(self, samples: np.ndarray, first_seq: int, stable: bool = False):
        """stable=True: `samples` stays unchanged until finish() (or
        push_fence()), so a DMA out of it is only queued (ss_engine_push_async)
        and consecutive pushes' copies overlap; else push returns once the
        samples have left the buffer (the reference's synchronous writers)."""
        per = self.F * (2 if self.fmt == N.SS_FMT_I16 else 1)
        if samples.size % per:
            raise ValidationError("push takes whole chunks")
        fn = self.lib.ss_engine_push_async if stable else self.lib.ss_engine_push
        self._check(fn(self.h, C.c_void_p(samples.ctypes.data), samples.size // per, first_seq))

    def push_fence(self):
        self._check(self.lib.ss_engine_push_fence(self.h))

    def mark_lost(self, first: int, last: int):
        self._check(self.lib.ss_engine_mark_lost(self.h, first, last))

    def finish(self):
        self._check(self.lib.ss_engine_finish(self.h))
        self._finished = True

    def poll(self, wait_ms: int = -1):
        """(PlotRecord, boxes (n,4) f64 [f0,f1,t0,t1], bin_boxes (n,4) i32) or None."""
        rec = N.PlotRecord()
        got = C.c_int(0)
        st = self.lib.ss_engine_poll(self.h, wait_ms, C.byref(rec), self._boxes, self._bins, self.cap, C.byref(got))
        if not got.value:
            self._check(st)
            return None
        n = min(rec.n_boxes, self.cap)
        boxes = np.ctypeslib.as_array(C.cast(self._boxes, C.POINTER(C.c_double)), shape=(self.cap, 4))[:n].copy()
        bins = np.ctypeslib.as_array(C.cast(self._bins, C.POINTER(C.c_int32)), shape=(self.cap, 4))[:n].copy()
        r = PlotRecord(int(rec.plot_index), int(rec.start_seq), rec.latency_s, rec.deadline_s, bool(rec.met),
                       int(rec.n_boxes), int(rec.n_active), float(rec.noise_floor), float(rec.threshold),
                       rec.complete_s, rec.done_s, rec.gpu_s)
        self._check(st)
        return r, boxes, bins

    def finished_and_drained(self) -> bool:
        """True once finish() was called and every launched window was polled."""
        st = self.stats()
        return self._finished and st["pending"] == 0

    def stats(self) -> dict:
        v = [C.c_uint64() for _ in range(4)]
        self._check(self.lib.ss_engine_stats(self.h, *(C.byref(x) for x in v)))
        return dict(zip(("windows_completed", "overruns", "rows_retired", "pending"), (x.value for x in v)))

    def close(self):
        if getattr(self, "h", None):
            self.lib.ss_engine_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def run(source, frontend_config: FrontendConfig, detector_config: DetectorConfig | None = None,
        runtime_config: RuntimeConfig | None = None, on_detections=None, hop: int = 0, window: int = 0,
        devices=None) -> RunReport:
    """runtime::run (runtime.hpp:103-110): ingest thread -> HBM banks -> GPU
    sensing, one PlotRecord per window handed to on_detections(record, boxes)
    before its bank is released.  Worker errors abort the run and rethrow."""
    rc = runtime_config or RuntimeConfig()
    devices = list(devices) if devices else [0]
    G = len(devices)
    engines = [Engine(frontend_config, detector_config, rc, fmt=source.fmt, paced=source.paced(), device=d, hop=hop,
                      window=window, shard=(g, G)) for g, d in enumerate(devices)]
    eng = engines[0]
    errors = []
    wall0 = time.perf_counter()  # after the engine's one-time setup (banks, graphs, warm-up window)

    stable = bool(getattr(source, "stable", False))

    def ingest():
        expected = 0
        try:
            for seq, block in source.blocks():
                for e_ in engines:  # each engine keeps only its own windows' samples
                    if seq > expected:
                        e_.mark_lost(expected, seq)
                    e_.push(block, seq, stable=stable)
                expected = seq + block.size // (frontend_config.n_fft * (2 if source.fmt == N.SS_FMT_I16 else 1))
        except Exception as e:  # noqa: BLE001
            errors.append(e)
        finally:
            for e_ in engines:
                try:
                    e_.finish()
                except Exception as e:  # noqa: BLE001
                    errors.append(e)

    th = threading.Thread(target=ingest, daemon=True)
    th.start()
    records = []
    ok = False
    try:
        if G == 1:
            while (got := eng.poll(-1)) is not None:
                records.append(got[0])
                if on_detections is not None:
                    on_detections(got[0], got[1])
        else:
            # each engine returns its own windows in order; across engines the
            # handler sees them as they complete (the report is sorted by window)
            live = set(range(G))
            while live:
                for g in list(live):
                    got = engines[g].poll(1)
                    if got is None:
                        if engines[g].finished_and_drained():
                            live.discard(g)
                        continue
                    records.append(got[0])
                    if on_detections is not None:
                        on_detections(got[0], got[1])
        ok = True
    finally:
        if not ok:
            # the manager failed (handler error, capacity): end the stream so a
            # push blocked on a held bank returns, and drain what is in flight
            # (runtime.cpp:466-478 rethrows after joining the workers)
            for e_ in engines:
                try:
                    e_.finish()
                    while e_.poll(-1) is not None:
                        pass
                except Exception:  # noqa: BLE001
                    pass
        th.join()
    if errors:
        raise Error(f"engine aborted, {errors[0]}")
    overruns = sum(e_.stats()["overruns"] for e_ in engines)
    span = frontend_config.plot_rows * (hop or frontend_config.n_fft) / frontend_config.sample_rate_hz
    deadline = rc.deadline_s if rc.deadline_s > 0 else span
    for e_ in engines:
        e_.close()
    rep = summarize(records, overruns, deadline)
    rep.wall_time_s = time.perf_counter() - wall0
    return rep
