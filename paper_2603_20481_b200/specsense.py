"""Python mirror of the reference's hot-path API, over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++
functions (proj/include/specsense/frontend.hpp:45-84,
proj/include/specsense/detector.hpp:57-169), so parity tests read like the
reference's own tests.  Host inputs are numpy arrays; device memory is torch
CUDA storage (PyTorch is plumbing here).  Every call runs on the GPU through
``_lib/libspecsense_b200.so``; nothing falls back to the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


# ---- error hierarchy (proj/include/specsense/types.hpp:43-70)
class Error(RuntimeError):
    pass


class ValidationError(Error):
    pass


class FormatError(Error):
    pass


class SchemaError(Error):
    pass


class IoError(Error):
    pass


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise Error("specsense-b200 needs a CUDA device (no CPU fallback)")
    return torch


class Context:
    """One ss_ctx per device (ss_open / ss_close)."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int = 0):
        self.lib = N.load()
        torch = _torch()
        torch.cuda.set_device(device)
        torch.cuda.init()
        h = C.c_void_p()
        rc = self.lib.ss_open(device, C.byref(h))
        if rc != N.SS_OK:
            raise Error(f"ss_open({device}) failed with status {rc}")
        self.h = h
        self.device = device

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls._by_device[device] = Context(device)
        return ctx

    def check(self, rc: int):
        if rc == N.SS_OK:
            return
        msg = self.lib.ss_last_error(self.h).decode()
        if rc == N.SS_EVALIDATION:
            raise ValidationError(msg)
        if rc == N.SS_EFORMAT:
            raise FormatError(msg)
        raise Error(f"status {rc}: {msg}")

    def set_stream(self, stream_ptr: int | None):
        self.check(self.lib.ss_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def launches(self) -> int:
        return int(self.lib.ss_launch_count(self.h))

    def sync(self):
        self.check(self.lib.ss_synchronize(self.h))


def _ctx() -> Context:
    """The device-0 context, bound to torch's current stream so the H2D/D2H
    copies torch issues and our kernels are ordered on one stream."""
    ctx = Context.get(0)
    torch = _torch()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    return ctx


def _dev(a: np.ndarray, dtype=None):
    torch = _torch()
    a = np.ascontiguousarray(a if dtype is None else a.astype(dtype, copy=False))
    return torch.from_numpy(a).cuda()


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _host(t) -> np.ndarray:
    return t.cpu().numpy()


# ---------------------------------------------------------------- config

@dataclass
class DetectorConfig:
    """proj/include/specsense/detector.hpp:11-23 (same defaults)."""

    savgol_window: int = 31
    savgol_order: int = 3
    psd_margin_db: float = 3.0
    min_component_area: int = 4
    one_d_opening_along_time: bool = False

    def c(self) -> N.DetectorCfg:
        return N.DetectorCfg(self.savgol_window, self.savgol_order, float(self.psd_margin_db),
                             self.min_component_area, int(self.one_d_opening_along_time))


@dataclass
class PsdProfile:
    raw: np.ndarray
    smoothed: np.ndarray = None
    noise_floor: float = 0.0
    threshold: float = 0.0


@dataclass
class Detections:
    boxes: np.ndarray       # (n, 4) f0_hz, f1_hz, t0_s, t1_s
    bin_boxes: np.ndarray   # (n, 4) t0, t1, f0, f1
    psd: PsdProfile
    active_columns: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))


class MorphOp:
    Erode, Dilate, Open, Close = 0, 1, 2, 3


# ---------------------------------------------------------------- frontend

def make_plots_device(iq, n_fft: int, rows: int, n_plots: int, fmt: int = N.SS_FMT_F32):
    """IQ (torch CUDA tensor, interleaved) -> torch (n_plots, rows, n_fft) float32 TF plots."""
    torch = _torch()
    ctx = _ctx()
    tf = torch.empty((n_plots, rows, n_fft), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.ss_tf_plots(ctx.h, _ptr(iq), fmt, n_fft, rows, n_plots, _ptr(tf)))
    return tf


def make_plot(samples: np.ndarray, sample_rate_hz: float, n_fft: int, start_seq: int = 0) -> np.ndarray:
    """frontend::make_plot (frontend.cpp:157-171): rows = len // n_fft."""
    if n_fft < 8 or n_fft & (n_fft - 1):
        raise ValidationError(f"FFT size must be a power of two >= 8, got {n_fft}")
    if not sample_rate_hz > 0:
        raise ValidationError("sample_rate_hz must be positive")
    rows = len(samples) // n_fft
    if rows == 0:
        return np.zeros((0, n_fft), np.float32)
    x = np.ascontiguousarray(samples[: rows * n_fft].astype(np.complex64)).view(np.float32)
    return _host(make_plots_device(_dev(x), n_fft, rows, 1))[0]


def make_plots(samples: np.ndarray, sample_rate_hz: float, n_fft: int, plot_rows: int,
               fmt: int = N.SS_FMT_F32) -> np.ndarray:
    """frontend::make_plots (frontend.cpp:173-183); trailing partial window dropped.

    ``samples``: complex64 (f32 IQ) or interleaved int16 (fmt = SS_FMT_I16)."""
    if not sample_rate_hz > 0:
        raise ValidationError("sample_rate_hz must be positive")
    if n_fft < 8 or n_fft & (n_fft - 1):
        raise ValidationError(f"FFT size must be a power of two >= 8, got {n_fft}")
    if plot_rows < 1:
        raise ValidationError("plot_rows must be >= 1")
    if fmt == N.SS_FMT_I16:
        raw = np.ascontiguousarray(samples, np.int16)
        n = len(raw) // 2
    else:
        raw = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        n = len(samples)
    per = plot_rows * n_fft
    n_plots = n // per
    if n_plots == 0:
        return np.zeros((0, plot_rows, n_fft), np.float32)
    raw = raw[: n_plots * per * 2]
    return _host(make_plots_device(_dev(raw), n_fft, plot_rows, n_plots, fmt))


def stft_plots(samples: np.ndarray, sample_rate_hz: float, n_fft: int, hop: int, window: int, plot_rows: int,
               fmt: int = N.SS_FMT_F32) -> np.ndarray:
    """STFT extension of make_plots (BASELINE config 5 as written): frames every
    `hop` samples, window 0 = rectangular / 1 = periodic Hann; consecutive plots
    of `plot_rows` frames."""
    if fmt == N.SS_FMT_I16:
        raw = np.ascontiguousarray(samples, np.int16)
        n = len(raw) // 2
    else:
        raw = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        n = len(samples)
    frames = (n - n_fft) // hop + 1 if n >= n_fft else 0
    n_plots = frames // plot_rows
    if n_plots == 0:
        return np.zeros((0, plot_rows, n_fft), np.float32)
    torch = _torch()
    ctx = _ctx()
    span = (n_plots * plot_rows - 1) * hop + n_fft
    d = _dev(raw[: 2 * span])
    tf = torch.empty((n_plots, plot_rows, n_fft), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.ss_stft_plots(ctx.h, _ptr(d), fmt, n_fft, hop, window, plot_rows, n_plots, _ptr(tf)))
    return _host(tf)


def fft_row(chunk: np.ndarray) -> np.ndarray:
    """frontend::fft_row (frontend.cpp:127-149)."""
    n = len(chunk)
    if n < 8 or n & (n - 1):
        raise ValidationError(f"FFT size must be a power of two >= 8, got {n}")
    return make_plot(chunk, 1.0, n)[0]


# ---------------------------------------------------------------- detector stages

def estimate_psd_into(tf: np.ndarray, col_begin: int, col_end: int) -> np.ndarray:
    ctx = _ctx()
    rows, cols = tf.shape
    d = _dev(tf, np.float32)
    torch = _torch()
    out = torch.empty(max(col_end - col_begin, 1), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.ss_psd_cols(ctx.h, _ptr(d), rows, cols, col_begin, col_end, _ptr(out)))
    return _host(out)[: col_end - col_begin]


def estimate_psd(tf: np.ndarray) -> np.ndarray:
    return estimate_psd_into(tf, 0, tf.shape[1])


def savgol_smooth(values: np.ndarray, window: int, order: int) -> np.ndarray:
    ctx = _ctx()
    d = _dev(values, np.float32)
    out = d.clone()
    ctx.check(ctx.lib.ss_savgol_smooth(ctx.h, _ptr(d), len(values), window, order, _ptr(out)))
    return _host(out)


def smooth_and_floor(profile: PsdProfile, config: DetectorConfig) -> np.ndarray:
    """Fills profile.smoothed / noise_floor / threshold; returns prune_columns()."""
    ctx = _ctx()
    torch = _torch()
    raw = _dev(profile.raw, np.float32)
    n = len(profile.raw)
    sm = torch.empty(n, dtype=torch.float32, device="cuda")
    ft = torch.empty(2, dtype=torch.float32, device="cuda")
    act = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    na = C.c_int32(0)
    cfg = config.c()
    ctx.check(ctx.lib.ss_floor(ctx.h, _ptr(raw), n, C.byref(cfg), _ptr(sm), _ptr(ft), _ptr(act), C.byref(na)))
    profile.smoothed = _host(sm)
    f = _host(ft)
    profile.noise_floor, profile.threshold = float(f[0]), float(f[1])
    return _host(act)[: na.value]


def otsu_threshold(values: np.ndarray) -> tuple[bool, float]:
    ctx = _ctx()
    v = _dev(values, np.float32) if len(values) else None
    valid = C.c_int32(0)
    thr = C.c_float(0.0)
    ctx.check(ctx.lib.ss_otsu(ctx.h, _ptr(v) if v is not None else None, len(values), C.byref(valid),
                              C.byref(thr)))
    return bool(valid.value), float(thr.value)


def binarize_columns(tf: np.ndarray, active, col_begin: int, col_end: int, out: np.ndarray) -> np.ndarray:
    ctx = _ctx()
    rows, cols = tf.shape
    if out.shape != tf.shape:
        raise ValidationError("binarize output mask shape mismatch")
    d = _dev(tf, np.float32)
    m = _dev(out, np.uint8)
    act = np.ascontiguousarray(np.asarray(active, np.int32))
    ctx.check(ctx.lib.ss_binarize_cols(ctx.h, _ptr(d), rows, cols, act.ctypes.data_as(C.c_void_p), len(act),
                                       col_begin, col_end, _ptr(m)))
    return _host(m)


def binarize(tf: np.ndarray, active) -> np.ndarray:
    return binarize_columns(tf, active, 0, tf.shape[1], np.zeros(tf.shape, np.uint8))


def morphology_cols(src: np.ndarray, dst: np.ndarray, op: int, se: tuple[int, int], col_begin: int,
                    col_end: int) -> np.ndarray:
    ctx = _ctx()
    rows, cols = src.shape
    if dst.shape != src.shape:
        raise ValidationError("morphology output mask shape mismatch")
    s = _dev(src, np.uint8)
    d = _dev(dst, np.uint8)
    ctx.check(ctx.lib.ss_morph_cols(ctx.h, _ptr(s), rows, cols, op, se[0], se[1], col_begin, col_end, _ptr(d)))
    return _host(d)


def morphology(mask: np.ndarray, op: int, se: tuple[int, int]) -> np.ndarray:
    return morphology_cols(mask, np.zeros_like(mask, dtype=np.uint8), op, se, 0, mask.shape[1])


def consolidate(mask: np.ndarray, one_d_opening_along_time: bool = False) -> np.ndarray:
    ctx = _ctx()
    rows, cols = mask.shape
    s = _dev(mask, np.uint8)
    d = s.clone()
    ctx.check(ctx.lib.ss_consolidate(ctx.h, _ptr(s), rows, cols, int(one_d_opening_along_time), _ptr(d)))
    return _host(d)


def label_components(mask: np.ndarray, min_component_area: int, with_labels: bool = True):
    """Returns (extents (n,5) int64 [min_t,max_t,min_f,max_f,area], labels int32 or None)."""
    ctx = _ctx()
    torch = _torch()
    rows, cols = mask.shape
    m = _dev(mask, np.uint8)
    cap = min(rows * cols // 2 + 2, 1 << 20)
    ext = np.zeros((cap, 5), np.int64)
    lab = torch.empty((rows, cols), dtype=torch.int32, device="cuda") if with_labels else None
    n = C.c_int64(0)
    ctx.check(ctx.lib.ss_components(ctx.h, _ptr(m), rows, cols, min_component_area,
                                    _ptr(lab) if lab is not None else None, ext.ctypes.data_as(C.c_void_p), cap,
                                    C.byref(n)))
    return ext[: n.value].copy(), (_host(lab) if lab is not None else None)


def component_extents(mask: np.ndarray, min_component_area: int) -> np.ndarray:
    return label_components(mask, min_component_area, with_labels=False)[0]


def extent_to_bin_box(e) -> tuple[int, int, int, int]:
    """detector.cpp:622-624: (t0, t1, f0, f1) half-open."""
    return int(e[0]), int(e[1]) + 1, int(e[2]), int(e[3]) + 1


def bin_box_to_physical(b, cols: int, sample_rate_hz: float, start_seq: int = 0):
    """detector.cpp:626-635: (f0_hz, f1_hz, t0_s, t1_s)."""
    dt = cols / sample_rate_hz
    df = sample_rate_hz / cols
    return ((b[2] - cols // 2) * df, (b[3] - cols // 2) * df, (float(start_seq) + b[0]) * dt,
            (float(start_seq) + b[1]) * dt)


# ---------------------------------------------------------------- fused

def _batch_out(torch, n_plots, cols, cap):
    t = dict(
        psd_raw=torch.empty((n_plots, cols), dtype=torch.float32, device="cuda"),
        psd_smoothed=torch.empty((n_plots, cols), dtype=torch.float32, device="cuda"),
        floor_thr=torch.empty((n_plots, 2), dtype=torch.float32, device="cuda"),
        active=torch.empty((n_plots, cols), dtype=torch.int32, device="cuda"),
        n_active=torch.empty(n_plots, dtype=torch.int32, device="cuda"),
        boxes=torch.empty((n_plots, cap, 4), dtype=torch.float64, device="cuda"),
        bin_boxes=torch.empty((n_plots, cap, 4), dtype=torch.int32, device="cuda"),
        n_boxes=torch.empty(n_plots, dtype=torch.int32, device="cuda"),
    )
    out = N.BatchOut(*(C.c_void_p(v.data_ptr()) for v in t.values()), cap)
    return t, out


def _unpack_batch(t, n_plots) -> list[Detections]:
    h = {k: _host(v) for k, v in t.items()}
    dets = []
    for p in range(n_plots):
        nb = int(h["n_boxes"][p])
        na = int(h["n_active"][p])
        psd = PsdProfile(h["psd_raw"][p].copy(), h["psd_smoothed"][p].copy(), float(h["floor_thr"][p, 0]),
                         float(h["floor_thr"][p, 1]))
        dets.append(Detections(h["boxes"][p, :nb].copy(), h["bin_boxes"][p, :nb].copy(), psd,
                               h["active"][p, :na].copy()))
    return dets


def detect_batch(tf: np.ndarray, sample_rate_hz: float, config: DetectorConfig | None = None,
                 start_seq=None, box_capacity: int = 1024) -> list[Detections]:
    """detector::detect (detector.cpp:637-670) over a (P, T, F) stack of TF plots."""
    config = config or DetectorConfig()
    ctx = _ctx()
    torch = _torch()
    tf = np.asarray(tf, np.float32)
    if tf.ndim == 2:
        tf = tf[None]
    P, T, F = tf.shape
    d = _dev(tf, np.float32)
    t, out = _batch_out(torch, P, F, box_capacity)
    seq = np.ascontiguousarray(np.zeros(P, np.uint64) if start_seq is None else np.asarray(start_seq, np.uint64))
    cfg = config.c()
    ctx.check(ctx.lib.ss_detect_batch(ctx.h, _ptr(d), P, T, F, seq.ctypes.data_as(C.c_void_p),
                                      float(sample_rate_hz), C.byref(cfg), C.byref(out)))
    return _unpack_batch(t, P)


def detect(tf: np.ndarray, config: DetectorConfig | None = None, sample_rate_hz: float = 1e6,
           start_seq: int = 0) -> Detections:
    return detect_batch(tf[None], sample_rate_hz, config, [start_seq])[0]


def sense(samples: np.ndarray, sample_rate_hz: float, n_fft: int, plot_rows: int,
          config: DetectorConfig | None = None, fmt: int = N.SS_FMT_F32, first_seq: int = 0,
          box_capacity: int = 1024, return_tf: bool = False, hop: int | None = None, window: int = 0):
    """IQ -> Detections per full window (make_plots + detect, the runtime's per-plot work).
    hop / window select the STFT extension (default: the reference's rect, hop = n_fft)."""
    config = config or DetectorConfig()
    ctx = _ctx()
    torch = _torch()
    if fmt == N.SS_FMT_I16:
        raw = np.ascontiguousarray(samples, np.int16)
        n = len(raw) // 2
    else:
        raw = np.ascontiguousarray(samples.astype(np.complex64)).view(np.float32)
        n = len(samples)
    hop = n_fft if hop is None else hop
    frames = (n - n_fft) // hop + 1 if n >= n_fft else 0
    P = frames // plot_rows
    if P == 0:
        return ([], None) if return_tf else []
    span = (P * plot_rows - 1) * hop + n_fft
    raw = raw[: 2 * span]
    d = _dev(raw)
    tf = torch.empty((P, plot_rows, n_fft), dtype=torch.float32, device="cuda") if return_tf else None
    t, out = _batch_out(torch, P, n_fft, box_capacity)
    cfg = config.c()
    if hop == n_fft and window == 0:
        ctx.check(ctx.lib.ss_sense_batch(ctx.h, _ptr(d), fmt, n_fft, plot_rows, P, first_seq, float(sample_rate_hz),
                                         C.byref(cfg), _ptr(tf) if tf is not None else None, C.byref(out)))
    else:
        ctx.check(ctx.lib.ss_stft_sense_batch(ctx.h, _ptr(d), fmt, n_fft, hop, window, plot_rows, P, first_seq,
                                              float(sample_rate_hz), C.byref(cfg),
                                              _ptr(tf) if tf is not None else None, C.byref(out)))
    dets = _unpack_batch(t, P)
    return (dets, _host(tf)) if return_tf else dets


def test_libm(x: np.ndarray, which: int, variant: int = -1) -> np.ndarray:
    ctx = _ctx()
    d = _dev(x, np.float32)
    out = d.clone()
    ctx.check(ctx.lib.ss_test_libm(ctx.h, _ptr(d), len(x), which, variant, _ptr(out)))
    return _host(out)
