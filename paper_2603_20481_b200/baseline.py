"""Python mirror of specsense::baseline (proj/include/specsense/baseline.hpp):
the Searchlight-style comparison detector on the GPU (ss_baseline_detect:
SAT + dyadic kernel bank on the device, greedy growth on the host, bit-identical
to the reference) and the pipeline-vs-baseline comparison table."""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import metrics
from .specsense import DetectorConfig, Error, ValidationError, _ctx, _dev, _ptr, detect


@dataclass
class BaselineConfig:
    conv_threshold: float = 2.0
    rate_change_threshold: float = 0.5
    noise_offset_db: float = 3.0
    max_kernel_rows: int = 0
    max_kernel_cols: int = 0

    def c(self) -> N.BaselineCfg:
        return N.BaselineCfg(self.conv_threshold, self.rate_change_threshold, self.noise_offset_db,
                             self.max_kernel_rows, self.max_kernel_cols)

    def validate(self):
        if not self.conv_threshold > 0:
            raise ValidationError("conv_threshold must be > 0")
        if not self.rate_change_threshold > 0:
            raise ValidationError("rate_change_threshold must be > 0")
        if self.max_kernel_rows < 0 or self.max_kernel_cols < 0:
            raise ValidationError("kernel caps must be >= 0")


def kernel_sizes(rows: int, cols: int, config: BaselineConfig | None = None) -> list[tuple[int, int]]:
    """baseline::kernel_sizes (host-only ABI call)."""
    config = config or BaselineConfig()
    config.validate()
    if rows < 1 or cols < 1:
        raise ValidationError("plot must be non-empty")
    lib = N.load()
    out = (C.c_int32 * (2 * 4096))()
    n = lib.ss_baseline_kernel_sizes(rows, cols, C.byref(config.c()), out, 4096)
    if n < 0:
        raise ValidationError("kernel_sizes failed")
    return [(out[2 * i], out[2 * i + 1]) for i in range(n)]


def baseline_detect(tf: np.ndarray, sample_rate_hz: float = 1e6, start_seq: int = 0,
                    config: BaselineConfig | None = None, cap: int = 1 << 16):
    """Boxes (n, 4) f64 [f0, f1, t0, t1] and bin boxes (n, 4) i32, sorted by (t0, f0, t1, f1)."""
    config = config or BaselineConfig()
    ctx = _ctx()
    tf = np.ascontiguousarray(tf, np.float32)
    rows, cols = tf.shape
    d = _dev(tf)
    boxes = np.zeros((cap, 4), np.float64)
    bins = np.zeros((cap, 4), np.int32)
    n = C.c_int(0)
    ctx.check(ctx.lib.ss_baseline_detect(ctx.h, _ptr(d), rows, cols, start_seq, float(sample_rate_hz),
                                         C.byref(config.c()), boxes.ctypes.data_as(C.c_void_p),
                                         bins.ctypes.data_as(C.c_void_p), cap, C.byref(n)))
    return boxes[: n.value].copy(), bins[: n.value].copy()


@dataclass
class CompareRow:
    detector: str
    mean_latency_s: float
    p_d: float
    p_fa: float
    mean_iou: float


def make_compare_row(name: str, detections_per_plot, truth_per_plot, theta: float,
                     mean_latency_s: float) -> CompareRow:
    """baseline.cpp:178-205: pooled P_D / P_FA / mean IoU over plots."""
    if len(detections_per_plot) != len(truth_per_plot):
        raise ValidationError("detections/truth plot counts differ")
    n_gt = n_det = n_true = n_false = 0
    iou_sum = 0.0
    for det, gt in zip(detections_per_plot, truth_per_plot):
        m = metrics.iou_matrix(gt, det)
        t, f = metrics.count_matches(m, theta)
        n_gt += m.n_gt
        n_det += m.n_det
        n_true += t
        n_false += f
        for g in range(m.n_gt):
            iou_sum += m.row_max(g)
    return CompareRow(name, mean_latency_s, n_true / n_gt if n_gt else 0.0, n_false / n_det if n_det else 0.0,
                      iou_sum / n_gt if n_gt else 0.0)


def compare(plots, truth_per_plot, sample_rate_hz: float, detector_config: DetectorConfig | None = None,
            baseline_config: BaselineConfig | None = None, theta: float = 0.5, start_seqs=None):
    """baseline::compare (baseline.cpp:207-232) with both detectors on the GPU:
    rows [pipeline, baseline] and speedup = baseline / pipeline mean latency."""
    if len(plots) != len(truth_per_plot):
        raise ValidationError("plots/truth counts differ")
    if not len(plots):
        raise ValidationError("compare needs at least one plot")
    import torch

    start_seqs = start_seqs or [0] * len(plots)
    pipe, base = [], []
    pipe_s = base_s = 0.0
    for tf, s0 in zip(plots, start_seqs):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pipe.append(detect(tf, detector_config, sample_rate_hz=sample_rate_hz, start_seq=s0).boxes)
        torch.cuda.synchronize()
        pipe_s += time.perf_counter() - t0
        t0 = time.perf_counter()
        base.append(baseline_detect(tf, sample_rate_hz, s0, baseline_config)[0])
        torch.cuda.synchronize()
        base_s += time.perf_counter() - t0
    n = len(plots)
    rows = [make_compare_row("pipeline", pipe, truth_per_plot, theta, pipe_s / n),
            make_compare_row("baseline", base, truth_per_plot, theta, base_s / n)]
    return rows, (base_s / pipe_s if pipe_s > 0 else 0.0)
