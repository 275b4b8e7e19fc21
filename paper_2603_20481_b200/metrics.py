"""Evaluation metrics (mirror of specsense::metrics, proj/include/specsense/
metrics.hpp:7-56): IoU of boxes in continuous seconds x Hz, the dense IoU
matrix, strict-theta match counts, P_D / P_FA / mean IoU and theta sweeps.
Host code: the GPU produces the boxes, these score them."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def iou(a, b) -> float:
    """a, b: (f0, f1, t0, t1).  Zero if either box has zero area (metrics.cpp:7-15)."""
    area_a = (a[1] - a[0]) * (a[3] - a[2])
    area_b = (b[1] - b[0]) * (b[3] - b[2])
    if area_a <= 0.0 or area_b <= 0.0:
        return 0.0
    fi = max(0.0, min(a[1], b[1]) - max(a[0], b[0]))
    ti = max(0.0, min(a[3], b[3]) - max(a[2], b[2]))
    inter = fi * ti
    return inter / (area_a + area_b - inter)


@dataclass
class IoUMatrix:
    n_gt: int
    n_det: int
    v: np.ndarray  # n_gt x n_det

    def row_max(self, g: int) -> float:
        return float(max(0.0, self.v[g].max())) if self.n_det else 0.0

    def col_max(self, d: int) -> float:
        return float(max(0.0, self.v[:, d].max())) if self.n_gt else 0.0


def iou_matrix(gt, detections) -> IoUMatrix:
    gt = np.asarray(gt, np.float64).reshape(-1, 4)
    det = np.asarray(detections, np.float64).reshape(-1, 4)
    # iou() broadcast over all pairs (same IEEE operations, same order)
    ga = ((gt[:, 1] - gt[:, 0]) * (gt[:, 3] - gt[:, 2]))[:, None]
    da = ((det[:, 1] - det[:, 0]) * (det[:, 3] - det[:, 2]))[None, :]
    fi = np.maximum(0.0, np.minimum(gt[:, None, 1], det[None, :, 1]) - np.maximum(gt[:, None, 0], det[None, :, 0]))
    ti = np.maximum(0.0, np.minimum(gt[:, None, 3], det[None, :, 3]) - np.maximum(gt[:, None, 2], det[None, :, 2]))
    inter = fi * ti
    with np.errstate(divide="ignore", invalid="ignore"):
        v = inter / (ga + da - inter)
    v = np.where((ga <= 0.0) | (da <= 0.0), 0.0, v).reshape(len(gt), len(det))
    return IoUMatrix(len(gt), len(det), v)


def count_matches(m: IoUMatrix, theta: float) -> tuple[int, int]:
    """(n_true, n_false): strict comparisons on both sides (metrics.hpp:27-33)."""
    n_true = sum(1 for g in range(m.n_gt) if m.row_max(g) > theta)
    n_false = sum(1 for d in range(m.n_det) if m.col_max(d) < theta)
    return n_true, n_false


@dataclass
class EvalResult:
    theta: float
    n_gt: int
    n_det: int
    n_true: int
    n_false: int
    p_d: float
    p_fa: float
    mean_iou: float


def evaluate(m_or_gt, detections=None, theta: float = 0.5) -> EvalResult:
    m = m_or_gt if isinstance(m_or_gt, IoUMatrix) else iou_matrix(m_or_gt, detections)
    t, f = count_matches(m, theta)
    s = 0.0
    for g in range(m.n_gt):
        s += m.row_max(g)
    return EvalResult(theta, m.n_gt, m.n_det, t, f, t / m.n_gt if m.n_gt else 0.0,
                      f / m.n_det if m.n_det else 0.0, s / m.n_gt if m.n_gt else 0.0)


def sweep(gt, detections, thetas) -> list[EvalResult]:
    m = iou_matrix(gt, detections)
    return [evaluate(m, theta=th) for th in thetas]
