"""CPU tests of the baseline's host-side pieces: kernel_sizes (host-only ABI)
against the reference's baseline::kernel_sizes, config validation
(baseline.cpp:89-94), and the metrics mirror against the reference's iou."""
import numpy as np
import pytest

from paper_2603_20481_b200 import baseline as bl
from paper_2603_20481_b200 import metrics
from paper_2603_20481_b200.specsense import ValidationError


@pytest.mark.parametrize("rows,cols,mkr,mkc", [(2000, 1024, 0, 0), (500, 1024, 0, 0), (1, 1, 0, 0), (7, 300, 0, 0),
                                               (2441, 4096, 64, 256), (128, 256, 200, 3)])
def test_kernel_sizes_match_reference(ref, rows, cols, mkr, mkc):
    cfg = bl.BaselineConfig(max_kernel_rows=mkr, max_kernel_cols=mkc)
    assert np.array_equal(np.array(bl.kernel_sizes(rows, cols, cfg)).reshape(-1, 2),
                          ref.kernel_sizes(rows, cols, mkr=mkr, mkc=mkc))


def test_baseline_config_validation():
    for bad in (dict(conv_threshold=0.0), dict(rate_change_threshold=-1.0), dict(max_kernel_rows=-1),
                dict(max_kernel_cols=-2)):
        with pytest.raises(ValidationError):
            bl.kernel_sizes(10, 10, bl.BaselineConfig(**bad))
    with pytest.raises(ValidationError):
        bl.kernel_sizes(0, 10)


def test_iou_matches_reference(ref):
    rng = np.random.default_rng(5)
    for _ in range(300):
        a = np.sort(rng.uniform(-5, 5, 2)).tolist() + np.sort(rng.uniform(0, 3, 2)).tolist()
        b = np.sort(rng.uniform(-5, 5, 2)).tolist() + np.sort(rng.uniform(0, 3, 2)).tolist()
        if rng.random() < 0.1:
            b = list(a)
        if rng.random() < 0.05:
            a[1] = a[0]                      # zero area
        assert metrics.iou(a, b) == ref.iou(np.array(a), np.array(b))


def test_metrics_counts():
    gt = [[0, 10, 0, 1], [20, 30, 0, 1]]
    det = [[0, 10, 0, 1], [100, 110, 5, 6], [20, 30, 0, 0.5]]
    m = metrics.iou_matrix(gt, det)
    assert m.v.shape == (2, 3) and m.v[0, 0] == 1.0 and m.v[1, 2] == 0.5
    assert metrics.count_matches(m, 0.5) == (1, 1)          # strict on both sides: 0.5 is neither
    r = metrics.evaluate(m, theta=0.4)
    assert (r.n_true, r.n_false, r.p_d, r.p_fa, r.mean_iou) == (2, 1, 1.0, 1 / 3, 0.75)
    assert [e.n_true for e in metrics.sweep(gt, det, [0.2, 0.6, 0.99])] == [2, 1, 1]
    row = bl.make_compare_row("x", [det], [gt], 0.4, 1e-3)
    assert (row.p_d, row.p_fa, row.mean_iou) == (1.0, 1 / 3, 0.75)
