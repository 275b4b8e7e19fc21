"""GPU parity of the baseline detector (ss_baseline_detect: SAT + kernel bank on
the device, greedy growth on the host) against the reference's own
baseline::baseline_detect (proj/src/baseline.cpp:103-176) on the same TF
plots: every box bit-identical, for default and non-default configs."""
import numpy as np
import pytest

from paper_2603_20481_b200 import baseline as bl
from paper_2603_20481_b200 import signals

pytestmark = pytest.mark.gpu


def _cmp(tf, fs, start_seq, cfg, ref):
    got, bins = bl.baseline_detect(tf, fs, start_seq, cfg)
    exp = ref.baseline_detect(tf, start_seq, fs, cfg.conv_threshold, cfg.rate_change_threshold, cfg.noise_offset_db,
                              cfg.max_kernel_rows, cfg.max_kernel_cols)
    assert got.shape == exp.shape
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    assert np.all(bins[:, 0] < bins[:, 1]) and np.all(bins[:, 2] < bins[:, 3])
    return len(got)


def test_baseline_paper_plot(ss, ref):
    sc = signals.paper_scenario(rows=1000)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    tf = ref.make_plots(iq, 100e6, 1024, 500)
    for p in range(2):
        assert _cmp(tf[p], 100e6, p * 500, bl.BaselineConfig(), ref) > 0


@pytest.mark.parametrize("cfg", [bl.BaselineConfig(conv_threshold=3.0, rate_change_threshold=0.7, noise_offset_db=6.0),
                                 bl.BaselineConfig(max_kernel_rows=16, max_kernel_cols=64),
                                 bl.BaselineConfig(conv_threshold=1.2, rate_change_threshold=0.3)])
def test_baseline_configs(ss, ref, cfg):
    sc = signals.paper_scenario(rows=500)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    tf = ref.make_plots(iq, 100e6, 1024, 500)[0]
    _cmp(tf, 100e6, 7, cfg, ref)


def test_baseline_small_plots(ss, ref):
    rng = np.random.default_rng(3)
    for rows, cols in [(128, 256), (40, 64), (1, 32), (33, 31)]:
        tf = rng.exponential(1.0, (rows, cols)).astype(np.float32)
        tf[rows // 3: rows // 2 + 1, cols // 4: cols // 3 + 1] *= 30
        _cmp(np.sqrt(tf), 1e6, 0, bl.BaselineConfig(), ref)


def test_baseline_compare_table(ss, ref):
    """compare(): pipeline and baseline on the same plots, pooled P_D/P_FA/IoU."""
    sc = signals.paper_scenario(rows=1000)
    iq, truth = ref.synthesize(signals.scenario_json(sc))
    tf = ref.make_plots(iq, 100e6, 1024, 500)
    gt = []
    for p in range(2):
        t0, t1 = p * 500 * 1024 / 100e6, (p + 1) * 500 * 1024 / 100e6
        g = [b[:4] for b in truth if b[2] < t1 and b[3] > t0]
        gt.append([[b[0], b[1], max(b[2], t0), min(b[3], t1)] for b in g])
    rows, speedup = bl.compare(list(tf), gt, 100e6, theta=0.5, start_seqs=[0, 500])
    assert [r.detector for r in rows] == ["pipeline", "baseline"] and speedup > 0
    assert 0.0 <= rows[0].p_d <= 1.0 and rows[0].mean_latency_s > 0
