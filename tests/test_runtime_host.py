"""CPU tests of the streaming-runtime host logic (paper_2603_20481_b200/runtime.py):
the report arithmetic against the reference's own runtime::summarize /
RunReport::ccdf (proj/src/runtime.cpp:166-214) built in oracle/_ref, config
validation (runtime.hpp:13-24), and that the engine entry points fail
loudly without a GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_20481_b200 import _native as N
from paper_2603_20481_b200 import runtime as rt
from paper_2603_20481_b200.specsense import ValidationError


@pytest.mark.parametrize("n", [1, 7, 99, 100, 101, 1000])
def test_summarize_matches_reference(ref, n):
    rng = np.random.default_rng(n)
    lat = np.round(rng.exponential(0.004, n), 4)        # rounding makes ties
    idx = rng.permutation(n).astype(np.uint64) + 5
    deadline = 0.005
    met = (lat <= deadline).astype(np.int32)
    recs = [rt.PlotRecord(int(i), 0, float(l), deadline, bool(m), 0) for i, l, m in zip(idx, lat, met)]
    got = rt.summarize(recs, 3, deadline)
    exp, ccdf = ref.summarize(idx, lat, met, 3, deadline)
    assert got.plots == exp["plots"] and got.overruns == exp["overruns"]
    assert got.fraction_met == exp["fraction_met"] and got.realtime_met == bool(exp["realtime_met"])
    assert (got.p50_s, got.p90_s, got.p99_s, got.max_s) == (exp["p50_s"], exp["p90_s"], exp["p99_s"], exp["max_s"])
    assert got.percentiles_valid == bool(exp["percentiles_valid"])
    assert got.ccdf() == ccdf
    assert [r.plot_index for r in got.records] == sorted(idx.tolist())


def test_summarize_empty(ref):
    got = rt.summarize([], 2, 0.02)
    exp, ccdf = ref.summarize([], [], [], 2, 0.02)
    assert got.plots == 0 and got.overruns == 2 and got.fraction_met == exp["fraction_met"] == 0.0
    assert got.realtime_met is False and got.ccdf() == ccdf == []


def test_nearest_rank():
    """runtime.hpp:92-94: element ceil(q*n), 1-based, clamped to [1, n]."""
    v = [1.0, 2.0, 3.0, 4.0, 5.0]
    assert rt.nearest_rank(v, 0.0) == 1.0 and rt.nearest_rank(v, 0.5) == 3.0 and rt.nearest_rank(v, 1.0) == 5.0
    assert rt.nearest_rank(v, 0.99) == 5.0 and rt.nearest_rank(v, 0.2) == 1.0
    assert rt.nearest_rank([], 0.5) == 0.0      # runtime.cpp:171


def test_runtime_config_validation():
    rt.RuntimeConfig().validate()
    for bad in (dict(n_compute_workers=0), dict(n_sensing_workers=0), dict(halo_bins=2), dict(deadline_s=-1.0),
                dict(chunk_queue_capacity=-1)):
        with pytest.raises(ValidationError):
            rt.RuntimeConfig(**bad).validate()


def test_memory_source_blocks():
    x = (np.arange(10 * 16) + 1j).astype(np.complex64)
    src = rt.MemorySource(x, 16, total_chunks=25, block=4, pinned=False)
    seqs, total = [], 0
    for seq, blk in src.blocks():
        k = blk.size // 16
        assert np.array_equal(blk, np.concatenate([x[((seq + i) % 10) * 16:((seq + i) % 10 + 1) * 16]
                                                   for i in range(k)]))
        seqs.append(seq)
        total += k
    assert total == 25 and seqs[0] == 0 and all(b > a for a, b in zip(seqs, seqs[1:]))
    i16 = np.zeros(2 * 16 * 3, np.int16)
    assert rt.MemorySource(i16, 16, pinned=False).chunks == 3


def test_engine_open_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    lib = N.load()
    h = C.c_void_p()
    cfg = N.EngineCfg(1024, 100, 0, 1e6, 2, 0, 0.0, 64)
    det = N.DetectorCfg()
    lib.ss_default_detector_cfg(C.byref(det))
    assert lib.ss_engine_open(0, C.byref(cfg), C.byref(det), C.byref(h)) == N.SS_ECUDA
    assert not h.value
    with pytest.raises(Exception):
        rt.Engine(rt.FrontendConfig(1e6, 1024, 100))
