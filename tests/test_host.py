"""CPU tests of the host side: the C-ABI library loads and exports every symbol
include/specsense_b200.h declares, the C++ drop-in exports the reference's API,
host-only entry points behave, the workload generator is valid, and the N>1
capture-sharding + detection gather runs on gloo with world_size 2."""
import ctypes as C
import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2603_20481_b200 import _native as N, parallel, signals

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    hdr = (ROOT / "include" / "specsense_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", hdr)))


def test_header_symbols_exported():
    lib = N.load()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.SIGNATURES), "ctypes binding must cover the header exactly"


def test_cpp_dropin_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", str(N.lib_path())], capture_output=True, text=True).stdout
    for sym in ["specsense::frontend::fft_row(", "specsense::frontend::make_plot(", "specsense::frontend::make_plots(",
                "specsense::detector::estimate_psd(", "specsense::detector::estimate_psd_into(",
                "specsense::detector::savgol_smooth(", "specsense::detector::smooth_and_floor(",
                "specsense::detector::prune_columns(", "specsense::detector::otsu_threshold(",
                "specsense::detector::binarize(", "specsense::detector::binarize_columns(",
                "specsense::detector::morphology(", "specsense::detector::morphology_cols(",
                "specsense::detector::consolidate(", "specsense::detector::label_components(",
                "specsense::detector::component_extents(", "specsense::detector::extent_to_bin_box(",
                "specsense::detector::bin_box_to_physical(", "specsense::detector::detect(",
                "specsense::detector::DetectorConfig::validate(", "specsense::frontend::FrontendConfig::validate(",
                "specsense::runtime::run(", "specsense::runtime::summarize(", "specsense::runtime::nearest_rank(",
                "specsense::runtime::partition(", "specsense::runtime::consolidate_sliced(",
                "specsense::runtime::RunReport::ccdf(", "specsense::runtime::RuntimeConfig::validate(",
                "specsense::baseline::baseline_detect(", "specsense::baseline::kernel_sizes(",
                "specsense::baseline::BaselineConfig::validate("]:
        assert sym in out, sym


def test_host_only_entry_points(ora):
    lib = N.load()
    assert lib.ss_abi_version() == 1
    cfg = N.DetectorCfg()
    lib.ss_default_detector_cfg(C.byref(cfg))
    assert (cfg.savgol_window, cfg.savgol_order, cfg.psd_margin_db, cfg.min_component_area,
            cfg.one_d_opening_along_time) == (31, 3, 3.0, 4, 0)
    assert lib.ss_fft_twiddle_count(1000) == -1
    # the device twiddle table is the SSFFT-1 canonical table re-laid out per pass
    canon = ora.ssfft_table(4096)
    n = lib.ss_fft_twiddle_count(4096)
    tw = np.empty((n, 2), np.float64)
    assert lib.ss_fft_twiddles(4096, tw.ctypes.data_as(C.c_void_p)) == 0
    # pass 1 (Ns=16, R=16): entry (r-1)*16 + k = tw[r*k*16]
    for r in range(1, 16):
        for k in range(16):
            assert np.array_equal(tw[(r - 1) * 16 + k], canon[r * k * 16])
    off = 15 * 16
    for r in (1, 7, 15):
        for k in (0, 1, 100, 255):
            assert np.array_equal(tw[off + (r - 1) * 256 + k], canon[r * k])


def test_open_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    lib = N.load()
    h = C.c_void_p()
    assert lib.ss_open(0, C.byref(h)) == N.SS_ECUDA
    from paper_2603_20481_b200 import specsense as ss
    with pytest.raises(ss.Error):
        ss.make_plots(np.zeros(2048, np.complex64), 1e6, 1024, 1)


def test_c5_scenarios_valid(ref):
    """The config-5 sampler stays inside the reference's Scenario::validate
    (signals.cpp:128-146) and its ranges."""
    for i in range(16):
        sc = signals.c5_scenario(i)
        assert len(sc["signals"]) == 16
        for s in sc["signals"]:
            assert 5e6 <= s["bandwidth_hz"] <= 40e6 and 0.1e-3 <= s["duration_s"] <= 5e-3
            assert -50e6 <= s["center_freq_hz"] - s["bandwidth_hz"] / 2
            assert s["center_freq_hz"] + s["bandwidth_hz"] / 2 <= 50e6
            assert 0 <= s["t_start_s"] and s["t_start_s"] + s["duration_s"] <= 0.1
    small = dict(sample_rate_hz=1e6, duration_s=0.002, noise_power=1.0, seed=5,
                 signals=[dict(kind="ofdm-like", center_freq_hz=c, bandwidth_hz=50e3, t_start_s=2e-4,
                               duration_s=1e-3, power=1.0) for c in (-1e5, 0.0, 2e5)])
    iq, truth = ref.synthesize(signals.scenario_json(small))
    assert len(iq) == 2000 and truth.shape == (3, 5)
    assert np.allclose(truth[:, :4], signals.truth_boxes(small))


def test_capture_shard():
    for total in (0, 1, 7, 296, 1000):
        for world in (1, 2, 3, 8):
            shards = [parallel.capture_shard(total, r, world) for r in range(world)]
            assert sum(len(s) for s in shards) == total
            assert [i for s in shards for i in s] == list(range(total))
            assert max(len(s) for s in shards) - min(len(s) for s in shards) <= 1


def _gloo_worker(rank, world, port, q):
    """One rank of bench.py's exchange step: detections (counts + fixed-capacity
    records, as ss_sense_batch writes them) gathered to rank 0 with the exact
    function bench.measure() calls each timed step."""
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, K = 3, 5
    n = torch.tensor([rank + 1, 0, 7 if rank else 2], dtype=torch.int32)   # 7 > K: clamped like the device capacity
    b = torch.full((P, K, 4), float(rank), dtype=torch.float64)
    b[:, :, 0] += torch.arange(P, dtype=torch.float64)[:, None]
    b[:, :, 1] += torch.arange(K, dtype=torch.float64)[None, :]
    g = parallel.gather_detections(n, b)
    if rank == 0:
        flat = parallel.flatten_detections(g)
        q.put(json.dumps({"counts": [c.tolist() for c, _ in g], "sizes": [list(p.shape) for _, p in g],
                          "lens": [len(x) for x in flat], "first": flat[0].tolist(), "last": flat[-1].tolist()}))
    else:
        assert g is None
    dist.destroy_process_group()


def test_gather_detections_gloo_world2():
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = json.loads(q.get(timeout=300))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["counts"] == [[1, 0, 2], [2, 0, 5]]
    assert res["sizes"] == [[3, 4], [7, 4]]                # only the boxes that exist travel
    assert res["lens"] == [1, 0, 2, 2, 0, 5]
    assert res["first"] == [[0.0, 0.0, 0.0, 0.0]]
    assert res["last"] == [[3.0, 1.0, 1.0, 1.0], [3.0, 2.0, 1.0, 1.0], [3.0, 3.0, 1.0, 1.0], [3.0, 4.0, 1.0, 1.0],
                           [3.0, 5.0, 1.0, 1.0]]
