"""GPU tests of the streaming engine (ss_engine_*, csrc/engine.cpp) -- the
B200 form of runtime::run + PingPongBuffer (proj/src/runtime.cpp:221-487,
proj/include/specsense/frontend.hpp:86-135).  Every window's boxes must be
bit-identical to the batch pipeline on the same samples and to the
reference engine itself (oracle/_ref runtime::run over a MemorySource);
bank/overrun accounting follows the PingPongBuffer rules."""
import threading
import time

import numpy as np
import pytest

from paper_2603_20481_b200 import runtime as rt
from paper_2603_20481_b200 import signals

# a blocked push never returns to Python: kill the process instead of hanging the suite
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(240, method="thread")]

FS, F, T = 100e6, 1024, 500


def _stream(ref, rows_total):
    sc = signals.paper_scenario(rows=rows_total)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    return np.ascontiguousarray(iq[: rows_total * F])


def _drain(eng, n, wait_ms=5000):
    out = []
    for _ in range(n):
        got = eng.poll(wait_ms)
        assert got is not None
        out.append(got)
    return out


def test_engine_windows_match_batch_and_reference(ss, ref):
    iq = _stream(ref, 6 * T)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), runtime_config=rt.RuntimeConfig(box_capacity=2048))
    recs = []
    for w in range(6):                      # push a window, poll it (ping-pong never fills)
        eng.push(iq[w * T * F:(w + 1) * T * F], w * T)
        recs += _drain(eng, 1)
    eng.finish()
    assert eng.poll(100) is None
    st = eng.stats()
    assert st["windows_completed"] == 6 and st["overruns"] == 0 and st["pending"] == 0
    dets = ss.sense(iq, FS, F, T, box_capacity=2048)
    exp_ref, seen = ref.run_engine_boxes(iq, FS, F, T, 6)
    assert seen == 6
    for w, (rec, boxes, bins) in enumerate(recs):
        assert rec.plot_index == w and rec.start_seq == w * T
        assert 0 < rec.latency_s < 1.0 and rec.complete_s <= rec.done_s
        assert rec.met == (rec.latency_s <= rec.deadline_s)
        assert rec.deadline_s == pytest.approx(T * F / FS)
        d = dets[w]
        assert rec.n_boxes == len(d.boxes) and rec.n_active == len(d.active_columns)
        assert np.array_equal(boxes.view(np.uint64), d.boxes.view(np.uint64))
        assert np.array_equal(bins, d.bin_boxes)
        e = exp_ref.get(w, np.zeros((0, 4)))
        assert np.array_equal(boxes.view(np.uint64), np.asarray(e, np.float64).reshape(-1, 4).view(np.uint64))
    eng.close()


def test_engine_chunk_granular_pushes(ss, ref):
    """Rows arriving in odd-sized pushes that straddle window boundaries (3 banks:
    nobody polls until the end, and an unpaced push waits for a held bank)."""
    iq = _stream(ref, 3 * T)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), runtime_config=rt.RuntimeConfig(n_banks=3))
    seq = 0
    sizes = [1, 7, 300, 191, 2, 499, 250, 250]
    for k in sizes:
        eng.push(iq[seq * F:(seq + k) * F], seq)
        seq += k
    assert seq == 3 * T
    eng.finish()
    recs = []
    while (got := eng.poll(2000)) is not None:
        recs.append(got)
    dets = ss.sense(iq, FS, F, T)
    assert [r.plot_index for r, _, _ in recs] == [0, 1, 2]
    for (r, boxes, _), d in zip(recs, dets):
        assert np.array_equal(boxes, d.boxes)
    eng.close()


def test_paced_overrun_accounting(ref):
    """Paced: rows of a window whose bank is still held are shed and counted once (PingPongBuffer)."""
    iq = _stream(ref, 8 * T)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), paced=True)
    for w in range(6):                     # nobody polls: windows 0, 1 hold both banks
        eng.push(iq[w * T * F:(w + 1) * T * F], w * T)
    st = eng.stats()
    assert st["windows_completed"] == 2 and st["overruns"] == 4 and st["rows_retired"] == 6 * T
    got = _drain(eng, 2)
    assert [g[0].plot_index for g in got] == [0, 1]
    for w in (6, 7):                       # banks free again
        eng.push(iq[w * T * F:(w + 1) * T * F], w * T)
    got = _drain(eng, 2)
    assert [g[0].plot_index for g in got] == [6, 7]
    assert eng.stats()["overruns"] == 4
    eng.close()


def test_unpaced_back_pressure_no_loss(ss, ref):
    """Unpaced: the writer blocks on a held bank instead of dropping (row_slot_blocking)."""
    iq = _stream(ref, 6 * T)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T))

    def writer():
        for w in range(6):
            eng.push(iq[w * T * F:(w + 1) * T * F], w * T)
        eng.finish()

    th = threading.Thread(target=writer)
    th.start()
    recs = []
    while True:
        time.sleep(0.01)                   # a slow reader
        got = eng.poll(5000)
        if got is None:
            break
        recs.append(got)
    th.join()
    assert [r.plot_index for r, _, _ in recs] == list(range(6))
    assert eng.stats()["overruns"] == 0
    dets = ss.sense(iq, FS, F, T)
    for (r, boxes, _), d in zip(recs, dets):
        assert np.array_equal(boxes, d.boxes)
    eng.close()


def test_lost_range_drops_window(ss, ref):
    iq = _stream(ref, 4 * T)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), runtime_config=rt.RuntimeConfig(n_banks=4))
    eng.push(iq[: T * F], 0)
    eng.push(iq[T * F:(T + 100) * F], T)
    eng.mark_lost(T + 100, T + 120)       # 20 rows of window 1 never arrive
    eng.push(iq[(T + 120) * F:2 * T * F], T + 120)
    eng.push(iq[2 * T * F:4 * T * F], 2 * T)
    eng.finish()
    recs = []
    while (got := eng.poll(2000)) is not None:
        recs.append(got)
    assert [r.plot_index for r, _, _ in recs] == [0, 2, 3]
    assert eng.stats()["overruns"] == 1
    dets = ss.sense(iq, FS, F, T)
    for r, boxes, _ in recs:
        assert np.array_equal(boxes, dets[r.plot_index].boxes)
    eng.close()


def test_run_report_and_handler(ss, ref):
    """runtime::run mirror: unpaced MemorySource cycling 3 windows of samples over 12 windows."""
    iq = _stream(ref, 3 * T)
    seen = {}
    rep = rt.run(rt.MemorySource(iq, F, total_chunks=12 * T, block=97), rt.FrontendConfig(FS, F, T),
                 on_detections=lambda r, b: seen.setdefault(r.plot_index, b))
    assert rep.plots == 12 and rep.overruns == 0 and sorted(seen) == list(range(12))
    assert rep.p50_s <= rep.p90_s <= rep.p99_s <= rep.max_s and rep.fraction_met == 1.0 and rep.realtime_met
    dets = ss.sense(iq, FS, F, T)
    for w in range(12):
        d = dets[w % 3]
        assert len(seen[w]) == len(d.boxes)
        # start_seq differs per cycle: times move, frequencies are identical
        assert np.array_equal(seen[w][:, :2], d.boxes[:, :2])


def test_run_aborts_cleanly_on_manager_error(ref):
    """A failing detection handler (or a window over the box capacity) must end
    run() with the error, not deadlock: the unpaced ingest thread is then
    blocked on a bank only the (gone) reader would release.  runtime.cpp:466-478
    rethrows worker failures after joining."""
    iq = _stream(ref, 3 * T)

    def handler(r, b):
        if r.plot_index == 1:
            raise RuntimeError("handler failed")

    t0 = time.perf_counter()
    with pytest.raises(RuntimeError, match="handler failed"):
        rt.run(rt.MemorySource(iq, F, total_chunks=40 * T, block=97), rt.FrontendConfig(FS, F, T),
               on_detections=handler)
    # capacity below the window's box count: the engine reports it, run() returns the error
    with pytest.raises(rt.Error, match="capacity"):
        rt.run(rt.MemorySource(iq, F, total_chunks=40 * T, block=97), rt.FrontendConfig(FS, F, T),
               runtime_config=rt.RuntimeConfig(box_capacity=1))
    assert time.perf_counter() - t0 < 120


def test_int16_engine(ss, ref):
    iq = _stream(ref, 2 * T)
    v = np.clip(iq.view(np.float32) * np.float32(2.0 ** -6) * np.float32(32768.0), -32768, 32767)
    q = np.rint(v).astype(np.int16)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), fmt=1)
    eng.push(q, 0)
    got = _drain(eng, 2)
    dets = ss.sense(q, FS, F, T, fmt=1)
    for (r, boxes, _), d in zip(got, dets):
        assert np.array_equal(boxes, d.boxes)
    eng.close()


def test_engine_validation():
    from paper_2603_20481_b200.specsense import ValidationError
    with pytest.raises(ValidationError):
        rt.Engine(rt.FrontendConfig(FS, 1000, T))
    with pytest.raises(ValidationError):
        rt.Engine(rt.FrontendConfig(FS, F, T), runtime_config=rt.RuntimeConfig(n_banks=1))


@pytest.mark.parametrize("hop,window", [(512, 1), (256, 1), (1024, 1)])
def test_stft_engine_matches_batch(ss, ref, hop, window):
    """The engine with the STFT extension (frames every hop samples, Hann):
    windows overlap by F - hop samples, so boundary chunks feed two banks.
    Every window equals ss_stft_sense_batch on the same stream."""
    n_win, T = 4, 300
    n = n_win * T * hop + F - hop
    n_chunks = (n + F - 1) // F
    iq = np.resize(_stream(ref, 3 * T), n_chunks * F).astype(np.complex64)
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), hop=hop, window=window)
    out = []

    def reader():
        while (got := eng.poll(10000)) is not None:
            out.append(got)

    th = threading.Thread(target=reader)
    th.start()
    seq, k, sizes = 0, 0, [5, 97, 1, 300, 2, 64, 128, 700, 33]
    while seq < n_chunks:
        m = min(sizes[k % len(sizes)], n_chunks - seq)
        eng.push(iq[seq * F:(seq + m) * F], seq)
        seq += m
        k += 1
    eng.finish()
    th.join()
    dets = ss.sense(iq, FS, F, T, hop=hop, window=window, box_capacity=1024)
    assert [r.plot_index for r, _, _ in out] == list(range(len(dets))) and len(dets) >= n_win
    for r, boxes, bins in out:
        d = dets[r.plot_index]
        assert r.start_seq == r.plot_index * T
        assert np.array_equal(boxes.view(np.uint64), d.boxes.view(np.uint64)), r.plot_index
        assert np.array_equal(bins, d.bin_boxes)
    assert eng.stats()["overruns"] == 0
    eng.close()


def test_sharded_engines_cover_every_window(ss, ref):
    """Multi-GPU form of the engine: windows dealt round-robin over shard_count
    engines (here two engines on the one visible device): every window sensed
    exactly once, each bit-identical to the batch pipeline."""
    iq = _stream(ref, 3 * T)
    seen = {}
    rep = rt.run(rt.MemorySource(iq, F, total_chunks=9 * T, block=61), rt.FrontendConfig(FS, F, T),
                 on_detections=lambda r, b: seen.setdefault(r.plot_index, []).append(b), devices=[0, 0])
    assert rep.plots == 9 and rep.overruns == 0 and sorted(seen) == list(range(9))
    assert all(len(v) == 1 for v in seen.values())
    dets = ss.sense(iq, FS, F, T)
    for w in range(9):
        assert np.array_equal(seen[w][0][:, :2], dets[w % 3].boxes[:, :2])
    # one shard alone: only its own windows, no overruns for the skipped ones
    eng = rt.Engine(rt.FrontendConfig(FS, F, T), shard=(1, 3))
    eng.push(iq[: 3 * T * F], 0)
    eng.push(iq[: 3 * T * F], 3 * T)
    eng.finish()
    got = []
    while (g := eng.poll(2000)) is not None:
        got.append(g[0].plot_index)
    assert got == [1, 4] and eng.stats()["overruns"] == 0
    eng.close()
    with pytest.raises(Exception):
        rt.Engine(rt.FrontendConfig(FS, F, T), shard=(3, 3))


def test_async_pushes_match_synchronous(ss, ref):
    """ss_engine_push_async (DMAs out of an unchanging pinned buffer only queue;
    push_fence waits for them) delivers the same windows as synchronous pushes."""
    import torch

    iq = _stream(ref, 4 * T)
    pinned = torch.from_numpy(iq.view(np.float32)).pin_memory()
    host = pinned.numpy().view(np.complex64)
    out = {}
    for stable in (False, True):
        eng = rt.Engine(rt.FrontendConfig(FS, F, T), runtime_config=rt.RuntimeConfig(n_banks=4))
        for s0 in range(0, 4 * T, 250):  # 250-row pushes: DMA'd straight from the pinned buffer
            eng.push(host[s0 * F:(s0 + 250) * F], s0, stable=stable)
        if stable:
            eng.push_fence()
        eng.finish()
        recs = []
        while (got := eng.poll(2000)) is not None:
            recs.append(got)
        eng.close()
        out[stable] = recs
    assert [r.plot_index for r, _, _ in out[True]] == [0, 1, 2, 3]
    for (ra, ba, ia), (rb, bb, ib) in zip(out[False], out[True]):
        assert ra.plot_index == rb.plot_index and ra.n_boxes == rb.n_boxes
        assert np.array_equal(ba.view(np.uint64), bb.view(np.uint64)) and np.array_equal(ia, ib)
    dets = ss.sense(iq, FS, F, T)
    for (r, boxes, _), d in zip(out[True], dets):
        assert np.array_equal(boxes.view(np.uint64), d.boxes.view(np.uint64))
