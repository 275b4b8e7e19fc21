"""GPU parity end to end: IQ -> TF plot -> PSD/floor/prune -> Otsu -> morphology
-> CCL -> boxes through the fused C-ABI pipeline (ss_sense_batch), against the
reference's make_plots + detect run on identical bytes rendered by the
reference's own signals::synthesize.  Every output is compared bit for bit."""
import numpy as np
import pytest

from paper_2603_20481_b200 import signals

pytestmark = pytest.mark.gpu


def _check(det, exp, tf_got=None, tf_exp=None):
    if tf_got is not None:
        assert np.array_equal(tf_got.view(np.uint32), tf_exp.view(np.uint32))
    assert np.array_equal(det.psd.raw.view(np.uint32), exp["raw"].view(np.uint32))
    assert np.array_equal(det.psd.smoothed.view(np.uint32), exp["smoothed"].view(np.uint32))
    assert np.float32(det.psd.noise_floor) == np.float32(exp["noise_floor"])
    assert np.float32(det.psd.threshold) == np.float32(exp["threshold"])
    assert np.array_equal(det.active_columns, exp["active"])
    assert np.array_equal(det.bin_boxes, exp["bin_boxes"])
    assert np.array_equal(det.boxes.view(np.uint64), exp["boxes"].view(np.uint64))


def _run(ss, ref, sc, n_fft, rows, fmt=0):
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    fs = sc["sample_rate_hz"]
    dets, tf = ss.sense(iq, fs, n_fft, rows, return_tf=True)
    exp_tf = ref.make_plots(iq, fs, n_fft, rows)
    assert len(dets) == len(exp_tf) > 0
    nb = 0
    for p, det in enumerate(dets):
        exp = ref.detect(exp_tf[p], start_seq=p * rows, fs=fs)
        _check(det, exp, tf[p], exp_tf[p])
        nb += len(det.boxes)
    return nb


def test_paper_config_T500(ss, ref):
    """(T, F) = (500, 1024) @ 100 MS/s -- the acceptance suite grid (acceptance.cpp:93)."""
    sc = signals.paper_scenario(rows=2000)
    assert _run(ss, ref, sc, 1024, 500) > 0


def test_paper_config_T2000(ss, ref):
    """(T, F) = (2000, 1024): the paper's real-time configuration."""
    sc = signals.paper_scenario(rows=4000)
    assert _run(ss, ref, sc, 1024, 2000) > 0


@pytest.mark.parametrize("capture", [0, 1])
def test_c5_rect_capture(ss, ref, capture):
    """BASELINE config 5 in reference-parity mode: 100 ms fp32 @ 100 MS/s, F = 4096
    rectangular, hop 4096 -> T = 2441 (tail dropped)."""
    sc = signals.c5_scenario(capture)
    _run(ss, ref, sc, 4096, 2441)


def test_c5_short_plots(ss, ref):
    """Config-5 captures cut into T = 500 plots (20.48 ms at F = 4096): more bursts clear the prune."""
    sc = signals.c5_scenario(5, duration_s=0.1)
    assert _run(ss, ref, sc, 4096, 500) > 0


def test_single_burst_iou(ss, ref):
    """test_detector.cpp:608-650: one 20 dB burst in a (128, 256) plot -> one box, IoU >= 0.6."""
    fs = 1e6
    bw = 100e3
    snr = 20.0
    sc = dict(sample_rate_hz=fs, duration_s=0.0328, noise_power=1.0, seed=77,
              signals=[dict(kind="ofdm-like", center_freq_hz=120e3, bandwidth_hz=bw, t_start_s=0.008,
                            duration_s=0.016, power=10 ** (snr / 10) * (1.0 / fs) * bw)])
    iq, truth = ref.synthesize(signals.scenario_json(sc))
    dets = ss.sense(iq, fs, 256, 128)
    assert len(dets) == 1 and len(dets[0].boxes) == 1
    assert ref.iou(dets[0].boxes[0], truth[0, :4]) >= 0.6
    _run(ss, ref, sc, 256, 128)


def test_noise_only(ss, ref):
    """test_detector.cpp:582-606: noise only -> no boxes, <= 5 % active columns."""
    sc = dict(sample_rate_hz=1e6, duration_s=0.1, noise_power=1.0, seed=2024, signals=[])
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    dets = ss.sense(iq, 1e6, 256, 128)
    assert len(dets) >= 3
    assert all(len(d.boxes) == 0 for d in dets)
    assert sum(len(d.active_columns) for d in dets) / (len(dets) * 256) <= 0.05
    _run(ss, ref, sc, 256, 128)


def test_int16_path(ss, ref):
    """int16 IQ (quantised with the reference's rule) through the fused pipeline."""
    sc = signals.paper_scenario(rows=1000)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    v = np.clip(np.asarray(iq).view(np.float32) * np.float32(2.0 ** -6) * np.float32(32768.0), -32768, 32767)
    q = np.rint(v).astype(np.int16)
    dets, tf = ss.sense(q, 100e6, 1024, 500, fmt=1, return_tf=True)
    as_f32 = (q.astype(np.float32) * np.float32(1 / 32768)).view(np.complex64)
    exp_tf = ref.make_plots(as_f32, 100e6, 1024, 500)
    for p, det in enumerate(dets):
        _check(det, ref.detect(exp_tf[p], start_seq=p * 500, fs=100e6), tf[p], exp_tf[p])


def test_detect_batch_matches_sense(ss, ref):
    sc = signals.paper_scenario(rows=1500)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    exp_tf = ref.make_plots(iq, 100e6, 1024, 500)
    dets = ss.detect_batch(exp_tf, 100e6, start_seq=[0, 500, 1000])
    for p, det in enumerate(dets):
        _check(det, ref.detect(exp_tf[p], start_seq=p * 500, fs=100e6))


def test_config_variants(ss, ref):
    """Non-default DetectorConfig: window/order/margin/min_area/vertical line opening."""
    sc = signals.paper_scenario(rows=1000)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    tf = ref.make_plots(iq, 100e6, 1024, 500)
    for cfg in [ss.DetectorConfig(savgol_window=15, savgol_order=2, psd_margin_db=1.5, min_component_area=9,
                                  one_d_opening_along_time=True),
                ss.DetectorConfig(savgol_window=51, savgol_order=4, psd_margin_db=0.5, min_component_area=1)]:
        dets = ss.detect_batch(tf, 100e6, cfg, start_seq=[0, 500])
        for p, det in enumerate(dets):
            exp = ref.detect(tf[p], start_seq=p * 500, fs=100e6, window=cfg.savgol_window,
                             order=cfg.savgol_order, margin_db=cfg.psd_margin_db,
                             min_area=cfg.min_component_area, along_time=cfg.one_d_opening_along_time)
            _check(det, exp)


def test_config_validation(ss):
    tf = np.ones((1, 10, 16), np.float32)
    with pytest.raises(ss.ValidationError):
        ss.detect_batch(tf, 1e6)                        # window 31 > 16 columns
    with pytest.raises(ss.ValidationError):
        ss.detect_batch(np.ones((1, 10, 64), np.float32), 1e6, ss.DetectorConfig(savgol_window=30))
    with pytest.raises(ss.ValidationError):
        ss.detect_batch(np.ones((1, 10, 64), np.float32), 1e6, ss.DetectorConfig(min_component_area=0))


def test_stft_hann_detect(ss, ref, ora):
    """Config 5 as written (4096-pt Hann, 50 % overlap) end to end on the device
    vs the oracle restatement: TF plot, PSD, active set, bin boxes bit-exact;
    box times on the hop/fs frame grid."""
    sc = signals.c5_scenario(7, duration_s=0.025)
    iq, _ = ref.synthesize(signals.scenario_json(sc))
    fs, n_fft, hop, rows = 100e6, 4096, 2048, 600
    dets, tf = ss.sense(iq, fs, n_fft, rows, hop=hop, window=1, return_tf=True, first_seq=0)
    assert len(dets) == 2
    exp_tf = ora.stft_plot(iq, n_fft, hop, 1, 2 * rows).reshape(2, rows, n_fft)
    for p, det in enumerate(dets):
        assert np.array_equal(tf[p].view(np.uint32), exp_tf[p].view(np.uint32))
        exp = ora.detect(exp_tf[p], start_seq=p * rows, fs=fs)
        assert np.array_equal(det.psd.raw, exp["raw"]) and np.array_equal(det.active_columns, exp["active"])
        assert np.array_equal(det.bin_boxes, exp["bin_boxes"])
        bb = exp["bin_boxes"].astype(np.float64)
        dt, df = hop / fs, fs / n_fft
        assert np.array_equal(det.boxes[:, 0], (bb[:, 2] - n_fft // 2) * df)
        assert np.array_equal(det.boxes[:, 2], (p * rows + bb[:, 0]) * dt)
        assert np.array_equal(det.boxes[:, 3], (p * rows + bb[:, 1]) * dt)


def _host_sense(ss, src, n_fft, hop, window, rows, P, fs, K=2048):
    """ss_(stft_)sense_batch with HOST input and HOST outputs: the chunked
    copy-stream pipeline (capi.cu sense_impl) instead of the device-resident path."""
    import ctypes as C
    from paper_2603_20481_b200 import _native as NAT
    ctx = ss.Context.get(0)
    o = dict(raw=np.empty((P, n_fft), np.float32), sm=np.empty((P, n_fft), np.float32),
             ft=np.empty((P, 2), np.float32), act=np.empty((P, n_fft), np.int32), nact=np.empty(P, np.int32),
             boxes=np.empty((P, K, 4), np.float64), bins=np.empty((P, K, 4), np.int32), nb=np.empty(P, np.int32))
    bout = NAT.BatchOut(*(C.c_void_p(v.ctypes.data) for v in o.values()), K)
    cfg = ss.DetectorConfig().c()
    src = np.ascontiguousarray(src)
    ctx.check(ctx.lib.ss_stft_sense_batch(ctx.h, C.c_void_p(src.ctypes.data), NAT.SS_FMT_F32, n_fft, hop, window,
                                          rows, P, C.c_uint64(0), C.c_double(fs), C.byref(cfg), None, C.byref(bout)))
    return o


@pytest.mark.parametrize("hop,window,rows", [(4096, 0, 2441), (2048, 1, 4881)])
def test_host_input_pipeline_matches_device(ss, hop, window, rows):
    """4 x 80 MB plots from host memory -> 2 staging chunks (3 + 1 plots, the STFT
    chunks overlapping by n_fft - hop samples) == the device-resident result."""
    import torch
    n_fft, P, fs = 4096, 4, 100e6
    n = P * rows * hop + n_fft - hop
    iq = np.concatenate([signals.synthesize_torch(signals.c5_scenario(40 + i), device="cuda").cpu().numpy()
                         for i in range((n + 9_999_999) // 10_000_000)])[:n]
    got = _host_sense(ss, iq, n_fft, hop, window, rows, P, fs)
    dets = ss.sense(iq, fs, n_fft, rows, hop=hop, window=window, box_capacity=2048)
    assert len(dets) == P
    for p, d in enumerate(dets):
        k = int(got["nb"][p])
        assert k == len(d.boxes)
        assert np.array_equal(got["raw"][p], d.psd.raw) and np.array_equal(got["sm"][p], d.psd.smoothed)
        assert np.array_equal(got["act"][p][: got["nact"][p]], d.active_columns)
        assert np.array_equal(got["bins"][p][:k], d.bin_boxes)
        assert np.array_equal(got["boxes"][p][:k], d.boxes)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n_fft,rows", [(8192, 60), (32, 700), (64, 1), (2048, 3), (1024, 6200), (512, 3264), (512, 3265),
                                         (256, 12288), (256, 12289)])
def test_size_edges(ss, ref, n_fft, rows):
    """Extreme geometries through the fused pipeline vs the reference: the largest
    device FFT, the smallest F the default window accepts, single-row plots,
    and a plot taller than the K4 tile limit (generic binarize path)."""
    rng = np.random.default_rng(n_fft + rows)
    n = 2 * rows * n_fft
    x = (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex64)
    # a strong band in the second half of each plot so components exist
    for p in range(2):
        s0 = (p * rows + rows // 2) * n_fft
        t = np.arange(s0, s0 + max(1, rows // 3) * n_fft)
        x[t] += (8 * np.exp(2j * np.pi * 0.2 * t)).astype(np.complex64)
    fs = 1e6
    dets, tf = ss.sense(x, fs, n_fft, rows, return_tf=True, box_capacity=4096)
    exp_tf = ref.make_plots(x, fs, n_fft, rows)
    assert len(dets) == len(exp_tf) == 2
    for p, det in enumerate(dets):
        _check(det, ref.detect(exp_tf[p], start_seq=p * rows, fs=fs), tf[p], exp_tf[p])


def test_all_zero_and_constant_plots(ss, ref):
    """Degenerate spectra: zero input (PSD 0 -> -3000 dB floor path) and a pure
    tone (constant columns -> invalid Otsu scale)."""
    n_fft, rows = 256, 64
    z = np.zeros(rows * n_fft, np.complex64)
    tone = np.exp(2j * np.pi * 0.25 * np.arange(rows * n_fft)).astype(np.complex64)
    for x in (z, tone):
        dets, tf = ss.sense(x, 1e6, n_fft, rows, return_tf=True)
        exp_tf = ref.make_plots(x, 1e6, n_fft, rows)
        _check(dets[0], ref.detect(exp_tf[0], fs=1e6), tf[0], exp_tf[0])


@pytest.mark.parametrize("n_fft,rows", [(16384, 40), (65536, 12)])
def test_large_fft_detect(ss, ref, n_fft, rows):
    """Wide plots through the whole chain (large-N FFT, K2 PSD, global-scratch
    floor for F > 25,000 columns, K4-K6) vs the reference."""
    rng = np.random.default_rng(n_fft + rows)
    n = 2 * rows * n_fft
    x = (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex64)
    t = np.arange(n)
    x[(t // n_fft) % rows > rows // 3] += (6 * np.exp(2j * np.pi * 0.1 * t[(t // n_fft) % rows > rows // 3])).astype(np.complex64)
    dets, tf = ss.sense(x, 1e6, n_fft, rows, return_tf=True, box_capacity=8192)
    exp_tf = ref.make_plots(x, 1e6, n_fft, rows)
    for p, det in enumerate(dets):
        _check(det, ref.detect(exp_tf[p], start_seq=p * rows, fs=1e6), tf[p], exp_tf[p])


def _k2_ms(ss):
    """Stage-timer reading of K2 (the separate PSD kernel): zero when K1 fused it."""
    import ctypes as C
    ctx = ss.Context.get(0)
    st = (C.c_double * 8)()
    ctx.lib.ss_stage_times(ctx.h, st)
    return st[1]


@pytest.mark.parametrize("n_fft,rows,P,fmt", [(4096, 12, 296, 0), (4096, 12, 296, 1), (8192, 6, 148, 0),
                                              (1024, 8, 592, 0)])
def test_fused_full_wave(ss, ref, n_fft, rows, P, fmt):
    """Batches that fill whole waves of plot slots take K1's fused-PSD form (one
    plot per row group, row-order column sums -- in TMEM for N >= 4096; the
    int16 form's first DFT4 layer in integer arithmetic) and the bench's
    K4 -> K6 chain: every plot vs the reference, bit for bit."""
    rng = np.random.default_rng(n_fft * 7 + P + fmt)
    n = P * rows * n_fft
    x = (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex64)
    t = np.arange(n)
    x += (6 * np.exp(2j * np.pi * 0.23 * t) * ((t // (rows * n_fft)) % 3 == 0)).astype(np.complex64)
    fs = 1e6
    ctx = ss.Context.get(0)
    ctx.lib.ss_enable_stage_timing(ctx.h, 1)  # resets the stage timers
    try:
        if fmt == 1:
            v = np.clip(x.view(np.float32) * np.float32(2048.0), -32768, 32767)
            q = np.rint(v).astype(np.int16)
            dets, tf = ss.sense(q, fs, n_fft, rows, fmt=1, return_tf=True, box_capacity=4096)
            x = (q.astype(np.float32) * np.float32(1 / 32768)).view(np.complex64)
        else:
            dets, tf = ss.sense(x, fs, n_fft, rows, return_tf=True, box_capacity=4096)
        assert _k2_ms(ss) == 0.0, "batch did not take the fused-PSD K1"
    finally:
        ctx.lib.ss_enable_stage_timing(ctx.h, 0)
    exp_tf = ref.make_plots(x, fs, n_fft, rows)
    assert len(dets) == len(exp_tf) == P
    for p, det in enumerate(dets):
        _check(det, ref.detect(exp_tf[p], start_seq=p * rows, fs=fs), tf[p], exp_tf[p])


def test_fused_full_wave_hann(ss, ora):
    """Config 5 as written on a full wave (296 plots): the fused K1 with the
    window, vs the oracle's STFT restatement."""
    n_fft, hop, rows, P, fs = 4096, 2048, 6, 296, 100e6
    rng = np.random.default_rng(2961)
    n = P * rows * hop + n_fft - hop
    iq = (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex64)
    dets, tf = ss.sense(iq, fs, n_fft, rows, hop=hop, window=1, return_tf=True, first_seq=0, box_capacity=4096)
    exp_tf = ora.stft_plot(iq, n_fft, hop, 1, P * rows).reshape(P, rows, n_fft)
    assert len(dets) == P
    for p in range(0, P, 37):
        assert np.array_equal(tf[p].view(np.uint32), exp_tf[p].view(np.uint32)), p
        exp = ora.detect(exp_tf[p], start_seq=p * rows, fs=fs)
        assert np.array_equal(dets[p].psd.raw.view(np.uint32), exp["raw"].view(np.uint32)), p
        assert np.array_equal(dets[p].active_columns, exp["active"]), p
        assert np.array_equal(dets[p].bin_boxes, exp["bin_boxes"]), p


SCEN_DIR = __import__("pathlib").Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "suite" / "scenarios"
REF_SCENARIOS = ["sparse", "default", "control", "dense_mixed", "dense_noise_like"]


@pytest.mark.parametrize("name", REF_SCENARIOS)
@pytest.mark.parametrize("rows", [2000, 500])
def test_reference_scenario_fixtures(ss, ref, name, rows):
    """The reference's own scenario fixtures (proj/scenarios/*.json, SURVEY.md
    §8(d) P-parity set; copied next to the suite binaries by oracle/Makefile),
    rendered by the reference's signals::synthesize, through ss_sense_batch:
    2 plots at (2000, 1024) and 8 at (500, 1024) per scenario (10 and 40 over
    the five), every output
    bit-identical to the reference's make_plots + detect."""
    text = (SCEN_DIR / f"{name}.json").read_text()
    iq, _ = ref.synthesize(text)
    fs = 100e6
    dets, tf = ss.sense(iq, fs, 1024, rows, return_tf=True)
    exp_tf = ref.make_plots(iq, fs, 1024, rows)
    assert len(dets) == len(exp_tf) == (2 if rows == 2000 else 8)
    for p, det in enumerate(dets):
        exp = ref.detect(exp_tf[p], start_seq=p * rows, fs=fs)
        _check(det, exp, tf[p], exp_tf[p])


def test_async_batches_match_sync(ss, ref):
    """ss_set_async: back-to-back batches from pinned host IQ into pinned host
    outputs queue without a host synchronisation; after ss_wait their results
    equal the synchronous calls bit for bit, and an exceeded box capacity is
    reported by ss_wait (not by the call)."""
    import ctypes as C

    import torch

    from paper_2603_20481_b200 import _native as NAT
    ctx = ss.Context.get(0)
    lib = ctx.lib
    fs, n_fft, rows, P = 100e6, 1024, 500, 4
    iqs = []
    for k in range(2):
        iq, _ = ref.synthesize(signals.scenario_json(signals.paper_scenario(rows=P * rows, seed=11 + k)))
        h = torch.from_numpy(np.ascontiguousarray(iq[: P * rows * n_fft])).pin_memory()
        iqs.append(h)
    cfg = ss.DetectorConfig().c()

    def outs(K):
        o = dict(raw=torch.empty((P, n_fft), dtype=torch.float32), sm=torch.empty((P, n_fft), dtype=torch.float32),
                 ft=torch.empty((P, 2), dtype=torch.float32), act=torch.empty((P, n_fft), dtype=torch.int32),
                 nact=torch.empty(P, dtype=torch.int32), boxes=torch.empty((P, K, 4), dtype=torch.float64),
                 bins=torch.empty((P, K, 4), dtype=torch.int32), nb=torch.empty(P, dtype=torch.int32))
        o = {k: v.pin_memory() for k, v in o.items()}
        return o, NAT.BatchOut(*(C.c_void_p(v.data_ptr()) for v in o.values()), K)

    def call(h, bo):
        return lib.ss_sense_batch(ctx.h, C.c_void_p(h.data_ptr()), NAT.SS_FMT_F32, n_fft, rows, P, C.c_uint64(0),
                                  C.c_double(fs), C.byref(cfg), None, C.byref(bo))

    sync = []
    for h in iqs:
        o, bo = outs(1024)
        ctx.check(call(h, bo))
        sync.append(o)
    ctx.check(lib.ss_set_async(ctx.h, 1))
    try:
        a = [outs(1024) for _ in iqs]
        for h, (o, bo) in zip(iqs, a):
            ctx.check(call(h, bo))         # queued, returns before the work is done
        ctx.check(lib.ss_wait(ctx.h))
        for (o, _), e in zip(a, sync):
            for k in ("raw", "sm", "ft", "nact", "nb"):
                assert torch.equal(o[k], e[k]), k
            for p in range(P):
                n = int(e["nb"][p])
                assert torch.equal(o["bins"][p, :n], e["bins"][p, :n])
                assert torch.equal(o["boxes"][p, :n].view(torch.int64), e["boxes"][p, :n].view(torch.int64))
        # a capacity below the true box count is reported at ss_wait
        small, bs = outs(1)
        ctx.check(call(iqs[0], bs))
        assert lib.ss_wait(ctx.h) == NAT.SS_ECAPACITY
        assert lib.ss_wait(ctx.h) == NAT.SS_OK          # the flags were consumed
    finally:
        lib.ss_set_async(ctx.h, 0)


def test_fused_tall_plots_take_k1_extremes(ss, ora):
    """Config 5 as written at full size (296 plots x 4881 rows, Hann, hop 2048):
    the fused K1 also writes the column extremes and K4's 2-CTA cluster form
    bins each box as it lands (no min / max sweep).  Three plots carrying the
    seeded tone burst (early, middle, late) against the oracle's STFT
    restatement, bit for bit."""
    import ctypes as C

    import torch

    from paper_2603_20481_b200 import _native as NAT
    from paper_2603_20481_b200.specsense import DetectorConfig, _batch_out, _unpack_batch

    n_fft, hop, rows, P, fs = 4096, 2048, 4881, 296, 100e6
    n = P * rows * hop + n_fft - hop
    g = torch.Generator(device="cuda").manual_seed(4881)
    iq = torch.randn(2 * n, generator=g, device="cuda", dtype=torch.float32)
    t = torch.arange(n, device="cuda", dtype=torch.float64)
    burst = ((t // (rows * hop)) % 5 == 1) & ((t % (rows * hop)) < rows * hop // 3)
    ph = 2 * np.pi * 0.17 * t
    iq[0::2] += (4 * torch.cos(ph) * burst).float()
    iq[1::2] += (4 * torch.sin(ph) * burst).float()
    del t, burst, ph
    tf = torch.empty((P, rows, n_fft), dtype=torch.float32, device="cuda")
    out_t, out = _batch_out(torch, P, n_fft, 4096)
    ctx = ss.Context.get(0)
    cfg = DetectorConfig().c()
    ctx.check(ctx.lib.ss_stft_sense_batch(ctx.h, C.c_void_p(iq.data_ptr()), NAT.SS_FMT_F32, n_fft, hop, 1, rows, P, 0,
                                          fs, C.byref(cfg), C.c_void_p(tf.data_ptr()), C.byref(out)))
    torch.cuda.synchronize()
    dets = _unpack_batch(out_t, P)
    for p in (1, 146, 291):  # plots p % 5 == 1 carry the burst
        seg = iq[2 * p * rows * hop: 2 * (p * rows * hop + (rows - 1) * hop + n_fft)].cpu().numpy().view(np.complex64)
        exp_tf = ora.stft_plot(seg, n_fft, hop, 1, rows)
        assert np.array_equal(tf[p].cpu().numpy().view(np.uint32), exp_tf.view(np.uint32)), p
        exp = ora.detect(exp_tf, start_seq=p * rows, fs=fs)
        assert np.array_equal(dets[p].psd.raw.view(np.uint32), exp["raw"].view(np.uint32)), p
        assert np.array_equal(dets[p].active_columns, exp["active"]), p
        assert np.array_equal(dets[p].bin_boxes, exp["bin_boxes"]), p
        assert len(dets[p].bin_boxes) > 0, p
