"""Seeded synthetic workloads for the spectrum-occupancy path.

* ``c5_scenarios`` -- BASELINE.json config 5 stand-in:
  100 ms of complex fp32 IQ at 100 MS/s, unit noise power, 16 rectangular
  time-frequency bursts per capture ("ofdm-like": brick-wall band-limited
  noise, proj/src/signals.cpp:190-196): bandwidth U[5, 40] MHz, duration
  U[0.1, 5] ms, centre inside +/- fs/2, start U[0, 100 ms - dur], SNR U[0, 20] dB
  resolved to power by the reference's rule (signals.cpp:462-466:
  power = 10^(snr/10) * noise_power/fs * bandwidth).  Our own sampler
  (numpy PCG64, seed 2603 + capture); no external dataset exists or is used.
* ``paper_scenario`` -- the reference acceptance criterion-1 recipe
  (proj/tests/acceptance.cpp:213-233): one plot span, noise 1.0, seed 404,
  three 3 MHz ofdm-like bursts at -25/+5/+32 MHz over 15-75 % of the span,
  power 60.
* ``synthesize_torch`` renders a scenario on the GPU (torch RNG + FFT): a fast
  generator for benchmark inputs.  Parity tests use the reference's own
  signals::synthesize through the oracle instead, so both sides see identical
  bytes.
"""
from __future__ import annotations

import json
import math

import numpy as np


def c5_scenario(capture: int, duration_s: float = 0.1, fs: float = 100e6, n_bursts: int = 16,
                seed0: int = 2603) -> dict:
    rng = np.random.Generator(np.random.PCG64(seed0 + capture))
    noise_power = 1.0
    sigs = []
    for _ in range(n_bursts):
        bw = float(rng.uniform(5e6, 40e6))
        dur = float(rng.uniform(0.1e-3, 5e-3))
        dur = min(dur, duration_s * 0.999)
        fc = float(rng.uniform(-fs / 2 + bw / 2, fs / 2 - bw / 2))
        t0 = float(rng.uniform(0.0, duration_s - dur))
        snr = float(rng.uniform(0.0, 20.0))
        power = 10.0 ** (snr / 10.0) * (noise_power / fs) * bw
        sigs.append(dict(kind="ofdm-like", center_freq_hz=fc, bandwidth_hz=bw, t_start_s=t0, duration_s=dur,
                         power=power))
    return dict(sample_rate_hz=fs, duration_s=duration_s, noise_power=noise_power, seed=seed0 + capture,
                signals=sigs)


def paper_scenario(fs: float = 100e6, n_fft: int = 1024, rows: int = 2000, seed: int = 404) -> dict:
    span = rows * n_fft / fs
    sigs = [dict(kind="ofdm-like", center_freq_hz=c, bandwidth_hz=3e6, t_start_s=span * 0.15,
                 duration_s=span * 0.6, power=60.0) for c in (-25e6, 5e6, 32e6)]
    return dict(sample_rate_hz=fs, duration_s=span, noise_power=1.0, seed=seed, signals=sigs)


def scenario_json(sc: dict) -> str:
    """The reference's scenario schema (proj/src/signals.cpp:415-470)."""
    return json.dumps(sc)


def truth_boxes(sc: dict) -> np.ndarray:
    """Ground-truth boxes (f0, f1, t0, t1) as synthesize() labels them (signals.cpp:213-219)."""
    return np.array([[s["center_freq_hz"] - s["bandwidth_hz"] / 2, s["center_freq_hz"] + s["bandwidth_hz"] / 2,
                      s["t_start_s"], s["t_start_s"] + s["duration_s"]] for s in sc["signals"]], np.float64)


def synthesize_torch(sc: dict, device="cuda", seed: int | None = None):
    """Render a scenario to complex64 baseband on `device` (benchmark inputs)."""
    import torch

    fs = sc["sample_rate_hz"]
    n = int(round(sc["duration_s"] * fs))
    g = torch.Generator(device=device)
    g.manual_seed(int(sc["seed"] if seed is None else seed))
    std = math.sqrt(sc["noise_power"] / 2.0)
    x = torch.complex(torch.randn(n, generator=g, device=device, dtype=torch.float32) * std,
                      torch.randn(n, generator=g, device=device, dtype=torch.float32) * std)
    for s in sc["signals"]:
        i0 = max(0, min(n, int(round(s["t_start_s"] * fs))))
        i1 = max(i0, min(n, int(round((s["t_start_s"] + s["duration_s"]) * fs))))
        m = i1 - i0
        if m == 0:
            continue
        f = torch.fft.fftfreq(m, d=1.0 / fs, device=device, dtype=torch.float64)
        band = (f - s["center_freq_hz"]).abs() < s["bandwidth_hz"] / 2
        spec = torch.complex(torch.randn(m, generator=g, device=device, dtype=torch.float64),
                             torch.randn(m, generator=g, device=device, dtype=torch.float64)) * band
        if not bool(band.any()):
            spec[int((f - s["center_freq_hz"]).abs().argmin())] = 1.0
        b = torch.fft.ifft(spec)
        ms = (b.abs() ** 2).mean()
        b = b * torch.sqrt(s["power"] / ms)
        x[i0:i1] += b.to(torch.complex64)
    return x


def quantize_i16(x, gain: float = 2.0 ** -6):
    """The reference's int16 quantiser (proj/src/frontend.cpp:563-568:
    clamp(x * 32768) -> lrintf) after a power-of-two gain; returns (int16
    interleaved tensor, n_clipped)."""
    import torch

    v = torch.view_as_real(x * gain).reshape(-1) * 32768.0
    clipped = int(((v < -32768.0) | (v > 32767.0)).sum())
    q = torch.round(v.clamp(-32768.0, 32767.0)).to(torch.int16)
    return q, clipped
