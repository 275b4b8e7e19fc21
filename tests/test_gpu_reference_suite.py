"""The reference's OWN test programs, unmodified, linked against the B200
drop-in (oracle/Makefile `suite`): proj/tests/test_{frontend,detector,runtime,
baseline,signals}.cpp (doctest API via oracle/doctest/doctest.h) and the
acceptance gate proj/tests/acceptance.cpp (six criteria).

In the *_b200 binaries every hot-path symbol (fft_row, make_plot(s),
detector::*, runtime::*, baseline_detect ...) binds to libspecsense_b200.so;
only the reference's out-of-scope code (signals, metrics, the I/O classes of
frontend.cpp, compare/make_compare_row of baseline.cpp) is linked from the
reference objects, with the replaced symbols localized.

The acceptance gate's accuracy criteria are deterministic functions of the
detections, so their evidence lines must equal the reference's own run
(tests/golden/acceptance_ref.log, produced by oracle/_ref/suite/acceptance_ref
on the CPU): bit-identical detections give identical IoU / p_d lines.
"""
from __future__ import annotations

import os
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "oracle" / "_ref" / "suite"
GOLDEN = ROOT / "tests" / "golden" / "acceptance_ref.log"
UNITS = ["test_frontend", "test_detector", "test_runtime", "test_baseline", "test_signals"]


def _run(binary: Path, timeout: int) -> subprocess.CompletedProcess:
    assert binary.exists(), f"{binary} missing: build() runs `make -C oracle suite`"
    env = dict(os.environ)
    return subprocess.run([str(binary)], capture_output=True, text=True, timeout=timeout, env=env, cwd=str(ROOT))


def _bound_to_b200(binary: Path) -> None:
    """The drop-in binary resolves its hot path from libspecsense_b200.so."""
    ldd = subprocess.run(["ldd", str(binary)], capture_output=True, text=True).stdout
    assert "libspecsense_b200.so" in ldd, ldd
    nm = subprocess.run(["nm", "-C", str(binary)], capture_output=True, text=True).stdout
    for sym in ("specsense::frontend::fft_row(", "specsense::detector::detect(", "specsense::runtime::run("):
        lines = [ln for ln in nm.splitlines() if sym in ln]
        # undefined in the executable ("U") or file-local ("t"); never a global text definition
        assert all(" T " not in ln for ln in lines), lines


@pytest.mark.gpu
@pytest.mark.parametrize("unit", UNITS)
def test_reference_unit_suite_on_b200(unit, tmp_path):
    binary = SUITE / f"{unit}_b200"
    _bound_to_b200(binary)
    r = _run(binary, 900)
    out = r.stdout + r.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"suite_{unit}.log").write_text(out)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| checks: (\d+) \| (\d+) failed", out)
    assert m, out[-2000:]
    assert r.returncode == 0 and m.group(3) == "0" and m.group(5) == "0", out[-4000:]


def _criteria(log: str) -> dict[int, str]:
    return {int(m.group(1)): m.group(2) for m in re.finditer(r"^criterion (\d) \([^)]*\): (PASS|FAIL)", log, re.M)}


def _deterministic_lines(log: str) -> list[str]:
    """Evidence lines of criteria 2, 3 and the IoU line of 4, plus criterion 5's
    check lines: functions of the detections only (no timing)."""
    keep = []
    for ln in log.splitlines():
        s = ln.strip()
        if re.match(r"^(sparse|default|control|dense_mixed|dense_noise_like)\s+n_gt", s) or s.startswith("snr ") \
                or s.startswith("mean IoU:") or re.match(r"^(otsu|labeling|morphology|sliced consolidate|worker invariance|fft energy)\s", s) \
                or s.startswith("criterion 2") or s.startswith("criterion 3") or s.startswith("criterion 5"):
            keep.append(s)
    return keep


@pytest.mark.gpu
def test_reference_acceptance_gate_on_b200():
    binary = SUITE / "acceptance_b200"
    _bound_to_b200(binary)
    r = _run(binary, 1500)
    log = r.stdout
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "acceptance_b200.log").write_text(log + r.stderr)
    crit = _criteria(log)
    assert sorted(crit) == [1, 2, 3, 4, 5, 6], log[-3000:]
    # accuracy, baseline comparison and every stage-equivalence oracle pass on the GPU path
    for c in (1, 2, 3, 4, 5):
        assert crit[c] == "PASS", f"criterion {c}: {log[-3000:]}"
    # bit-identical detections => the reference's own evidence lines, verbatim
    exp = _deterministic_lines(GOLDEN.read_text())
    got = _deterministic_lines(log)
    assert got == exp, "\n".join(f"{a!r} vs {b!r}" for a, b in zip(got, exp) if a != b)
