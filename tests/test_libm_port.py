"""The floor stage's libm is glibc 2.39 (third-party; proj/src/detector.cpp:217,
222).  oracle/libm_port.c restates glibc's log10f / powf; pin it against the
live glibc on a strided sweep of all 2^32 bit patterns (the full sweep is
tools/libm_exhaustive.c, result in DESIGN.md)."""
import numpy as np
import pytest


def _sweep(stride, offset):
    return np.arange(offset, 1 << 32, stride, dtype=np.uint64).astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("variant", [1, 0])
def test_log10f_port(ora, variant):
    x = _sweep(4099, 7)
    x = x[(x > 0) & np.isfinite(x)]
    assert np.array_equal(ora.log10f(x, variant).view(np.uint32), ora.glibc_log10f(x).view(np.uint32))


@pytest.mark.parametrize("variant", [1, 0])
def test_powf10_port(ora, variant):
    y = np.concatenate([_sweep(4099, 11), np.array([0, -0.0, np.inf, -np.inf, -300, -149.5, 38.6], np.float32)])
    a, b = ora.powf10(y, variant), ora.glibc_powf10(y)
    nan = np.isnan(b)
    assert np.array_equal(np.isnan(a), nan)
    assert np.array_equal(a[~nan].view(np.uint32), b[~nan].view(np.uint32))


def test_db_range_dense(ora):
    lo, hi = np.float32(1.0).view(np.uint32), np.float32(1e9).view(np.uint32)
    x = np.arange(lo, hi, 61, dtype=np.uint32).view(np.float32)
    assert np.array_equal(ora.log10f(x).view(np.uint32), ora.glibc_log10f(x).view(np.uint32))
    y = np.linspace(-310, 130, 2_000_000, dtype=np.float32)
    assert np.array_equal(ora.powf10(y).view(np.uint32), ora.glibc_powf10(y).view(np.uint32))
