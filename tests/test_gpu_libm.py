"""GPU parity of the device glibc ports (csrc/glibc_libm.cuh) against the live
glibc log10f / powf(10, y) the reference calls (proj/src/detector.cpp:217,
222), over a strided sweep of all 2^32 float bit patterns plus the special
values."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sweep(stride, offset):
    u = np.arange(offset, 1 << 32, stride, dtype=np.uint64).astype(np.uint32)
    return u.view(np.float32)


SPECIAL = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, 10.0, 1e-45, 1.17549435e-38, 3.4028235e38,
                    -300.0, -150.0, -149.5, -45.0, 38.5, 38.6, 1e-3, 0.1], np.float32)


@pytest.mark.parametrize("variant", [1, 0])
def test_log10f_matches_glibc(ss, ora, variant):
    x = np.concatenate([_sweep(97, 13), SPECIAL])
    x = x[(x > 0) & np.isfinite(x)]
    got = ss.test_libm(x, 0, variant)
    exp = ora.glibc_log10f(x)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("variant", [1, 0])
def test_powf10_matches_glibc(ss, ora, variant):
    y = np.concatenate([_sweep(97, 29), SPECIAL])
    got = ss.test_libm(y, 1, variant)
    exp = ora.glibc_powf10(y)
    nan = np.isnan(exp)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint32), exp[~nan].view(np.uint32))


def test_db_range_dense(ss, ora):
    """Every float in the dB range the floor stage actually sees (raw in [1e-3, 1e12])."""
    lo, hi = np.float32(1e-3).view(np.uint32), np.float32(1e12).view(np.uint32)
    x = np.arange(lo, hi, 3, dtype=np.uint32).view(np.float32)
    assert np.array_equal(ss.test_libm(x, 0).view(np.uint32), ora.glibc_log10f(x).view(np.uint32))
    y = np.linspace(-310, 130, 20_000_000, dtype=np.float32)
    assert np.array_equal(ss.test_libm(y, 1).view(np.uint32), ora.glibc_powf10(y).view(np.uint32))
