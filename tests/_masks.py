"""Seeded test-mask generators (the shapes proj/tests/oracles.cpp:270-301 draws:
Bernoulli speckle, and a few filled rectangles plus 2 % speckle)."""
import numpy as np


def random_mask(rng, rows, cols, density):
    return (rng.random((rows, cols)) < density).astype(np.uint8)


def random_blob_mask(rng, rows, cols):
    m = np.zeros((rows, cols), np.uint8)
    for _ in range(int(rng.integers(1, 6))):
        r0 = int(rng.integers(0, rows))
        c0 = int(rng.integers(0, cols))
        r1 = min(rows, r0 + int(rng.integers(2, max(2, rows // 3) + 1)))
        c1 = min(cols, c0 + int(rng.integers(2, max(2, cols // 3) + 1)))
        m[r0:r1, c0:c1] = 1
    flip = rng.random((rows, cols)) < 0.02
    m[flip] ^= 1
    return m


def random_plot(rng, rows, cols, hi=4.0):
    return rng.uniform(0.0, hi, (rows, cols)).astype(np.float32)


def burst_plot(rng, rows, cols, n_bursts=4):
    """Rayleigh-like noise magnitudes with a few bright rectangles."""
    tf = np.abs(rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))).astype(np.float32)
    for _ in range(n_bursts):
        r0 = int(rng.integers(0, rows - 8))
        c0 = int(rng.integers(0, cols - 8))
        r1 = min(rows, r0 + int(rng.integers(8, rows // 2)))
        c1 = min(cols, c0 + int(rng.integers(4, max(5, cols // 10))))
        tf[r0:r1, c0:c1] *= np.float32(rng.uniform(3, 10))
    return tf
