"""CPU restatement of the reference's KSG estimator (oracle only; test
infrastructure -- the product runs csrc/ksg.cu).

Follows `ifr.py:27-48` (digamma) and `ifr.py:59-104` (ksg_mi: PCG64 jitter of
amplitude 1e-10 x per-coordinate range, Chebyshev distances, k-th smallest
joint distance with self excluded, strict-inequality marginal counts with the
self distance subtracted when eps > 0).  Pinned bit-for-bit to the
reference's own outputs in tests/golden/ifr.npz.
"""

from __future__ import annotations

import numpy as np


def digamma(x):
    arr = np.atleast_1d(np.asarray(x, dtype=np.float64)).copy()
    acc = np.zeros_like(arr)
    small = arr < 6.0
    while small.any():
        acc[small] -= 1.0 / arr[small]
        arr[small] += 1.0
        small = arr < 6.0
    inv2 = 1.0 / (arr * arr)
    series = (-1.0 / 12.0 + inv2 * (1.0 / 120.0 + inv2 * (-1.0 / 252.0 + inv2 * (
        1.0 / 240.0 + inv2 * (-1.0 / 132.0 + inv2 * (691.0 / 32760.0))))))
    return acc + np.log(arr) - 0.5 / arr + inv2 * series


def jitter(z, y, seed):
    rng = np.random.Generator(np.random.PCG64(seed))

    def amp(a):
        span = a.max(axis=0) - a.min(axis=0)
        span[span == 0.0] = 1.0
        return 1e-10 * span
    z = z + amp(z) * rng.uniform(-1.0, 1.0, size=z.shape)
    y = y + amp(y) * rng.uniform(-1.0, 1.0, size=y.shape)
    return z, y


def ksg_counts(z, y, k):
    n = z.shape[0]
    cz = np.empty(n, np.int64)
    cy = np.empty(n, np.int64)
    degenerate = 0
    for i in range(n):
        dz = np.abs(z[i] - z).max(axis=1)
        dy = np.abs(y[i] - y).max(axis=1)
        dj = np.maximum(dz, dy)
        dj[i] = np.inf
        eps = np.partition(dj, k - 1)[k - 1]
        degenerate += int(eps == 0.0)
        self_ = int(eps > 0.0)
        cz[i] = int((dz < eps).sum()) - self_
        cy[i] = int((dy < eps).sum()) - self_
    return cz, cy, degenerate


def ksg_mi(z, y, k=5, jitter_seed=0):
    z, y = jitter(np.asarray(z, np.float64), np.asarray(y, np.float64), jitter_seed)
    cz, cy, deg = ksg_counts(z, y, k)
    n = z.shape[0]
    value = float(digamma(k)[0] + digamma(n)[0] - np.mean(digamma(cz + 1) + digamma(cy + 1)))
    return value, value < 0.0 or deg > 0
