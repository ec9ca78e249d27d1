"""Synthetic instances at BASELINE scale (SURVEY.md 8(d) "Synthetic inputs"), shared by the
golden generator (tests/golden/make_golden_scale.py, run against the reference) and the GPU
tests (tests/test_gpu_scale.py).  Pure numpy, seeded: the box regenerates the same bytes, and
every fixture records a digest of its inputs to prove it."""

from __future__ import annotations

import hashlib

import numpy as np


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def c2(variant: str = "planted"):
    """C2: values (600, 1000) ~ U(0.5, 2), seed 1, one task, n = 3 (35,820,200 tuples).
    planted: y = 2 f17 - f211 + 0.5 f499 + 0.75 + 0.01 N(0,1); random: y ~ N(0,1) (dense near-ties)."""
    rng = np.random.default_rng(1)
    v = rng.uniform(0.5, 2.0, size=(600, 1000))
    if variant == "planted":
        y = 2.0 * v[17] - v[211] + 0.5 * v[499] + 0.75 + 0.01 * rng.standard_normal(1000)
    else:
        y = rng.standard_normal(1000)
    return v, y, None


def c3(variant: str = "planted"):
    """C3: values (2000, 10000) ~ U(0.5, 2), seed 2, 4 round-robin tasks, n = 3.
    planted: bench.py's y (per-task coefficients on f17, f911, f1499); random: y ~ N(0,1)."""
    M, S, T = 2000, 10000, 4
    rng = np.random.default_rng(2)
    v = rng.uniform(0.5, 2.0, size=(M, S))
    slices = [np.arange(t, S, T) for t in range(T)]
    y = np.empty(S)
    if variant == "planted":
        for t, sl in enumerate(slices):
            y[sl] = (2.0 + 0.5 * t) * v[17, sl] - (1.0 + 0.25 * t) * v[911, sl] + 0.5 * v[1499, sl] + 0.75 \
                + 0.01 * rng.standard_normal(len(sl))
    else:
        y[:] = rng.standard_normal(S)
    return v, y, slices


def c4():
    """C4: values (1000, 5000) ~ U(0.5, 2), seed 3, one task, n = 4 (41,417,124,750 tuples), with
    near-copies spanning the reference's 1e-10 rank rule, near-constant features colliding with
    the intercept (two resolvable, two always rejected) and exact duplicates; y planted on four
    well-conditioned features + 1e-3 noise (the shape tools/run_configs.py times)."""
    rng = np.random.default_rng(3)
    m, s = 1000, 5000
    v = rng.uniform(0.5, 2.0, size=(m, s))
    deltas = [1e-4, 1e-6, 1e-8, 1e-9, 1e-10, 1e-12]
    for c in range(12):  # near-copies of features 0..11 placed at 900..911
        v[900 + c] = v[c] + deltas[c % len(deltas)] * rng.standard_normal(s)
    for c, d in enumerate([1e-4, 1e-6, 1e-12, 1e-13]):
        v[950 + c] = 1.0 + c + d * rng.standard_normal(s)
    v[960] = v[100]
    v[961] = v[200]
    y = 1.5 * v[100] - 0.8 * v[300] + 0.6 * v[500] + 0.4 * v[700] + 1e-3 * rng.standard_normal(s)
    return v, y, None
