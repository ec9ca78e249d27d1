"""Parity at BASELINE scale (SURVEY.md 8(c) checks 1-3) and a seeded stress loop.

* C2 in full: every one of the 35,820,200 tuples, planted y and y ~ N(0,1), against top-10
  lists the reference itself produced (tests/golden/make_golden_scale.py).
* C3 with y ~ N(0,1) and C4 (ill-conditioned, n = 4): 10^6 uniformly random tuples scored on
  the device (l0s_fit_tuples) and by the oracle (score_tuples restated), bit for bit; on the
  same sample the screen's lower bound never exceeds the reference's SSR, and no sampled tuple
  beats the search's keep-th model without being in the returned list.
* 200 mid-size instances (random, planted, exact ties, near-collinear, large-mean, mixed
  scales, noiseless; 1-8 tasks; n = 2..4; fp64 and fp32), each searched exhaustively by the
  oracle and compared model by model.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
from math import comb

import numpy as np
import pytest

import scale_cases
from conftest import GOLDEN, bits_equal, check_models

pytestmark = pytest.mark.gpu

THREADS = len(os.sched_getaffinity(0))


def _partition(s, slices):
    from paper_2502_20072_b200.search import _partition as part

    return part(s, slices)


def _oracle_scores(oracle, vals, y, bounds, tuples, tol):
    """score_tuples on every host thread (the C kernel releases the GIL)."""
    parts = np.array_split(np.arange(len(tuples)), THREADS * 4)
    out = np.empty(len(tuples))

    def run(ix):
        if len(ix):
            out[ix] = oracle.score_tuples(vals, y, bounds, tuples[ix], tol)

    with cf.ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(run, parts))
    return out


def _random_subsets(rng, m, n, count):
    """`count` uniformly random n-subsets of [0, m), ascending (uniform over combinations)."""
    out = np.empty((0, n), dtype=np.int64)
    while len(out) < count:
        t = np.sort(rng.integers(0, m, size=(2 * (count - len(out)) + 16, n)), axis=1)
        t = t[np.all(np.diff(t, axis=1) > 0, axis=1)]
        out = np.concatenate([out, t])
    return np.ascontiguousarray(out[:count])


@pytest.mark.parametrize("variant", ["planted", "random"])
@pytest.mark.parametrize("mode", ["auto", "fast"])
def test_c2_full_search_matches_reference(variant, mode):
    """C2 (600 x 1000, n = 3): the whole search, top 10 bit for bit against the reference's run."""
    from paper_2502_20072_b200 import L0Config, SearchStats, l0_search

    path = os.path.join(GOLDEN, f"scale_c2_{variant}.npz")
    g = np.load(path)
    v, y, slices = scale_cases.c2(variant)
    assert scale_cases.digest(v, y) == str(g["digest"]), "regenerated C2 inputs differ from the fixture's"
    st = SearchStats()
    models = l0_search(v, y, slices, L0Config(dimension=3, n_models_store=10), stats=st, mode=mode)
    check_models(models, {k: g[k] for k in ("exp_indices", "exp_score", "exp_coef", "exp_rmse")})
    assert st.device["certified"] == 1
    assert st.n_tuples == comb(600, 3)


@pytest.mark.parametrize("case", ["c3_random", "c4"])
def test_random_rank_sample_bitwise_and_bounds(oracle, case):
    """10^6 random tuples: device exact scores == oracle bits; lb <= s * score_ref on every tuple
    the screen certifies; no sampled tuple beats the returned keep-th model unseen."""
    from paper_2502_20072_b200 import L0Config, SearchStats, _lib, l0_search
    from paper_2502_20072_b200.search import rank_tuple

    if case == "c3_random":
        (v, y, slices), n = scale_cases.c3("random"), 3
    else:
        (v, y, slices), n = scale_cases.c4(), 4
    m, s = v.shape
    perm, bounds, _ = _partition(s, slices)
    rng = np.random.default_rng(20260822 + n)
    tuples = _random_subsets(rng, m, n, 1_000_000)

    eng = _lib.engine(0)
    eng.stage(v, y, perm, bounds, "fp64")
    ok, got, _, _ = eng.fit_tuples(tuples)
    lb, flags = eng.screen_tuples(tuples)
    vals, yy, ob, _ = oracle.prepare(v, y, slices, "fp64")
    want = _oracle_scores(oracle, vals, yy, ob, tuples, 1e-10)
    assert bits_equal(got, want)
    assert np.array_equal(ok.astype(bool), np.isfinite(want) | np.isnan(want))
    sel = (flags == 3) & np.isfinite(want)
    assert sel.sum() > 0.5 * len(tuples)
    viol = lb[sel] > want[sel] * s
    assert not viol.any(), float(np.max(lb[sel] / (want[sel] * s)))

    st = SearchStats()
    models = l0_search(v, y, slices, L0Config(dimension=n, n_models_store=10), stats=st, mode="fast")
    assert st.device["certified"] == 1 and len(models) == 10
    kept = {rank_tuple(md.indices, m, n) for md in models}
    k_score, k_rank = models[-1].score, rank_tuple(models[-1].indices, m, n)
    fin = np.isfinite(want)
    better = np.nonzero(fin & (want <= k_score))[0]
    for i in better:
        r = rank_tuple(tuples[i], m, n)
        if want[i] < k_score or r < k_rank:
            assert r in kept, (tuples[i], want[i], k_score)


KINDS = ("random", "planted", "tie", "collinear", "large_mean", "scales", "noiseless")


def _stress_instance(k):
    rng = np.random.default_rng(7000 + k)
    n = (2, 3, 4)[k % 3]
    T = 1 + (k // 3) % 12  # more than 8 tasks: the sweep bounds with 8 of them
    kind = KINDS[(k // 24 + k) % len(KINDS)]
    precision = "fp32" if k % 5 == 4 else "fp64"
    m = int(rng.integers(*{2: (60, 301), 3: (40, 121), 4: (24, 51)}[n]))
    r = int(rng.integers(max(n + 3, 8), 70))
    s = T * r + int(rng.integers(0, T))  # ragged tasks
    v = rng.uniform(0.5, 2.0, size=(m, s))
    pick = rng.choice(m, size=n, replace=False)
    coef = rng.uniform(0.5, 2.0, size=n) * rng.choice([-1.0, 1.0], size=n)
    noise = 0.02 * rng.standard_normal(s)
    if kind == "random":
        y = rng.standard_normal(s)
    elif kind == "noiseless":
        y = coef @ v[pick] + 0.3
    else:
        if kind == "tie":  # exact duplicates: bitwise-equal systems, order decided by rank
            for a, b in rng.choice(m, size=(3, 2), replace=False):
                v[b] = v[a]
        elif kind == "collinear":
            for c, d in enumerate((1e-5, 1e-8, 1e-10, 1e-12)):
                a, b = rng.choice(m, size=2, replace=False)
                v[b] = v[a] + d * rng.standard_normal(s)
            v[pick[-1]] = v[pick[0]] + 1e-9 * rng.standard_normal(s)
        elif kind == "large_mean":
            v[: m // 3] = 1e3 + rng.uniform(0.0, 1.0, size=(m // 3, s))
        elif kind == "scales":
            v *= np.logspace(-4, 4, m)[rng.permutation(m)][:, None]
        y = coef @ v[pick] + noise
    order = rng.permutation(s)
    cuts = np.linspace(0, s, T + 1).astype(int)
    slices = [np.sort(order[cuts[t]:cuts[t + 1]]) for t in range(T)]
    keep = int(rng.integers(1, 41)) if k % 7 else int(rng.integers(97, 300))  # > 96: global candidate list
    return dict(v=v, y=y, slices=slices, n=n, keep=keep, precision=precision, kind=kind)


@pytest.mark.parametrize("block", range(10))
def test_stress_loop_matches_oracle(oracle, block):
    """20 seeded instances per block (200 in all), each exhaustively against the oracle."""
    from paper_2502_20072_b200 import L0Config, SearchStats, l0_search

    for k in range(20 * block, 20 * block + 20):
        c = _stress_instance(k)
        want = oracle.l0_search(c["v"], c["y"], c["slices"], c["n"], c["keep"], c["precision"], threads=THREADS)
        st = SearchStats()
        cfg = L0Config(dimension=c["n"], n_models_store=c["keep"], precision=c["precision"], autotune=False)
        got = l0_search(c["v"], c["y"], c["slices"], cfg, stats=st, mode="fast")
        tag = (k, c["kind"], c["n"], len(c["slices"]), c["precision"], c["v"].shape)
        assert st.device["certified"] == 1, tag
        exp = {"exp_indices": np.array([w["indices"] for w in want]).reshape(len(want), c["n"]),
               "exp_score": np.array([w["score"] for w in want]),
               "exp_coef": np.array([w["coefficients"] for w in want]),
               "exp_rmse": np.array([w["rmse_per_task"] for w in want])}
        try:
            check_models(got, exp)
        except AssertionError as e:
            raise AssertionError(f"instance {tag}: {e}") from e


@pytest.mark.parametrize("keep", [97, 250, 1000])
@pytest.mark.parametrize("n", [2, 3, 4])
def test_large_keep_matches_oracle(oracle, n, keep):
    """keep > 96: the screened path collects candidates globally below the histogram threshold."""
    from paper_2502_20072_b200 import L0Config, SearchStats, l0_search

    rng = np.random.default_rng(keep + n)
    m, s, T = {2: 160, 3: 60, 4: 32}[n], 240, 3
    v = rng.uniform(0.5, 2.0, size=(m, s))
    y = rng.standard_normal(s) if keep != 250 else v[1] - v[7] + 0.5 * v[m - 2] + 0.1 * rng.standard_normal(s)
    slices = [np.arange(t, s, T) for t in range(T)]
    want = oracle.l0_search(v, y, slices, n, keep, "fp64", threads=THREADS)
    st = SearchStats()
    got = l0_search(v, y, slices, L0Config(dimension=n, n_models_store=keep), stats=st, mode="fast")
    assert st.device["mode_used"] == 1 and st.device["certified"] == 1
    exp = {"exp_indices": np.array([w["indices"] for w in want]), "exp_score": np.array([w["score"] for w in want]),
           "exp_coef": np.array([w["coefficients"] for w in want]),
           "exp_rmse": np.array([w["rmse_per_task"] for w in want])}
    check_models(got, exp)
