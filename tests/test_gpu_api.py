"""The reference's own API tests for fit_tuple / l0_search / SearchStats, run on the drop-in.

Mirrors /root/reference/pkg/tests/test_search.py (TestFitTuple :73-107, TestL0Search
:110-197) with the reference's assertions; brute force is the CPU oracle (bit for bit).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture()
def rng():
    return np.random.default_rng(20260822)


def test_frozen_line():
    """x = [0, 1, 2] against y = [1, 2, 4]: slope 3/2, intercept 5/6 (test_search.py:73-82).
    One sample per coefficient + 1: the smallest system the device kernel takes (s = 3)."""
    from paper_2502_20072_b200 import fit_tuple

    model = fit_tuple((0,), np.array([[0.0, 1.0, 2.0]]), [1.0, 2.0, 4.0])
    assert model.indices == (0,)
    assert model.coefficients.shape == (1, 2)
    assert model.coefficients[0, 0] == pytest.approx(1.5, abs=1e-14)
    assert model.coefficients[0, 1] == pytest.approx(5.0 / 6.0, abs=1e-14)
    assert model.score == pytest.approx(1.0 / 18.0, abs=1e-15)
    assert model.rmse_per_task[0] == pytest.approx(np.sqrt(1.0 / 18.0), abs=1e-15)
    assert model.task_labels == ("0",)


def test_frozen_line_bitwise_vs_oracle(oracle):
    from paper_2502_20072_b200 import fit_tuple

    v, y = np.array([[0.0, 1.0, 2.0]]), np.array([1.0, 2.0, 4.0])
    got = fit_tuple((0,), v, y)
    want = oracle.fit_tuple((0,), v, y)
    assert bits_equal(got.coefficients, want["coefficients"]) and bits_equal(got.score, want["score"])
    assert bits_equal(got.rmse_per_task, want["rmse_per_task"])


def test_rank_deficient_raises(rng):
    from paper_2502_20072_b200 import RankDeficient, fit_tuple

    values = rng.uniform(0.5, 2.0, size=(3, 12))
    values[2] = values[0]
    with pytest.raises(RankDeficient):
        fit_tuple((0, 2), values, rng.standard_normal(12))


def test_validates_tuple(rng):
    from paper_2502_20072_b200 import RankOutOfRange, fit_tuple

    values = rng.uniform(0.5, 2.0, size=(4, 8))
    y = rng.standard_normal(8)
    with pytest.raises(RankOutOfRange):
        fit_tuple((2, 1), values, y)
    with pytest.raises(RankOutOfRange):
        fit_tuple((1, 4), values, y)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_task_labels_and_per_task_fit(rng, oracle, precision):
    from paper_2502_20072_b200 import fit_tuple

    values = rng.uniform(0.5, 2.0, size=(3, 20))
    y = rng.standard_normal(20)
    slices = [np.arange(0, 12), np.arange(12, 20)]
    model = fit_tuple((0, 2), values, y, task_slices=slices, task_labels=["a", "b"], precision=precision)
    assert model.task_labels == ("a", "b")
    assert model.coefficients.shape == (2, 3)
    assert model.coefficients.dtype == np.float64
    assert model.rmse_per_task.shape == (2,)
    want = oracle.fit_tuple((0, 2), values, y, slices, precision)
    assert bits_equal(model.coefficients, want["coefficients"]) and bits_equal(model.score, want["score"])


def test_fit_tuple_subspace_and_expressions(rng):
    """A SelectedSubspace-like object: expressions of the tuple come back on the model."""
    from types import SimpleNamespace

    from paper_2502_20072_b200 import fit_tuple

    v = rng.uniform(0.5, 2.0, size=(5, 30))
    entries = [SimpleNamespace(values=v[i], expression=f"x{i}") for i in range(5)]
    sub = SimpleNamespace(entries=entries, expressions=[e.expression for e in entries],
                          values_matrix=lambda: np.stack([e.values for e in entries]))
    md = fit_tuple((1, 3), sub, rng.standard_normal(30))
    assert md.expressions == ("x1", "x3")


def _instance(rng, m=10, s=25):
    return rng.uniform(0.5, 2.0, size=(m, s)), rng.standard_normal(s)


@pytest.mark.parametrize("n", [1, 2, 3])
@pytest.mark.parametrize("mode", ["auto", "exact"])
def test_matches_brute_force(rng, oracle, n, mode):
    from paper_2502_20072_b200 import L0Config, l0_search

    for _ in range(4):
        values, y = _instance(rng, m=8, s=20)
        models = l0_search(values, y, config=L0Config(dimension=n, autotune=False), mode=mode)
        want = oracle.l0_search(values, y, None, n, 10, "fp64")
        assert [md.indices for md in models] == [w["indices"] for w in want]
        assert bits_equal([md.score for md in models], [w["score"] for w in want])
        assert [md.score for md in models] == sorted(md.score for md in models)


def test_matches_brute_force_multitask(rng, oracle):
    from paper_2502_20072_b200 import L0Config, l0_search

    values, y = _instance(rng, m=7, s=22)
    slices = [np.arange(0, 9), np.arange(9, 22)]
    models = l0_search(values, y, task_slices=slices, config=L0Config(dimension=2, autotune=False))
    want = oracle.l0_search(values, y, slices, 2, 10, "fp64")
    assert models[0].indices == want[0]["indices"]
    assert bits_equal(models[0].score, want[0]["score"])


def test_batch_and_worker_invariance(rng):
    from paper_2502_20072_b200 import L0Config, l0_search

    values, y = _instance(rng, m=12, s=18)
    ref = None
    for batch in (7, 45, 131072):
        for workers in (1, 3):
            cfg = L0Config(dimension=2, batch_size=batch, autotune=False, n_models_store=8)
            got = [(m.indices, m.score) for m in l0_search(values, y, config=cfg, workers=workers)]
            if ref is None:
                ref = got
            assert got == ref


def test_autotune_same_result(rng):
    from paper_2502_20072_b200 import L0Config, l0_search

    values, y = _instance(rng)
    plain = l0_search(values, y, config=L0Config(dimension=2, autotune=False))
    tuned = l0_search(values, y, config=L0Config(dimension=2, autotune=True))
    assert [(m.indices, m.score) for m in tuned] == [(m.indices, m.score) for m in plain]


@pytest.mark.parametrize("mode", ["auto", "fast"])
def test_score_tie_goes_to_smaller_rank(rng, mode):
    from paper_2502_20072_b200 import L0Config, l0_search

    values = rng.uniform(0.5, 2.0, size=(3, 15))
    values[2] = values[1]
    y = rng.standard_normal(15)
    models = l0_search(values, y, config=L0Config(dimension=2, autotune=False, n_models_store=5), mode=mode)
    assert [m.indices for m in models] == [(0, 1), (0, 2)]
    assert models[0].score == models[1].score


@pytest.mark.parametrize("mode", ["auto", "fast"])
def test_all_deficient_returns_empty(rng, mode):
    from paper_2502_20072_b200 import L0Config, l0_search

    values = rng.uniform(0.5, 2.0, size=(2, 10))
    values[1] = values[0]
    y = rng.standard_normal(10)
    assert l0_search(values, y, config=L0Config(dimension=2, autotune=False), mode=mode) == []


def test_fp32_runs_and_reports_float64_models(rng):
    from paper_2502_20072_b200 import L0Config, l0_search

    values, y = _instance(rng, m=6)
    models = l0_search(values, y, config=L0Config(dimension=2, precision="fp32", autotune=False))
    assert models
    assert models[0].coefficients.dtype == np.float64
    assert np.isfinite(models[0].score)


@pytest.mark.parametrize("autotune", [False, True])
def test_stats_filled(rng, autotune):
    """SearchStats semantics (search.py:231-256, :305-308; test_search.py:174-183)."""
    from paper_2502_20072_b200 import L0Config, SearchStats, count_models, l0_search

    values, y = _instance(rng, m=9)
    stats = SearchStats()
    cfg = L0Config(dimension=2, batch_size=10, autotune=autotune)
    l0_search(values, y, config=cfg, stats=stats)
    assert stats.n_tuples == count_models(9, 2)
    assert stats.seconds > 0.0
    assert stats.tuples_per_second > 0.0
    n_batches = -(-count_models(9, 2) // 10)
    if autotune:
        # the first batch is timed once per chunk candidate; the choice is a candidate
        assert stats.chosen_chunk in {min(c, cfg.batch_size) for c in cfg.chunk_candidates}
        assert len(stats.batch_seconds) == n_batches - 1 + len(cfg.chunk_candidates)
    else:
        assert stats.chosen_chunk == 10  # min(chunk_candidates[0], batch_size)
        assert len(stats.batch_seconds) == n_batches
    assert len(stats.batch_seconds) >= count_models(9, 2) // 10
    # seconds covers scan + merge only (the reference excludes _prepare and the refit)
    assert stats.seconds <= sum(stats.batch_seconds) * (1 + 1e-9) + 1e-9


def test_n_models_store_caps_output(rng):
    from paper_2502_20072_b200 import L0Config, l0_search

    values, y = _instance(rng, m=9)
    assert len(l0_search(values, y, config=L0Config(dimension=2, n_models_store=3, autotune=False))) == 3
    # n_models_store < 1 keeps one model (search.py:229)
    assert len(l0_search(values, y, config=L0Config(dimension=2, n_models_store=0, autotune=False))) == 1


def test_rejects_undersized_subspace(rng):
    from paper_2502_20072_b200 import L0Config, l0_search

    values, y = _instance(rng, m=2)
    with pytest.raises(ValueError):
        l0_search(values, y, config=L0Config(dimension=3))
    with pytest.raises(ValueError):
        l0_search(values, y, config=None)


@pytest.mark.gpu
@pytest.mark.parametrize("m,dup", [(40, 6), (120, 10)])
def test_exact_mode_sort_with_ties_matches_oracle(oracle, m, dup):
    """The exact path sorts each chunk of scores on the device (sort.cu: one shared-memory
    block for <= 8192 entries, merge rounds above): C(40, 3) = 9880 and C(120, 3) = 280840
    tuples, with duplicated features so that many scores tie exactly and the rank decides
    (search.py:303)."""
    from paper_2502_20072_b200 import L0Config, l0_search

    rng = np.random.default_rng(1000 + m)
    values = rng.uniform(0.5, 2.0, size=(m, 30))
    values[m - dup:] = values[:dup]  # exact duplicates: tuples differing by a twin tie
    y = rng.standard_normal(30)
    cfg = L0Config(dimension=3, autotune=False, n_models_store=60)
    got = l0_search(values, y, config=cfg, mode="exact")
    want = oracle.l0_search(values, y, None, 3, 60, "fp64")
    assert [g.indices for g in got] == [w["indices"] for w in want]
    assert bits_equal([g.score for g in got], [w["score"] for w in want])
