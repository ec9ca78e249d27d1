"""Pins the CPU oracle (oracle/l0_oracle.c) to the reference's own outputs.

Every comparison is on exact float bits: the golden vectors in tests/golden
were produced by the reference's numba kernels (make_golden.py), and the
reference's own known-answer tests (test_lsq.py / test_search.py) are
restated at the bottom.
"""

from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import bits_equal, golden_names, load_golden, search_case, slices_of


@pytest.mark.parametrize("name", golden_names("lsq"))
def test_score_tuples_bitwise(oracle, name):
    g = load_golden("lsq", name)
    prec = str(g["precision"])
    got = oracle.score_tuples(g["values"], g["y"], g["bounds"], g["tuples"], oracle.RANK_TOL_FACTOR[prec])
    assert bits_equal(got, g["scores"])


@pytest.mark.parametrize("name", golden_names("lsq"))
def test_fit_tuple_kernel_bitwise(oracle, name):
    g = load_golden("lsq", name)
    prec = str(g["precision"])
    for i, t in enumerate(g["fit_pick"]):
        ok, coef, ssr = oracle.fit_tuple_kernel(g["values"], g["y"], g["bounds"], g["tuples"][t],
                                                oracle.RANK_TOL_FACTOR[prec])
        assert ok == bool(g["fit_ok"][i])
        if ok:
            assert bits_equal(coef, g["fit_coef"][i])
            assert bits_equal(ssr, g["fit_ssr"][i])


@pytest.mark.parametrize("name", golden_names("search"))
def test_l0_search_matches_reference(oracle, name):
    c = search_case(name)
    models = oracle.l0_search(c["values"], c["y"], c["slices"], c["n"], c["keep"], c["precision"])
    assert len(models) == len(c["exp_score"])
    for i, md in enumerate(models):
        assert md["indices"] == tuple(c["exp_indices"][i])
        assert bits_equal(md["score"], c["exp_score"][i])
        assert bits_equal(md["coefficients"], c["exp_coef"][i])
        assert bits_equal(md["rmse_per_task"], c["exp_rmse"][i])


@pytest.mark.parametrize("name", [n for n in golden_names("search") if search_case(n)["all_scores"] is not None])
def test_all_scores_bitwise(oracle, name):
    c = search_case(name)
    vals, y, bounds, _ = oracle.prepare(c["values"], c["y"], c["slices"], c["precision"])
    m, n = vals.shape[0], c["n"]
    tup = np.array(list(itertools.combinations(range(m), n)), dtype=np.int64)
    got = oracle.score_tuples(vals, y, bounds, tup, oracle.RANK_TOL_FACTOR[c["precision"]])
    assert bits_equal(got, c["all_scores"])


def test_pipeline_inputs_reproduce(oracle):
    g = load_golden("pipe", "c1")
    from conftest import slices_of

    for d in range(1, int(g["n_dims"]) + 1):
        sl = slices_of(g[f"d{d}_task_id"], g[f"d{d}_order"])
        models = oracle.l0_search(g[f"d{d}_values"], g[f"d{d}_y"], sl, d, int(g["keep"]), str(g["precision"]))
        assert [md["indices"] for md in models] == [tuple(r) for r in g[f"d{d}_exp_indices"]]
        assert bits_equal([md["score"] for md in models], g[f"d{d}_exp_score"])


# ---- the reference's own known-answer tests, restated against the oracle ----

def test_frozen_line(oracle):
    # test_search.py:73-82 / test_lsq.py:118-129: x=[0,1,2], y=[1,2,4]
    ok, coef, ssr = oracle.fit_tuple_kernel(np.array([[0.0, 1.0, 2.0]]), np.array([1.0, 2.0, 4.0]),
                                            np.array([0, 3]), np.array([0]), 1e-10)
    assert ok
    assert coef[0, 0] == pytest.approx(1.5, abs=1e-14)
    assert coef[0, 1] == pytest.approx(5.0 / 6.0, abs=1e-14)
    assert ssr[0] == pytest.approx(1.0 / 6.0, abs=1e-14)


@pytest.mark.parametrize("m,n", [(5, 2), (7, 3), (6, 1), (6, 6), (9, 4)])
def test_fill_combinations_matches_itertools(oracle, m, n):
    # test_lsq.py:184-188
    want = list(itertools.combinations(range(m), n))
    cur = np.arange(n, dtype=np.int64)
    got = oracle.fill_combinations(cur, m, len(want))
    assert list(map(tuple, got)) == want


@pytest.mark.parametrize("m,n", [(6, 2), (8, 3), (5, 1), (7, 7), (9, 4)])
def test_rank_unrank(oracle, m, n):
    # test_search.py:39-48
    want = list(itertools.combinations(range(m), n))
    assert [oracle.unrank_tuple(r, m, n) for r in range(len(want))] == want
    assert all(oracle.rank_tuple(t, m, n) == r for r, t in enumerate(want))


def test_duplicate_and_constant_score_inf(oracle, rng):
    # test_lsq.py:72-87
    values = rng.uniform(0.5, 2.0, size=(4, 30))
    values[3] = values[1]
    values[2] = 4.25
    y = rng.standard_normal(30)
    out = oracle.score_tuples(values, y, np.array([0, 30]), np.array([[0, 1], [1, 3], [0, 2]]), 1e-10)
    assert np.isfinite(out[0]) and out[1] == np.inf and out[2] == np.inf


def test_threaded_scan_is_thread_invariant(oracle, rng):
    values = rng.uniform(0.5, 2.0, size=(25, 40))
    y = rng.standard_normal(40)
    vals, yy, bounds, _ = oracle.prepare(values, y)
    one = oracle.scan(vals, yy, bounds, 25, 3, 1e-10, 0, 2300, 10, threads=1)
    four = oracle.scan(vals, yy, bounds, 25, 3, 1e-10, 0, 2300, 10, threads=4)
    assert one == four


@pytest.mark.parametrize("name", golden_names("sis"))
def test_sis_oracle_matches_reference_golden(name):
    """oracle/sis.py == the reference's _chunk_scores, bit for bit."""
    from oracle import sis

    g = load_golden("sis", name)
    slices = slices_of(g["task_id"], g["order"])
    got = sis.chunk_scores(g["F"], list(g["targets"]), slices)
    assert bits_equal(got, g["scores"])
