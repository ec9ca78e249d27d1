"""Host-side API semantics of the drop-in (no device needed): argument
validation and error types happen before any device work, exactly where the
reference raises them (search.py:217-226, 113-121), and the counting /
ranking helpers restate test_search.py:24-69."""

from __future__ import annotations

import itertools

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2502_20072_b200 import (
    CapacityError,
    L0Config,
    RankOutOfRange,
    SearchStats,
    count_models,
    l0_search,
    rank_tuple,
    unrank_tuple,
)
from paper_2502_20072_b200.search import _partition


def test_exact_big_counts():
    assert count_models(100000, 2) == 4_999_950_000
    assert count_models(5000, 3) == 20_820_835_000
    assert count_models(10, 1) == 10
    assert count_models(3, 5) == 0
    with pytest.raises(ValueError):
        count_models(5, 0)
    with pytest.raises(ValueError):
        count_models(-1, 2)


@pytest.mark.parametrize("m,n", [(6, 2), (8, 3), (5, 1), (7, 7)])
def test_unrank_walks_lexicographic_order(m, n):
    want = list(itertools.combinations(range(m), n))
    assert [unrank_tuple(r, m, n) for r in range(len(want))] == want
    assert [rank_tuple(t, m, n) for t in want] == list(range(len(want)))


@given(st.integers(1, 60), st.integers(1, 6), st.data())
@settings(max_examples=60, deadline=None)
def test_round_trip_property(m, n, data):
    total = count_models(m, n)
    if total == 0:
        return
    r = data.draw(st.integers(0, total - 1))
    assert rank_tuple(unrank_tuple(r, m, n), m, n) == r


def test_out_of_range():
    with pytest.raises(RankOutOfRange):
        unrank_tuple(-1, 5, 2)
    with pytest.raises(RankOutOfRange):
        unrank_tuple(10, 5, 2)
    with pytest.raises(RankOutOfRange):
        rank_tuple((3, 2), 5, 2)
    with pytest.raises(RankOutOfRange):
        rank_tuple((1, 5), 5, 2)
    with pytest.raises(ValueError):
        rank_tuple((1, 2, 3), 5, 2)


def test_guards_before_device():
    rng = np.random.default_rng(1)
    values = rng.uniform(0.5, 2.0, size=(2, 9))
    with pytest.raises(ValueError):
        l0_search(values, rng.standard_normal(9), config=L0Config(dimension=3))
    with pytest.raises(ValueError):
        l0_search(values, rng.standard_normal(9), config=None)
    with pytest.raises(CapacityError):
        l0_search(np.zeros((20000, 2)), np.zeros(2), config=L0Config(dimension=5))


def test_partition_validation():
    perm, bounds, _ = _partition(6, [np.array([0, 2, 4]), np.array([1, 3, 5])])
    assert perm.tolist() == [0, 2, 4, 1, 3, 5]
    assert bounds.tolist() == [0, 3, 6]
    with pytest.raises(ValueError):
        _partition(6, [np.array([0, 1, 2]), np.array([2, 3, 4, 5])])
    with pytest.raises(ValueError):
        _partition(6, [np.array([0, 1, 2])])


def test_config_defaults_match_reference():
    cfg = L0Config(dimension=3)
    assert (cfg.batch_size, cfg.precision, cfg.n_models_store, cfg.autotune, cfg.chunk_candidates) == (
        131072, "fp64", 10, True, (4096, 16384, 65536))
    assert SearchStats().tuples_per_second == 0.0
