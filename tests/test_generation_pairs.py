"""pair_arrays (the device stream's candidate enumeration) against the reference's
generate_pairs (generation.py:205-242): same pairs, same order -- CPU only."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _reference():
    if os.path.isdir(REF) and REF not in sys.path:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_l0s")
        sys.path.append(REF)
    try:
        import descsearch  # noqa: F401
    except Exception:
        pytest.skip("reference package not importable here")


def _pool(units, ops, seed):
    from descsearch.expressions import get_operator
    from descsearch.generation import FeatureSpace, GenerationConfig, generate_rung

    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, size=(40, len(units)))
    x[:5, 1] = 0.0  # a child with exact zeros: div never takes it second
    pool = FeatureSpace.from_primaries([f"x{i}" for i in range(len(units))], units, x)
    gcfg = GenerationConfig(operators=[get_operator(o) for o in ops], max_rung=3)
    generate_rung(pool, 1, gcfg)
    return pool


@pytest.mark.parametrize("seed", [0, 1])
def test_pair_arrays_equal_generate_pairs(seed):
    _reference()
    from descsearch.expressions import get_operator
    from descsearch.generation import generate_pairs
    from descsearch.units import Unit

    from paper_2502_20072_b200.generation import pair_arrays

    units = [Unit.of(m=1), Unit.of(m=1), Unit.of(s=1), Unit(), Unit.of(m=1, s=-1), Unit()]
    ops = ["add", "sub", "mul", "div", "abs_diff", "sqrt", "inv", "exp", "log"]
    pool = _pool(units, ops, seed)
    for rung in (1, 2):
        for name in ops:
            op = get_operator(name)
            want = generate_pairs(op, pool, rung).pairs
            pi, pj = pair_arrays(op, pool, rung)
            got = [(i, None if j < 0 else j) for i, j in zip(pi.tolist(), pj.tolist())]
            assert got == want, (name, rung)
