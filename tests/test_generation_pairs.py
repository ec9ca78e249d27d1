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


@pytest.mark.parametrize("seed", [0, 1])
def test_keys_and_pending_records_match_apply(seed):
    """The device stream's canonical keys (generation._key) are expressions.apply's, and the
    index-pair records rebuild the same nodes; their taken test agrees with the key test."""
    _reference()
    from descsearch.expressions import apply, get_operator
    from descsearch.screening import SelectedSubspace, SubspaceEntry
    from descsearch.units import Unit

    from paper_2502_20072_b200.generation import PendingExprs, _key, pair_arrays

    units = [Unit.of(m=1), Unit.of(m=1), Unit.of(s=1), Unit(), Unit.of(m=1, s=-1), Unit()]
    pool = _pool(units, ["add", "sub", "mul", "div", "sqrt", "inv"], seed)
    feats = pool.features
    index_of = {f.key: i for i, f in enumerate(feats)}
    for name in ["add", "sub", "mul", "div", "abs_diff", "sqrt", "inv", "exp"]:
        op = get_operator(name)
        pi, pj = pair_arrays(op, pool, 2)
        if len(pi) == 0:
            continue
        rec = PendingExprs(op, pi, pj, feats, index_of)
        nodes = [apply(op, feats[i]) if j < 0 else apply(op, feats[i], feats[j])
                 for i, j in zip(pi.tolist(), pj.tolist())]
        for k in range(0, len(nodes), max(1, len(nodes) // 50)):
            i, j = int(pi[k]), int(pj[k])
            assert _key(op, feats[i].key, None if j < 0 else feats[j].key) == nodes[k].key
            assert rec[k].key == nodes[k].key and rec[k].build().key == nodes[k].key
        chosen = nodes[:: max(1, len(nodes) // 7)]
        prior = SelectedSubspace([SubspaceEntry(e, 0.5, np.zeros(3)) for e in chosen + feats[:3]])
        taken = prior.keys()
        want = np.array([n.key not in taken for n in nodes])
        assert np.array_equal(rec.not_taken(prior.entries), want)
