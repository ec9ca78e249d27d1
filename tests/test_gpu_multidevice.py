"""Several devices in one process (l0s_group_*, search.l0_search(device=[...])) and the host
input paths (pageable numpy through the pinned ring, pinned memory, row pointers).

The driver's GPU box has one B200, so a group repeats device 0: every member is its own
context with its own part of the search, the block exchange is a device-to-device copy, and the
merge is the one a multi-GPU group runs.  Every result must equal the single-device search bit
for bit (parts certify their own lists exactly; the (score, rank) merge is exact).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert [md.indices for md in a] == [md.indices for md in b]
    assert bits_equal([md.score for md in a], [md.score for md in b])
    assert bits_equal(np.array([md.coefficients for md in a]), np.array([md.coefficients for md in b]))
    assert bits_equal(np.array([md.rmse_per_task for md in a]), np.array([md.rmse_per_task for md in b]))


def _case(name, rng):
    if name == "planted3":
        m, s, T, n = 300, 800, 4, 3
        v = rng.uniform(0.5, 2.0, size=(m, s))
        y = 2 * v[7] - v[150] + 0.5 * v[299] + 0.01 * rng.standard_normal(s)
    elif name == "random3":
        m, s, T, n = 150, 400, 2, 3
        v = rng.uniform(0.5, 2.0, size=(m, s))
        y = rng.standard_normal(s)
    elif name == "ill4":
        m, s, T, n = 60, 300, 1, 4
        v = rng.uniform(0.5, 2.0, size=(m, s))
        v[40] = v[3] + 1e-9 * rng.standard_normal(s)
        y = v[3] - v[10] + 0.5 * v[20] + 0.2 * v[33] + 1e-3 * rng.standard_normal(s)
    elif name == "n1":
        m, s, T, n = 40, 120, 3, 1
        v = rng.uniform(0.5, 2.0, size=(m, s))
        y = rng.standard_normal(s)
    elif name == "n5":
        m, s, T, n = 18, 90, 2, 5
        v = rng.uniform(0.5, 2.0, size=(m, s))
        y = v[1] + v[2] - v[5] + 0.3 * v[9] + 0.1 * v[17] + 0.01 * rng.standard_normal(s)
    elif name == "tasks12":
        m, s, T, n = 80, 12 * 40, 12, 3
        v = rng.uniform(0.5, 2.0, size=(m, s))
        y = v[4] - 2 * v[30] + v[77] + 0.05 * rng.standard_normal(s)
    else:
        raise KeyError(name)
    slices = [np.arange(t, s, T) for t in range(T)]
    return v, y, slices, n


@pytest.mark.parametrize("name", ["planted3", "random3", "ill4", "n1", "n5", "tasks12"])
@pytest.mark.parametrize("members", [2, 3, 8])
def test_group_equals_single_device(name, members):
    from paper_2502_20072_b200 import L0Config, SearchStats, l0_search

    rng = np.random.default_rng(members * 100 + len(name))
    v, y, slices, n = _case(name, rng)
    cfg = L0Config(dimension=n, n_models_store=7)
    one = l0_search(v, y, slices, cfg)
    st = SearchStats()
    many = l0_search(v, y, slices, cfg, device=[0] * members, stats=st)
    _same(one, many)
    assert st.device["certified"] == 1
    assert st.n_tuples == st.device["n_tuples"]


def test_group_from_env(monkeypatch):
    """L0S_DEVICES selects the group."""
    from paper_2502_20072_b200 import L0Config, l0_search

    rng = np.random.default_rng(5)
    v, y, slices, n = _case("planted3", rng)
    cfg = L0Config(dimension=n)
    one = l0_search(v, y, slices, cfg)
    monkeypatch.setenv("L0S_DEVICES", "0,0,0,0")
    many = l0_search(v, y, slices, cfg)
    _same(one, many)


class _Sub:
    def __init__(self, v):
        from types import SimpleNamespace

        self.entries = [SimpleNamespace(values=np.array(r), expression=f"f{i}") for i, r in enumerate(v)]
        self.expressions = [e.expression for e in self.entries]

    def values_matrix(self):
        return np.stack([e.values for e in self.entries])

    def __len__(self):
        return len(self.entries)


def test_group_selected_subspace():
    from paper_2502_20072_b200 import L0Config, l0_search

    rng = np.random.default_rng(6)
    v, y, slices, n = _case("random3", rng)
    cfg = L0Config(dimension=n)
    one = l0_search(v, y, slices, cfg)
    many = l0_search(_Sub(v), y, slices, cfg, device=[0, 0])
    _same(one, many)
    assert many[0].expressions == tuple(f"f{i}" for i in many[0].indices)


@pytest.mark.parametrize("shape", [(300, 900), (1100, 4000)])  # unchunked and chunked (>= 32 MB) stage
def test_pageable_pinned_device_inputs_agree(shape):
    """The same search from pageable numpy (pinned ring), pinned memory and device memory."""
    import torch

    from paper_2502_20072_b200 import L0Config, _lib, l0_search
    from paper_2502_20072_b200.search import _partition

    rng = np.random.default_rng(shape[0])
    m, s = shape
    v = rng.uniform(0.5, 2.0, size=(m, s))
    y = v[3] - 0.5 * v[m - 1] + 0.25 * v[m // 2] + 0.01 * rng.standard_normal(s)
    slices = [np.arange(0, s, 2), np.arange(1, s, 2)]
    cfg = L0Config(dimension=3)
    pageable = l0_search(v, y, slices, cfg)
    pinned = l0_search(torch.from_numpy(v).pin_memory().numpy(), torch.from_numpy(y).pin_memory().numpy(), slices, cfg)
    _same(pageable, pinned)
    eng = _lib.engine(0)
    perm, bounds, _ = _partition(s, slices)
    vd, yd, pd = (torch.from_numpy(a).cuda() for a in (v, y, perm))
    torch.cuda.synchronize()
    eng.stage((m, s), None, None, bounds, "fp64", device_ptrs=(vd.data_ptr(), yd.data_ptr(), pd.data_ptr()))
    sc, rk, _, _, _ = eng.search(3, 10)
    assert bits_equal(sc, [md.score for md in pageable])
