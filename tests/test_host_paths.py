"""Host-side paths of the drop-in on CPU, with the device engine replaced by a stand-in that
returns fixed results: argument handling, device selection (one device, a group, L0S_DEVICES,
workers), Model assembly, SearchStats bookkeeping and the residual dispatch.  No numbers here
are checked against the reference -- the GPU tests do that -- only that every host branch runs."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2502_20072_b200 import L0Config, SearchStats, _lib, search


class _FakeStats:
    ms_records = 0.0

    def as_dict(self):
        return {"certified": 1, "ms_records": 0.0}


class _Fake:
    """Engine / Group stand-in: the best tuples are the first `keep` ranks."""

    def __init__(self):
        self.calls = []
        self.subspace_cache = None
        self.T = 1
        self.s = 0

    def stage(self, values, y, perm, bounds, precision, device_ptrs=None):
        self.calls.append("stage")
        self.T = len(bounds) - 1
        self.s = len(y)

    def stage_rows(self, arrays, y, perm, bounds, precision):
        self.calls.append("stage_rows")
        self.T = len(bounds) - 1
        self.s = len(y)

    def search(self, n, keep, *args):
        self.calls.append("search")
        k = min(keep, 3)
        return (np.arange(k, dtype=float), np.arange(k, dtype=np.int64), np.ones((k, self.T, n + 1)),
                np.ones((k, self.T)), _FakeStats())

    def residuals(self, tup, coef):
        self.calls.append("residuals")
        return np.zeros((len(tup), self.s))


@pytest.fixture()
def fake(monkeypatch):
    f = _Fake()
    monkeypatch.setattr(_lib, "engine", lambda device=None: f)
    monkeypatch.setattr(_lib, "group", lambda devices: f)
    monkeypatch.setattr(_lib, "device_count", lambda: 4)
    monkeypatch.delenv("L0S_DEVICES", raising=False)
    return f


def test_one_device_models_and_stats(fake):
    v = np.random.default_rng(0).uniform(size=(6, 20))
    st = SearchStats()
    models = search.l0_search(v, v[0], None, L0Config(dimension=2, n_models_store=2), stats=st)
    assert [m.indices for m in models] == [(0, 1), (0, 2)]
    assert st.n_tuples == 15 and st.seconds > 0 and st.device["certified"] == 1
    assert fake.calls == ["stage", "search"]
    assert search._last_stage[0] is fake


@pytest.mark.parametrize("how", ["list", "env", "workers"])
def test_group_selection(fake, monkeypatch, how):
    v = np.random.default_rng(1).uniform(size=(6, 20))
    kw = {}
    if how == "list":
        kw["device"] = [0, 1]
    elif how == "env":
        monkeypatch.setenv("L0S_DEVICES", "0,1,2")
    else:
        kw["workers"] = 3
    models = search.l0_search(v, v[0], None, L0Config(dimension=2), **kw)
    assert len(models) == 3 and fake.calls == ["stage", "search"]
    assert search._devices(kw.get("device"), kw.get("workers", 1)) is not None


def test_residuals_dispatch(fake):
    from types import SimpleNamespace

    rng = np.random.default_rng(2)
    v = rng.uniform(size=(5, 12))
    entries = [SimpleNamespace(values=v[i], expression=object()) for i in range(5)]

    class Sub:
        def __init__(self):
            self.entries = entries
            self.expressions = [e.expression for e in entries]

        def values_matrix(self):
            return np.stack([e.values for e in self.entries])

        def __len__(self):
            return len(self.entries)

    y = v[1] - v[3]
    models = search.l0_search(Sub(), y, None, L0Config(dimension=2))
    res = search.residuals(models, y, None, None, 2)
    assert len(res) == 2 and fake.calls[-1] == "residuals"
