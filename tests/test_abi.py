"""CPU-side checks of the C ABI: the library loads, exports what the header
declares, its host-only helpers agree with the reference's counting and
ranking (test_search.py:24-69), and it refuses to run without a device."""

from __future__ import annotations

import ctypes
import itertools
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "l0search.h")


@pytest.fixture(scope="module")
def L():
    from paper_2502_20072_b200 import _lib

    return _lib.lib()


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(l0s_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_exports():
    from paper_2502_20072_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_cdylib_has_sm100a_code():
    from paper_2502_20072_b200 import _lib

    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def _count(L, m, n):
    v = ctypes.c_int64()
    rc = L.l0s_count(m, n, ctypes.byref(v))
    return rc, v.value


def test_count_matches_reference(L):
    # test_search.py:25-29 exact big counts
    assert _count(L, 100000, 2) == (0, 4_999_950_000)
    assert _count(L, 5000, 3) == (0, 20_820_835_000)
    assert _count(L, 10, 1) == (0, 10)
    assert _count(L, 3, 5) == (0, 0)
    assert _count(L, 1000, 4) == (0, 41_417_124_750)
    assert _count(L, 20000, 5)[0] == 2  # >= 2^63 -> capacity
    assert _count(L, 5, 0)[0] == 1


@pytest.mark.parametrize("m,n", [(6, 2), (8, 3), (5, 1), (7, 7), (9, 4)])
def test_unrank_rank_lexicographic(L, m, n):
    want = list(itertools.combinations(range(m), n))
    out = np.zeros(n, dtype=np.int64)
    for r, tup in enumerate(want):
        assert L.l0s_unrank(r, m, n, out.ctypes.data) == 0
        assert tuple(out) == tup
        t = np.array(tup, dtype=np.int64)
        rk = ctypes.c_int64()
        assert L.l0s_rank(t.ctypes.data, m, n, ctypes.byref(rk)) == 0
        assert rk.value == r


def test_unrank_large(L):
    from math import comb

    m, n = 2000, 3
    out = np.zeros(n, dtype=np.int64)
    for r in (0, 1, 12345678, comb(m, n) - 1):
        assert L.l0s_unrank(r, m, n, out.ctypes.data) == 0
        from paper_2502_20072_b200 import unrank_tuple

        assert tuple(out) == unrank_tuple(r, m, n)


def test_no_device_means_no_fallback(L):
    n = ctypes.c_int(-1)
    L.l0s_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a device is visible")
    h = ctypes.c_void_p()
    assert L.l0s_create(0, ctypes.byref(h)) == 5  # L0S_ENODEV
    from paper_2502_20072_b200 import L0Config, l0_search

    with pytest.raises(RuntimeError):
        l0_search(np.random.default_rng(0).uniform(size=(5, 12)), np.zeros(12), config=L0Config(dimension=2))
