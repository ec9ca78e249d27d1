"""CPU oracle for the l0 (SO) search -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg /
``--impl reference`` arm may import this module.  The product package
(paper_2502_20072_b200) never imports it.

It drives ``liborc.so`` (l0_oracle.c, a restatement of
/root/reference/pkg/src/descsearch/lsq.py:61-215) the way
``descsearch.search`` drives its numba kernels:

* ``prepare``      <- search._prepare          search.py:113-127
* ``l0_search``    <- search.l0_search         search.py:202-322 (scan + merge
                      by (score, rank), then the per-model refit of
                      search.fit_tuple, search.py:136-171)
* ``fit_tuple``    <- search.fit_tuple         search.py:136-171
* ``unrank/rank``  <- search.unrank_tuple / rank_tuple  search.py:66-104

Models are returned as plain dicts with the reference's Model fields
(models.py:23-41) so the checker does not depend on either package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from math import comb

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
RANK_TOL_FACTOR = {"fp64": 1e-10, "fp32": 1e-5}  # lsq.py:23

_lib = None


def build(force: bool = False) -> str:
    """Compile liborc.so from l0_oracle.c (gcc, -ffp-contract=off)."""
    src = os.path.join(_HERE, "l0_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liborc.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.orc_score_tuples.argtypes = [vp, i32, i64, vp, vp, i32, vp, i64, i32, dbl, vp]
        L.orc_score_tuples.restype = None
        L.orc_fit_tuple.argtypes = [vp, i32, i64, vp, vp, i32, vp, i32, dbl, vp, vp]
        L.orc_fit_tuple.restype = i32
        L.orc_fill_combinations.argtypes = [vp, i32, i64, vp, i64]
        L.orc_fill_combinations.restype = None
        L.orc_scan.argtypes = [vp, i32, i64, vp, vp, i32, i64, i32, dbl, i64, i64, i32, i32, vp, vp]
        L.orc_scan.restype = i32
        L.orc_binom.argtypes = [i64, i64]
        L.orc_binom.restype = i64
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def prepare(values, property_values, task_slices=None, precision="fp64"):
    """search._prepare (search.py:113-127): cast + task-contiguous permutation."""
    values = np.asarray(values)
    dtype = np.float32 if precision == "fp32" else np.float64
    s = values.shape[1]
    if task_slices is None:
        task_slices = [np.arange(s)]
    perm = np.concatenate([np.asarray(sl, dtype=np.intp) for sl in task_slices])
    if perm.shape[0] != s or not np.array_equal(np.sort(perm), np.arange(s)):
        raise ValueError("task_slices must partition the sample axis")
    bounds = np.zeros(len(task_slices) + 1, dtype=np.int64)
    np.cumsum([len(sl) for sl in task_slices], out=bounds[1:])
    vals = np.ascontiguousarray(values[:, perm], dtype=dtype)
    y = np.ascontiguousarray(np.asarray(property_values, dtype=np.float64)[perm], dtype=dtype)
    return vals, y, bounds, list(task_slices)


def score_tuples(vals, y, bounds, tuples, tol):
    """lsq.score_tuples on prepared arrays; returns float64 scores."""
    vals = np.ascontiguousarray(vals)
    y = np.ascontiguousarray(y, dtype=vals.dtype)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    tuples = np.ascontiguousarray(tuples, dtype=np.int64)
    out = np.empty(tuples.shape[0], dtype=np.float64)
    lib().orc_score_tuples(_ptr(vals), int(vals.dtype == np.float32), vals.shape[1], _ptr(y), _ptr(bounds),
                           bounds.shape[0] - 1, _ptr(tuples), tuples.shape[0], tuples.shape[1], float(tol), _ptr(out))
    return out


def fit_tuple_kernel(vals, y, bounds, tup, tol):
    """lsq.fit_tuple_kernel; returns (ok, coef (ntasks, n+1) working dtype, ssr float64)."""
    vals = np.ascontiguousarray(vals)
    y = np.ascontiguousarray(y, dtype=vals.dtype)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    tup = np.ascontiguousarray(tup, dtype=np.int64)
    T = bounds.shape[0] - 1
    coef = np.zeros((T, tup.shape[0] + 1), dtype=vals.dtype)
    ssr = np.zeros(T, dtype=np.float64)
    ok = lib().orc_fit_tuple(_ptr(vals), int(vals.dtype == np.float32), vals.shape[1], _ptr(y), _ptr(bounds), T,
                             _ptr(tup), tup.shape[0], float(tol), _ptr(coef), _ptr(ssr))
    return bool(ok), coef, ssr


def fill_combinations(cur: np.ndarray, m: int, count: int) -> np.ndarray:
    out = np.empty((count, cur.shape[0]), dtype=np.int64)
    lib().orc_fill_combinations(_ptr(cur), cur.shape[0], m, _ptr(out), count)
    return out


def unrank_tuple(rank: int, m: int, n: int) -> tuple:
    """search.unrank_tuple (search.py:66-85), Python ints."""
    out, r, nxt = [], rank, 0
    for k in range(n):
        rem = n - k - 1
        e = nxt
        while True:
            c = comb(m - 1 - e, rem)
            if r < c:
                break
            r -= c
            e += 1
        out.append(e)
        nxt = e + 1
    return tuple(out)


def rank_tuple(tup, m: int, n: int) -> int:
    """search.rank_tuple (search.py:88-104)."""
    r, nxt = 0, 0
    for k, e in enumerate(tup):
        for v in range(nxt, e):
            r += comb(m - 1 - v, n - k - 1)
        nxt = e + 1
    return r


def scan(vals, y, bounds, m, n, tol, rank_begin, rank_end, keep, threads=1):
    """Exhaustive scores over ranks [rank_begin, rank_end); best `keep` (score, rank)."""
    vals = np.ascontiguousarray(vals)
    y = np.ascontiguousarray(y, dtype=vals.dtype)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    sc = np.empty(keep, dtype=np.float64)
    rk = np.empty(keep, dtype=np.int64)
    got = lib().orc_scan(_ptr(vals), int(vals.dtype == np.float32), vals.shape[1], _ptr(y), _ptr(bounds),
                         bounds.shape[0] - 1, m, n, float(tol), int(rank_begin), int(rank_end), keep, threads,
                         _ptr(sc), _ptr(rk))
    if got < 0:
        raise ValueError("bad scan arguments")
    return [(float(sc[i]), int(rk[i])) for i in range(got)]


def fit_tuple(tup, values, property_values, task_slices=None, precision="fp64"):
    """search.fit_tuple (search.py:136-171) as a dict, or None if rank deficient."""
    vals, y, bounds, slices = prepare(values, property_values, task_slices, precision)
    ok, coef, ssr = fit_tuple_kernel(vals, y, bounds, np.asarray(tup), RANK_TOL_FACTOR[precision])
    if not ok:
        return None
    sizes = np.diff(bounds).astype(np.float64)
    return {
        "indices": tuple(int(i) for i in tup),
        "coefficients": coef.astype(np.float64),
        "score": float(ssr.sum() / vals.shape[1]),
        "rmse_per_task": np.sqrt(ssr / sizes),
    }


def l0_search(values, property_values, task_slices=None, dimension=2, n_models_store=10,
              precision="fp64", threads=1, rank_range=None):
    """search.l0_search semantics (search.py:202-322) on the C kernels.

    Ranking is the exact total order (score, rank); the reference's own merge
    uses the same order (search.py:195-197, 303).
    """
    values = np.asarray(values)
    m = values.shape[0]
    if m < dimension:
        raise ValueError(f"subspace holds {m} features, need at least {dimension}")
    total = comb(m, dimension)
    vals, y, bounds, slices = prepare(values, property_values, task_slices, precision)
    keep = max(1, n_models_store)
    lo, hi = (0, total) if rank_range is None else rank_range
    best = scan(vals, y, bounds, m, dimension, RANK_TOL_FACTOR[precision], lo, hi, keep, threads)
    out = []
    for score, rank in best:
        tup = unrank_tuple(rank, m, dimension)
        md = fit_tuple(tup, values, property_values, task_slices, precision)
        md["rank"] = rank
        md["scan_score"] = score
        out.append(md)
    return out
