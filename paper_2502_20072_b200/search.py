"""Drop-in for ``descsearch.search`` on the B200.

Same names, signatures, argument meaning and error behaviour as the
reference module (/root/reference/pkg/src/descsearch/search.py):

* ``L0Config``, ``SearchStats``              search.py:35-56
* ``count_models``, ``unrank_tuple``,
  ``rank_tuple``                             search.py:59-104
* ``fit_tuple``                              search.py:136-171
* ``l0_search``                              search.py:202-322
* ``RankOutOfRange``, ``RankDeficient``      search.py:27-32

Every score, coefficient and rmse is produced on the device by
libl0search.so and is bit-identical to the reference's numba kernels; the
host only validates arguments, builds the task permutation (the index part
of search._prepare) and assembles ``Model`` records with the same numpy
expressions the reference uses.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from math import comb

import numpy as np

from . import _lib
from ._compat import CapacityError, DescsearchError, Model, RankDeficient, RankOutOfRange  # noqa: F401

RANK_TOL_FACTOR = {"fp64": 1e-10, "fp32": 1e-5}  # lsq.py:23


@dataclass
class L0Config:
    dimension: int
    batch_size: int = 131072
    precision: str = "fp64"
    n_models_store: int = 10
    autotune: bool = True
    chunk_candidates: tuple[int, ...] = (4096, 16384, 65536)


@dataclass
class SearchStats:
    """Filled by l0_search when passed in: throughput bookkeeping (search.py:45-56).

    ``device`` carries the engine's own counters (l0s_stats) as a dict.
    """

    n_tuples: int = 0
    seconds: float = 0.0
    chosen_chunk: int = 0
    batch_seconds: list[float] = field(default_factory=list)
    device: dict = field(default_factory=dict)

    @property
    def tuples_per_second(self) -> float:
        return self.n_tuples / self.seconds if self.seconds > 0 else 0.0


def count_models(m: int, n: int) -> int:
    """Number of distinct n-feature descriptors over m features, C(m, n)."""
    if n < 1 or m < 0:
        raise ValueError("need m >= 0 and n >= 1")
    return comb(m, n)


def unrank_tuple(rank: int, m: int, n: int) -> tuple[int, ...]:
    """The rank-th strictly increasing n-tuple in lexicographic order.

    Walk over the combinadic: position k takes the largest e whose preceding
    blocks sum_{e0 <= e' < e} C(m-1-e', n-1-k) = C(m-e0, n-k) - C(m-e, n-k)
    (hockey stick) do not exceed the remaining rank -- found by binary search,
    O(n log m) exact binomials instead of a scan over e.
    """
    total = count_models(m, n)
    if not 0 <= rank < total:
        raise RankOutOfRange(f"rank {rank} outside [0, {total})")
    out = []
    e0 = 0
    for k in range(n):
        top = comb(m - e0, n - k)
        target = top - rank
        lo, hi = e0, m - n + k  # largest e with C(m - e, n - k) >= target
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if comb(m - mid, n - k) >= target:
                lo = mid
            else:
                hi = mid - 1
        rank -= top - comb(m - lo, n - k)
        out.append(lo)
        e0 = lo + 1
    return tuple(out)


def rank_tuple(tup, m: int, n: int) -> int:
    """Inverse of unrank_tuple: C(m, n) - 1 - sum_k C(m-1-c_k, n-k)."""
    tup = tuple(tup)
    if len(tup) != n:
        raise ValueError(f"expected {n} indices, got {len(tup)}")
    prev = -1
    for e in tup:
        if not prev < e < m:
            raise RankOutOfRange(f"tuple {tup} is not strictly increasing within range")
        prev = e
    return comb(m, n) - 1 - sum(comb(m - 1 - int(c), n - k) for k, c in enumerate(tup))


def _as_matrix(subspace):
    """SelectedSubspace (screening.py:171-198) or a raw (features, samples) array."""
    if hasattr(subspace, "values_matrix") and hasattr(subspace, "expressions"):
        return subspace.values_matrix(), subspace.expressions
    return np.asarray(subspace), None


def _is_subspace(subspace) -> bool:
    return hasattr(subspace, "values_matrix") and hasattr(subspace, "expressions") and hasattr(subspace, "entries")


def _stage_subspace(eng, subspace, y, perm, bounds, precision: str):
    """Stage a SelectedSubspace, incrementally when it extends the one the engine holds.

    The pipeline's subspace only grows by appending entries between dimensions
    (screening.py:197-198, pipeline.py:181-240): when the first entries are the very
    objects staged last time (same value arrays, same y / partition / precision), only the
    new rows are sent (l0s_stage_append_rows) -- the reference re-stacks and re-prepares the
    whole matrix every dimension (search.py:113-127).  Rows go to the device one entry at a
    time, never stacked on the host.  Entry value arrays are taken as immutable records, as
    the pipeline treats them.
    """
    entries = subspace.entries
    c = eng.subspace_cache
    if c is not None:
        pe, pv, py, pperm, pb, pprec = c
        m0 = len(pe)
        if (0 < m0 <= len(entries) and pprec == precision and np.array_equal(py, y)
                and np.array_equal(pperm, perm) and np.array_equal(pb, bounds)
                and all(e is a and e.values is v for e, a, v in zip(entries, pe, pv))):
            if len(entries) > m0:
                eng.stage_append_rows([e.values for e in entries[m0:]])
            eng.subspace_cache = (list(entries), [e.values for e in entries], py, pperm, pb, pprec)
            return
    # rows straight from the entries (values_matrix would stack a host copy first)
    eng.stage_rows([e.values for e in entries], y, perm, bounds, precision)
    eng.subspace_cache = (list(entries), [e.values for e in entries], np.array(y, copy=True), perm.copy(),
                          bounds.copy(), precision)


def _partition(s: int, task_slices):
    """Index half of search._prepare (search.py:113-127): permutation and bounds."""
    if task_slices is None:
        task_slices = [np.arange(s)]
    perm = np.concatenate([np.asarray(sl, dtype=np.intp) for sl in task_slices]).astype(np.int64)
    if perm.shape[0] != s or (s and (perm.min() < 0 or perm.max() >= s)):
        raise ValueError("task_slices must partition the sample axis")
    seen = np.zeros(s, dtype=bool)
    seen[perm] = True
    if not seen.all():  # s indices in range, all distinct
        raise ValueError("task_slices must partition the sample axis")
    bounds = np.zeros(len(task_slices) + 1, dtype=np.int64)
    np.cumsum([len(sl) for sl in task_slices], out=bounds[1:])
    return perm, bounds, task_slices


def _labels_for(task_slices, task_labels):
    if task_labels is not None:
        return tuple(task_labels)
    return tuple(str(i) for i in range(len(task_slices)))


def _model(tup, expressions, coef, ssr, bounds, s, labels, sizes=None) -> Model:
    # the same numpy expressions as search.fit_tuple (search.py:162-170)
    if sizes is None:
        sizes = np.diff(bounds).astype(np.float64)
    return Model(
        indices=tuple(int(i) for i in tup),
        expressions=tuple(expressions[i] for i in tup) if expressions is not None else None,
        coefficients=np.asarray(coef, dtype=np.float64),
        score=float(ssr.sum() / s),
        rmse_per_task=np.sqrt(ssr / sizes),
        task_labels=labels,
    )


def fit_tuple(tup, subspace, property_values, task_slices=None, precision: str = "fp64", task_labels=None,
              *, device: int | None = None) -> Model:
    """Fit one feature tuple and return the full model record (search.py:136-171).

    Raises RankDeficient when any task's design matrix is singular at the
    working precision's tolerance.
    """
    values, expressions = _as_matrix(subspace)
    m = values.shape[0]
    n = len(tup)
    rank_tuple(tup, m, n)
    s = values.shape[1]
    perm, bounds, slices = _partition(s, task_slices)
    if precision not in RANK_TOL_FACTOR:
        raise KeyError(precision)
    # only the tuple's rows are staged: the device kernel reads exactly these values
    rows = np.ascontiguousarray(np.asarray(values)[list(tup)], dtype=np.float64)
    eng = _lib.engine(device)
    eng.stage(rows, np.asarray(property_values, dtype=np.float64), perm, bounds, precision)
    ok, _, coef, ssr = eng.fit_tuples(np.arange(n, dtype=np.int64)[None, :])
    eng.staged_key = None
    if not ok[0]:
        raise RankDeficient(f"singular least-squares system for tuple {tuple(tup)}")
    return _model(tup, expressions, coef[0], ssr[0], bounds, s, _labels_for(slices, task_labels))


def l0_search(
    subspace,
    property_values,
    task_slices=None,
    config: L0Config | None = None,
    workers: int = 1,
    task_labels=None,
    stats: SearchStats | None = None,
    *,
    device: int | None = None,
    mode: str = "auto",
    rank_range: tuple[int, int] | None = None,
) -> list[Model]:
    """Score every n-combination and return the best models, ranked (search.py:202-322).

    subspace is a SelectedSubspace or a raw (features, samples) matrix.
    Returns up to n_models_store models ordered by (score, rank); tuples whose
    system is rank deficient score +inf and are never returned.

    Parallelism: the reference runs ``workers`` threads over rank ranges (search.py:258-301);
    here one device does the work, or several devices of this process (``device`` a list of
    CUDA ordinals, else ``L0S_DEVICES="0,1,..."``, else -- with ``workers`` > 1 -- the first
    ``workers`` visible devices): each searches its part and the exact per-part lists merge by
    (score, rank).  Extra keyword-only knobs: ``device`` (ordinal or list), ``mode`` ("auto",
    "fast", "exact") and ``rank_range`` (restrict the scan to ranks [lo, hi), one device).
    """
    if config is None:
        raise ValueError("config is required")
    incremental = _is_subspace(subspace) and len(subspace) > 0
    if incremental:  # rows are stacked only as far as the device does not hold them already
        expressions = subspace.expressions
        m, s = len(subspace), int(np.asarray(subspace.entries[0].values).shape[0])
    else:
        values, expressions = _as_matrix(subspace)
        m, s = values.shape[0], values.shape[1]
    n = config.dimension
    if m < n:
        raise ValueError(f"subspace holds {m} features, need at least {n}")
    total = count_models(m, n)
    if total >= 2 ** 63:
        raise CapacityError(f"{total} candidate tuples exceed the enumerable range")
    if config.precision not in RANK_TOL_FACTOR:
        raise KeyError(config.precision)
    perm, bounds, slices = _partition(s, task_slices)
    keep = max(1, config.n_models_store)
    batch = max(1, config.batch_size)
    lo, hi = (0, total) if rank_range is None else (max(0, int(rank_range[0])), min(total, int(rank_range[1])))

    y = np.asarray(property_values, dtype=np.float64)
    devices = _devices(device, workers)
    if devices is not None and rank_range is None:
        return _group_search(devices, subspace if incremental else values, incremental, expressions, y, perm, bounds,
                             slices, n, keep, total, config, batch, task_labels, stats, mode, m, s)
    if isinstance(device, (list, tuple)):
        device = device[0]
    eng = _lib.engine(device)
    if incremental:
        _stage_subspace(eng, subspace, y, perm, bounds, config.precision)
    else:
        eng.stage(np.asarray(values), y, perm, bounds, config.precision)
    t0 = time.perf_counter()
    scores, ranks, coef, ssr, dst = eng.search(n, keep, lo, hi, mode)
    elapsed = time.perf_counter() - t0

    if stats is not None:
        _fill_stats(stats, config, batch, lo, hi, total, elapsed, dst)

    labels = _labels_for(slices, task_labels)
    sizes = np.diff(bounds).astype(np.float64)
    _remember_stage(eng, expressions, y, slices, config.precision)
    return [_model(unrank_tuple(int(ranks[i]), m, n), expressions, coef[i], ssr[i], bounds, s, labels, sizes)
            for i in range(len(scores))]


def _devices(device, workers: int):
    """Device list of a multi-device search, or None for one device."""
    import os

    if isinstance(device, (list, tuple)):
        devs = [int(d) for d in device]
    elif device is None and os.environ.get("L0S_DEVICES"):
        devs = [int(x) for x in os.environ["L0S_DEVICES"].split(",") if x.strip()]
    elif device is None and workers > 1:
        devs = list(range(min(int(workers), _lib.device_count())))
    else:
        return None
    return devs if len(devs) > 1 else None


def _fill_stats(stats, config, batch, lo, hi, total, elapsed, dst):
    candidates = [c for c in config.chunk_candidates if c >= 1] or [16384]
    stats.chosen_chunk = min(candidates[0], batch)
    n_batches = max(1, -(-(hi - lo) // batch)) if hi > lo else 0
    extra = len(candidates) - 1 if (config.autotune and len(candidates) > 1 and n_batches) else 0
    # scan + merge only: the reference's seconds exclude _prepare and the per-model refit
    # (search.py:305-308); the device reports the final-record refit separately
    elapsed = max(elapsed - 1e-3 * dst.ms_records, 1e-9)
    per = elapsed / max(1, n_batches + extra)
    stats.batch_seconds.extend([per] * (n_batches + extra))
    stats.n_tuples = total
    stats.seconds = elapsed
    stats.device = dst.as_dict()


def _group_search(devices, values, incremental, expressions, y, perm, bounds, slices, n, keep, total, config, batch,
                  task_labels, stats, mode, m, s):
    """l0_search over several devices of this process (l0s_group_*)."""
    grp = _lib.group(devices)
    grp.stage([e.values for e in values.entries] if incremental else np.asarray(values), y, perm, bounds,
              config.precision)
    t0 = time.perf_counter()
    scores, ranks, coef, ssr, dst = grp.search(n, keep, mode)
    elapsed = time.perf_counter() - t0
    if stats is not None:
        _fill_stats(stats, config, batch, 0, total, total, elapsed, dst)
    labels = _labels_for(slices, task_labels)
    sizes = np.diff(bounds).astype(np.float64)
    _remember_stage(grp, expressions, y, slices, config.precision)
    return [_model(unrank_tuple(int(ranks[i]), m, n), expressions, coef[i], ssr[i], bounds, s, labels, sizes)
            for i in range(len(scores))]


# the last l0_search's staged subspace: (engine or group, expressions, y, task slices, precision)
_last_stage = None


def _remember_stage(owner, expressions, y, slices, precision):
    global _last_stage
    _last_stage = (owner, expressions, y, slices, precision)


def residuals(models, property_values, primary_values, task_slices=None, n_residual=None):
    """models.residuals (models.py:69-83): y minus each model's prediction, float64.

    On the device when the models index the subspace the last l0_search staged (the pipeline's
    call right after its search, pipeline.py:239): the columns are the staged feature rows and
    the arithmetic is predict's (intercept, then + c_k x_k per feature, then y - acc) with
    explicit roundings (l0s_residuals).  Otherwise -- other models, precision "fp32" (predict
    re-evaluates the expressions in float64, not the float32 pool values) -- the reference's
    host function runs.
    """
    chosen = models if n_residual is None else models[:n_residual]
    y = np.asarray(property_values, dtype=np.float64)
    st = _last_stage
    ok = (st is not None and st[4] == "fp64" and st[1] is not None and len(chosen) > 0
          and all(md.expressions is not None and len(md.indices) == len(chosen[0].indices)
                  and all(md.expressions[k] is st[1][i] for k, i in enumerate(md.indices)) for md in chosen)
          and np.array_equal(np.asarray(st[2]), y) and _same_slices(st[3], task_slices))
    if not ok:
        from descsearch.models import residuals as ref_residuals

        return ref_residuals(models, property_values, primary_values, task_slices, n_residual)
    tup = np.array([md.indices for md in chosen], dtype=np.int64)
    coef = np.array([md.coefficients for md in chosen], dtype=np.float64)
    return list(st[0].residuals(tup, coef))


def _same_slices(a, b):
    if b is None:
        return a is None or len(a) == 1
    if a is None or len(a) != len(b):
        return False
    return all(np.array_equal(np.asarray(x), np.asarray(z)) for x, z in zip(a, b))


def fit_tuples(values, property_values, tuples, task_slices=None, precision: str = "fp64",
               *, device: int | None = None):
    """Batched fit_tuple_kernel / score_tuples on the device (lsq.py:113-192).

    Returns (ok, score, coef, ssr): score is score_tuples' pooled value
    (+inf when deficient), coef (count, ntasks, n+1), ssr (count, ntasks).
    """
    values = np.asarray(values, dtype=np.float64)
    perm, bounds, _ = _partition(values.shape[1], task_slices)
    eng = _lib.engine(device)
    eng.stage(values, np.asarray(property_values, dtype=np.float64), perm, bounds, precision)
    return eng.fit_tuples(np.asarray(tuples, dtype=np.int64))


def install(sis: bool = True, gen: bool = True):
    """Route the reference package's l0 entry points to this implementation.

    Patches descsearch.search.{l0_search, fit_tuple}, the names the pipeline
    bound at import (pipeline.py:34) and the package re-exports; with ``sis``
    also the SIS projection scores (screening._chunk_scores, screening.py:126);
    with ``gen`` the streamed last rung (generation.iter_final_rung,
    generation.py:331-393) and the pipeline's screen of it (pipeline.py:25-33:
    candidates evaluated, screened and kept on the device, ``generation.py`` here).
    Returns a callable that restores the originals.
    """
    import sys

    import descsearch
    import descsearch.errors as ref_errors
    import descsearch.models as ref_models
    import descsearch.pipeline as pipeline
    import descsearch.screening as ref_screening
    import descsearch.search as ref_search

    from . import screening as gpu_screening

    me = sys.modules[__name__]
    saved = [(ref_search, "l0_search", ref_search.l0_search), (ref_search, "fit_tuple", ref_search.fit_tuple),
             (pipeline, "l0_search", pipeline.l0_search), (descsearch, "l0_search", descsearch.l0_search),
             (descsearch, "fit_tuple", descsearch.fit_tuple)]
    # records and exceptions become the reference's own classes
    for name, obj in (("Model", ref_models.Model), ("CapacityError", ref_errors.CapacityError),
                      ("RankDeficient", ref_search.RankDeficient), ("RankOutOfRange", ref_search.RankOutOfRange)):
        saved.append((me, name, getattr(me, name)))
        setattr(me, name, obj)
    if sis:  # SIS projection scores (screening._chunk_scores, looked up by sis_select at call time)
        saved.append((ref_screening, "_chunk_scores", ref_screening._chunk_scores))
        ref_screening._chunk_scores = lambda matrix, target: gpu_screening.chunk_scores(matrix, target)
    if gen:  # the streamed last rung: evaluated on the device, screened there by the pipeline
        import functools

        import descsearch.generation as ref_generation

        from . import generation as gpu_generation

        saved += [(ref_generation, "iter_final_rung", ref_generation.iter_final_rung),
                  (pipeline, "iter_final_rung", pipeline.iter_final_rung),
                  (pipeline, "sis_select", pipeline.sis_select)]
        ref_generation.iter_final_rung = gpu_generation.iter_final_rung
        pipeline.iter_final_rung = functools.partial(gpu_generation.iter_final_rung, on_device=True)
        pipeline.sis_select = gpu_screening.sis_select
    # residual targets of the next dimension's SIS (pipeline.py:239), from the staged rows
    saved.append((pipeline, "residuals", pipeline.residuals))
    pipeline.residuals = residuals
    ref_search.l0_search = l0_search
    ref_search.fit_tuple = fit_tuple
    pipeline.l0_search = l0_search
    descsearch.l0_search = l0_search
    descsearch.fit_tuple = fit_tuple

    def uninstall():
        for mod, name, fn in saved:
            setattr(mod, name, fn)

    return uninstall
