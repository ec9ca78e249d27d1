"""SIS projection scores on the B200 -- drop-in for descsearch.screening._chunk_scores.

The reference ranks candidate features by the sample-weighted mean over tasks of
|Pearson(feature, target)|, best over targets, clipped to [0, 1], with every sum taken by a
fixed-shape pairwise tree so that scores do not depend on chunking
(/root/reference/pkg/src/descsearch/screening.py:102-155).  ``chunk_scores`` computes the
same values, bit for bit, in libl0search.so (csrc/sis.cu); ``sis_select`` itself (the
running top list ordered by (score desc, canonical key asc), screening.py:201-257) stays the
reference's host code and reaches this through ``install()``.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

from . import _lib

_MAX_TARGETS = 8  # per device pass (l0s_sis_prepare); more targets are folded with np.maximum
_lock = threading.Lock()  # sis_select may score chunks from a thread pool; a context is single-threaded


def _partition(target):
    slices = [np.asarray(sl, dtype=np.int64) for sl in target.task_slices]
    perm = np.concatenate(slices) if slices else np.zeros(0, dtype=np.int64)
    bounds = np.zeros(len(slices) + 1, dtype=np.int64)
    np.cumsum([len(sl) for sl in slices], out=bounds[1:])
    return perm, bounds


def chunk_scores(matrix, target, *, device: int | None = None) -> np.ndarray:
    """Projection scores of a (features, samples) chunk (screening._chunk_scores).

    ``target`` is a descsearch ScreeningTarget (or anything with ``targets``,
    ``task_slices`` and ``n_samples``).  Returns float64 scores, bit-identical to the
    reference's.
    """
    F = np.ascontiguousarray(matrix, dtype=np.float64)
    if F.ndim != 2:
        raise ValueError("expected a (features, samples) matrix")
    k = F.shape[0]
    if k == 0:
        return np.zeros(0)
    if F.shape[1] != target.n_samples:
        raise ValueError(f"matrix has {F.shape[1]} samples, target {target.n_samples}")
    with _lock:
        return _scores_locked(F, target, device)


def _scores_locked(F, target, device, eng=None, dev=None):
    eng = eng if eng is not None else _lib.engine(device)
    groups = [target.targets[i:i + _MAX_TARGETS] for i in range(0, len(target.targets), _MAX_TARGETS)]
    out = None
    for g, tg in enumerate(groups):
        key = (g, len(groups))
        ref = getattr(eng, "_sis_target", None)
        if len(groups) > 1 or ref is None or ref() is not target or getattr(eng, "_sis_key", None) != key:
            perm, bounds = _partition(target)
            eng.sis_prepare(np.stack([np.asarray(t, dtype=np.float64) for t in tg]), perm, bounds)
            eng._sis_target = weakref.ref(target)
            eng._sis_key = key
        sc = eng.sis_scores(F) if dev is None else eng.sis_scores(None, device_ptr=dev[0], k=dev[1])
        out = sc if out is None else np.maximum(out, sc)
    return out


def device_chunk_scores(eng, dev_ptr: int, k: int, target) -> np.ndarray:
    """Scores of k fp64 rows already on the engine's device (a generation.DeviceChunk)."""
    if k == 0:
        return np.zeros(0)
    with _lock:
        return _scores_locked(None, target, None, eng=eng, dev=(dev_ptr, k))


def sis_select(source, target, n_sis_select: int, already_selected=None, workers: int = 1, chunk_size: int = 65536):
    """Screen a candidate stream and grow the selected subspace (screening.sis_select,
    screening.py:201-257): the same entries, scores and order -- the top ``n_sis_select`` new
    candidates by (score desc, canonical key asc).

    Chunks may be host matrices (scored through ``chunk_scores``) or ``DeviceChunk`` blocks
    from ``generation.iter_final_rung(on_device=True)``, scored where they lie; a row's
    values are copied out only when it enters the running top list (the reference copies
    every new row of every chunk).  ``workers`` is accepted for the signature.
    """
    from descsearch.generation import FeatureSpace
    from descsearch.screening import EmptySpace, SelectedSubspace, SubspaceEntry

    from .generation import DeviceChunk, PendingExpr, PendingExprs

    if n_sis_select < 1:
        raise ValueError("n_sis_select must be positive")
    prior = already_selected if already_selected is not None else SelectedSubspace()
    taken = prior.keys()
    chunks = source.iter_batches(chunk_size) if isinstance(source, FeatureSpace) else iter(source)
    best: list = []  # [-score, key, expr, values or None, row] ascending
    n_new_seen = 0
    for exprs, matrix in chunks:
        on_dev = isinstance(matrix, DeviceChunk)
        scores = np.asarray(matrix.sis_scores(target) if on_dev else chunk_scores(matrix, target))
        if isinstance(exprs, PendingExprs):  # device stream: the taken test on index pairs
            new = exprs.not_taken(prior.entries) if taken else np.ones(len(exprs), dtype=bool)
        else:
            new = np.fromiter((e.key not in taken for e in exprs), dtype=bool, count=len(exprs))
        n_new_seen += int(new.sum())
        # only a score at or above the current n-th can enter the list (ties go by key)
        ok = new & (scores >= -best[-1][0]) if len(best) >= n_sis_select else new
        cand = [[-float(scores[i]), exprs[i].key, exprs[i], None, i] for i in np.flatnonzero(ok).tolist()]
        if not cand:
            continue
        best = sorted(best + cand, key=lambda item: (item[0], item[1]))[:n_sis_select]
        fresh = [item for item in best if item[3] is None]
        if fresh:
            if on_dev:
                rows = matrix.rows([item[4] for item in fresh])
                for item, r in zip(fresh, rows):
                    item[3] = np.array(r, copy=True)
            else:
                for item in fresh:
                    item[3] = np.array(matrix[item[4]], copy=True)
    if n_new_seen == 0:
        raise EmptySpace("no unselected candidates in the screened space")
    return prior.extended([SubspaceEntry(expr.build() if isinstance(expr, PendingExpr) else expr, -neg, vals)
                           for neg, _, expr, vals, _ in best])


def projection_score(feature_values, target, *, device: int | None = None) -> float:
    """Score of one feature vector (screening.projection_score, screening.py:158-161)."""
    v = np.asarray(feature_values, dtype=np.float64)
    return float(chunk_scores(v[None, :], target, device=device)[0])


__all__ = ["chunk_scores", "device_chunk_scores", "projection_score", "sis_select"]
