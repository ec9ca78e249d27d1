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


def _scores_locked(F, target, device):
    eng = _lib.engine(device)
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
        sc = eng.sis_scores(F)
        out = sc if out is None else np.maximum(out, sc)
    return out


def projection_score(feature_values, target, *, device: int | None = None) -> float:
    """Score of one feature vector (screening.projection_score, screening.py:158-161)."""
    v = np.asarray(feature_values, dtype=np.float64)
    return float(chunk_scores(v[None, :], target, device=device)[0])


__all__ = ["chunk_scores", "projection_score"]
