"""Final-rung candidates on the B200 -- drop-in for descsearch.generation.iter_final_rung.

The reference streams the last rung instead of storing it
(/root/reference/pkg/src/descsearch/generation.py:331-393): per operator it enumerates the
child pairs (``generate_pairs``), evaluates every candidate's value vector in chunks
(``_chunk_values``), drops the invalid ones (``_validity_mask``), then, in candidate order,
the ones whose canonical key or rounded-value fingerprint was seen before, and yields the
survivors.  Here the pool stays resident on the device and csrc/gen.cu evaluates a chunk of
candidates -- values, validity and a 128-bit fingerprint of the rounded values -- one warp
per candidate; the host keeps only what is symbolic: the pair enumeration and the
expression keys (the reference's own ``generate_pairs`` / ``apply``) and the ordered
dedup walk over the device's flags and fingerprints.

Values are bit-identical to numpy's for the IEEE operators (add, sub, mul, div, abs_diff,
sqrt, sq, cb, inv, abs: one correctly rounded operation per step, no contraction).  The
libm operators (exp, log, sin, cos, cbrt, six_pow) are evaluated by the reference's own
``apply_operator_values`` and only their validity and fingerprints are computed on the
device: a GPU libm differs from numpy's in the last ulp, which would move the validity and
dedup decisions.

``on_device=True`` (what ``install()`` wires into the pipeline together with
``screening.sis_select``) yields ``DeviceChunk`` blocks instead of host matrices: the kept
rows never leave the device unless the screen selects them.
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib

DEVICE_KINDS = {"add": 1, "sub": 2, "mul": 3, "div": 4, "abs_diff": 5, "sqrt": 6, "sq": 7, "cb": 8, "inv": 9,
                "abs": 10}
GEN_COPY, GEN_VALUES = 0, 11
SUB_CHUNK = 65536  # candidates per device pass


class DeviceChunk:
    """The kept candidate rows of one device pass (valid until the generator advances).

    ``sis_scores(target)`` scores them on the device; ``rows(idx)`` copies selected rows
    to the host in the pool's dtype.  ``np.asarray(chunk)`` copies all of them.
    """

    def __init__(self, eng, dev_ptr: int, k: int, s: int, dtype):
        self._eng = eng
        self._ptr = dev_ptr
        self.shape = (k, s)
        self.dtype = np.dtype(dtype)

    def __len__(self):
        return self.shape[0]

    def sis_scores(self, target) -> np.ndarray:
        from .screening import device_chunk_scores

        return device_chunk_scores(self._eng, self._ptr, self.shape[0], target)

    def rows(self, idx) -> np.ndarray:
        return self._eng.gen_fetch(np.asarray(idx, dtype=np.int32))

    def __getitem__(self, i):
        return self.rows([int(i)])[0]

    def __array__(self, dtype=None, copy=None):
        a = self.rows(np.arange(self.shape[0]))
        return a if dtype is None else a.astype(dtype)


def pool_fingerprints(eng, pool) -> set:
    """The pool's own fingerprints, in the device's scheme (pool.dedup_state()'s role)."""
    n = len(pool)
    if n == 0:
        return set()
    _, h = eng.gen_eval(GEN_COPY, pi=np.arange(n, dtype=np.int32), tol=pool.dedup_tolerance, min_abs=0.0,
                        max_abs=np.inf, dedup_tol=0.0)
    return {h[16 * r:16 * r + 16] for r in range(n)}


def iter_final_rung(pool, config, workers: int = 1, timer=None, stats=None, *, device: int | None = None,
                    on_device: bool = False):
    """Generator over the surviving rung ``config.max_rung`` features, never stored
    (generation.iter_final_rung, generation.py:331-393): same (expressions, values) chunks in
    the same order, same ``stats`` counters; ``workers`` is accepted for the signature."""
    from descsearch.expressions import apply, apply_operator_values
    from descsearch.generation import RungStats, generate_pairs

    target_rung = config.max_rung
    if stats is None:
        stats = RungStats(rung=target_rung)
    t0 = time.perf_counter()
    keys = set(pool.dedup_state()[0])
    eng = _lib.engine(device)
    eng.gen_pool(pool.values_matrix())
    fps = pool_fingerprints(eng, pool)
    feats = pool.features
    vals = pool.values
    tol = config.dedup_tolerance
    limits = dict(tol=tol, min_abs=config.min_abs_value, max_abs=config.max_abs_value, dedup_tol=tol)
    batch = max(1, config.value_batch_size)
    spent = time.perf_counter() - t0

    for op in config.operators:
        t0 = time.perf_counter()
        pairs = generate_pairs(op, pool, target_rung).pairs
        stats.n_pairs += len(pairs)
        kind = DEVICE_KINDS.get(op.kind)
        spent += time.perf_counter() - t0
        for start in range(0, len(pairs), batch):  # the reference's value batches
            t0 = time.perf_counter()
            chunk = pairs[start:start + batch]
            out_exprs, out_rows = [], []
            for sub in range(0, len(chunk), SUB_CHUNK):
                sc = chunk[sub:sub + SUB_CHUNK]
                if kind is None:
                    host = np.stack([apply_operator_values(op.kind, vals[i]) if j is None
                                     else apply_operator_values(op.kind, vals[i], vals[j]) for i, j in sc])
                    valid, h = eng.gen_eval(GEN_VALUES, values=host, **limits)
                else:
                    pi = np.fromiter((p[0] for p in sc), dtype=np.int32, count=len(sc))
                    pj = np.fromiter((-1 if p[1] is None else p[1] for p in sc), dtype=np.int32, count=len(sc))
                    valid, h = eng.gen_eval(kind, pi=pi, pj=pj, **limits)
                exprs, kept = [], []
                for row, (i, j) in enumerate(sc):
                    if not valid[row]:
                        stats.n_invalid += 1
                        continue
                    expr = apply(op, feats[i]) if j is None else apply(op, feats[i], feats[j])
                    if expr.key in keys:
                        stats.n_dup_key += 1
                        continue
                    fp = h[16 * row:16 * row + 16]
                    if fp in fps:
                        stats.n_dup_value += 1
                        continue
                    keys.add(expr.key)
                    fps.add(fp)
                    exprs.append(expr)
                    kept.append(row)
                    stats.n_kept += 1
                if not exprs:
                    continue
                if on_device:
                    _, ptr = eng.gen_take(kept)
                    spent += time.perf_counter() - t0
                    if timer is not None:
                        timer.add(spent)
                        spent = 0.0
                    yield exprs, DeviceChunk(eng, ptr, len(kept), eng.gen_s, eng.gen_dtype)
                    t0 = time.perf_counter()
                else:
                    rows, _ = eng.gen_take(kept, host=True)
                    out_exprs.extend(exprs)
                    out_rows.append(rows)
            spent += time.perf_counter() - t0
            if out_exprs:
                if timer is not None:
                    timer.add(spent)
                    spent = 0.0
                yield out_exprs, np.ascontiguousarray(np.concatenate(out_rows))
    if timer is not None and spent:
        timer.add(spent)


__all__ = ["DeviceChunk", "iter_final_rung", "pool_fingerprints", "DEVICE_KINDS"]
