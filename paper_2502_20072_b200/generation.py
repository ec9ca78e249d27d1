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
``screening.sis_select``) yields ``DeviceChunk`` blocks instead of host matrices, and
``PendingExpr`` records (canonical key now, expression node on ``build()``): the kept rows
never leave the device and the nodes are never built unless the screen selects them.
"""

from __future__ import annotations

import time
import weakref

import numpy as np

from . import _lib
from .screening import _lock  # one context per device is shared with the SIS scores (threads)

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
        with _lock:
            return self._eng.gen_fetch(np.asarray(idx, dtype=np.int32))

    def __getitem__(self, i):
        return self.rows([int(i)])[0]

    def __array__(self, dtype=None, copy=None):
        a = self.rows(np.arange(self.shape[0]))
        return a if dtype is None else a.astype(dtype)


def _key(op, ka: str, kb: str | None) -> str:
    """expressions.apply's canonical key (expressions.py:152-161), without building the node."""
    if kb is None:
        return f"{op.kind}({ka})"
    if op.commutative:
        ab, ba = ka + "," + kb, kb + "," + ka
        return f"{op.kind}({ab if ab <= ba else ba})"
    return f"{op.kind}({ka},{kb})"


class PendingExpr:
    """A kept candidate of the device stream: the canonical key on first access, the
    expression node (expressions.apply) when ``build()`` is called -- sis_select builds only
    the ones it keeps."""

    __slots__ = ("op", "a", "b", "_key")

    def __init__(self, op, a, b, key=None):
        self.op, self.a, self.b, self._key = op, a, b, key

    @property
    def key(self) -> str:
        if self._key is None:
            self._key = _key(self.op, self.a.key, None if self.b is None else self.b.key)
        return self._key

    def build(self):
        from descsearch.expressions import apply

        return apply(self.op, self.a) if self.b is None else apply(self.op, self.a, self.b)


class PendingExprs:
    """The kept candidates of one device pass as index arrays; items (``PendingExpr``) are
    made on access.  ``not_taken(entries)`` masks out candidates that are the expressions of
    already-selected entries without building any key (sis_select's ``taken`` test)."""

    def __init__(self, op, pi, pj, feats, index_of):
        self.op, self.pi, self.pj, self._feats, self._index_of = op, pi, pj, feats, index_of

    def __len__(self):
        return len(self.pi)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[x] for x in range(*k.indices(len(self)))]
        i, j = int(self.pi[k]), int(self.pj[k])
        return PendingExpr(self.op, self._feats[i], None if j < 0 else self._feats[j])

    def __iter__(self):
        return (self[k] for k in range(len(self)))

    def not_taken(self, entries) -> np.ndarray:
        n = len(self._feats)
        codes = []
        for e in entries:
            ex = e.expression
            if ex.op is None or ex.op.kind != self.op.kind:
                continue
            ch = [self._index_of.get(c.key) for c in ex.children]
            if any(c is None for c in ch):
                continue
            codes.append(ch[0] * (n + 1) + (ch[1] + 1 if len(ch) > 1 else 0))
        mine = self.pi.astype(np.int64) * (n + 1) + (self.pj.astype(np.int64) + 1)
        return ~np.isin(mine, np.asarray(codes, dtype=np.int64)) if codes else np.ones(len(self), dtype=bool)


_PAIRS = weakref.WeakKeyDictionary()  # pool -> {(len, operator, rung): (pi, pj)}


def pair_arrays(op, pool, target_rung: int):
    """generation.generate_pairs (generation.py:205-242) as index arrays (pj = -1: unary):
    the same pairs in the same order (first child ascending, second ascending within it),
    built with numpy masks over the eligible features instead of a Python double loop; the
    unit rule (expressions.check_unit) is evaluated once per distinct unit pair.  The pool only
    grows by appending, so the arrays are kept per (pool, its length, operator, rung): the
    pipeline streams the same last rung once per dimension (pipeline.py:181-240)."""
    key = (len(pool), op.kind, op.arity, bool(getattr(op, "commutative", False)), int(target_rung))
    try:
        cache = _PAIRS.setdefault(pool, {})
    except TypeError:  # a pool that cannot be weakly referenced: no cache
        cache = {}
    hit = cache.get(key)
    if hit is None:
        hit = _pair_arrays(op, pool, target_rung)
        for x in hit:
            x.setflags(write=False)  # shared between calls
        cache[key] = hit
    return hit


def _pair_arrays(op, pool, target_rung: int):
    from descsearch.expressions import check_unit

    prev = target_rung - 1
    if prev < 0:
        raise ValueError("target_rung must be at least 1")
    feats = pool.features
    if op.arity == 1:
        idx = [i for i in pool.rung_indices(prev) if check_unit(op, (feats[i].unit,)) is not None]
        return np.asarray(idx, dtype=np.int32), np.full(len(idx), -1, dtype=np.int32)
    elig = [i for i in range(len(pool)) if feats[i].rung <= prev]
    if not elig:
        return np.zeros(0, dtype=np.int32), np.zeros(0, dtype=np.int32)
    units, uid = {}, []
    for i in elig:
        uid.append(units.setdefault(feats[i].unit, len(units)))
    ulist = list(units)
    ok = np.array([[check_unit(op, (ua, ub)) is not None for ub in ulist] for ua in ulist], dtype=bool)
    e = np.asarray(elig, dtype=np.int64)
    u = np.asarray(uid, dtype=np.int64)
    r = np.asarray([feats[i].rung for i in elig], dtype=np.int64)
    zero_b = np.asarray([pool._has_zero[i] for i in elig], dtype=bool) if op.kind == "div" else None
    n = len(elig)
    out_i, out_j = [], []
    step = max(1, (1 << 22) // max(n, 1))  # first children per block: ~4M candidate cells
    for a0 in range(0, n, step):
        a1 = min(n, a0 + step)
        A = np.arange(a0, a1)[:, None]
        B = np.arange(n)[None, :]
        m = np.maximum(r[A], r[B]) == prev
        if op.commutative:
            m &= B >= A
        m &= ok[u[A], u[B]]
        if zero_b is not None:
            m &= ~zero_b[B]
        aa, bb = np.nonzero(m)  # row-major: first child, then second
        out_i.append(e[aa + a0])
        out_j.append(e[bb])
    return (np.concatenate(out_i).astype(np.int32), np.concatenate(out_j).astype(np.int32))


def pool_fingerprints(eng, pool) -> set:
    """The pool's own fingerprints, in the device's scheme (pool.dedup_state()'s role)."""
    n = len(pool)
    if n == 0:
        return set()
    with _lock:
        _, h = eng.gen_eval(GEN_COPY, pi=np.arange(n, dtype=np.int32), tol=pool.dedup_tolerance, min_abs=0.0,
                            max_abs=np.inf, dedup_tol=0.0)
    return {h[16 * r:16 * r + 16] for r in range(n)}


def iter_final_rung(pool, config, workers: int = 1, timer=None, stats=None, *, device: int | None = None,
                    on_device: bool = False):
    """Generator over the surviving rung ``config.max_rung`` features, never stored
    (generation.iter_final_rung, generation.py:331-393): same (expressions, values) chunks in
    the same order, same ``stats`` counters; ``workers`` is accepted for the signature."""
    from descsearch.expressions import apply, apply_operator_values
    from descsearch.generation import RungStats

    target_rung = config.max_rung
    if stats is None:
        stats = RungStats(rung=target_rung)
    t0 = time.perf_counter()
    keys = set(pool.dedup_state()[0])
    eng = _lib.engine(device)
    with _lock:
        eng.gen_pool(pool.values_matrix())
    fps = pool_fingerprints(eng, pool)
    kinds0 = [op.kind for op in config.operators]
    device_walk = len(set(kinds0)) == len(kinds0) and (len(pool) == 0 or pool.max_rung() < target_rung)
    if device_walk:  # the value dedup runs on the device, seeded with the pool's fingerprints
        with _lock:
            eng.gen_dedup_reset(fps)
    feats = pool.features
    fkeys = [f.key for f in feats]
    index_of = {k: x for x, k in enumerate(fkeys)}
    vals = pool.values
    # A final-rung key is op(child keys): its nesting depth is its rung, so it never equals a
    # pool key (rungs < max), and it is unique per (operator, pair).  With distinct operator
    # kinds the key test can therefore never fire: keys are then built only on demand.
    kinds = [op.kind for op in config.operators]
    keys_free = len(set(kinds)) == len(kinds) and (len(pool) == 0 or pool.max_rung() < target_rung)
    # fingerprints: the first 64 bits index the set, the full 128 bits decide
    fp64 = {}
    for fp in fps:
        fp64.setdefault(int.from_bytes(fp[:8], "little"), []).append(fp)
    tol = config.dedup_tolerance
    limits = dict(tol=tol, min_abs=config.min_abs_value, max_abs=config.max_abs_value, dedup_tol=tol)
    batch = max(1, config.value_batch_size)
    spent = time.perf_counter() - t0

    for op in config.operators:
        t0 = time.perf_counter()
        all_i, all_j = pair_arrays(op, pool, target_rung)
        stats.n_pairs += len(all_i)
        kind = DEVICE_KINDS.get(op.kind)
        spent += time.perf_counter() - t0
        for start in range(0, len(all_i), batch):  # the reference's value batches
            t0 = time.perf_counter()
            stop = min(len(all_i), start + batch)
            out_exprs, out_rows = [], []
            for sub in range(start, stop, SUB_CHUNK):
                pi, pj = all_i[sub:min(stop, sub + SUB_CHUNK)], all_j[sub:min(stop, sub + SUB_CHUNK)]
                if kind is None:
                    host = np.stack([apply_operator_values(op.kind, vals[i]) if j < 0
                                     else apply_operator_values(op.kind, vals[i], vals[j])
                                     for i, j in zip(pi.tolist(), pj.tolist())])
                    with _lock:
                        valid, h = eng.gen_eval(GEN_VALUES, values=host, **limits)
                else:
                    with _lock:
                        valid, h = eng.gen_eval(kind, pi=pi, pj=pj, **limits)
                rows_ok = np.flatnonzero(valid)
                stats.n_invalid += len(pi) - len(rows_ok)
                if device_walk:
                    # keys cannot collide (distinct operator kinds): only the value test remains, and
                    # the device's ordered-first-owner set decides it (dedup.cu)
                    with _lock:
                        kept = np.flatnonzero(eng.gen_dedup())  # an index array: never a Python list
                    stats.n_dup_value += len(rows_ok) - len(kept)
                    rows_ok = rows_ok[:0]
                else:
                    kept = []
                h64 = np.frombuffer(h, dtype="<u8")[0::2][rows_ok].tolist()
                hv = np.frombuffer(h, dtype="V16")[rows_ok].tolist() if len(rows_ok) else []
                li, lj = pi[rows_ok].tolist(), pj[rows_ok].tolist()
                # the reference's ordered walk (generation.py:364-385): invalid, key, fingerprint
                for x, row in enumerate(rows_ok.tolist()):
                    key = None
                    if not keys_free:
                        i, j = li[x], lj[x]
                        key = _key(op, fkeys[i], None if j < 0 else fkeys[j])
                        if key in keys:
                            stats.n_dup_key += 1
                            continue
                    fp, f = hv[x], h64[x]
                    same = fp64.get(f)
                    if same is not None and fp in same:
                        stats.n_dup_value += 1
                        continue
                    if key is not None:
                        keys.add(key)
                    if same is None:
                        fp64[f] = [fp]
                    else:
                        same.append(fp)
                    kept.append(row)
                kept = np.asarray(kept, dtype=np.int64)
                stats.n_kept += len(kept)
                if len(kept) == 0:
                    continue
                if on_device:
                    exprs = PendingExprs(op, pi[kept], pj[kept], feats, index_of)
                    with _lock:
                        _, ptr = eng.gen_take(kept)
                    spent += time.perf_counter() - t0
                    if timer is not None:
                        timer.add(spent)
                        spent = 0.0
                    yield exprs, DeviceChunk(eng, ptr, len(kept), eng.gen_s, eng.gen_dtype)
                    t0 = time.perf_counter()
                else:
                    with _lock:
                        rows, _ = eng.gen_take(kept, host=True)
                    out_exprs.extend(apply(op, feats[i]) if j < 0 else apply(op, feats[i], feats[j])
                                     for i, j in zip(pi[kept].tolist(), pj[kept].tolist()))
                    out_rows.append(rows)
            spent += time.perf_counter() - t0
            if out_exprs:
                if timer is not None:
                    timer.add(spent)
                    spent = 0.0
                yield out_exprs, np.ascontiguousarray(np.concatenate(out_rows))
    if timer is not None and spent:
        timer.add(spent)


__all__ = ["DeviceChunk", "PendingExpr", "PendingExprs", "iter_final_rung", "pair_arrays", "pool_fingerprints", "DEVICE_KINDS"]
