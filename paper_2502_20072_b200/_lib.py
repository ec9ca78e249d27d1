"""ctypes binding of libl0search.so (include/l0search.h).

The shared library is built in-tree (``python -m paper_2502_20072_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library or
a B200 device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _compat

HERE = os.path.dirname(os.path.abspath(__file__))
# L0S_LIB selects a tuning variant built by tools/tune_fit.py (same ABI, in-tree .so)
LIB_PATH = os.environ.get("L0S_LIB") or os.path.join(HERE, "libl0search.so")

L0S_OK, L0S_EINVAL, L0S_ECAPACITY, L0S_ECUDA, L0S_ENOMEM, L0S_ENODEV, L0S_ESTATE = range(7)
PREC = {"fp64": 0, "fp32": 1}
MODES = {"auto": 0, "fast": 1, "exact": 2}

# every symbol include/l0search.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "l0s_last_error", "l0s_version", "l0s_device_count", "l0s_create", "l0s_destroy", "l0s_stage",
    "l0s_search", "l0s_fit_tuples", "l0s_screen_tuples", "l0s_get_gram", "l0s_unrank", "l0s_rank",
    "l0s_count", "l0s_fp64_peak", "l0s_rcp_check", "l0s_gram_shard_size", "l0s_stage_shard",
    "l0s_stage_finish", "l0s_sis_prepare", "l0s_sis_scores", "l0s_set_gram_mode", "l0s_stage_info", "l0s_stage_loose_rows", "l0s_stage_timings", "l0s_qr_tuples", "l0s_residuals",
    "l0s_gen_dedup_reset", "l0s_gen_dedup",
    "l0s_group_create", "l0s_group_destroy", "l0s_group_size", "l0s_group_ctx", "l0s_group_stage", "l0s_group_search",
    "l0s_stage_append", "l0s_search_part", "l0s_set_part_exchange", "l0s_stage_rows", "l0s_stage_append_rows", "l0s_gen_pool", "l0s_gen_eval", "l0s_gen_take", "l0s_gen_fetch",
)


# l0s_exchange_fn: double (*)(const double* scores, int64_t count, void* user)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_void_p)


class Stats(ctypes.Structure):
    """Mirror of l0s_stats."""

    _fields_ = [
        ("n_tuples", ctypes.c_int64),
        ("ms_total", ctypes.c_double),
        ("ms_fit", ctypes.c_double),
        ("ms_exact", ctypes.c_double),
        ("ms_gram", ctypes.c_double),
        ("theta", ctypes.c_double),
        ("n_candidates", ctypes.c_int64),
        ("n_ill", ctypes.c_int64),
        ("n_rescan", ctypes.c_int64),
        ("n_fit_launches", ctypes.c_int64),
        ("n_launches", ctypes.c_int64),
        ("mode_used", ctypes.c_int32),
        ("certified", ctypes.c_int32),
        ("margin", ctypes.c_double),
        ("ms_qr", ctypes.c_double),
        ("n_ill_refit", ctypes.c_int64),
        ("ms_gram_kernel", ctypes.c_double),
        ("ms_records", ctypes.c_double),
        ("n_eval", ctypes.c_int64),
        ("n_screen", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def lib():
    """Load and type the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2502_20072_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        P = ctypes.POINTER
        L.l0s_last_error.restype = ctypes.c_char_p
        L.l0s_last_error.argtypes = []
        L.l0s_version.restype = i32
        L.l0s_device_count.argtypes = [P(i32)]
        L.l0s_create.argtypes = [i32, P(vp)]
        L.l0s_destroy.argtypes = [vp]
        L.l0s_stage.argtypes = [vp, vp, i64, i64, vp, vp, vp, i32, i32, i32]
        L.l0s_gram_shard_size.argtypes = [i64, i32, i32, P(i64)]
        L.l0s_stage_shard.argtypes = [vp, vp, i64, i64, vp, vp, vp, i32, i32, i32, i32, i32, vp]
        L.l0s_stage_finish.argtypes = [vp, vp]
        L.l0s_stage_append.argtypes = [vp, vp, i64]
        L.l0s_stage_rows.argtypes = [vp, vp, i64, i64, vp, vp, vp, i32, i32]
        L.l0s_stage_append_rows.argtypes = [vp, vp, i64]
        L.l0s_gen_pool.argtypes = [vp, vp, i64, i64, i32]
        L.l0s_gen_eval.argtypes = [vp, i32, vp, vp, i64, vp, dbl, dbl, dbl, dbl, vp, vp]
        L.l0s_gen_take.argtypes = [vp, vp, i64, vp, P(vp)]
        L.l0s_gen_fetch.argtypes = [vp, vp, i64, vp]
        L.l0s_set_gram_mode.argtypes = [vp, i32]
        L.l0s_stage_info.argtypes = [vp, vp, vp]
        L.l0s_stage_loose_rows.argtypes = [vp, vp]
        L.l0s_set_part_exchange.argtypes = [vp, vp, vp]
        L.l0s_stage_timings.argtypes = [vp, vp]
        L.l0s_qr_tuples.argtypes = [vp, i32, vp, i64, vp, vp]
        L.l0s_residuals.argtypes = [vp, i32, vp, vp, i64, vp]
        L.l0s_gen_dedup_reset.argtypes = [vp, vp, i64]
        L.l0s_gen_dedup.argtypes = [vp, vp, P(i64)]
        L.l0s_sis_prepare.argtypes = [vp, vp, i32, i64, vp, vp, i32]
        L.l0s_sis_scores.argtypes = [vp, vp, i64, i32, vp]
        L.l0s_search.argtypes = [vp, i32, i64, i64, i64, i32, vp, vp, vp, vp, P(i64), P(Stats)]
        L.l0s_search_part.argtypes = [vp, i32, i64, i32, i32, i32, vp, vp, vp, vp, P(i64), P(Stats)]
        L.l0s_fit_tuples.argtypes = [vp, i32, vp, i64, vp, vp, vp, vp]
        L.l0s_screen_tuples.argtypes = [vp, i32, vp, i64, vp, vp]
        L.l0s_get_gram.argtypes = [vp, i32, vp]
        L.l0s_unrank.argtypes = [i64, i64, i32, vp]
        L.l0s_rank.argtypes = [vp, i64, i32, P(i64)]
        L.l0s_count.argtypes = [i64, i32, P(i64)]
        L.l0s_fp64_peak.argtypes = [vp, P(dbl)]
        L.l0s_rcp_check.argtypes = [i64, P(dbl)]
        L.l0s_group_create.argtypes = [i32, vp, P(vp)]
        L.l0s_group_destroy.argtypes = [vp]
        L.l0s_group_size.argtypes = [vp, P(i32)]
        L.l0s_group_ctx.argtypes = [vp, i32, P(vp)]
        L.l0s_group_stage.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, i32, i32]
        L.l0s_group_search.argtypes = [vp, i32, i64, i32, vp, vp, vp, vp, P(i64), P(Stats)]
        for name in EXPORTS:
            if name not in ("l0s_last_error",):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map an l0s status to the reference's exception types."""
    if rc == L0S_OK:
        return
    msg = lib().l0s_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == L0S_EINVAL:
        raise ValueError(msg)
    if rc == L0S_ECAPACITY:
        raise _compat.CapacityError(msg)
    raise RuntimeError(f"l0search error {rc}: {msg}")


def ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class Engine:
    """One device context (owns device memory, a stream and events)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = ctypes.c_void_p()
        check(L.l0s_create(int(device), ctypes.byref(h)), "l0s_create")
        self.handle = h
        self.device = device
        self.staged_key = None
        # (entries, their value arrays, y, perm, bounds, precision) of the SelectedSubspace the
        # context holds (search.l0_search's incremental stage); any other stage clears it
        self.subspace_cache = None

    def close(self):
        if self.handle:
            lib().l0s_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage(self, values: np.ndarray, y: np.ndarray, perm: np.ndarray, bounds: np.ndarray, precision: str,
              device_ptrs: tuple | None = None) -> None:
        """Host arrays (or, with device_ptrs=(values, y, perm) data pointers, device-resident inputs)."""
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        m, s = values.shape if device_ptrs is None else (values[0], values[1])
        if device_ptrs is None:
            values = np.ascontiguousarray(values, dtype=np.float64)
            y = np.ascontiguousarray(y, dtype=np.float64)
            perm = np.ascontiguousarray(perm, dtype=np.int64)
            args = (ptr(values), m, s, ptr(y), ptr(perm))
            is_dev = 0
        else:
            args = (ctypes.c_void_p(device_ptrs[0]), m, s, ctypes.c_void_p(device_ptrs[1]),
                    ctypes.c_void_p(device_ptrs[2]))
            is_dev = 1
        self.subspace_cache = None
        check(lib().l0s_stage(self.handle, *args, ptr(bounds), bounds.shape[0] - 1, PREC[precision], is_dev),
              "l0s_stage")
        self.m, self.s, self.T = int(m), int(s), bounds.shape[0] - 1

    @staticmethod
    def _row_pointers(arrays, s: int):
        rows = [np.ascontiguousarray(a, dtype=np.float64) for a in arrays]
        for r in rows:
            if r.ndim != 1 or r.shape[0] != s:
                raise ValueError(f"every row must hold {s} samples")
        return rows, (ctypes.c_void_p * len(rows))(*[r.ctypes.data for r in rows])

    def stage_rows(self, arrays, y: np.ndarray, perm: np.ndarray, bounds: np.ndarray, precision: str) -> None:
        """Stage host feature rows given as separate arrays (no host stacking; l0s_stage_rows)."""
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        s = y.shape[0]
        keep, ptrs = self._row_pointers(arrays, s)
        self.subspace_cache = None
        check(lib().l0s_stage_rows(self.handle, ptrs, len(keep), s, ptr(y), ptr(perm), ptr(bounds),
                                   bounds.shape[0] - 1, PREC[precision]), "l0s_stage_rows")
        self.m, self.s, self.T = len(keep), int(s), bounds.shape[0] - 1

    def stage_append_rows(self, arrays) -> None:
        """Append feature rows given as separate host arrays (l0s_stage_append_rows)."""
        keep, ptrs = self._row_pointers(arrays, self.s)
        check(lib().l0s_stage_append_rows(self.handle, ptrs, len(keep)), "l0s_stage_append_rows")
        self.m += len(keep)

    def stage_append(self, rows: np.ndarray) -> None:
        """Append feature rows (host, (m_new, s)) to the staged host problem (l0s_stage_append)."""
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        if rows.ndim != 2 or rows.shape[1] != self.s:
            raise ValueError(f"rows must be (m_new, {self.s})")
        check(lib().l0s_stage_append(self.handle, ptr(rows), rows.shape[0]), "l0s_stage_append")
        self.m += rows.shape[0]

    @staticmethod
    def gram_shard_size(m: int, ntasks: int, nshards: int) -> int:
        """Doubles in one rank's Gram pack (l0s_gram_shard_size)."""
        out = ctypes.c_int64(0)
        check(lib().l0s_gram_shard_size(int(m), int(ntasks), int(nshards), ctypes.byref(out)), "l0s_gram_shard_size")
        return out.value

    def stage_shard(self, shape: tuple, bounds: np.ndarray, precision: str, device_ptrs: tuple, shard: int,
                    nshards: int, pack_ptr: int) -> None:
        """Stage device-resident inputs and compute this rank's Gram shard into pack_ptr (device)."""
        self.subspace_cache = None
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        m, s = shape
        check(lib().l0s_stage_shard(self.handle, ctypes.c_void_p(device_ptrs[0]), m, s, ctypes.c_void_p(device_ptrs[1]),
                                    ctypes.c_void_p(device_ptrs[2]), ptr(bounds), bounds.shape[0] - 1,
                                    PREC[precision], 1, int(shard), int(nshards), ctypes.c_void_p(pack_ptr)),
              "l0s_stage_shard")
        self.m, self.s, self.T = int(m), int(s), bounds.shape[0] - 1

    def stage_finish(self, gathered_ptr: int) -> None:
        """Scatter the all-gathered packs (device pointer, nshards x pack doubles) into the Gram."""
        check(lib().l0s_stage_finish(self.handle, ctypes.c_void_p(gathered_ptr)), "l0s_stage_finish")

    def set_gram_mode(self, mode: str) -> None:
        """'auto' | 'dmma' | 'ozaki' (INT8 tensor cores) for subsequent stages."""
        check(lib().l0s_set_gram_mode(self.handle, {"auto": 0, "dmma": 1, "ozaki": 2}[mode]), "l0s_set_gram_mode")

    def stage_info(self):
        """(per-task Gram entry error bound eta, whether the INT8 path produced the Gram)."""
        eta = np.zeros(self.T, dtype=np.float64)
        oz = ctypes.c_int(0)
        check(lib().l0s_stage_info(self.handle, ptr(eta), ctypes.byref(oz)), "l0s_stage_info")
        return eta, bool(oz.value)

    def stage_loose_rows(self) -> int:
        """Rows of the last INT8 Gram recomputed in fp64 (their own error term was too large)."""
        n = ctypes.c_int(0)
        check(lib().l0s_stage_loose_rows(self.handle, ctypes.byref(n)), "l0s_stage_loose_rows")
        return int(n.value)

    def residuals(self, tuples: np.ndarray, coef: np.ndarray) -> np.ndarray:
        """y - prediction of each model (tuple of staged features, (T, n+1) coefficients), float64 (count, s)."""
        tuples = np.ascontiguousarray(np.atleast_2d(tuples), dtype=np.int64)
        coef = np.ascontiguousarray(coef, dtype=np.float64).reshape(len(tuples), self.T, tuples.shape[1] + 1)
        out = np.empty((len(tuples), self.s), dtype=np.float64)
        check(lib().l0s_residuals(self.handle, tuples.shape[1], ptr(tuples), ptr(coef), len(tuples), ptr(out)),
              "l0s_residuals")
        return out

    def qr_tuples(self, tuples: np.ndarray):
        """Device QR screen of explicit tuples: (pooled score, min rank-rule ratio over tasks)."""
        tuples = np.ascontiguousarray(np.atleast_2d(tuples), dtype=np.int64)
        sc = np.empty(len(tuples))
        rt = np.empty(len(tuples))
        check(lib().l0s_qr_tuples(self.handle, tuples.shape[1], ptr(tuples), len(tuples), ptr(sc), ptr(rt)),
              "l0s_qr_tuples")
        return sc, rt

    def stage_timings(self) -> dict:
        """Device ms of the last device-resident stage: gather, normalize, gram, flags."""
        out = np.zeros(4, dtype=np.float64)
        check(lib().l0s_stage_timings(self.handle, ptr(out)), "l0s_stage_timings")
        return dict(zip(("gather", "normalize", "gram", "flags"), out.tolist()))

    def sis_prepare(self, targets: np.ndarray, perm: np.ndarray, bounds: np.ndarray) -> None:
        targets = np.ascontiguousarray(np.atleast_2d(targets), dtype=np.float64)
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        check(lib().l0s_sis_prepare(self.handle, ptr(targets), targets.shape[0], targets.shape[1], ptr(perm),
                                    ptr(bounds), bounds.shape[0] - 1), "l0s_sis_prepare")

    def sis_scores(self, F, device_ptr: int | None = None, k: int | None = None) -> np.ndarray:
        """Scores of the rows of F (host array), or of k device rows at device_ptr."""
        if device_ptr is None:
            F = np.ascontiguousarray(F, dtype=np.float64)
            k = F.shape[0]
            src, is_dev = ptr(F), 0
        else:
            src, is_dev = ctypes.c_void_p(device_ptr), 1
        out = np.empty(int(k), dtype=np.float64)
        check(lib().l0s_sis_scores(self.handle, src, int(k), is_dev, ptr(out)), "l0s_sis_scores")
        return out

    # ---- final-rung candidates (csrc/gen.cu) ----
    def gen_pool(self, values: np.ndarray) -> None:
        """The pool's rows ((n_pool, s), float32 or float64: the pool's dtype) to the device."""
        fp32 = values.dtype == np.float32
        values = np.ascontiguousarray(values, dtype=np.float32 if fp32 else np.float64)
        check(lib().l0s_gen_pool(self.handle, ptr(values), values.shape[0], values.shape[1], int(fp32)), "l0s_gen_pool")
        self.gen_dtype = values.dtype
        self.gen_s = values.shape[1]

    def gen_eval(self, kind: int, pi=None, pj=None, values=None, *, tol: float, min_abs: float, max_abs: float,
                 dedup_tol: float):
        """Evaluate one chunk of candidates; returns (valid bool (k,), fingerprints bytes (16 k))."""
        if values is not None:
            values = np.ascontiguousarray(values, dtype=self.gen_dtype)
            k = values.shape[0]
            a = b = None
        else:
            a = np.ascontiguousarray(pi, dtype=np.int32)
            b = None if pj is None else np.ascontiguousarray(pj, dtype=np.int32)
            k = a.shape[0]
        valid = np.empty(k, dtype=np.uint8)
        h = np.empty(2 * k, dtype=np.uint64)
        check(lib().l0s_gen_eval(self.handle, int(kind), None if a is None else ptr(a), None if b is None else ptr(b), k,
                                 None if values is None else ptr(values), float(tol), float(min_abs), float(max_abs),
                                 float(dedup_tol), ptr(valid), ptr(h)), "l0s_gen_eval")
        self._gen_last_count = k
        return valid.view(bool), h.tobytes()

    def gen_take(self, rows, host: bool = False):
        """Compact rows of the last evaluation on the device; returns (host rows or None, device pointer)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        out = np.empty((rows.shape[0], self.gen_s), dtype=self.gen_dtype) if host else None
        dev = ctypes.c_void_p()
        check(lib().l0s_gen_take(self.handle, ptr(rows), rows.shape[0], None if out is None else ptr(out),
                                 ctypes.byref(dev)), "l0s_gen_take")
        return out, dev.value

    def gen_dedup_reset(self, fingerprints) -> None:
        """Seed the device fingerprint set (iterable of 16-byte fingerprints, or a (k, 2) uint64 array)."""
        if isinstance(fingerprints, np.ndarray):
            seed = np.ascontiguousarray(fingerprints, dtype=np.uint64).reshape(-1, 2)
        else:
            seed = np.frombuffer(b"".join(bytes(f) for f in fingerprints), dtype="<u8").reshape(-1, 2)
            seed = np.ascontiguousarray(seed)
        check(lib().l0s_gen_dedup_reset(self.handle, ptr(seed) if len(seed) else None, len(seed)), "l0s_gen_dedup_reset")

    def gen_dedup(self) -> np.ndarray:
        """Kept flags of the last gen_eval's candidates (valid, fingerprint not seen earlier in the stream)."""
        n = self._gen_last_count
        kept = np.zeros(n, dtype=np.uint8)
        cnt = ctypes.c_int64(0)
        check(lib().l0s_gen_dedup(self.handle, ptr(kept), ctypes.byref(cnt)), "l0s_gen_dedup")
        return kept.astype(bool)

    def gen_fetch(self, rows) -> np.ndarray:
        """Rows of the taken block to the host (pool dtype)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        out = np.empty((rows.shape[0], self.gen_s), dtype=self.gen_dtype)
        check(lib().l0s_gen_fetch(self.handle, ptr(rows), rows.shape[0], ptr(out)), "l0s_gen_fetch")
        return out

    def search(self, n: int, keep: int, rank_begin: int = 0, rank_end: int = 2**63 - 1, mode: str = "auto"):
        keep = int(keep)
        scores = np.zeros(keep, dtype=np.float64)
        ranks = np.zeros(keep, dtype=np.int64)
        coef = np.zeros((keep, self.T, n + 1), dtype=np.float64)
        ssr = np.zeros((keep, self.T), dtype=np.float64)
        cnt = ctypes.c_int64(0)
        st = Stats()
        check(lib().l0s_search(self.handle, n, keep, int(rank_begin), int(rank_end), MODES[mode], ptr(scores),
                               ptr(ranks), ptr(coef), ptr(ssr), ctypes.byref(cnt), ctypes.byref(st)), "l0s_search")
        k = cnt.value
        return scores[:k], ranks[:k], coef[:k], ssr[:k], st

    def search_part(self, n: int, keep: int, part: int, nparts: int, mode: str = "auto"):
        """Part `part` of `nparts` disjoint parts of the whole search (l0s_search_part)."""
        keep = int(keep)
        scores = np.zeros(keep, dtype=np.float64)
        ranks = np.zeros(keep, dtype=np.int64)
        coef = np.zeros((keep, self.T, n + 1), dtype=np.float64)
        ssr = np.zeros((keep, self.T), dtype=np.float64)
        cnt = ctypes.c_int64(0)
        st = Stats()
        check(lib().l0s_search_part(self.handle, n, keep, int(part), int(nparts), MODES[mode], ptr(scores), ptr(ranks),
                                    ptr(coef), ptr(ssr), ctypes.byref(cnt), ctypes.byref(st)), "l0s_search_part")
        k = cnt.value
        return scores[:k], ranks[:k], coef[:k], ssr[:k], st

    def set_part_exchange(self, fn) -> None:
        """fn(scores: np.ndarray) -> float: the collective of l0s_set_part_exchange (the keep-th
        score of the union of every part's best exact scores); None clears it."""
        if fn is None:
            check(lib().l0s_set_part_exchange(self.handle, None, None), "l0s_set_part_exchange")
            self._exchange = None
            return

        def cb(scores, count, _user):
            try:
                arr = np.ctypeslib.as_array(scores, shape=(count,)).copy() if count > 0 else np.zeros(0)
                return float(fn(arr))
            except Exception:  # noqa: BLE001 -- never unwind through the C caller
                return float("inf")

        self._exchange = EXCHANGE_FN(cb)  # kept alive while registered
        check(lib().l0s_set_part_exchange(self.handle, ctypes.cast(self._exchange, ctypes.c_void_p), None),
              "l0s_set_part_exchange")

    def fit_tuples(self, tuples: np.ndarray):
        tuples = np.ascontiguousarray(tuples, dtype=np.int64)
        count, n = tuples.shape
        ok = np.zeros(count, dtype=np.int32)
        score = np.zeros(count, dtype=np.float64)
        coef = np.zeros((count, self.T, n + 1), dtype=np.float64)
        ssr = np.zeros((count, self.T), dtype=np.float64)
        check(lib().l0s_fit_tuples(self.handle, n, ptr(tuples), count, ptr(ok), ptr(score), ptr(coef), ptr(ssr)),
              "l0s_fit_tuples")
        return ok.astype(bool), score, coef, ssr

    def screen_tuples(self, tuples: np.ndarray):
        tuples = np.ascontiguousarray(tuples, dtype=np.int64)
        count, n = tuples.shape
        lb = np.zeros(count, dtype=np.float64)
        flags = np.zeros(count, dtype=np.int32)
        check(lib().l0s_screen_tuples(self.handle, n, ptr(tuples), count, ptr(lb), ptr(flags)), "l0s_screen_tuples")
        return lb, flags

    def gram(self, task: int = 0) -> np.ndarray:
        out = np.zeros((self.m + 1, self.m + 1), dtype=np.float64)
        check(lib().l0s_get_gram(self.handle, task, ptr(out)), "l0s_get_gram")
        return out

    def fp64_peak(self) -> float:
        v = ctypes.c_double(0.0)
        check(lib().l0s_fp64_peak(self.handle, ctypes.byref(v)), "l0s_fp64_peak")
        return v.value


class Group:
    """Several devices of this process searching one problem (l0s_group_*: row blocks uploaded per
    device and exchanged device to device, part g of the search on device g, (score, rank) merge)."""

    def __init__(self, devices):
        L = lib()
        self.devices = tuple(int(d) for d in devices)
        arr = np.asarray(self.devices, dtype=np.int32)
        h = ctypes.c_void_p()
        check(L.l0s_group_create(len(arr), ptr(arr), ctypes.byref(h)), "l0s_group_create")
        self.handle = h
        self.T = 0
        self.m = 0

    def close(self):
        if self.handle:
            lib().l0s_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage(self, values, y, perm, bounds, precision: str) -> None:
        """values: an (m, s) array, or a list of m row arrays (a SelectedSubspace's entries)."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        s = y.shape[0]
        if isinstance(values, np.ndarray):
            values = np.ascontiguousarray(values, dtype=np.float64)
            m = values.shape[0]
            rc = lib().l0s_group_stage(self.handle, ptr(values), None, m, s, ptr(y), ptr(perm), ptr(bounds),
                                       len(bounds) - 1, PREC[precision])
        else:
            keep, rows = Engine._row_pointers(values, s)
            m = len(keep)
            rc = lib().l0s_group_stage(self.handle, None, rows, m, s, ptr(y), ptr(perm), ptr(bounds),
                                       len(bounds) - 1, PREC[precision])
        check(rc, "l0s_group_stage")
        self.T = len(bounds) - 1
        self.m = m
        self.s = s

    def residuals(self, tuples: np.ndarray, coef: np.ndarray) -> np.ndarray:
        """l0s_residuals on member 0 (every member staged the whole problem)."""
        h = ctypes.c_void_p()
        check(lib().l0s_group_ctx(self.handle, 0, ctypes.byref(h)), "l0s_group_ctx")
        tuples = np.ascontiguousarray(np.atleast_2d(tuples), dtype=np.int64)
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        out = np.empty((len(tuples), self.s), dtype=np.float64)
        check(lib().l0s_residuals(h, tuples.shape[1], ptr(tuples), ptr(coef), len(tuples), ptr(out)), "l0s_residuals")
        return out

    def search(self, n: int, keep: int, mode: str = "auto"):
        keep = int(keep)
        scores = np.zeros(keep, dtype=np.float64)
        ranks = np.zeros(keep, dtype=np.int64)
        coef = np.zeros((keep, self.T, n + 1), dtype=np.float64)
        ssr = np.zeros((keep, self.T), dtype=np.float64)
        cnt = ctypes.c_int64(0)
        st = Stats()
        check(lib().l0s_group_search(self.handle, n, keep, MODES[mode], ptr(scores), ptr(ranks), ptr(coef), ptr(ssr),
                                     ctypes.byref(cnt), ctypes.byref(st)), "l0s_group_search")
        k = cnt.value
        return scores[:k], ranks[:k], coef[:k], ssr[:k], st


_groups: dict[tuple, Group] = {}


def group(devices) -> Group:
    """Process-wide device group per device tuple."""
    key = tuple(int(d) for d in devices)
    g = _groups.get(key)
    if g is None or g.handle is None:
        g = Group(key)
        _groups[key] = g
    return g


_engines: dict[int, Engine] = {}


def device_count() -> int:
    n = ctypes.c_int(0)
    lib().l0s_device_count(ctypes.byref(n))
    return n.value


def engine(device: int | None = None) -> Engine:
    """Process-wide engine per device (LOCAL_RANK or 0 by default)."""
    if device is None:
        device = int(os.environ.get("L0S_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    eng = _engines.get(device)
    if eng is None or eng.handle is None:
        eng = Engine(device)
        _engines[device] = eng
    return eng
