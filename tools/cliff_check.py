"""Timing of the shapes the screened path used to leave to the exact kernel (run under gpurun):
C3 with keep 10 / 200 / 1000, C3 with 4 / 12 tasks, and an n = 5 search.

    python tools/cliff_check.py > gpurun_out/cliff.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import scale_cases  # noqa: E402
from paper_2502_20072_b200 import _lib  # noqa: E402
from paper_2502_20072_b200.search import _partition, count_models  # noqa: E402


def c3_tasks(T, seed=2):
    M, S = 2000, 10000
    rng = np.random.default_rng(seed)
    v = rng.uniform(0.5, 2.0, size=(M, S))
    slices = [np.arange(t, S, T) for t in range(T)]
    y = np.empty(S)
    for t, sl in enumerate(slices):
        y[sl] = (2.0 + 0.1 * t) * v[17, sl] - (1.0 + 0.05 * t) * v[911, sl] + 0.5 * v[1499, sl] + 0.75 \
            + 0.01 * rng.standard_normal(len(sl))
    return v, y, slices


def timed(v, y, slices, n, keep, mode="auto", reps=3):
    eng = _lib.engine(0)
    m, s = v.shape
    perm, bounds, _ = _partition(s, slices)
    vd, yd, pd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (v, y, perm))
    torch.cuda.synchronize()
    out = []
    for _ in range(reps + 1):
        eng.stage((m, s), None, None, bounds, "fp64", device_ptrs=(vd.data_ptr(), yd.data_ptr(), pd.data_ptr()))
        sc, rk, _, _, st = eng.search(n, keep, 0, 2**63 - 1, mode)
        out.append(st)
    st = out[-1]
    ms = min(o.ms_total + o.ms_gram for o in out[1:])
    return {"n": n, "keep": keep, "T": len(slices) if slices else 1, "m": m, "s": s, "tuples": count_models(m, n), "ms": ms,
            "fit_ms": st.ms_fit, "mode_used": int(st.mode_used), "certified": int(st.certified),
            "n_candidates": int(st.n_candidates), "n_rescan": int(st.n_rescan), "best": float(sc[0]) if len(sc) else None}


class _Rows(list):
    def append(self, r):
        print(json.dumps(r), flush=True)
        super().append(r)


def main():
    rows = _Rows()
    v, y, sl = scale_cases.c3("planted")
    for keep in (10, 200, 1000):
        rows.append(dict(case=f"C3 keep={keep}", **timed(v, y, sl, 3, keep)))
    v, y, sl = scale_cases.c3("random")
    for keep in (10, 200):
        rows.append(dict(case=f"C3 random y keep={keep}", **timed(v, y, sl, 3, keep)))
    for T in (4, 12):
        v, y, sl = c3_tasks(T)
        rows.append(dict(case=f"C3 T={T}", **timed(v, y, sl, 3, 10)))
    rng = np.random.default_rng(5)
    v = rng.uniform(0.5, 2.0, size=(60, 1000))
    y = v[1] + v[2] - v[5] + 0.3 * v[9] + 0.1 * v[17] + 0.01 * rng.standard_normal(1000)
    rows.append(dict(case="n=5 m=60 s=1000", **timed(v, y, None, 5, 10, reps=1)))


if __name__ == "__main__":
    main()
