"""Tuning sweep for the dim-3 fit kernel's (P, IB, CTAs/SM, unroll) choice.

    python tools/tune_fit.py build            # here: compile the variants
    python tools/tune_fit.py run [--m 2000]   # GPU box: time each variant on C3

Each variant is a full libl0search.so built with a different L0S_CFG34 /
L0S_CFG12 define; `run` loads each in its own process (L0S_LIB=...) and
times the screened fit on the bench workload, checking that every variant
returns the same models.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2502_20072_b200", "variants")

VARIANTS = {
    "base": (),
    "ich256": ("L0S_ICH4=256",),
    "ich512": ("L0S_ICH4=512",),
    "ich1024": ("L0S_ICH4=1024",),
}
if os.environ.get("L0S_TUNE_ONLY"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["L0S_TUNE_ONLY"].split(",")}


def build_all():
    from paper_2502_20072_b200 import build as b

    os.makedirs(VDIR, exist_ok=True)
    for name, defs in VARIANTS.items():
        out = os.path.join(VDIR, f"lib_{name}.so")
        b.build(force=True, defines=defs, out=out)
        print(name, out)


def time_one(steps: int = 5):
    import numpy as np

    import bench
    from paper_2502_20072_b200 import _lib
    from paper_2502_20072_b200.search import _partition

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import scale_cases

    v, y, slices = scale_cases.c3(os.environ.get("L0S_TUNE_Y", "planted"))
    tasks = int(os.environ.get("L0S_TUNE_T", "4"))
    if tasks != 4:  # the same features, y re-planted on `tasks` round-robin tasks
        slices = [np.arange(t, bench.S, tasks) for t in range(tasks)]
    perm, bounds, _ = _partition(bench.S, slices)
    eng = _lib.engine(0)
    eng.stage(v, y, perm, bounds, "fp64")
    res = []
    for _ in range(steps + 2):
        sc, rk, coef, ssr, st = eng.search(3, 10, 0, 2**62, "fast")
        res.append((st.ms_fit, st.ms_total, st.n_candidates, st.n_eval, st.n_rescan))
    fit = sorted(r[0] for r in res[2:])
    print(json.dumps({"fit_ms_min": fit[0], "fit_ms_med": fit[len(fit) // 2], "total_ms": res[-1][1],
                      "n_eval": res[-1][3], "n_cand": res[-1][2], "n_rescan": res[-1][4],
                      "ranks": rk.tolist(), "scores": [float(x) for x in sc]}))


def run_all():
    out = {}
    rounds = int(os.environ.get("L0S_TUNE_ROUNDS", "1"))
    for name in [v for _ in range(rounds) for v in VARIANTS]:  # interleaved rounds: min over rounds
        path = os.path.join(VDIR, f"lib_{name}.so")
        env = dict(os.environ, L0S_LIB=path)
        r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True, timeout=600)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        o = json.loads(line[-1]) if line else {"error": r.stderr[-400:]}
        if name in out and "fit_ms_min" in out[name] and "fit_ms_min" in o:
            o["fit_ms_min"] = min(o["fit_ms_min"], out[name]["fit_ms_min"])
        out[name] = o
        print(name, {k: v for k, v in o.items() if k not in ("ranks", "scores")}, flush=True)
    ref = next((o for o in out.values() if "ranks" in o), None)
    for name, o in out.items():
        if "ranks" in o:
            assert o["ranks"] == ref["ranks"] and o["scores"] == ref["scores"], name
    print("all variants agree")


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    {"build": build_all, "run": run_all, "one": time_one}[cmd]()
