"""Variants of the staging pass (k_stage_rows): python tools/tune_stage.py build | run
Each variant is a full libl0search.so with different defines; `run` times the fused staging
kernel (l0s_stage_timings[0]) on C3 in its own process and checks the searches agree."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2502_20072_b200", "variants")
VARIANTS = {"t256": (), "t128": ("L0S_SR_THREADS=128",), "t64": ("L0S_SR_THREADS=64",)}


def build_all():
    from paper_2502_20072_b200 import build as b

    os.makedirs(VDIR, exist_ok=True)
    for name, defs in VARIANTS.items():
        b.build(force=True, defines=defs, out=os.path.join(VDIR, f"lib_{name}.so"))


def time_one():
    import torch

    import bench
    from paper_2502_20072_b200 import _lib
    from paper_2502_20072_b200.search import _partition

    v, y, slices = bench.make_c3()
    perm, bounds, _ = _partition(bench.S, slices)
    eng = _lib.engine(0)
    vd, yd, pd = (torch.from_numpy(x).cuda() for x in (v, y, perm))
    ms = []
    for _ in range(10):
        eng.stage((bench.M, bench.S), None, None, bounds, "fp64", device_ptrs=(vd.data_ptr(), yd.data_ptr(), pd.data_ptr()))
        ms.append(eng.stage_timings()["gather"])
    sc, rk, *_ = eng.search(3, 10, 0, 2**62, "fast")
    print(json.dumps({"stage_rows_ms": sorted(ms)[len(ms) // 2], "ranks": rk.tolist(), "scores": sc.tolist()}))


def run_all():
    out = {}
    for name in VARIANTS:
        env = dict(os.environ, L0S_LIB=os.path.join(VDIR, f"lib_{name}.so"))
        r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True, timeout=600)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        out[name] = json.loads(line[-1]) if line else {"error": r.stderr[-400:]}
        print(name, out[name].get("stage_rows_ms", out[name].get("error")), flush=True)
    ref = next(o for o in out.values() if "ranks" in o)
    assert all(o.get("ranks") == ref["ranks"] and o.get("scores") == ref["scores"] for o in out.values())
    print("all variants agree")


if __name__ == "__main__":
    {"build": build_all, "run": run_all, "one": time_one}[sys.argv[1] if len(sys.argv) > 1 else "run"]()
