"""Per-part device time of the multi-GPU split, emulated on one GPU (the max over parts is
what N GPUs would wait for): l0s_search_part (every N-th unit) vs contiguous rank ranges.

    python tools/parts_balance.py [c3|c4] [N]
"""
import json
import os
import sys
from math import comb

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_20072_b200 import _lib  # noqa: E402
from paper_2502_20072_b200.search import _partition  # noqa: E402
from tools.run_configs import make_c4  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c3"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    if which == "c3":
        v, y, slices = bench.make_c3()
        n = 3
    else:
        v, y, slices, n = make_c4()
    s = v.shape[1]
    perm, bounds, _ = _partition(s, slices)
    eng = _lib.engine(0)
    eng.stage(v, y, perm, bounds, "fp64")
    total = comb(v.shape[0], n)
    eng.search(n, 10, 0, 2**63 - 1, "fast")  # warm-up
    out = {"config": which, "parts": N}
    # the parts' exchange (l0s_set_part_exchange) emulated in two passes: the scores every part
    # brings, then each part again receiving the keep-th of their union (what the collective
    # returns when the parts run concurrently on N GPUs)
    brought = []
    eng.set_part_exchange(lambda x: (brought.append(np.array(x)), float("inf"))[1])
    for p in range(N):
        eng.search_part(n, 10, p, N, "fast")
    union = np.sort(np.concatenate(brought)) if brought else np.zeros(0)
    g = float(union[9]) if len(union) >= 10 else float("inf")
    eng.set_part_exchange(None)

    def with_exchange(p):
        eng.set_part_exchange(lambda x: g)
        try:
            return eng.search_part(n, 10, p, N, "fast")
        finally:
            eng.set_part_exchange(None)

    for label, run in (("units_exchange", with_exchange), ("units", lambda p: eng.search_part(n, 10, p, N, "fast")),
                       ("ranges", lambda p: eng.search(n, 10, total * p // N, total * (p + 1) // N, "fast"))):
        ms, ill, fit, ex, cand, resc = [], [], [], [], [], []
        for p in range(N):
            run(p)  # warm-up: per-part tables and buffers
            st = run(p)[4].as_dict()
            ms.append(st["ms_total"])
            ill.append(st["n_ill"])
            fit.append(round(st["ms_fit"], 3))
            ex.append(round(st["ms_exact"], 3))
            cand.append(st["n_candidates"])
            resc.append(st["n_rescan"])
        out[label] = {"max_ms": max(ms), "mean_ms": float(np.mean(ms)), "ill_per_part": ill, "fit_ms": fit,
                      "exact_ms": ex, "candidates": cand, "rescans": resc}
    st = eng.search(n, 10, 0, 2**63 - 1, "fast")[4].as_dict()
    out["whole_ms"] = st["ms_total"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
