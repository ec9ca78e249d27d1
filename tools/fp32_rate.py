"""C3 with precision="fp32" (the reference's float32 mode): public l0_search timing and stats."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_20072_b200 import L0Config, SearchStats, l0_search  # noqa: E402

v, y, sl = bench.make_c3()
for prec in ("fp32", "fp64"):
    cfg = L0Config(dimension=3, precision=prec)
    l0_search(v, y, sl, cfg)
    st = SearchStats()
    t0 = time.perf_counter()
    m = l0_search(v, y, sl, cfg, stats=st)
    dt = time.perf_counter() - t0
    d = st.device
    print(json.dumps({"precision": prec, "wall_ms": 1e3 * dt, "device_search_ms": d["ms_total"], "gram_ms": d["ms_gram"],
                      "fit_ms": d["ms_fit"], "exact_ms": d["ms_exact"], "n_ill": d["n_ill"], "n_ill_refit": d["n_ill_refit"],
                      "candidates": d["n_candidates"], "rescans": d["n_rescan"], "best": list(m[0].indices)}))
