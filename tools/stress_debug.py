import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import test_gpu_scale as t
from oracle import oracle as orc
from paper_2502_20072_b200 import L0Config, SearchStats, l0_search, _lib
from paper_2502_20072_b200.search import _partition, rank_tuple
k = int(sys.argv[1]) if len(sys.argv) > 1 else 131
c = t._stress_instance(k)
orc.build()
n = c["n"]
want = orc.l0_search(c["v"], c["y"], c["slices"], n, c["keep"], c["precision"], threads=8)
res = {}
for mode in ("exact", "fast"):
    st = SearchStats()
    got = res[mode] = l0_search(c["v"], c["y"], c["slices"], L0Config(dimension=n, n_models_store=c["keep"], precision=c["precision"]), stats=st, mode=mode)
    print(mode, {k2: v for k2, v in st.device.items() if k2.startswith("n_") or k2 in ("certified", "theta", "margin")})
    for i in range(max(len(got), len(want))):
        g = got[i] if i < len(got) else None
        w = want[i] if i < len(want) else None
        print(i, g.indices if g else None, g.score if g else None, w["indices"] if w else None, w["score"] if w else None,
              "" if (g and w and g.indices == w["indices"]) else "<<<")
gi = {md.indices for md in got}
miss = [w for w in want if w["indices"] not in gi]
m, s = c["v"].shape
perm, bounds, _ = _partition(s, c["slices"])
eng = _lib.engine(0)
eng.stage(c["v"], c["y"], perm, bounds, c["precision"])
for w in miss:
    tup = np.array([w["indices"]], dtype=np.int64)
    ok, score, _, _ = eng.fit_tuples(tup)
    lb, fl = eng.screen_tuples(tup)
    qs, qr = eng.qr_tuples(tup)
    print("missing", w["indices"], "rank", rank_tuple(w["indices"], m, n), "ref", w["score"] * s, "dev", score[0] * s, "lb", lb[0], "flags", fl[0], "qr", qs[0], qr[0])
