import sys, time, json
sys.path.insert(0, '/root/repo')
from tools.run_configs import make_c2
from paper_2502_20072_b200 import L0Config, SearchStats, l0_search
v, y, sl, n = make_c2()
for mode in ("exact", "fast"):
    l0_search(v, y, sl, L0Config(dimension=n), mode=mode)
    st = SearchStats(); t0 = time.perf_counter()
    m = l0_search(v, y, sl, L0Config(dimension=n), mode=mode, stats=st)
    dt = time.perf_counter() - t0
    print(json.dumps({"config": "c2", "mode": mode, "wall_s": dt, "tuples": 35820200, "tuples_per_s": 35820200 / dt,
                      "device_ms": st.device["ms_total"], "best": list(m[0].indices)}))
