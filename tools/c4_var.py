import os, sys
sys.path.insert(0, "/root/repo")
from tools.run_configs import make_c4
from paper_2502_20072_b200 import L0Config, SearchStats, l0_search
v, y, slices, n = make_c4()
for it in range(6):
    st = SearchStats()
    l0_search(v, y, slices, L0Config(dimension=n), stats=st)
    d = st.device
    print(it, round(d["ms_fit"], 1), round(d["ms_exact"], 1), d["n_candidates"], d["n_ill"], round(d["theta"], 6) if "theta" in d else None, d.get("n_rescan"))
