"""C4 timing variants: python tools/c4_var.py [planted|random|mt4] [iters]
planted: BASELINE C4 (tools/run_configs.make_c4); random: the same features, y ~ N(0,1);
mt4: the same features and y on 4 round-robin tasks."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20072_b200 import L0Config, SearchStats, l0_search  # noqa: E402
from tools.run_configs import make_c4  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "planted"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
v, y, slices, n = make_c4()
if which == "random":
    y = np.random.default_rng(9).standard_normal(v.shape[1])
elif which == "mt4":
    slices = [np.arange(t, v.shape[1], 4) for t in range(4)]
for it in range(iters):
    st = SearchStats()
    models = l0_search(v, y, slices, L0Config(dimension=n), stats=st)
    d = st.device
    print(which, it, "total", round(d["ms_total"], 1), "fit", round(d["ms_fit"], 1), "exact", round(d["ms_exact"], 1),
          "qr", round(d["ms_qr"], 1), "cand", d["n_candidates"], "ill", d["n_ill"], "ill_refit", d["n_ill_refit"],
          "rescan", d.get("n_rescan"), "best", models[0].indices, flush=True)
