"""Device time of stage + Gram on the C3 bench problem (inputs resident): python tools/time_stage.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_20072_b200 import _lib  # noqa: E402
from paper_2502_20072_b200.search import _partition  # noqa: E402

v, y, slices = bench.make_c3()
perm, bounds, _ = _partition(bench.S, slices)
eng = _lib.engine(0)
eng.set_gram_mode(os.environ.get("L0S_GRAM_MODE", "auto"))
vd, yd, pd = (torch.from_numpy(x).cuda() for x in (v, y, perm))
ms = []
for _ in range(8):
    eng.stage((bench.M, bench.S), None, None, bounds, "fp64", device_ptrs=(vd.data_ptr(), yd.data_ptr(), pd.data_ptr()))
    sc, rk, coef, ssr, st = eng.search(3, 10, 0, 2**62, "fast")
    ms.append(st.ms_gram)
print(json.dumps({"gram_mode": os.environ.get("L0S_GRAM_MODE", "auto"), "stage_gram_ms": sorted(ms)[len(ms) // 2],
                  "gram_kernel_ms": st.ms_gram_kernel, "eta": eng.stage_info()[0].tolist(),
                  "best": rk[:3].tolist()}))
