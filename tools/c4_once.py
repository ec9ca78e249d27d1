"""One C4 search (for profiling): python tools/c4_once.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20072_b200 import L0Config, SearchStats, l0_search  # noqa: E402
from tools.run_configs import make_c4  # noqa: E402

v, y, slices, n = make_c4()
st = SearchStats()
l0_search(v, y, slices, L0Config(dimension=n), stats=st)
t0 = time.perf_counter()
st = SearchStats()
l0_search(v, y, slices, L0Config(dimension=n), stats=st)
print(time.perf_counter() - t0, st.device)
