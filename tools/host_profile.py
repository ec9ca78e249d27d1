"""cProfile of the public l0_search on C3 (pinned host inputs): where host time goes."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_20072_b200 import L0Config, l0_search  # noqa: E402

v, y, slices = bench.make_c3()
vh = torch.from_numpy(v).pin_memory().numpy()
yh = torch.from_numpy(y).pin_memory().numpy()
cfg = L0Config(dimension=3)
for _ in range(3):
    l0_search(vh, yh, slices, cfg)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    l0_search(vh, yh, slices, cfg)
    ts.append(1e3 * (time.perf_counter() - t0))
print("l0_search ms:", [round(t, 3) for t in ts])
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    l0_search(vh, yh, slices, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
