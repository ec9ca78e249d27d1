"""Incremental stage across dimensions: a SelectedSubspace grown by appending
(C3 shape: 1000 + 1000 features x 10k samples, 4 tasks) searched at dim 3, staged in full vs
through l0s_stage_append.  One JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_20072_b200 import L0Config, _lib, l0_search  # noqa: E402


class Entry:
    def __init__(self, key, values):
        self.expression = key
        self.values = values


class Subspace:
    def __init__(self, entries):
        self.entries = list(entries)

    def __len__(self):
        return len(self.entries)

    @property
    def expressions(self):
        return [e.expression for e in self.entries]

    def values_matrix(self):
        return np.stack([e.values for e in self.entries])

    def extended(self, new):
        return Subspace(self.entries + list(new))


def main():
    v, y, slices = bench.make_c3()
    vh = torch.from_numpy(v).pin_memory().numpy()
    entries = [Entry(f"f{i}", vh[i]) for i in range(v.shape[0])]
    half = v.shape[0] // 2
    cfg = L0Config(dimension=3)
    full, incr = [], []
    for _ in range(4):
        sub0 = Subspace(entries[:half])
        sub1 = sub0.extended(entries[half:])
        _lib.engine(0).subspace_cache = None
        l0_search(sub0, y, slices, L0Config(dimension=2))  # the previous dimension's search
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = l0_search(sub1, y, slices, cfg)  # appends 1000 rows
        torch.cuda.synchronize()
        incr.append(time.perf_counter() - t0)
        _lib.engine(0).subspace_cache = None
        t0 = time.perf_counter()
        b = l0_search(sub1, y, slices, cfg)  # full stage (cache cleared)
        torch.cuda.synchronize()
        full.append(time.perf_counter() - t0)
        assert [m.indices for m in a] == [m.indices for m in b]
    print(json.dumps({"shape": "C3: 1000 + 1000 features x 10k samples, 4 tasks, dim 3",
                      "full_stage_ms": 1e3 * min(full[1:]), "incremental_ms": 1e3 * min(incr[1:]),
                      "rows_sent_incremental": v.shape[0] - half, "rows_sent_full": v.shape[0],
                      "best": list(a[0].indices)}))


if __name__ == "__main__":
    main()
