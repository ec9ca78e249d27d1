"""SIS projection throughput on the BASELINE C5 shape (synthetic features generated on the device).

    python tools/sis_bench.py [--features 10000000] [--samples 2000] [--targets 10] [--tasks 1]

Features are generated chunk by chunk on the GPU (uniform, torch) and scored by
l0s_sis_scores straight from device memory; a running top-k (n_sis_select) is kept on the
device.  Reports features/s and the HBM roofline of the scoring kernel (8 B per sample read
once per feature).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20072_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--features", type=int, default=10_000_000)
    ap.add_argument("--samples", type=int, default=2000)
    ap.add_argument("--targets", type=int, default=10)
    ap.add_argument("--tasks", type=int, default=1)
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--select", type=int, default=2000)
    args = ap.parse_args()
    s, T = args.samples, args.tasks
    rng = np.random.default_rng(5)
    targets = rng.standard_normal((args.targets, s))
    slices = [np.arange(t, s, T) for t in range(T)]
    perm = np.concatenate(slices).astype(np.int64)
    bounds = np.zeros(T + 1, dtype=np.int64)
    np.cumsum([len(x) for x in slices], out=bounds[1:])
    eng = _lib.engine(0)
    eng.sis_prepare(targets[: min(8, args.targets)], perm, bounds)
    gen = torch.Generator(device="cuda").manual_seed(0)
    buf = torch.empty((args.chunk, s), dtype=torch.float64, device="cuda")
    best_v = torch.full((args.select,), -1.0, dtype=torch.float64, device="cuda")
    best_i = torch.zeros(args.select, dtype=torch.int64, device="cuda")
    # warm-up
    buf.uniform_(0.5, 2.0, generator=gen)
    eng.sis_scores(None, device_ptr=buf.data_ptr(), k=args.chunk)
    t_score = 0.0
    done = 0
    t0 = time.perf_counter()
    while done < args.features:
        k = min(args.chunk, args.features - done)
        buf[:k].uniform_(0.5, 2.0, generator=gen)
        torch.cuda.synchronize()
        ts = time.perf_counter()
        sc = eng.sis_scores(None, device_ptr=buf.data_ptr(), k=k)  # synchronous
        t_score += time.perf_counter() - ts
        v = torch.from_numpy(sc).cuda()
        allv = torch.cat([best_v, v])
        alli = torch.cat([best_i, torch.arange(done, done + k, device="cuda")])
        top = torch.topk(allv, args.select)
        best_v, best_i = top.values, alli[top.indices]
        done += k
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    bytes_per_feature = 8 * s
    gbs = args.features * bytes_per_feature / t_score / 1e9
    print(json.dumps({"features": args.features, "samples": s, "tasks": T, "targets": min(8, args.targets),
                      "score_s": t_score, "features_per_s": args.features / t_score, "wall_s": wall,
                      "hbm_gbs": gbs, "note": "score_s includes the 8 B/feature D2H of the scores per chunk",
                      "top": [int(x) for x in best_i[:5].tolist()]}))


if __name__ == "__main__":
    main()
