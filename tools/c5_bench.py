"""BASELINE config C5 on the device: SIS projection sweep over 10^7 features x 2k samples,
top-k screening, then the dim-3 l0 search on the selected subspace.

    python tools/c5_bench.py [--features 10000000] [--samples 2000] [--select 2000]
    torchrun --nproc-per-node N tools/c5_bench.py ...   (features sharded by chunk across ranks)

The features are synthetic, generated chunk by chunk on the GPU (uniform(0.5, 2), chunk c from
seed c, so every rank can regenerate any chunk); the property is planted on three features of
chunk 0 (global indices 17, 911, 1499) plus 0.01 N(0,1) noise.  SIS scores come from
l0s_sis_scores (bit-identical to screening._chunk_scores), the running top list is kept on the
device (score desc, index asc), and the selected rows go straight into l0s_stage (device
pointers) for l0s_search (n = 3).  Prints one JSON line (rank 0).
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
from paper_2502_20072_b200.search import unrank_tuple  # noqa: E402

PLANT = (17, 911, 1499)


def chunk(c, rows, s, dev):
    g = torch.Generator(device=dev).manual_seed(1000 + c)
    return torch.empty((rows, s), dtype=torch.float64, device=dev).uniform_(0.5, 2.0, generator=g)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--features", type=int, default=10_000_000)
    ap.add_argument("--samples", type=int, default=2000)
    ap.add_argument("--select", type=int, default=2000)
    ap.add_argument("--chunk", type=int, default=65536)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    s, K, CH = args.samples, args.select, args.chunk
    nchunks = -(-args.features // CH)
    c0 = chunk(0, CH, s, dev)
    gen = torch.Generator(device=dev).manual_seed(7)
    y = (2.0 * c0[PLANT[0]] - c0[PLANT[1]] + 0.5 * c0[PLANT[2]]
         + 0.01 * torch.randn(s, dtype=torch.float64, device=dev, generator=gen)).cpu().numpy()
    del c0
    eng = _lib.engine(local)
    eng.sis_prepare(y[None, :], np.arange(s, dtype=np.int64), np.array([0, s], dtype=np.int64))
    best_s = torch.full((K,), -1.0, dtype=torch.float64, device=dev)
    best_i = torch.full((K,), -1, dtype=torch.int64, device=dev)
    best_v = torch.zeros((K, s), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t_sis = 0.0
    for c in range(rank, nchunks, world):
        rows = min(CH, args.features - c * CH)
        F = chunk(c, CH, s, dev)[:rows]
        torch.cuda.synchronize()
        ts = time.perf_counter()
        sc = torch.from_numpy(eng.sis_scores(None, device_ptr=F.data_ptr(), k=rows)).to(dev)
        t_sis += time.perf_counter() - ts
        idx = torch.arange(c * CH, c * CH + rows, device=dev)
        all_s, all_i = torch.cat([best_s, sc]), torch.cat([best_i, idx])
        # (score desc, index asc): sort by index first, then a stable sort by score
        o = torch.argsort(all_i, stable=True)
        o = o[torch.argsort(-all_s[o], stable=True)][:K]
        src = torch.cat([best_v, F])
        best_s, best_i, best_v = all_s[o], all_i[o], src[o]
    torch.cuda.synchronize()
    t_sweep = time.perf_counter() - t0
    if world > 1:  # merge the per-rank top lists (NCCL all-gather of scores, indices, rows)
        gs = [torch.empty_like(best_s) for _ in range(world)]
        gi = [torch.empty_like(best_i) for _ in range(world)]
        gv = [torch.empty_like(best_v) for _ in range(world)]
        dist.all_gather(gs, best_s)
        dist.all_gather(gi, best_i)
        dist.all_gather(gv, best_v)
        all_s, all_i, all_v = torch.cat(gs), torch.cat(gi), torch.cat(gv)
        o = torch.argsort(all_i, stable=True)
        o = o[torch.argsort(-all_s[o], stable=True)][:K]
        best_s, best_i, best_v = all_s[o], all_i[o], all_v[o]
    # the l0 search on the selected subspace (rows in selection order, like SelectedSubspace)
    t1 = time.perf_counter()
    best_v = best_v.contiguous()
    yd = torch.from_numpy(y).to(dev)
    pd = torch.arange(s, dtype=torch.int64, device=dev)
    eng.stage((K, s), None, None, np.array([0, s], dtype=np.int64), "fp64",
              device_ptrs=(best_v.data_ptr(), yd.data_ptr(), pd.data_ptr()))
    sc, rk, coef, ssr, st = eng.search(3, 10, 0, 2**62, "auto")
    torch.cuda.synchronize()
    t_l0 = time.perf_counter() - t1
    sel = best_i.cpu().numpy()
    top = [int(sel[i]) for i in unrank_tuple(int(rk[0]), K, 3)] if len(rk) else None
    if rank == 0:
        print(json.dumps({
            "config": "C5: SIS sweep + top-k + l0 dim 3", "features": args.features, "samples": s, "select": K,
            "gpus": world, "sis_sweep_s": t_sweep, "sis_kernel_s_rank0": t_sis,
            "sis_features_per_s": args.features / t_sweep, "l0_s": t_l0, "total_s": t_sweep + t_l0,
            "l0_tuples": K * (K - 1) * (K - 2) // 6, "best_tuple_global_indices": sorted(top) if top else None,
            "planted": list(PLANT), "best_mse": float(sc[0]) if len(sc) else None,
            "data": "synthetic features generated on the device (uniform(0.5,2), seeded per chunk)"}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
