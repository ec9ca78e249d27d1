"""Multi-GPU l0 search: contiguous rank ranges, one per rank, merged by (score, rank).

The reference's worker pool hands out contiguous rank ranges (search.py:258-301)
and merges per-worker top lists by the total order (score, rank) (search.py:303).
Across GPUs the same discipline applies: rank g of G searches
[floor(g N / G), floor((g+1) N / G)) and certifies its own top-k exactly
(every score is the bit-exact kernel's), so the global answer is the
(score, rank) merge of the per-rank lists -- a single all-gather of
keep x (score, rank) per search, no data-path collective.

``sharded_l0_search`` runs on top of ``torch.distributed`` (NCCL on the GPU
box; gloo in the CPU tests, where ``local_search`` is injected).
"""

from __future__ import annotations

from math import comb

import numpy as np


def rank_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of [0, total) for `rank` of `world` (sizes differ by at most one)."""
    return total * rank // world, total * (rank + 1) // world


def merge_candidates(parts, keep: int):
    """(score, rank, payload) lists from every rank -> best `keep` by (score, rank)."""
    allc = [c for part in parts for c in part if np.isfinite(c[0])]
    allc.sort(key=lambda c: (c[0], c[1]))
    out, seen = [], set()
    for c in allc:
        if c[1] in seen:
            continue
        seen.add(c[1])
        out.append(c)
        if len(out) == keep:
            break
    return out


OZAKI_MIN_M = 256  # api.cu: the AUTO Gram is the INT8 one from this many features up (fp64)


def sharded_stage(eng, shape, bounds, precision, device_ptrs, group=None, all_gather=None, force_shard=False):
    """Collective stage: every rank stages the whole problem, computes 1/world of the Gram
    (l0s_stage_shard) and the shards are all-gathered over NCCL straight into the buffer
    l0s_stage_finish scatters from.  world == 1 is a plain stage, and so is every problem whose
    Gram runs on the INT8 tensor cores (cheaper than a shard plus the exchange) unless
    ``force_shard``.

    ``all_gather(out, inp)`` defaults to ``torch.distributed.all_gather_into_tensor``.
    """
    import torch
    import torch.distributed as dist

    from ._lib import Engine

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    me = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1 or (precision == "fp64" and int(shape[0]) >= OZAKI_MIN_M and not force_shard):
        # the INT8 tensor-core Gram (Ozaki digits) costs one GPU less than a 1/world DMMA shard
        # plus the exchange for world <= 8 (C3: 0.25 ms vs 1.78/world + ~0.12 ms): stage locally
        eng.stage(shape, None, None, bounds, precision, device_ptrs=device_ptrs)
        return
    m, ntasks = int(shape[0]), len(bounds) - 1
    per = Engine.gram_shard_size(m, ntasks, world)
    key = (per, world)
    if getattr(eng, "_xbuf_key", None) != key:
        dev = torch.device("cuda", eng.device)
        eng._xbuf = (torch.empty(per, dtype=torch.float64, device=dev),
                     torch.empty(world * per, dtype=torch.float64, device=dev))
        eng._xbuf_key = key
    send, recv = eng._xbuf
    eng.stage_shard(shape, bounds, precision, device_ptrs, me, world, send.data_ptr())
    if all_gather is None:
        if dist.get_backend(group) == "gloo":  # CPU transport (tests / ranks sharing one GPU)
            def all_gather(o, i):
                oc = o.new_empty(o.shape, device="cpu")
                dist.all_gather_into_tensor(oc, i.cpu(), group=group)
                o.copy_(oc)
        else:
            def all_gather(o, i):
                dist.all_gather_into_tensor(o, i, group=group)
    torch.cuda.synchronize(send.device)  # shard written on the engine's stream
    all_gather(recv, send)
    torch.cuda.current_stream(send.device).synchronize()  # the engine runs on its own stream
    eng.stage_finish(recv.data_ptr())


def exchange_keepth(scores, keep: int, group=None) -> float:
    """The parts' exchange (l0s_set_part_exchange): all-gather every rank's best exact scores
    (at most keep, ascending) and return the keep-th of their union (+inf when fewer)."""
    import torch
    import torch.distributed as dist

    buf = torch.full((keep,), float("inf"), dtype=torch.float64)
    k = min(len(scores), keep)
    if k:
        buf[:k] = torch.from_numpy(np.asarray(scores[:k], dtype=np.float64))
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    out = [torch.empty_like(buf) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, buf, group=group)
    allv = torch.cat(out).cpu().numpy()
    allv.sort()
    return float(allv[keep - 1]) if len(allv) >= keep else float("inf")


def sharded_l0_search(values, property_values, task_slices=None, config=None, task_labels=None,
                      group=None, local_search=None, device=None):
    """Collective l0_search: every rank must call it with the same inputs; every rank
    receives the same merged list of ``Model`` records.

    Default path (one process per GPU): the inputs go to this rank's device, the stage is
    collective (``sharded_stage``), the rank searches its part (``l0s_search_part``: every
    world-th unit of the screened path, else its contiguous rank range) and certifies its own
    top list exactly, and the lists are merged by (score, rank).  ``local_search(values, y, task_slices, config, task_labels,
    rank_range) -> list of models`` replaces the device part (the CPU tests inject the oracle).
    """
    import torch.distributed as dist

    from . import _lib
    from .search import _as_matrix, _labels_for, _model, _partition, count_models, l0_search, rank_tuple, unrank_tuple

    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    vals, expressions = _as_matrix(values)
    m = vals.shape[0]
    n = config.dimension
    total = count_models(m, n)
    lo, hi = rank_range(total, me, world)
    keep = max(1, config.n_models_store)
    if local_search is not None:
        models = local_search(values, property_values, task_slices, config, task_labels, (lo, hi)) if hi > lo else []
    elif m < n:
        models = l0_search(values, property_values, task_slices, config, task_labels=task_labels)  # raises
    else:
        import torch

        s = vals.shape[1]
        perm, bounds, slices = _partition(s, task_slices)
        dev = torch.cuda.current_device() if device is None else int(device)
        eng = _lib.engine(dev)
        vd = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(dev)
        yd = torch.from_numpy(np.ascontiguousarray(property_values, dtype=np.float64)).to(dev)
        pd = torch.from_numpy(perm).to(dev)
        torch.cuda.synchronize(dev)
        sharded_stage(eng, (m, s), bounds, config.precision, (vd.data_ptr(), yd.data_ptr(), pd.data_ptr()), group)
        # this rank's part of the search: every world-th unit of the screened path (ill-
        # conditioned tuples cluster in rank ranges, C4), else the contiguous rank range; the
        # parts certify against the keep-th of the union of their best scores (one all-gather)
        if world > 1:
            eng.set_part_exchange(lambda scores: exchange_keepth(scores, keep, group))
        try:
            sc, rk, coef, ssr, _ = eng.search_part(n, keep, me, world, "auto")
        finally:
            if world > 1:
                eng.set_part_exchange(None)
        labels = _labels_for(slices, task_labels)
        # merge key: the device score (score_tuples' sequential task sum, search.py:303), not
        # Model.score (numpy's ssr.sum(), which may differ in the last bit for 8 tasks)
        mine = [(float(sc[i]), int(rk[i]),
                 _model(unrank_tuple(int(rk[i]), m, n), expressions, coef[i], ssr[i], bounds, s, labels))
                for i in range(len(sc))]
        models = None
    if models is not None:
        mine = [(float(md.score), rank_tuple(md.indices, m, n), md) for md in models]
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return [c[2] for c in merge_candidates(parts, keep)]


__all__ = ["rank_range", "merge_candidates", "sharded_stage", "sharded_l0_search", "exchange_keepth", "comb"]
