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


def sharded_stage(eng, shape, bounds, precision, device_ptrs, group=None, all_gather=None):
    """Collective stage: every rank stages the whole problem, computes 1/world of the Gram
    (l0s_stage_shard) and the shards are all-gathered over NCCL straight into the buffer
    l0s_stage_finish scatters from.  world == 1 is a plain stage.

    ``all_gather(out, inp)`` defaults to ``torch.distributed.all_gather_into_tensor``.
    """
    import torch
    import torch.distributed as dist

    from ._lib import Engine

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    me = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1:
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
    (all_gather or (lambda o, i: dist.all_gather_into_tensor(o, i, group=group)))(recv, send)
    torch.cuda.current_stream(send.device).synchronize()  # the engine runs on its own stream
    eng.stage_finish(recv.data_ptr())


def sharded_l0_search(values, property_values, task_slices=None, config=None, task_labels=None,
                      group=None, local_search=None):
    """Collective l0_search: every rank must call it with the same inputs; every rank
    receives the same merged list of ``Model`` records.

    local_search(values, y, task_slices, config, task_labels, rank_range) -> list of models
    (default: this package's device search).
    """
    import torch.distributed as dist

    from .search import count_models, l0_search, rank_tuple

    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    m = np.asarray(values).shape[0] if not hasattr(values, "values_matrix") else len(values.expressions)
    total = count_models(m, config.dimension)
    lo, hi = rank_range(total, me, world)
    search = local_search or (lambda v, y, sl, cfg, lab, rr: l0_search(v, y, sl, cfg, task_labels=lab,
                                                                          rank_range=rr))
    models = search(values, property_values, task_slices, config, task_labels, (lo, hi)) if hi > lo else []
    mine = [(float(md.score), rank_tuple(md.indices, m, config.dimension), md) for md in models]
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    keep = max(1, config.n_models_store)
    return [c[2] for c in merge_candidates(parts, keep)]


__all__ = ["rank_range", "merge_candidates", "sharded_stage", "sharded_l0_search", "comb"]
