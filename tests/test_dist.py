"""Multi-rank path on CPU: world size 2 over gloo.

The device search is replaced by the CPU oracle restricted to each rank's
contiguous rank range (the only thing a rank does differently on the GPU
box); the test checks that the sharded, all-gathered, (score, rank)-merged
result equals the oracle's single-process search bit for bit.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _M:  # minimal Model stand-in produced by the oracle-backed local search
    def __init__(self, d):
        self.indices = d["indices"]
        self.score = d["score"]
        self.coefficients = d["coefficients"]


def _worker(rank, world, port, out_q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2502_20072_b200.dist import sharded_l0_search
    from paper_2502_20072_b200.search import L0Config

    rng = np.random.default_rng(3)
    v = rng.uniform(0.5, 2.0, size=(14, 40))
    y = rng.standard_normal(40)
    slices = [np.arange(0, 40, 2), np.arange(1, 40, 2)]
    cfg = L0Config(dimension=3, n_models_store=7)

    def local(values, yy, sl, c, labels, rr):
        res = orc.l0_search(values, yy, sl, c.dimension, c.n_models_store, c.precision, rank_range=rr)
        return [_M(d) for d in res]

    got = sharded_l0_search(v, y, slices, cfg, group=None, local_search=local)
    if rank == 0:
        out_q.put([(md.indices, md.score) for md in got])
    dist.barrier()
    dist.destroy_process_group()


def test_rank_range_partition():
    from paper_2502_20072_b200.dist import rank_range

    for total in (0, 1, 7, 1331334000):
        for world in (1, 2, 3, 8):
            parts = [rank_range(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_merge_is_total_order():
    from paper_2502_20072_b200.dist import merge_candidates

    parts = [[(0.5, 7, "a"), (0.2, 9, "b")], [(0.2, 3, "c"), (float("nan"), 1, "x"), (0.9, 2, "d")]]
    assert [c[2] for c in merge_candidates(parts, 3)] == ["c", "b", "a"]


@pytest.mark.timeout(300)
def test_two_ranks_gloo_equals_single_process():
    from oracle import oracle as orc

    orc.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    v = rng.uniform(0.5, 2.0, size=(14, 40))
    y = rng.standard_normal(40)
    want = orc.l0_search(v, y, [np.arange(0, 40, 2), np.arange(1, 40, 2)], 3, 7, "fp64")
    assert [g[0] for g in got] == [w["indices"] for w in want]
    assert [np.float64(g[1]).view(np.int64) for g in got] == [np.float64(w["score"]).view(np.int64) for w in want]


def _exchange_worker(rank, world, port, out_q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_20072_b200.dist import exchange_keepth

    mine = [np.array([0.5, 1.0, 3.0]), np.array([0.7, 0.9])][rank]
    out_q.put((rank, exchange_keepth(mine, 3), exchange_keepth(mine, 6)))
    dist.barrier()
    dist.destroy_process_group()


def test_part_exchange_keepth_gloo():
    """The search parts' exchange (l0s_set_part_exchange's collective over torch.distributed):
    every rank receives the keep-th score of the union of the ranks' lists, +inf when fewer."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got == [(0, 0.9, float("inf")), (1, 0.9, float("inf"))]
