"""The multi-GPU path on CPU: candidate sharding (bench.py / nb_evaluate's
LPT) and the rank protocol -- every rank computes the same assignment
independently, the shards are disjoint and complete, and the step time is
the max over ranks -- with torch.distributed gloo, world_size 2."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_06599_b200.workloads import (fixture_path, load_candidates, resnet34_chain,
                                             shard_lpt)


def _costs(k):
    import paper_2102_06599_b200 as nb
    origin = resnet34_chain()
    pool = load_candidates(fixture_path("r34_candidates.json"), origin)[:k]
    return [nb.fisher_flops(n, 128) for n in pool]


def test_shard_lpt_balanced_and_complete():
    costs = _costs(64)
    for world in (1, 2, 4, 8):
        a = shard_lpt(costs, world, 64 // world)
        assert sorted(np.bincount(a, minlength=world)) == [64 // world] * world
        loads = np.bincount(a, weights=costs, minlength=world)
        # LPT bound (4/3 - 1/3m) * OPT <= that, with OPT >= mean load
        assert loads.max() <= (4 / 3) * loads.mean() + max(costs)
    assert shard_lpt(costs, 4, 16) == shard_lpt(list(costs), 4, 16)  # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, costs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    a = shard_lpt(costs, world, len(costs) // world)
    mine = [i for i, r in enumerate(a) if r == rank]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    t = torch.tensor([10.0 + rank])  # this rank's device-timed step ms
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((gathered, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_protocol_gloo():
    costs = _costs(16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, costs, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = gathered
    assert not set(a) & set(b) and sorted(a + b) == list(range(16))
    assert len(a) == len(b) == 8
    assert tmax == 11.0
