"""Multi-rank host logic on CPU (-m "not gpu"): world_size 2 and 3 over gloo.

Each rank takes its block-cyclic shard of the candidate space (the same rule
optimus_eval_candidates applies: blocks of `block` indices, block b to rank
b mod world), finds its (lat, index) minimum — here from the CPU oracle's lat
(test infrastructure; on a GPU box the kernel produces it) — and the
product's driver code gathers the 16-byte pairs (dist.gather_best, one
all_gather) and decodes the winner on every rank (optimus_best_plan through a
host-only context).  Every rank must agree with the single-rank answer.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, block, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__  # noqa: F401
        from oracle import oracle as O
        from paper_2408_03505_b200 import optimus_plan_only
        from paper_2408_03505_b200.dist import gather_best, rank_share
        from workload import config_problem, toy_problem
        prob = toy_problem() if cfg == 0 else config_problem(cfg)
        ctx = optimus_plan_only(prob)
        total, _ = ctx.num_candidates()
        mine = np.array([g for g in range(total) if (g // block) % world == rank], dtype=np.uint64)
        assert len(mine) == rank_share(0, total, rank, world, block)
        best2 = torch.tensor([2**63 - 1, -1], dtype=torch.int64)
        if len(mine):
            lat = O.Oracle(prob).eval(mine, threads=2)
            j = min(range(len(mine)), key=lambda i: (lat[i], mine[i]))
            best2 = torch.tensor([int(lat[j]), int(mine[j])], dtype=torch.int64)
        gathered = gather_best(best2)
        res = ctx.best_plan(gathered.numpy())
        q.put((rank, res["lat_ns"], res["index"], res["enc"], res["counts"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,block", [(2, 0, 64), (3, 0, 64), (2, 2, 4096), (3, 2, 640)])
def test_gloo_gather_and_decode(oracle_mod, world, cfg, block):
    from workload import config_problem, toy_problem
    prob = toy_problem() if cfg == 0 else config_problem(cfg)
    ref = oracle_mod.Oracle(prob).best(threads=4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, block, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lat, idx, enc, counts in out:
        assert (lat, idx) == ref, (rank, lat, idx, ref)
        assert sum(counts) == prob["n_mb"]
    assert len({(o[1], o[2], tuple(o[3]), tuple(o[4])) for o in out}) == 1
