"""Multi-GPU driver: one process per GPU, the candidate space
block-cyclically sharded over ranks inside optimus_eval_candidates, and ONE
collective — an all_gather of each rank's 16-byte (lat, index) — after which
every rank takes the lexicographic minimum (optimus_best_plan).  NCCL has no
argmin and (lat, index) does not fit a packed 64-bit min for config 5, hence
the gather.  torch.distributed is plumbing only.
"""
from __future__ import annotations


def rank_share(begin: int, end: int, rank: int, world: int, block: int = 4096) -> int:
    """Number of candidate indices rank `rank` owns (blocks b = rank mod world)."""
    n = end - begin
    nblocks = (n + block - 1) // block
    mine = 0
    for b in range(rank, nblocks, world):
        mine += min(block, n - b * block)
    return mine


def gather_best(best2, group=None):
    """all_gather of every rank's (lat, index) -> tensor [world, 2] on best2's device."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world, 2), dtype=best2.dtype, device=best2.device)
    dist.all_gather_into_tensor(out.view(-1), best2.view(-1), group=group)
    return out


def distributed_search(ctx, rank: int, world: int, block: int = 4096, stream=None, group=None) -> dict:
    """Evaluate this rank's shard of the whole space, gather, decode the winner."""
    import torch
    total, _ = ctx.num_candidates()
    best2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, best2, rank=rank, world=world, block=block, stream=stream)
    g = gather_best(best2, group) if world > 1 else best2.view(1, 2)
    return ctx.best_plan(g.cpu().numpy())
