"""Multi-GPU plumbing: the batch shards naturally.

Pairs are independent, so N GPUs process N contiguous, cell-balanced ranges of
the caller's batch with no collective on the data path (the
paper's experiments are single-GPU; this is the B200 build's own scaling).
torch.distributed (NCCL on B200 ranks, gloo in the CPU tests) is used only for
the timing barrier / max-over-ranks reduction and the optional result gather
(20 B per pair).
"""
from __future__ import annotations

import numpy as np

FIELDS = ("score", "q_end", "r_end", "q_start", "r_start")


def shard_cuts(q_offsets: np.ndarray, r_offsets: np.ndarray, world: int) -> np.ndarray:
    """Cell-count shard plan (host only): world + 1 cut indices (C ABI sw_plan_shards)."""
    from .sw import sw_plan_shards
    return sw_plan_shards(q_offsets, r_offsets, world)


def local_range(q_offsets: np.ndarray, r_offsets: np.ndarray, world: int, rank: int) -> tuple[int, int]:
    cuts = shard_cuts(q_offsets, r_offsets, world)
    return int(cuts[rank]), int(cuts[rank + 1])


def local_shard(batch, world: int, rank: int):
    """This rank's contiguous slice of a synth.Batch (a new CSR batch)."""
    from .synth import Batch
    lo, hi = local_range(batch.q_offsets, batch.r_offsets, world, rank)
    qo = batch.q_offsets[lo:hi + 1]
    ro = batch.r_offsets[lo:hi + 1]
    q = batch.queries[qo[0]:qo[-1]]
    r = batch.refs[ro[0]:ro[-1]]
    return Batch(np.ascontiguousarray(q), qo - qo[0], np.ascontiguousarray(r), ro - ro[0], dict(batch.scoring),
                 f"{batch.name}[rank {rank}/{world}]"), (lo, hi)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_results(local: dict, device=None) -> dict | None:
    """All-gather each rank's five int32 result arrays; returns the concatenation
    in rank order (= the caller's pair order, since shards are contiguous)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return {f: np.asarray(local[f]) for f in FIELDS}
    world = dist.get_world_size()
    n = int(len(local[FIELDS[0]]))
    sizes_t = torch.tensor([n], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(sizes, sizes_t)
    sizes = [int(s.item()) for s in sizes]
    width = max(max(sizes), 1)
    mine = torch.full((5, width), -3, dtype=torch.int32, device=device)
    if n:
        mine[:, :n] = torch.as_tensor(np.stack([np.asarray(local[f], dtype=np.int32) for f in FIELDS]),
                                      device=device)
    parts = [torch.empty((5, width), dtype=torch.int32, device=device) for _ in range(world)]
    dist.all_gather(parts, mine)
    cat = np.concatenate([p[:, :s].cpu().numpy() for p, s in zip(parts, sizes)], axis=1)
    return {f: cat[i] for i, f in enumerate(FIELDS)}
