"""Multi-rank host logic on CPU (world_size 2, gloo): cell-count sharding, the
max-over-ranks timing reduction and the result gather.  The per-rank compute
here is the oracle (tests may call it); on B200 ranks it is the CUDA path."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2208_12350_b200 import dist as swdist
from paper_2208_12350_b200 import synth


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out_dir: str):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = synth.generate("c1", 0, 240)
        shard, (lo, hi) = swdist.local_shard(batch, world, rank)
        res = oracle.align_batch(shard.queries, shard.q_offsets, shard.refs, shard.r_offsets, shard.scoring, threads=2)
        cells = shard.cells()
        total_cells = swdist.sum_over_ranks(cells)
        slowest = swdist.max_over_ranks(float(rank + 1))
        gathered = swdist.gather_results(res)
        if rank == 0:
            np.savez(os.path.join(out_dir, "gathered.npz"), **gathered, lo=lo, hi=hi,
                     total_cells=total_cells, slowest=slowest)
        np.save(os.path.join(out_dir, f"cells_{rank}.npy"), np.array([cells, lo, hi]))
    finally:
        dist.destroy_process_group()


def test_sharded_gather_equals_single_process(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    g = np.load(tmp_path / "gathered.npz")
    batch = synth.generate("c1", 0, 240)
    ref = oracle.align_batch(batch.queries, batch.q_offsets, batch.refs, batch.r_offsets, batch.scoring, threads=2)
    for f in swdist.FIELDS:
        np.testing.assert_array_equal(g[f], ref[f])
    assert float(g["total_cells"]) == batch.cells()
    assert float(g["slowest"]) == 2.0
    c0 = np.load(tmp_path / "cells_0.npy")
    c1 = np.load(tmp_path / "cells_1.npy")
    assert c0[1] == 0 and c0[2] == c1[1] and c1[2] == 240      # contiguous cover
    assert max(c0[0], c1[0]) / ((c0[0] + c1[0]) / 2) < 1.02    # cell-balanced


def test_local_shard_slices_are_contiguous_and_complete():
    batch = synth.generate("c1", 0, 100)
    seen = 0
    for rank in range(3):
        shard, (lo, hi) = swdist.local_shard(batch, 3, rank)
        assert lo == seen
        for k in range(shard.n_pairs):
            assert shard.pair(k) == batch.pair(lo + k)
        seen = hi
    assert seen == 100


def test_reductions_without_process_group():
    assert swdist.max_over_ranks(3.5) == 3.5
    out = swdist.gather_results({f: np.arange(4) for f in swdist.FIELDS})
    np.testing.assert_array_equal(out["score"], np.arange(4))


def test_bench_strong_scaling_shards():
    """bench.py's workload at N GPUs: BASELINE configs[3] (c4, 4 M pairs) cut into N contiguous
    cell-balanced shards by sw_plan_shards (strong scaling: the 1-GPU point is the whole batch)."""
    import bench
    from paper_2208_12350_b200 import synth as s
    n, m = s.batch_lengths(s.CONFIGS["c4"])
    assert n.size == 4_000_000
    for world in (1, 2, 4, 8):
        prev = 0
        for rank in range(world):
            lo, hi, total, shard_cells = bench.shard_range("c4", world, rank)
            assert lo == prev and total == n.size and len(shard_cells) == world
            assert shard_cells[rank] == int(np.sum(n[lo:hi] * m[lo:hi]))
            prev = hi
        assert prev == n.size
        assert max(shard_cells) / (sum(shard_cells) / world) < 1.0001
    # a rank's shard is byte-identical to the serial generator's pairs
    b = bench.make_shard("c4", 123_456, 123_456 + 3000, 2)
    assert s.batch_sha256(b) == s.batch_sha256(s.generate("c4", 123_456, 123_456 + 3000))
