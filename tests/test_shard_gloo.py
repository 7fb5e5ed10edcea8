"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic:
shard bounds, max-over-ranks timing and the optional grid gather.  The per
shard compute here is the CPU oracle standing in for the GPU launch, so the
test checks that assembling shards reproduces the unsharded grid bit for bit
(the analogue of the reference's worker invariance, test_batch.py:67-83)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_27830_b200.shard import gather_grid, max_over_ranks, shard_bounds


@pytest.mark.parametrize("n", list(range(0, 12)) + [9341, 100000])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_cover_disjoint_balanced(n, world):
    bounds = [shard_bounds(n, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in bounds]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cols, times, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sgp4_oracle as oracle
        n = cols.shape[1]
        lo, hi = shard_bounds(n, world, rank)
        planes, codes = oracle.grid(oracle.init_columns(cols[:, lo:hi], 64), times)
        slowest = max_over_ranks(10.0 * (rank + 1))
        got = gather_grid(torch.from_numpy(planes), torch.from_numpy(codes), n)
        if rank == 0:
            out["slowest"] = slowest
            out["planes"] = got[0].numpy()
            out["codes"] = got[1].numpy()
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shards_reassemble_bitwise(corpus_columns):
    from oracle import sgp4_oracle as oracle
    cols = corpus_columns[:, :37]
    times = np.linspace(0.0, 1440.0, 11)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, _free_port(), cols, times, out), nprocs=2, join=True)
    ref_planes, ref_codes = oracle.grid(oracle.init_columns(cols, 64), times)
    assert out["slowest"] == 20.0
    assert np.array_equal(out["planes"], ref_planes)
    assert np.array_equal(out["codes"], ref_codes)
