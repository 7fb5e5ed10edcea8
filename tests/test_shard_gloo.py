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

from paper_2603_27830_b200.shard import gather_grid, max_over_ranks, shard_bounds, shard_plan


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


@pytest.mark.parametrize("n,m,world", [(1, 1000, 8), (3, 10, 4), (9341, 1000, 8), (2, 1, 4), (0, 5, 2)])
def test_shard_plan_covers_grid(n, m, world):
    """Rows when there are at least as many satellites as ranks, otherwise
    time columns (C1: one satellite on 8 GPUs); either way the shards tile
    the grid exactly."""
    plans = [shard_plan(n, m, world, r) for r in range(world)]
    axes = {a for a, _, _ in plans}
    assert len(axes) == 1
    axis = axes.pop()
    total = n if axis == "rows" else m
    assert axis == ("cols" if (n < world <= m) else "rows")
    cov = sorted((lo, hi) for _, lo, hi in plans)
    assert cov[0][0] == 0 and cov[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(cov, cov[1:]))


def _col_worker(rank, world, port, cols, times, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sgp4_oracle as oracle
        axis, lo, hi = shard_plan(cols.shape[1], times.size, world, rank)
        assert axis == "cols"
        planes, codes = oracle.grid(oracle.init_columns(cols, 64), times[lo:hi])
        got = gather_grid(torch.from_numpy(planes), torch.from_numpy(codes), cols.shape[1],
                          axis="cols", m_total=times.size)
        if rank == 0:
            out["planes"] = got[0].numpy()
            out["codes"] = got[1].numpy()
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_time_shards_reassemble_bitwise(corpus_columns):
    """One satellite on two ranks: the time axis is split and reassembled."""
    from oracle import sgp4_oracle as oracle
    cols = corpus_columns[:, :1]
    times = np.linspace(0.0, 1440.0, 13)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_col_worker, args=(2, _free_port(), cols, times, out), nprocs=2, join=True)
    ref_planes, ref_codes = oracle.grid(oracle.init_columns(cols, 64), times)
    assert np.array_equal(out["planes"], ref_planes)
    assert np.array_equal(out["codes"], ref_codes)


def _empty_worker(rank, world, port, cols, times, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sgp4_oracle as oracle
        n = cols.shape[1]
        lo, hi = shard_bounds(n, world, rank)
        if hi > lo:
            planes, codes = oracle.grid(oracle.init_columns(cols[:, lo:hi], 64), times)
            planes, codes = torch.from_numpy(planes), torch.from_numpy(codes)
        else:                      # an empty shard still joins the collective
            planes = torch.empty((6, 0, times.size), dtype=torch.float64)
            codes = torch.empty((0, times.size), dtype=torch.int32)
        got = gather_grid(planes, codes, n)
        if rank == 0:
            out["planes"] = got[0].numpy()
            out["codes"] = got[1].numpy()
    finally:
        dist.destroy_process_group()


def test_gather_with_an_empty_shard(corpus_columns):
    """One satellite, two ranks (rank 1's row shard is empty): every rank
    joins the gather and rank 0 gets the full grid."""
    from oracle import sgp4_oracle as oracle
    cols = corpus_columns[:, :1]
    times = np.linspace(0.0, 60.0, 1)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_empty_worker, args=(2, _free_port(), cols, times, out), nprocs=2, join=True)
    ref_planes, ref_codes = oracle.grid(oracle.init_columns(cols, 64), times)
    assert np.array_equal(out["planes"], ref_planes)
    assert np.array_equal(out["codes"], ref_codes)


def _gpu_worker(rank, world, port, cols, times, precision, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_27830_b200.shard import propagate_sharded
        torch.cuda.set_device(0)
        res, (axis, lo, hi) = propagate_sharded(cols, times, precision=precision, device="cuda:0")
        got = gather_grid(res.planes.cpu(), res.error.cpu(), cols.shape[1], axis=axis,
                          m_total=len(times))
        if rank == 0:
            out["planes"] = got[0].numpy()
            out["codes"] = got[1].numpy()
            out["axis"] = axis
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,precision", [(301, 77, 32), (301, 77, 64), (1, 1000, 32), (1, 1, 64)])
def test_two_process_gpu_shards_bitwise_equal_single_launch(corpus_columns, n, m, precision):
    """Two processes (one per shard) each run init + propagate on the GPU for
    their satellite range (or time range, or an empty shard), the shards are
    gathered, and the grid equals one single-process launch bit for bit."""
    import paper_2603_27830_b200 as pkg
    cols = np.tile(corpus_columns, (1, 1))[:, :n]
    times = np.linspace(0.0, 1440.0, m)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_gpu_worker, args=(2, _free_port(), cols, times, precision, out), nprocs=2, join=True)
    full = pkg.propagate_batch(pkg.init_batch(cols, precision=precision), times)
    assert out["axis"] == ("cols" if n == 1 and m >= 2 else "rows")
    assert np.array_equal(out["planes"], full.planes)
    assert np.array_equal(out["codes"], full.error)
