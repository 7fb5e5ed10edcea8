"""Satellite sharding across the GPUs of one node.

Satellites are independent, so the path has NO exchange step: rank r takes
the contiguous satellite range ``shard_bounds(n, world, r)`` (sizes differ by
at most one — the reference's partition_work rule, batch.py:125-141), runs
its own init + grid launch on its own GPU and keeps its slice of the grid
resident in its HBM.  The only collectives here are optional consumers:
``max_over_ranks`` for timing and ``gather_grid`` for a caller that really
wants the whole grid on one rank (NVLink gather, not part of the timed path).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced satellite range of ``rank`` (empty if n < world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_plan(n: int, m: int, world: int, rank: int) -> tuple[str, int, int]:
    """What ``rank`` propagates: ``("rows", lo, hi)`` — a satellite range —
    normally, or ``("cols", lo, hi)`` — all satellites over a time range —
    when there are fewer satellites than ranks (e.g. C1, one ISS record),
    so no GPU idles."""
    if n >= world or m < world:
        return ("rows",) + shard_bounds(n, world, rank)
    return ("cols",) + shard_bounds(m, world, rank)


def world_info(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    world, _ = world_info(group)
    if world == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def propagate_sharded(columns: np.ndarray, times, precision: int = 32, group=None,
                      device=None):
    """Rank-local init + propagate of this rank's shard (``shard_plan``).

    ``columns`` is the full (7, n) catalogue (every rank may hold it; it is
    56 B per satellite).  Returns (BatchResult of device tensors or None,
    (axis, lo, hi)).
    """
    from .batch import init_batch, propagate_batch_device

    world, rank = world_info(group)
    times = np.asarray(times)
    axis, lo, hi = shard_plan(columns.shape[1], times.shape[0], world, rank)
    if hi <= lo:
        # an empty shard still takes part in collectives (gather_grid):
        # zero-row (or zero-column) grids on this rank's device
        from . import _device
        from .batch import BatchResult
        d = _device.require_cuda(device)
        n, m = (0, times.shape[0]) if axis == "rows" else (columns.shape[1], 0)
        planes = torch.empty((6, n, m), dtype=_device.torch_dtype(precision), device=d)
        error = torch.empty((n, m), dtype=torch.int32, device=d)
        return BatchResult(planes=planes, error=error, n=n, m=m), (axis, lo, hi)
    if axis == "rows":
        sats = init_batch(columns[:, lo:hi], precision=precision, device=device)
        return propagate_batch_device(sats, times), (axis, lo, hi)
    sats = init_batch(columns, precision=precision, device=device)
    return propagate_batch_device(sats, times[lo:hi]), (axis, lo, hi)


def gather_grid(planes: torch.Tensor, error: torch.Tensor, n_total: int, group=None,
                dst: int = 0, axis: str = "rows", m_total: int | None = None):
    """Assemble the full (6, N, M) / (N, M) grid on rank ``dst`` from the
    per-rank shards: row shards (``axis="rows"``, bounds from shard_bounds
    over ``n_total``) or time-column shards (``axis="cols"``, bounds over
    ``m_total``).  Returns the tensors on ``dst`` and None elsewhere.  Every
    rank must call it (empty shards pass zero-row tensors).  One
    ``dist.gather`` per plane set: gloo on CPU tensors, NCCL on device
    tensors (point-to-point under the hood), so only ``dst`` holds the
    world's shards."""
    world, rank = world_info(group)
    if world == 1:
        return planes, error
    if axis == "cols":
        # transpose to row form, reuse the row path, transpose back
        got = gather_grid(planes.transpose(1, 2).contiguous(), error.t().contiguous(),
                          int(m_total), group=group, dst=dst)
        if got is None:
            return None
        return got[0].transpose(1, 2).contiguous(), got[1].t().contiguous()
    m = planes.shape[2]
    bounds = [shard_bounds(n_total, world, r) for r in range(world)]
    rows_max = max(hi - lo for lo, hi in bounds)
    dev = planes.device

    def padded(x, shape):
        if tuple(x.shape) == tuple(shape):
            return x.contiguous()
        out = torch.zeros(shape, dtype=x.dtype, device=dev)
        out[tuple(slice(0, s) for s in x.shape)] = x
        return out

    p = padded(planes, (6, rows_max, m))
    e = padded(error, (rows_max, m))
    plist = [torch.empty_like(p) for _ in range(world)] if rank == dst else None
    elist = [torch.empty_like(e) for _ in range(world)] if rank == dst else None
    dist.gather(p, plist, dst=dst, group=group)
    dist.gather(e, elist, dst=dst, group=group)
    if rank != dst:
        return None
    full_p = torch.cat([plist[r][:, :hi - lo] for r, (lo, hi) in enumerate(bounds)], dim=1)
    full_e = torch.cat([elist[r][:hi - lo] for r, (lo, hi) in enumerate(bounds)], dim=0)
    return full_p, full_e
