"""Page-locked host blocks for result grids that cross PCIe.

The reference returns pageable ``np.empty`` grids that are freed when the
caller drops them (batch.py:177-183).  A D2H copy only runs at full PCIe rate
into page-locked memory, and page-locking is slow (it dominates a 200 MB
result if done per call), so blocks are pooled — but unlike torch's caching
host allocator they are sized exactly (rounded to 2 MiB, not to a power of
two) and the pool retains at most ``cache_limit()`` bytes of free blocks;
anything above is unpinned and freed as soon as the last array over it dies.
``empty_cache()`` releases every free block.

The memory comes from ``sgp4b_host_alloc`` (cudaHostAlloc, portable), so any
GPU of the process can DMA into it.
"""

from __future__ import annotations

import atexit
import collections
import ctypes
import os
import threading

import numpy as np

from . import _native

_ALIGN_LARGE = 2 << 20
_ALIGN_SMALL = 64 << 10
_DEFAULT_LIMIT = 4 << 30

_lock = threading.Lock()
_free: list[tuple[int, int, int]] = []     # (size, ptr, release order) of retained free blocks
# blocks released by PinnedBlock.__del__: a finalizer may run inside any
# allocation (GC), even while this module holds _lock, so it never takes the
# lock; it appends here (deque.append is atomic) and the next pool call
# drains the queue under the lock
_released: collections.deque = collections.deque()
_stats = {"pinned_bytes": 0, "cached_bytes": 0, "allocs": 0, "reuses": 0}


def cache_limit() -> int:
    """Bytes of free pinned blocks the pool may retain
    (``SGP4B_HOST_CACHE_BYTES``, default 4 GiB)."""
    v = os.environ.get("SGP4B_HOST_CACHE_BYTES")
    return int(v) if v else _DEFAULT_LIMIT


_PIN_EAGER = 256 << 20
_recent: collections.OrderedDict = collections.OrderedDict()   # recently requested sizes


def worth_pinning(nbytes: int) -> bool:
    """Whether a result of ``nbytes`` should land in a pinned block (fast
    D2H, pooled) rather than in pageable memory filled through the staging
    ring.  Page-locking costs ~0.4 s/GB, so a large block is pinned only
    when it will pay back: one of that size is already cached, or the same
    size was requested recently (a repeated call: the second pins, later
    ones reuse it).  Small results (<= 256 MiB) are always pinned.  Every
    call is remembered."""
    size = _round(max(int(nbytes), 1))
    if size > cache_limit():
        return False
    with _lock:
        excess = _drain()
        seen = size in _recent
        _recent[size] = None
        _recent.move_to_end(size)
        while len(_recent) > 16:
            _recent.popitem(last=False)
        cached = any(sz >= size and sz <= size + size // 2 for sz, _, _ in _free)
    for ptr in excess:
        _free_ptr(ptr)
    return size <= _PIN_EAGER or cached or seen


def _round(nbytes: int) -> int:
    a = _ALIGN_LARGE if nbytes >= _ALIGN_LARGE else _ALIGN_SMALL
    return -(-nbytes // a) * a


class PinnedBlock:
    """One page-locked region; numpy views keep it alive through
    ``__array_interface__`` (their ``.base``), and it goes back to the pool
    when the last one dies."""

    __slots__ = ("ptr", "size", "__weakref__")

    def __init__(self, ptr: int, size: int):
        self.ptr = ptr
        self.size = size

    @property
    def __array_interface__(self):
        return {"shape": (self.size,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}

    def __del__(self):
        if self.ptr:
            q = _released
            if q is not None:               # None at interpreter teardown
                q.append((self.size, self.ptr))
            self.ptr = 0


_age = [0]                                   # release order of the free blocks


def _drain() -> list[int]:
    """Move released blocks into the free list (caller holds _lock); returns
    the pointers to unpin outside the lock.  The most recently released
    blocks are kept: a block that does not fit under the cache limit evicts
    the least recently released free blocks first (a large grid that is
    re-requested call after call stays pinned even after smaller tiles
    filled the cache); only a block larger than the limit itself is freed."""
    excess = []
    limit = cache_limit()
    while _released:
        size, ptr = _released.popleft()
        if size > limit:
            _stats["pinned_bytes"] -= size
            excess.append(ptr)
            continue
        while _free and _stats["cached_bytes"] + size > limit:
            k = min(range(len(_free)), key=lambda i: _free[i][2])     # oldest
            osize, optr, _ = _free.pop(k)
            _stats["cached_bytes"] -= osize
            _stats["pinned_bytes"] -= osize
            excess.append(optr)
        _age[0] += 1
        _free.append((size, ptr, _age[0]))
        _stats["cached_bytes"] += size
    _free.sort()
    return excess


def _free_ptr(ptr: int) -> None:
    try:
        _native.load().sgp4b_host_free(ptr)
    except Exception:                       # interpreter teardown
        pass


def alloc(nbytes: int) -> PinnedBlock:
    """A pinned block of at least ``nbytes`` (reused from the pool when a free
    block is no more than 1.5x the rounded request)."""
    size = _round(max(int(nbytes), 1))
    hit = None
    with _lock:
        excess = _drain()
        for k, (sz, ptr, _) in enumerate(_free):
            if sz >= size and sz <= size + size // 2:
                del _free[k]
                _stats["cached_bytes"] -= sz
                _stats["reuses"] += 1
                hit = (ptr, sz)
                break
    for ptr in excess:
        _free_ptr(ptr)
    if hit is not None:
        return PinnedBlock(*hit)
    lib = _native.load()
    out = ctypes.c_void_p()
    status = lib.sgp4b_host_alloc(size, ctypes.byref(out))
    if status != 0:
        empty_cache()                       # retry once without the retained blocks
        status = lib.sgp4b_host_alloc(size, ctypes.byref(out))
        if status != 0:
            raise MemoryError(lib.sgp4b_last_error().decode(errors="replace"))
    with _lock:
        _stats["pinned_bytes"] += size
        _stats["allocs"] += 1
    return PinnedBlock(out.value, size)


def empty(shapes_dtypes) -> list[np.ndarray]:
    """Several C-contiguous arrays carved from ONE pinned block (each 256-B
    aligned), e.g. the planes and code plane of one result grid."""
    offs, total = [], 0
    for shape, dtype in shapes_dtypes:
        total = -(-total // 256) * 256
        offs.append(total)
        total += int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize
    raw = np.asarray(alloc(total))
    out = []
    for (shape, dtype), off in zip(shapes_dtypes, offs):
        nb = int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize
        out.append(raw[off:off + nb].view(dtype).reshape(shape))
    return out


_ZERO_CHUNK = 4 << 20
_fill_pool = None


def pool_threads() -> int:
    """Host threads for zero fills and staged copies (``SGP4B_HOST_THREADS``,
    default: every core the process may use, at most 32)."""
    v = os.environ.get("SGP4B_HOST_THREADS")
    if v:
        return max(1, int(v))
    try:
        n = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        n = os.cpu_count() or 2
    return max(1, min(32, n))


def _pool():
    global _fill_pool
    if _fill_pool is None:
        from concurrent.futures import ThreadPoolExecutor
        _fill_pool = ThreadPoolExecutor(max_workers=pool_threads(), thread_name_prefix="sgp4b-host")
    return _fill_pool


_ZERO_PARTS = 4


def zero_fill_async(arr: np.ndarray, lo: int, hi: int) -> list:
    """Zero rows lo..hi of a C-contiguous array on the host thread pool
    (``ctypes.memset`` releases the GIL, so the fill runs while the caller
    waits on a DMA), in at most ``_ZERO_PARTS`` pieces of at least
    ``_ZERO_CHUNK`` bytes: more concurrent fills only compete with the DMA
    for host memory bandwidth (C4: 4 threads 64 ms, 16 threads 67 ms, against
    a 60.4 ms planes copy).  Returns the futures."""
    if hi <= lo:
        return []
    row = arr.strides[0]
    base = arr.ctypes.data + lo * row
    total = (hi - lo) * row
    piece = max(_ZERO_CHUNK, -(-total // _ZERO_PARTS))
    pool = _pool()
    return [pool.submit(ctypes.memset, base + off, 0, min(piece, total - off))
            for off in range(0, total, piece)]


def empty_cache() -> None:
    """Unpin and free every retained free block."""
    with _lock:
        excess = _drain()
        blocks = list(_free)
        _free.clear()
        _stats["cached_bytes"] = 0
        _stats["pinned_bytes"] -= sum(b[0] for b in blocks)
    for ptr in excess + [b[1] for b in blocks]:
        _free_ptr(ptr)


def stats() -> dict:
    """pinned_bytes (live + cached), cached_bytes (free, retained), allocs, reuses."""
    with _lock:
        excess = _drain()
        out = dict(_stats)
    for ptr in excess:
        _free_ptr(ptr)
    return out


atexit.register(empty_cache)
