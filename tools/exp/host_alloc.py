"""Host-side costs of a large result grid: cudaHostAlloc (page-locking) vs
pageable np.empty + first touch (with and without MADV_HUGEPAGE), and
multi-threaded memcpy from a pinned staging buffer."""
import ctypes, json, mmap, sys, time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_27830_b200 import _hostmem, _native

out = {}
for gb in (1, 4, 8):
    nb = gb << 30
    t0 = time.perf_counter(); blk = _hostmem.alloc(nb); t1 = time.perf_counter()
    out[f"cudaHostAlloc_{gb}GB_s"] = round(t1 - t0, 3)
    del blk; _hostmem.empty_cache()
    t0 = time.perf_counter(); a = np.empty(nb, np.uint8); a[::4096] = 0; t1 = time.perf_counter()
    out[f"np_empty_touch_{gb}GB_s"] = round(t1 - t0, 3)
    del a
    m = mmap.mmap(-1, nb, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, np.uint8)
    t0 = time.perf_counter(); a[::4096] = 0; t1 = time.perf_counter()
    out[f"mmap_thp_touch_{gb}GB_s"] = round(t1 - t0, 3)
    del a; m.close()
# memcpy pinned staging (64 MB) -> pageable 4 GB with threads
nb = 4 << 30
dst = np.empty(nb, np.uint8)
stage = np.asarray(_hostmem.alloc(64 << 20))
for th in (1, 4, 8, 16):
    def cp(off):
        ctypes.memmove(dst.ctypes.data + off, stage.ctypes.data, 64 << 20)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(th) as ex:
        list(ex.map(cp, range(0, nb, 64 << 20)))
    t1 = time.perf_counter()
    out[f"memcpy_4GB_{th}threads_GBs"] = round(nb / (t1 - t0) / 1e9, 1)
print(json.dumps(out, indent=1))
