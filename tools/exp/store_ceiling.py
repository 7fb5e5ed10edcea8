"""Write-bandwidth ceilings on this B200: torch fill_ (pure sequential
writes) and store_kernel (the grid kernel's 7-stream layout, no math)."""
import ctypes
import json
import sys
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
lib = ctypes.CDLL(str(HERE / "store_ceiling.so"))
lib.launch_store.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
lib.launch_stream.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p]
lib.launch_store8.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
lib.launch_tma.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                           ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rd = torch.ones(256 << 18, dtype=torch.float32, device=dev)
sink = torch.empty((), device=dev)


def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        torch.sum(rd, 0, out=sink)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


out = {}
for name, n, m in (("c2", 9341, 1024), ("c5", 1000000, 1024)):
    nbytes = 28 * n * m
    buf = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    med, best = timeit(lambda: buf.fill_(0.5))
    out[f"{name}_fill_gbs"] = nbytes / med / 1e9
    planes = buf[: 6 * n * m]
    codes = buf[6 * n * m:].view(torch.int32)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for mode in (0,):
        for bpsm in (2, 8):
            med, best = timeit(lambda: lib.launch_store(planes.data_ptr(), codes.data_ptr(), n, m,
                                                        sms * bpsm, 256, mode,
                                                        torch.cuda.current_stream().cuda_stream))
            out[f"{name}_mode{mode}_{bpsm}bpsm_us"] = round(med * 1e6, 1)
    st = torch.cuda.current_stream().cuda_stream
    for ch in (1, 2):
        for bpsm, thr in ((2, 256), (1, 256), (4, 128)):
            r = lib.launch_tma(planes.data_ptr(), codes.data_ptr(), n, m, sms * bpsm, thr, ch, st)
            assert r == 0, r
            med, best = timeit(lambda: lib.launch_tma(planes.data_ptr(), codes.data_ptr(), n, m, sms * bpsm, thr, ch, st))
            out[f"{name}_tma_ch{ch}_{bpsm}x{thr}_us"] = round(med * 1e6, 1)
    ref = torch.arange(6 * n * m, dtype=torch.float32, device=dev)
    for mode in ():
        for bpsm in (2, 8, 32):
            med, best = timeit(lambda: lib.launch_stream(buf.data_ptr(), buf.numel(), sms * bpsm, 256, mode, st))
            out[f"{name}_stream_mode{mode}_{bpsm}bpsm_us"] = round(med * 1e6, 1)
    for bpsm in (2, 8):
        med, best = timeit(lambda: lib.launch_store8(planes.data_ptr(), codes.data_ptr(), n, m, sms * bpsm, 256, st))
        out[f"{name}_store8_{bpsm}bpsm_us"] = round(med * 1e6, 1)
    del buf, planes, codes
print(json.dumps(out, indent=1))
