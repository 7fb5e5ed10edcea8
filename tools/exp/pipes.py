"""Instruction throughput per SM per cycle for the pipes the fp32 cell uses."""
import ctypes
import json
from pathlib import Path

import torch

lib = ctypes.CDLL(str(Path(__file__).resolve().parent / "pipes.so"))
lib.run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda", 0)
out = torch.zeros(1024, device=dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
ITERS = 2048
# (name, warp-instructions of each class per thread-iteration)
spec = [("ffma2", {"FFMA2": 8}), ("ffma", {"FFMA": 16}), ("mufu_rcp", {"MUFU": 8, "FADD": 8}),
        ("dfma", {"DFMA": 8}), ("f2f_f32_f64", {"F2F": 8}), ("ffma2+dfma", {"FFMA2": 8, "DFMA": 4}),
        ("ffma2+mufu", {"FFMA2": 8, "MUFU": 2, "FADD": 2}), ("ffma+ffma2", {"FFMA2": 8, "FFMA": 8})]
res = {}
for which, (name, mix) in enumerate(spec):
    blocks, threads = sms * 8, 256
    st = torch.cuda.current_stream().cuda_stream
    lib.run(which, out.data_ptr(), blocks, threads, st)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); lib.run(which, out.data_ptr(), blocks, threads, st); b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    clk = 1.965e9
    cyc = best * clk
    thr = blocks * threads * ITERS
    res[name] = {k: round(v * thr / 32 / sms / cyc, 3) for k, v in mix.items()}   # warp-inst/SM/cycle
    res[name]["us"] = round(best * 1e6, 1)
print(json.dumps(res, indent=1))
