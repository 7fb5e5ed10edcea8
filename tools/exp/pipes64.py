"""FP64 issue/pipe interplay on this B200 (tools/exp/pipes64.cu): warp
instructions per SMSP per cycle for DFMA alone and DFMA mixed with ALU, LDS
and FFMA work, plus the dependent-DFMA latency."""
import ctypes
import json
from pathlib import Path

import torch

lib = ctypes.CDLL(str(Path(__file__).resolve().parent / "pipes64.so"))
lib.run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda", 0)
out = torch.zeros(1024, device=dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
ITERS = 1024
spec = [("dfma", 8, 0), ("dfma+8alu", 8, 8), ("dfma+16alu", 8, 16), ("dfma+4lds", 8, 4),
        ("dfma+8ffma", 8, 8), ("dfma_latency", 8, 0)]
res = {}
clk = 1.965e9
for which, (name, nd, no) in enumerate(spec):
    blocks, threads = (sms * 8, 256) if name != "dfma_latency" else (sms, 32)
    st = torch.cuda.current_stream().cuda_stream
    lib.run(which, out.data_ptr(), blocks, threads, st)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); lib.run(which, out.data_ptr(), blocks, threads, st); b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    cyc = best * clk
    if name == "dfma_latency":
        res[name] = {"cycles_per_dependent_dfma": round(cyc / (ITERS * 8), 2)}
        continue
    warp_iters = blocks * threads / 32 * ITERS / (sms * 4)       # per SMSP
    res[name] = {"dfma_per_smsp_cycle": round(nd * warp_iters / cyc, 3),
                 "other_per_smsp_cycle": round(no * warp_iters / cyc, 3),
                 "cycles_per_iter_per_warp": round(cyc / warp_iters, 2), "us": round(best * 1e6, 1)}
print(json.dumps(res, indent=1))

# ILP sweep at 4 warps per SMSP (148 x 512 threads) and 8 per SMSP; DMUL and
# register-operand DFMA at full occupancy
lib.run2.argtypes = lib.run.argtypes
sweep = {}
for which, name in enumerate(["chains1", "chains2", "chains3", "chains4", "dmul", "dfma_reg"]):
    for wps in ((4, 8) if name.startswith("chains") else (16,)):
        blocks, threads = (sms, 128 * wps) if wps <= 8 else (sms * 8, 256)
        st = torch.cuda.current_stream().cuda_stream
        lib.run2(which, out.data_ptr(), blocks, threads, st)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); lib.run2(which, out.data_ptr(), blocks, threads, st); b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3)
        ops = blocks * threads / 32 * ITERS * 8 / (sms * 4)
        sweep[f"{name}_w{wps}"] = round(ops / (best * clk), 3)
print(json.dumps({"fp64_warp_inst_per_smsp_cycle": sweep}, indent=1))
