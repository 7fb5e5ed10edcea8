"""Catalogue ingest: GPU read_catalog_columns vs the host vectorised decoder
(parse_catalog_columns on the file's lines) for a 1M-record 3-line file."""
import json, sys, tempfile, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200.catalog import starlink_like_lines
from paper_2603_27830_b200.ingest import _host_lines

base = starlink_like_lines(9341)
block = "".join(f"STARLINK-{i}\n{a}\n{b}\n" for i, (a, b) in enumerate(base))
text = block * 107                                  # 999,487 records
path = Path(tempfile.mkdtemp()) / "cat.tle"
path.write_text(text)
out = {"records": text.count("\n1 ") + (1 if text.startswith("1 ") else 0), "bytes": len(text)}
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cols = pkg.read_catalog_columns(path); torch.cuda.synchronize(); t1 = time.perf_counter()
out["gpu_read_catalog_columns_s"] = round(t1 - t0, 4)
t0 = time.perf_counter()
data = np.fromfile(path, dtype=np.uint8)
l1, l2 = _host_lines(data)
host = pkg.parse_catalog_columns(l1, l2)
t1 = time.perf_counter()
out["host_lines_plus_parse_catalog_columns_s"] = round(t1 - t0, 3)
out["bitwise_equal"] = bool(np.array_equal(cols.cpu().numpy().view(np.uint64), host.view(np.uint64)))
t0 = time.perf_counter()
sample = pkg.read_tle_file(path) if False else None
print(json.dumps(out))
