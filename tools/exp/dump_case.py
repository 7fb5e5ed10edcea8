"""Dump the GPU grid of a hard case (heavy drag, near-circular, +-14 days)
to gpurun_out/ for analysis against the oracle in the build container."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2603_27830_b200 as pkg  # noqa: E402
from paper_2603_27830_b200.tle import parse_catalog_columns  # noqa: E402
from tests.conftest import GOLDEN, read_tle_pairs  # noqa: E402

pairs = read_tle_pairs(GOLDEN / "leo_corpus.tle")[1]
cols = parse_catalog_columns([a for a, _ in pairs], [b for _, b in pairs])
base = cols[:, [137, 415, 391]].copy()
base[1] = 0.0029
base[6] = [1e-2, -1e-2, 1e-2]
times = np.linspace(-20160.0, 20160.0, 257)
out = {}
for p in (32, 64):
    res = pkg.propagate_batch(pkg.init_batch(base, precision=p), times)
    out[f"planes{p}"] = res.planes
    out[f"codes{p}"] = res.error
np.savez(ROOT / "gpurun_out" / "dump_case.npz", **out)
print("ok")
