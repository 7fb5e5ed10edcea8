"""Worst fp64 / fp32 cells of the parity campaign catalogues, with their
elements, for diagnosis."""
import json, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from oracle import sgp4_oracle as oracle
sys.path.insert(0, str(Path(__file__).resolve().parent))
from parity_campaign import catalogue, norms  # noqa: E402


def tempa_em(s64, i, t):
    """tempa and em of satellite i at t, as kernel.py:366-396 forms them."""
    g = {k: float(np.asarray(v)[i]) for k, v in s64.items() if k != "dtype"}
    if g["isimp"]:
        tempa = 1.0 - g["cc1"] * t
        tempe = g["bstar"] * g["cc4"] * t
    else:
        tempa = 1.0 - g["cc1"] * t - g["d2"] * t**2 - g["d3"] * t**3 - g["d4"] * t**4
        tempe = g["bstar"] * g["cc4"] * t          # + cc5 periodic (small)
    return tempa, g["ecco"] - tempe

rows = []
summary = {"fp64_cells_over_1mm": 0, "of_which_tempa_below_0.2_or_em_over_0.5": 0,
           "fp32_cells_over_1km": 0, "fp32_of_which_tempa_below_0.2_or_em_over_0.5": 0}
for seed in range(40):
    rng = np.random.default_rng(1000 + seed)
    cols = catalogue(rng, 400)
    times = np.sort(rng.uniform(-2880.0, 20160.0, 150))
    s64 = oracle.init_columns(cols, 64)
    r64, c64 = oracle.grid(s64, times, workers=8)
    g64 = pkg.propagate_batch(pkg.init_batch(cols, precision=64), times)
    g32 = pkg.propagate_batch(pkg.init_batch(cols, precision=32), times)
    ok = (c64 == 0) & (g64.error == 0)
    dr = np.linalg.norm(g64.planes[:3] - r64[:3], axis=0)
    dr = np.where(ok, dr, 0)
    d32 = np.linalg.norm(g32.planes[:3].astype(np.float64) - r64[:3], axis=0)
    d32 = np.where((c64 == 0) & (g32.error == 0), d32, 0)
    for name, d, thr in (("fp64", dr, 1e-6), ("fp32", d32, 1.0)):
        bad = np.argwhere(d > thr)
        key = "fp64_cells_over_1mm" if name == "fp64" else "fp32_cells_over_1km"
        key2 = ("of_which_tempa_below_0.2_or_em_over_0.5" if name == "fp64"
                else "fp32_of_which_tempa_below_0.2_or_em_over_0.5")
        summary[key] += len(bad)
        for bi, bj in bad:
            ta, em = tempa_em(s64, bi, times[bj])
            summary[key2] += int(ta < 0.2 or abs(em) > 0.5)
    for name, d in (("fp64", dr), ("fp32", d32)):
        i, j = np.unravel_index(np.argmax(d), d.shape)
        if d[i, j] > (1e-6 if name == "fp64" else 1.0):
            el = cols[:, i]
            rows.append({"seed": seed, "prec": name, "sat": int(i), "t": float(times[j]),
                         "err_km": float(d[i, j]), "n_bad_cells": int((d > (1e-6 if name == 'fp64' else 1.0)).sum()),
                         "no": el[0], "ecco": el[1], "incl": el[2], "bstar": el[6],
                         "period_min": 2 * np.pi / el[0], "isimp": bool(np.asarray(s64["isimp"])[i]),
                         "r_ref_km": float(np.linalg.norm(r64[:3, i, j])),
                         "tempa": tempa_em(s64, i, times[j])[0], "em": tempa_em(s64, i, times[j])[1]})
print(json.dumps({"summary": summary, "rows": rows}, indent=1))
