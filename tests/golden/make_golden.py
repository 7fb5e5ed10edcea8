"""Generate the golden fixtures from the REAL reference package.

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Outputs (committed, small): the reference's own corpora as TLE text, the
reference's TLE decode of them, and the reference's init constants, grid
states and error codes at fp64 and fp32.  Nothing on the GPU box reads
/root/reference; the tests there use these files plus oracle/.
"""

from __future__ import annotations

import dataclasses
import json
import math
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

import sgp4kit  # noqa: E402  (the reference)
from conftest import REAL_TLES, synthetic_tle_lines, with_checksums  # noqa: E402

import random  # noqa: E402

TWOPI = 2.0 * math.pi
INIT_FIELDS = [f.name for f in dataclasses.fields(sgp4kit.SatInit)
               if f.name not in ("grav", "dtype")]
ELEMENT_FIELDS = ("no_kozai", "ecco", "inclo", "nodeo", "argpo", "mo", "bstar")
PARSE_FIELDS = ("catalog_number", "epoch_year", "epoch_day_int", "epoch_day_frac",
                "ndot", "nddot", "bstar", "element_set_number", "inclination_deg",
                "raan_deg", "eccentricity", "argp_deg", "mean_anomaly_deg",
                "mean_motion_revday", "rev_number", "checksum1", "checksum2")

GRID_TIMES = np.concatenate([np.linspace(0.0, 1440.0, 41),
                             [-1440.0, -360.0, 4320.0, 10080.0, 20160.0]])


def write_tle(path: Path, records) -> None:
    with open(path, "w") as fh:
        for name, l1, l2 in records:
            if name:
                fh.write(name + "\n")
            fh.write(l1 + "\n" + l2 + "\n")


def main() -> None:
    # corpora ------------------------------------------------------------
    rng = random.Random(20230101)
    corpus = [synthetic_tle_lines(i, rng) for i in range(1200)]
    write_tle(OUT / "leo_corpus.tle", [("", a, b) for a, b in corpus])
    real = [(name,) + with_checksums(l1, l2) for name, l1, l2 in REAL_TLES]
    write_tle(OUT / "real_tles.tle", real)

    # reference TLE decode of every record --------------------------------
    recs = [sgp4kit.parse_tle(a, b, strict=True) for a, b in corpus]
    recs += [sgp4kit.parse_tle(a, b, strict=True) for _, a, b in real]
    parse = {f: np.array([getattr(r, f) for r in recs]) for f in PARSE_FIELDS}
    els = [sgp4kit.tle_to_elements(r) for r in recs]
    for f in ELEMENT_FIELDS:
        parse["el_" + f] = np.array([getattr(e, f) for e in els], dtype=np.float64)
    np.savez_compressed(OUT / "ref_parse.npz", **parse)

    # satellites for the state goldens: 4 near-Earth real + first 120 LEO --
    near = [e for (name, _, _), e in zip(real, els[1200:]) if name != "ECCENTRIC"]
    sats = near + els[:120]
    for precision in (64, 32):
        batch = sgp4kit.init_batch(sats, precision=precision)
        init = {f: np.asarray(getattr(batch.init, f)) for f in INIT_FIELDS}
        res = sgp4kit.propagate_batch(batch, GRID_TIMES)
        np.savez_compressed(OUT / f"ref_states_{precision}.npz",
                            times=GRID_TIMES, planes=res.planes, error=res.error,
                            **{"init_" + k: v for k, v in init.items()})

    # the documented failure modes -------------------
    by_name = dict(zip([r[0] for r in real], els[1200:]))
    iss, low = by_name["ISS"], by_name["LOWPERIGEE"]
    cases = {
        "iss_e015_b001": dataclasses.replace(iss, ecco=0.15, bstar=0.01),
        "lowperigee_b05": dataclasses.replace(low, bstar=0.5),
        "iss_e09999": dataclasses.replace(iss, ecco=0.9999),
        "n_zero": dataclasses.replace(iss, no_kozai=0.0),
        "e_15": dataclasses.replace(iss, ecco=1.5),
        "period_225": dataclasses.replace(iss, no_kozai=TWOPI / 225.0),
        "period_2249": dataclasses.replace(iss, no_kozai=TWOPI / 224.9),
        "eccentric": by_name["ECCENTRIC"],
        "period_226": dataclasses.replace(iss, no_kozai=TWOPI / 226.0),
        "period_718": dataclasses.replace(iss, no_kozai=2.0 * TWOPI / 1440.0),
        "e_neg": dataclasses.replace(iss, ecco=-0.002),
        "incl_180": dataclasses.replace(iss, inclo=math.pi),
    }
    fail_times = [0.0, 360.0, 720.0, 1440.0, 2880.0]
    table = {"times": fail_times, "cases": {}}
    for key, el in cases.items():
        row = {"elements": [float(getattr(el, f)) for f in ELEMENT_FIELDS]}
        for precision, dtype in ((64, np.float64), (32, np.float32)):
            init = sgp4kit.sgp4_init(el, dtype=dtype)
            st = sgp4kit.sgp4_propagate(init, np.asarray(fail_times, dtype=dtype))
            row[f"init_code_{precision}"] = int(np.asarray(init.error_code_at_init))
            row[f"codes_{precision}"] = [int(c) for c in np.asarray(st.error_code)]
            row[f"finite_{precision}"] = bool(np.isfinite(st.r).all() and np.isfinite(st.v).all())
        table["cases"][key] = row
    (OUT / "ref_failure_codes.json").write_text(json.dumps(table, indent=1) + "\n")

    # SGB1 bytes from the reference writer (batch.py:244-251) --------------
    sgb_times = np.array([0.0, 60.0, 120.0, 240.0, 480.0, 1440.0, -30.0])
    sgb_sats = near + els[:5] + [cases["lowperigee_b05"], cases["n_zero"]]
    for precision in (32, 64):
        res = sgp4kit.propagate_batch(sgp4kit.init_batch(sgb_sats, precision=precision),
                                      sgb_times)
        with open(OUT / f"ref_sgb1_{precision}.bin", "wb") as fh:
            sgp4kit.write_grid_binary(res, fh)
    np.save(OUT / "ref_sgb1_elements.npy",
            np.array([[getattr(e, f) for f in ELEMENT_FIELDS] for e in sgb_sats]).T)

    # the reference's drift_report (drift.py:52-100) on the acceptance corpus
    # (first 120 LEO records, test_acceptance.py:107-122 horizon/step) ----
    rep = sgp4kit.drift_report(els[:120], horizon_days=14.0, step_minutes=90.0)
    np.savez_compressed(
        OUT / "ref_drift.npz",
        **{k: np.asarray(getattr(rep, k)) for k in
           ("days", "p5_km", "p50_km", "p95_km", "p5_kms", "p50_kms", "p95_kms",
            "heuristic_km", "corpus_size", "excluded_cells", "included_cells")})
    (OUT / "ref_drift.csv").write_text(sgp4kit.emit_report_csv(rep))

    # the reference CLI (cli.py:160-184) on the real records file ---------
    import tempfile
    from sgp4kit import cli as ref_cli
    with tempfile.TemporaryDirectory() as tmp:
        for precision in (32, 64):
            path = Path(tmp) / f"b{precision}.bin"
            rc = ref_cli.main(["batch", str(OUT / "real_tles.tle"), "--tsince", "0:1500:300",
                               "--precision", str(precision), "--format", "binary",
                               "--out", str(path)])
            assert rc == 0
            (OUT / f"ref_cli_batch_{precision}.bin").write_bytes(path.read_bytes())
        path = Path(tmp) / "b.csv"
        rc = ref_cli.main(["batch", str(OUT / "real_tles.tle"), "--tsince-list",
                           "0,90.5,1440,-60", "--out", str(path)])
        assert rc == 0
        (OUT / "ref_cli_batch_64.csv").write_text(path.read_text())
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
