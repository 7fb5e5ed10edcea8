"""Deterministic synthetic catalogues.

``starlink_like(n)`` forges a Starlink-like constellation as real TLE lines
(so parse -> init -> propagate is exercised end to end), seed 20260113 (the
paper's TLE epoch date), template STARLINK-1007.  Shells as
(inclination deg, mean motion rev/day, fraction):

    (53.05, 15.06, 35%) (53.2, 15.09, 17%) (43.0, 15.12, 25%)
    (70.0, 14.99, 8%)   (97.6, 15.02, 5%)  (53.0, 15.14, 10%)

jitter: inclination ±0.05°, mean motion ±0.01 rev/day; e ~ U(1e-4, 3e-4);
B* log-uniform in [5e-5, 8e-4]; RAAN/argp/M ~ U(0, 360); epoch 2026 day 13
plus U(0, 1).  Every perigee is above 220 km, so no satellite is in
simplified-drag mode.
"""

from __future__ import annotations

import math
import random

import numpy as np

from .tle import checksum, parse_catalog_columns

SEED = 20260113
SHELLS = ((53.05, 15.06, 0.35), (53.2, 15.09, 0.17), (43.0, 15.12, 0.25),
          (70.0, 14.99, 0.08), (97.6, 15.02, 0.05), (53.0, 15.14, 0.10))


def _with_checksum(body: str) -> str:
    body = body.ljust(68)[:68]
    return body + str(checksum(body + "0"))


def _bstar_field(b: float) -> str:
    """B* in implied-exponent form ' 12345-4' (mantissa 0.12345)."""
    if b == 0.0:
        return " 00000-0"
    exp = math.floor(math.log10(abs(b))) + 1
    mant = int(round(abs(b) / 10.0 ** exp * 1e5))
    if mant >= 100000:
        mant //= 10
        exp += 1
    sign = "-" if b < 0 else " "
    return f"{sign}{mant:05d}{exp:+d}"


def starlink_like_lines(n: int, seed: int = SEED) -> list[tuple[str, str]]:
    rng = random.Random(seed)
    weights = [s[2] for s in SHELLS]
    out = []
    for i in range(n):
        incl0, mm0, _ = rng.choices(SHELLS, weights=weights)[0]
        incl = incl0 + rng.uniform(-0.05, 0.05)
        mm = mm0 + rng.uniform(-0.01, 0.01)
        ecc = rng.uniform(1e-4, 3e-4)
        bstar = math.exp(rng.uniform(math.log(5e-5), math.log(8e-4)))
        raan, argp, ma = (rng.uniform(0.0, 360.0) for _ in range(3))
        day = 13.0 + rng.random()
        cat = 44713 + i
        catf = f"{cat:05d}" if cat < 100000 else (
            "ABCDEFGHJKLMNPQRSTUVWXYZ"[cat // 10000 - 10] + f"{cat % 10000:04d}")
        l1 = (f"1 {catf}U 19074A   26{day:012.8f}  .00002182  00000-0 "
              f"{_bstar_field(bstar)} 0  999")
        l2 = (f"2 {catf} {incl:8.4f} {raan:8.4f} {int(round(ecc * 1e7)):07d} "
              f"{argp:8.4f} {ma:8.4f} {mm:11.8f}{(i % 99999) + 1:5d}")
        out.append((_with_checksum(l1), _with_checksum(l2)))
    return out


def starlink_like(n: int, seed: int = SEED, base: int = 9341) -> np.ndarray:
    """(7, n) fp64 element columns.  Above ``base`` satellites the base
    catalogue is tiled (as the paper tiled its 9,341 real TLEs)
    to keep generation O(base) in Python."""
    k = min(n, base)
    lines = starlink_like_lines(k, seed)
    cols = parse_catalog_columns([a for a, _ in lines], [b for _, b in lines])
    if n <= k:
        return cols
    reps = -(-n // k)
    return np.tile(cols, (1, reps))[:, :n].copy()


# C1 (BASELINE.json configs[0]): the reference's ISS fixture record
# (tests/conftest.py:77-79 of the reference; tests/golden/real_tles.tle here)
ISS_LINES = ("1 25544U 98067A   20344.91667824  .00016717  00000-0  10270-3 0  9003",
             "2 25544  51.6442  21.0000 0001882 345.0000  15.0000 15.49309239  1000")


def iss_columns() -> np.ndarray:
    """(7, 1) fp64 element columns of the C1 ISS record."""
    from .tle import parse_catalog_columns
    return parse_catalog_columns([ISS_LINES[0]], [ISS_LINES[1]])
