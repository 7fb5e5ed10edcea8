"""Earth constant sets (mirror of sgp4kit.gravity, gravity.py:13-50).

The kernels receive the eight constants as a flat fp64 vector in the order
of :data:`GRAV_ORDER` (include/sgp4b.h).
"""

from __future__ import annotations

import math
from dataclasses import astuple, dataclass

import numpy as np

GRAV_ORDER = ("mu", "radius_earth_km", "xke", "tumin", "j2", "j3", "j4", "j3oj2")


@dataclass(frozen=True)
class GravityModel:
    """Earth constants in the canonical SGP units.

    ``xke`` is sqrt(GM) in Earth-radii^1.5 per minute; ``tumin = 1/xke``.
    """

    mu: float
    radius_earth_km: float
    xke: float
    tumin: float
    j2: float
    j3: float
    j4: float
    j3oj2: float

    def as_array(self) -> np.ndarray:
        return np.array(astuple(self), dtype=np.float64)


def make_gravity_model(mu: float, radius_km: float, j2: float, j3: float,
                       j4: float) -> GravityModel:
    """Derive xke/tumin/j3oj2 from the primary constants."""
    # r*r*r (not r**3): matches the reference's rounding bit for bit
    xke = 60.0 / math.sqrt(radius_km * radius_km * radius_km / mu)
    return GravityModel(mu=mu, radius_earth_km=radius_km, xke=xke,
                        tumin=1.0 / xke, j2=j2, j3=j3, j4=j4, j3oj2=j3 / j2)


#: WGS-72 (the set SGP4 element sets are fitted with)
WGS72 = make_gravity_model(398600.8, 6378.135, 0.001082616, -0.00000253881,
                           -0.00000165597)
