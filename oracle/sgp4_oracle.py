"""CPU ORACLE — test infrastructure only, never shipped, never on the product path.

A NumPy restatement of the reference package's SGP4 hot path (sgp4kit,
/root/reference/pkg/src/sgp4kit), used as the parity checker for the CUDA
kernels and as the CPU baseline timed by ``bench.py``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline leg and
``--impl reference``) may import it.

It reproduces the reference BIT FOR BIT at both precisions: the same NumPy
ufuncs, the same expression grouping (so Python-float sub-expressions fold
in fp64 before meeting fp32 arrays, exactly as NEP 50 does in the
reference), the same guarded both-branch selects and the same floor-mod
conventions.  ``tests/test_oracle.py`` pins this against golden vectors the
real reference produced (tests/golden/make_golden.py).

Map to the reference (file:line under pkg/src/sgp4kit/):
  gravity constants ........ gravity.py:31-47       -> wgs72()
  _sgp4_init ............... kernel.py:154-322      -> init()
  solve_kepler ............. kernel.py:325-349      -> kepler()
  _propagate ............... kernel.py:352-510      -> propagate()
  _sgp4_propagate merge .... kernel.py:524-534      -> propagate_merged()
  propagate_batch tiling ... batch.py:144-205       -> grid()
  dmath selects/mod ........ dmath.py:180-221       -> _sel/_floor/_pow/_fmod2pi
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

TWOPI = 2.0 * math.pi
X2O3 = 2.0 / 3.0

ELEMENT_COLUMNS = ("no_kozai", "ecco", "inclo", "nodeo", "argpo", "mo", "bstar")

#: SatInit float fields (kernel.py:68-107) — the order of the device satrec
SATREC_FIELDS = (
    "no_kozai", "ecco", "inclo", "nodeo", "argpo", "mo", "bstar",
    "no_unkozai", "ao", "con41", "x1mth2", "x7thm1",
    "mdot", "argpdot", "nodedot", "nodecf",
    "cc1", "cc4", "cc5", "d2", "d3", "d4", "t2cof", "t3cof", "t4cof", "t5cof",
    "eta", "omgcof", "xmcof", "delmo", "sinmao", "aycof", "xlcof",
)


def wgs72() -> dict:
    """WGS-72 constants, same arithmetic as gravity.py:31-47."""
    mu, re = 398600.8, 6378.135
    xke = 60.0 / math.sqrt(re * re * re / mu)
    j2, j3, j4 = 0.001082616, -0.00000253881, -0.00000165597
    return {"mu": mu, "re": re, "xke": xke, "tumin": 1.0 / xke,
            "j2": j2, "j3": j3, "j4": j4, "j3oj2": j3 / j2}


# ---- select / guard primitives (dmath.py:180-221) -------------------------

def _sel(cond, a, b):
    return np.where(cond, a, b)


def _floor(x, f):
    """maximum(x, f) as the reference spells it: where(x >= f, x, f)."""
    return np.where(x >= f, x, f)


def _pow(x, p):
    """Always the array power loop (dmath.py:180-190)."""
    return np.power(np.asarray(x), p)


def _fmod2pi(x):
    """mod_twopi_signed: x % 2pi toward zero for negatives (dmath.py:218-221)."""
    return np.where(x >= 0.0, x % TWOPI, -((-x) % TWOPI))


def _first(*pairs):
    """First true condition wins (kernel.py:127-136)."""
    out = None
    for cond, val in reversed(pairs):
        cond = np.asarray(cond)
        out = np.where(cond, np.int32(val), np.int32(0) if out is None else out)
    return out


# ---- init -------------------------------------------------------------

def init(cols: dict, dtype, g: dict | None = None) -> dict:
    """Initialisation constants for element arrays (kernel.py:154-322).

    ``cols`` maps ELEMENT_COLUMNS names to arrays (already ``dtype``).
    Returns the SatInit fields plus 'isimp', 'error_code_at_init', 'dtype'.
    """
    g = g or wgs72()
    with np.errstate(all="ignore"):
        return _init(cols, dtype, g)


def _init(c: dict, dtype, g: dict) -> dict:
    n0 = np.asarray(c["no_kozai"], dtype=dtype)
    e0 = np.asarray(c["ecco"], dtype=dtype)
    i0 = np.asarray(c["inclo"], dtype=dtype)
    node0 = np.asarray(c["nodeo"], dtype=dtype)
    w0 = np.asarray(c["argpo"], dtype=dtype)
    m0 = np.asarray(c["mo"], dtype=dtype)
    bs = np.asarray(c["bstar"], dtype=dtype)

    xke = dtype(g["xke"])
    j2, j3oj2, j4, re = g["j2"], g["j3oj2"], g["j4"], g["re"]
    tiny = np.finfo(dtype).tiny

    bad_n = n0 <= 0.0
    bad_e = (e0 >= 1.0) | (e0 < -0.001)
    n_safe = _sel(bad_n, 1.0e-4, n0)

    # geometry and the un-Kozai step (kernel.py:181-193)
    omeosq = _floor(1.0 - e0 * e0, tiny)
    rteosq = np.sqrt(omeosq)
    cosio = np.cos(i0)
    cosio2 = cosio * cosio
    ak = _pow(xke / n_safe, X2O3)
    d1 = 0.75 * j2 * (3.0 * cosio2 - 1.0) / (rteosq * omeosq)
    dl = d1 / (ak * ak)
    adel = ak * (1.0 - dl * dl - dl * (1.0 / 3.0 + 134.0 * dl * dl / 81.0))
    dl = d1 / (adel * adel)
    no_unkozai = n_safe / (1.0 + dl)
    deep = TWOPI / no_unkozai >= 225.0

    ao = _pow(xke / no_unkozai, X2O3)
    sinio = np.sin(i0)
    po = ao * omeosq
    con42 = 1.0 - 5.0 * cosio2
    con41 = -con42 - cosio2 - cosio2
    posq = _floor(po * po, tiny)
    rp = ao * (1.0 - e0)
    isimp = rp < 220.0 / re + 1.0
    perige = (rp - 1.0) * re

    # atmosphere model parameters by perigee height (kernel.py:208-221)
    ss = 78.0 / re + 1.0
    qzms2t = _pow(np.asarray((120.0 - 78.0) / re, dtype=dtype), 4.0)
    low = perige < 156.0
    s4_low = _sel(perige < 98.0, np.asarray(20.0, dtype=dtype), perige - 78.0)
    qzms24 = _sel(low, _pow((120.0 - s4_low) / re, 4.0), qzms2t)
    sfour = _sel(low, s4_low / re + 1.0, ss)

    # drag and secular coefficients (kernel.py:223-275)
    pinvsq = 1.0 / posq
    den = ao - sfour
    tsi = 1.0 / _sel(den == 0.0, tiny, den)
    eta = ao * e0 * tsi
    etasq = eta * eta
    eeta = e0 * eta
    psisq = _floor(np.abs(1.0 - etasq), tiny)
    coef = qzms24 * _pow(tsi, 4.0)
    coef1 = coef / _pow(psisq, 3.5)
    cc2 = coef1 * no_unkozai * (ao * (1.0 + 1.5 * etasq + eeta * (4.0 + etasq)) +
                                0.375 * j2 * tsi / psisq * con41 *
                                (8.0 + 3.0 * etasq * (8.0 + etasq)))
    cc1 = bs * cc2
    circ = e0 <= 1.0e-4
    cc3 = _sel(circ, 0.0 * e0,
               -2.0 * coef * tsi * j3oj2 * no_unkozai * sinio / _floor(e0, 1.0e-4))
    x1mth2 = 1.0 - cosio2
    cc4 = 2.0 * no_unkozai * coef1 * ao * omeosq * \
        (eta * (2.0 + 0.5 * etasq) + e0 * (0.5 + 2.0 * etasq) -
         j2 * tsi / (ao * psisq) *
         (-3.0 * con41 * (1.0 - 2.0 * eeta + etasq * (1.5 - 0.5 * eeta)) +
          0.75 * x1mth2 * (2.0 * etasq - eeta * (1.0 + etasq)) * np.cos(2.0 * w0)))
    cc5 = 2.0 * coef1 * ao * omeosq * (1.0 + 2.75 * (etasq + eeta) + eeta * etasq)
    cosio4 = cosio2 * cosio2
    k1 = 1.5 * j2 * pinvsq * no_unkozai
    k2 = 0.5 * k1 * j2 * pinvsq
    k3 = -0.46875 * j4 * pinvsq * pinvsq * no_unkozai
    mdot = no_unkozai + 0.5 * k1 * rteosq * con41 + \
        0.0625 * k2 * rteosq * (13.0 - 78.0 * cosio2 + 137.0 * cosio4)
    argpdot = (-0.5 * k1 * con42 +
               0.0625 * k2 * (7.0 - 114.0 * cosio2 + 395.0 * cosio4) +
               k3 * (3.0 - 36.0 * cosio2 + 49.0 * cosio4))
    xhdot1 = -k1 * cosio
    nodedot = xhdot1 + (0.5 * k2 * (4.0 - 19.0 * cosio2) +
                        2.0 * k3 * (3.0 - 7.0 * cosio2)) * cosio
    omgcof = bs * cc3 * np.cos(w0)
    eeta_g = _sel(np.abs(eeta) < tiny, tiny, eeta)
    xmcof = _sel(circ, 0.0 * e0, -X2O3 * coef * bs / eeta_g)
    nodecf = 3.5 * omeosq * xhdot1 * cc1
    t2cof = 1.5 * cc1
    xl_den = _sel(np.abs(cosio + 1.0) > 1.5e-12, 1.0 + cosio, np.asarray(1.5e-12, dtype=dtype))
    xlcof = -0.25 * j3oj2 * sinio * (3.0 + 5.0 * cosio) / xl_den
    aycof = -0.5 * j3oj2 * sinio
    dmt = 1.0 + eta * np.cos(m0)
    delmo = dmt * dmt * dmt
    sinmao = np.sin(m0)
    x7thm1 = 7.0 * cosio2 - 1.0

    # higher-order drag terms, zeroed in simplified mode (kernel.py:277-294)
    cc1sq = cc1 * cc1
    d2 = 4.0 * ao * tsi * cc1sq
    td = d2 * tsi * cc1 / 3.0
    d3 = (17.0 * ao + sfour) * td
    d4 = 0.5 * td * ao * tsi * (221.0 * ao + 31.0 * sfour) * cc1
    t3cof = d2 + 2.0 * cc1sq
    t4cof = 0.25 * (3.0 * d3 + cc1 * (12.0 * d2 + 10.0 * cc1sq))
    t5cof = 0.2 * (3.0 * d4 + 12.0 * cc1 * d3 + 6.0 * d2 * d2 +
                   15.0 * cc1sq * (2.0 * d2 + cc1sq))
    z = 0.0 * cc1
    sat = {
        "dtype": dtype,
        "no_kozai": n0, "ecco": e0, "inclo": i0, "nodeo": node0, "argpo": w0,
        "mo": m0, "bstar": bs,
        "no_unkozai": no_unkozai, "ao": ao, "con41": con41, "x1mth2": x1mth2,
        "x7thm1": x7thm1, "mdot": mdot, "argpdot": argpdot, "nodedot": nodedot,
        "nodecf": nodecf, "isimp": isimp, "cc1": cc1, "cc4": cc4, "cc5": cc5,
        "d2": _sel(isimp, z, d2), "d3": _sel(isimp, z, d3), "d4": _sel(isimp, z, d4),
        "t2cof": t2cof, "t3cof": _sel(isimp, z, t3cof), "t4cof": _sel(isimp, z, t4cof),
        "t5cof": _sel(isimp, z, t5cof), "eta": eta, "omgcof": omgcof, "xmcof": xmcof,
        "delmo": delmo, "sinmao": sinmao, "aycof": aycof, "xlcof": xlcof,
    }
    code = _first((bad_n, 2), (bad_e, 1), (deep, 7))
    sat["error_code_at_init"] = code
    # epoch evaluation flags immediate decay (kernel.py:316-322)
    _, _, c0 = propagate(sat, np.asarray(0.0, dtype=dtype), g)
    sat["error_code_at_init"] = np.where(code != 0, code, c0)
    return sat


# ---- Kepler -----------------------------------------------------------

def kepler(axnl, aynl, u):
    """Newton on E - axnl sinE + aynl cosE = u (kernel.py:325-349)."""
    e = u
    live = np.ones(np.broadcast(axnl, aynl, u).shape, dtype=bool)
    for _ in range(10):
        if not live.any():
            break
        s = np.sin(e)
        c = np.cos(e)
        step = 1.0 - c * axnl - s * aynl
        step = (u - aynl * c + axnl * s - e) / step
        step = np.where(step >= 0.95, 0.95 + 0.0 * step,
                        np.where(step <= -0.95, -0.95 + 0.0 * step, step))
        e = np.where(live, e + step, e)
        live = live & (np.abs(step) >= 1.0e-12)
    return e


# ---- propagate --------------------------------------------------------

def propagate(s: dict, t, g: dict | None = None):
    """One broadcast evaluation of the near-Earth theory (kernel.py:352-510).

    Returns (r (...,3), v (...,3), code) without the init-code merge."""
    g = g or wgs72()
    with np.errstate(all="ignore"):
        return _propagate(s, t, g)


def _propagate(s: dict, t, g: dict):
    dtype = s["dtype"]
    tiny = np.finfo(dtype).tiny
    xke, j2, re = g["xke"], g["j2"], g["re"]
    vkms = re * xke / 60.0
    simp = s["isimp"]

    # secular gravity + drag, both branches then select (kernel.py:365-391)
    xmdf = s["mo"] + s["mdot"] * t
    argpdf = s["argpo"] + s["argpdot"] * t
    nodedf = s["nodeo"] + s["nodedot"] * t
    t2 = t * t
    nodem = nodedf + s["nodecf"] * t2
    tempa = 1.0 - s["cc1"] * t
    tempe = s["bstar"] * s["cc4"] * t
    templ = s["t2cof"] * t2
    dw = s["omgcof"] * t
    dm0 = 1.0 + s["eta"] * np.cos(xmdf)
    dm = s["xmcof"] * (dm0 * dm0 * dm0 - s["delmo"])
    corr = dw + dm
    mm_f = xmdf + corr
    argpm_f = argpdf - corr
    t3 = t2 * t
    t4 = t3 * t
    tempa_f = tempa - s["d2"] * t2 - s["d3"] * t3 - s["d4"] * t4
    tempe_f = tempe + s["bstar"] * s["cc5"] * (np.sin(mm_f) - s["sinmao"])
    templ_f = templ + s["t3cof"] * t3 + t4 * (s["t4cof"] + t * s["t5cof"])
    mm = _sel(simp, xmdf, mm_f)
    argpm = _sel(simp, argpdf, argpm_f)
    tempa = _sel(simp, tempa, tempa_f)
    tempe = _sel(simp, tempe, tempe_f)
    templ = _sel(simp, templ, templ_f)

    # mean motion and eccentricity (kernel.py:393-414)
    nm = s["no_unkozai"]
    bad_nm = nm <= 0.0
    am = _pow(xke / _sel(bad_nm, 1.0e-4, nm), X2O3) * tempa * tempa
    am = _floor(am, tiny)
    nm = xke / _pow(am, 1.5)
    em = s["ecco"] - tempe
    bad_em = (em >= 1.0) | (em < -0.001)
    em = _sel(em < 1.0e-6, 1.0e-6 + 0.0 * em, em)
    mm = mm + s["no_unkozai"] * templ
    xlm = mm + argpm + nodem
    nodem = _fmod2pi(nodem)
    argpm = argpm % TWOPI
    xlm = xlm % TWOPI
    mm = (xlm - argpm - nodem) % TWOPI

    sinip = np.sin(s["inclo"])
    cosip = np.cos(s["inclo"])

    # long-period periodics (kernel.py:419-431)
    axnl = em * np.cos(argpm)
    ilp = 1.0 / _floor(am * (1.0 - em * em), tiny)
    aynl = em * np.sin(argpm) + ilp * s["aycof"]
    xl = mm + argpm + nodem + ilp * s["xlcof"] * axnl

    # Kepler (kernel.py:434-437)
    u = (xl - nodem) % TWOPI
    eo1 = kepler(axnl, aynl, u)
    se = np.sin(eo1)
    ce = np.cos(eo1)

    # short-period preliminaries (kernel.py:440-460)
    ecose = axnl * ce + aynl * se
    esine = axnl * se - aynl * ce
    el2 = axnl * axnl + aynl * aynl
    pl = am * (1.0 - el2)
    bad_pl = pl < 0.0
    pl_s = _floor(pl, tiny)
    rl = am * (1.0 - ecose)
    rl_s = _sel(rl == 0.0, tiny, rl)
    rdotl = np.sqrt(am) * esine / rl_s
    rvdotl = np.sqrt(pl_s) / rl_s
    betal = np.sqrt(_floor(1.0 - el2, tiny))
    q = esine / (1.0 + betal)
    sinu = am / rl_s * (se - aynl - axnl * q)
    cosu = am / rl_s * (ce - axnl + aynl * q)
    su = np.arctan2(sinu, cosu)
    sin2u = (cosu + cosu) * sinu
    cos2u = 1.0 - 2.0 * sinu * sinu
    ipl = 1.0 / pl_s
    h1 = 0.5 * j2 * ipl
    h2 = h1 * ipl

    # short-period periodics (kernel.py:463-469)
    mrt = rl * (1.0 - 1.5 * h2 * betal * s["con41"]) + 0.5 * h1 * s["x1mth2"] * cos2u
    su = su - 0.25 * h2 * s["x7thm1"] * sin2u
    xnode = nodem + 1.5 * h2 * cosip * sin2u
    xinc = s["inclo"] + 1.5 * h2 * cosip * sinip * cos2u
    mvt = rdotl - nm * h1 * s["x1mth2"] * sin2u / xke
    rvdot = rvdotl + nm * h1 * (s["x1mth2"] * cos2u + 1.5 * s["con41"]) / xke

    # orientation (kernel.py:472-493)
    ssu, csu = np.sin(su), np.cos(su)
    snod, cnod = np.sin(xnode), np.cos(xnode)
    sinc, cinc = np.sin(xinc), np.cos(xinc)
    xmx = -snod * cinc
    xmy = cnod * cinc
    ux = xmx * ssu + cnod * csu
    uy = xmy * ssu + snod * csu
    uz = sinc * ssu
    vx = xmx * csu - cnod * ssu
    vy = xmy * csu - snod * ssu
    vz = sinc * csu
    mr = mrt * re
    r = np.stack(np.broadcast_arrays(mr * ux, mr * uy, mr * uz), axis=-1)
    v = np.stack(np.broadcast_arrays((mvt * ux + rvdot * vx) * vkms,
                                     (mvt * uy + rvdot * vy) * vkms,
                                     (mvt * uz + rvdot * vz) * vkms), axis=-1)
    code = _first((bad_nm, 2), (bad_em, 1), (bad_pl, 4), (mrt < 1.0, 6))
    return r, v, code


def propagate_merged(s: dict, t, g: dict | None = None):
    """Propagate + init-code merge (kernel.py:524-534): init codes other
    than 6 persist; 6 is recomputed per cell."""
    t = np.asarray(t, dtype=s["dtype"])
    r, v, code = propagate(s, t, g)
    ic = np.asarray(s["error_code_at_init"])
    keep = np.where(ic == 6, 0, ic)
    return r, v, np.where(keep != 0, keep, code)


# ---- batch grid (batch.py:144-205) -----------------------------------

def init_columns(cols: np.ndarray, precision: int, g: dict | None = None) -> dict:
    """(7, n) element columns -> satrec dict at the batch precision (the
    reference casts elements to the batch dtype BEFORE init, batch.py:97)."""
    dtype = np.float32 if precision == 32 else np.float64
    return init({k: np.asarray(cols[i], dtype=dtype) for i, k in enumerate(ELEMENT_COLUMNS)},
                dtype, g)


def _rows(s: dict, lo: int, hi: int) -> dict:
    out = {}
    for k, v in s.items():
        if k == "dtype":
            out[k] = v
        else:
            a = np.asarray(v)
            out[k] = a[lo:hi][:, None] if a.ndim else a
    return out


def grid(s: dict, times, workers: int = 1, tile_cells: int = 1 << 18,
         g: dict | None = None):
    """Dense (6, N, M) planes + (N, M) int32 codes, tiled over row bands of
    floor(2^18 / M) satellites and dealt to a thread pool, like
    propagate_batch; output is independent of ``workers``."""
    dtype = s["dtype"]
    t = np.asarray(times, dtype=dtype)
    n = np.asarray(s["mo"]).shape[0]
    m = t.size
    planes = np.empty((6, n, m), dtype=dtype)
    codes = np.empty((n, m), dtype=np.int32)
    step = max(1, min(n, tile_cells // max(m, 1)))
    bands = [(lo, min(lo + step, n)) for lo in range(0, n, step)]

    def work(band):
        lo, hi = band
        r, v, c = propagate_merged(_rows(s, lo, hi), t, g)
        planes[:3, lo:hi] = np.moveaxis(r, -1, 0)
        planes[3:, lo:hi] = np.moveaxis(v, -1, 0)
        codes[lo:hi] = np.broadcast_to(c, (hi - lo, m))

    if workers <= 1 or len(bands) == 1:
        for b in bands:
            work(b)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(work, bands))
    return planes, codes


def default_workers() -> int:
    return os.cpu_count() or 1
