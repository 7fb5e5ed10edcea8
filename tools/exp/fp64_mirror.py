"""NumPy mirror of the fp64 fast cell (cell64_c1 in csrc/sgp4b.cu) and its
record folding, checked against the oracle on CPU before a GPU run: catches
formula / constant mistakes in the series and table-trig rewrite.
    python tools/exp/fp64_mirror.py"""
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import sgp4_oracle as oracle  # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like, iss_columns  # noqa: E402

EXTRA = {}
N = 512
SCALE = 81.48733086305042
C1 = 0.012271846295334399
C2 = 7.750731091254222e-12
SHIFT = 6755399441055744.0
TAB_S = np.sin(2 * np.pi * np.arange(N) / N)
TAB_C = np.cos(2 * np.pi * np.arange(N) / N)


def trig(x, short=False):
    y = x * SCALE + SHIFT
    k = y - SHIFT
    idx = k.astype(np.int64) & (N - 1)
    r = x - k * C1
    r = r - k * C2
    z = r * r
    sr = r - r * z / 6.0 if short else r + r * z * (z / 120.0 - 1.0 / 6.0)
    cr = 1.0 + z * (z / 24.0 - 0.5)
    sa, ca = TAB_S[idx], TAB_C[idx]
    return sa * cr + ca * sr, ca * cr - sa * sr


def record(s, g):
    f = {k: np.asarray(v, dtype=np.float64) for k, v in s.items() if k != "dtype"}
    hj2 = 0.5 * g["j2"]
    vkm = g["re"] * g["xke"] / 60.0
    no = f["no_unkozai"]
    am0 = np.cbrt(g["xke"] / no) ** 2
    S = np.sqrt(am0)
    eta, xmcof = f["eta"], f["xmcof"]
    R = dict(ARGPO=f["argpo"], ARGPDOT=f["argpdot"], NODEO=f["nodeo"], NODEDOT=f["nodedot"],
             NODECF=f["nodecf"], MO=f["mo"], MDOT=f["mdot"],
             U0=np.mod(f["mo"] + f["argpo"], 2 * np.pi), UDOT=f["mdot"] + f["argpdot"],
             S=S, SC1=-S * f["cc1"], SD2=-S * f["d2"], SD3=-S * f["d3"], SD4=-S * f["d4"],
             N2=no * f["t2cof"], N3=no * f["t3cof"], N4=no * f["t4cof"], N5=no * f["t5cof"],
             A0=xmcof * (1 - f["delmo"]), A1=3 * xmcof * eta, A2=3 * xmcof * eta ** 2,
             A3=xmcof * eta ** 3, OMGCOF=f["omgcof"],
             E0=f["ecco"] + f["bstar"] * f["cc5"] * f["sinmao"], BC4=f["bstar"] * f["cc4"],
             BC5=f["bstar"] * f["cc5"], AYCOF=f["aycof"], XLCOF=f["xlcof"],
             K41R=-1.5 * f["con41"] * hj2 * g["re"], KXR=0.5 * f["x1mth2"] * hj2 * g["re"],
             QX=-0.25 * f["x7thm1"] * hj2, C15CO=1.5 * np.cos(f["inclo"]) * hj2,
             C15CS=1.5 * np.cos(f["inclo"]) * np.sin(f["inclo"]) * hj2,
             X1V=f["x1mth2"] * hj2 * vkm, C41V=1.5 * f["con41"] * hj2 * vkm,
             SINIO=np.sin(f["inclo"]), COSIO=np.cos(f["inclo"]), INCLO=f["inclo"])
    return {k: v[:, None] for k, v in R.items()}, g["re"], vkm


def cell_c1(R, t, re, vkm):
    argpdf = R["ARGPO"] + R["ARGPDOT"] * t
    t2 = t * t
    nodem = R["NODEO"] + R["NODEDOT"] * t + R["NODECF"] * t2
    usec = R["U0"] + R["UDOT"] * t
    xmdf = R["MO"] + R["MDOT"] * t
    sx, cx = trig(xmdf, True)
    temp = ((R["A3"] * cx + R["A2"]) * cx + R["A1"]) * cx + R["OMGCOF"] * t + R["A0"]
    argpm = argpdf - temp
    sqam = (((R["SD4"] * t + R["SD3"]) * t + R["SD2"]) * t + R["SC1"]) * t + R["S"]
    nol = t2 * (((R["N5"] * t + R["N4"]) * t + R["N3"]) * t + R["N2"])
    tt = temp * temp
    smm = sx * (1 - 0.5 * tt) + cx * temp * (1 - tt / 6)
    em = R["E0"] - R["BC4"] * t - R["BC5"] * smm
    assert (np.abs(em) < 0.004).all()
    em = np.where(em < 1e-6, 1e-6, em)
    am = sqam * sqam
    irs = 1 / np.abs(sqam)
    inv_am = irs * irs
    nmx = inv_am * irs
    sa, ca = trig(argpm, True)
    axnl = em * ca
    em2 = em * em
    ilp = inv_am * (1 + em2 + em2 * em2)
    aynl = em * sa + ilp * R["AYCOF"]
    u = usec + nol + ilp * R["XLCOF"] * axnl
    s0, c0 = trig(u)
    q = c0 * axnl + s0 * aynl
    num = axnl * s0 - aynl * c0
    d1 = num * (1 + q + q * q)
    dd = d1 * d1
    sd = d1 - d1 * dd / 6
    cd = 1 + dd * (dd / 24 - 0.5)
    s1, c1 = s0 * cd + c0 * sd, c0 * cd - s0 * sd
    q = c1 * axnl + s1 * aynl
    num = axnl * s1 - aynl * c1 - d1
    d2 = (num + num * q) * (1 + q * q)
    se, ce = s1 + c1 * d2, c1 - s1 * d2
    ecose = axnl * ce + aynl * se
    esine = axnl * se - aynl * ce
    el2 = axnl * axnl + aynl * aynl
    ome = 1 - ecose
    iome = 1 / ome
    rl = am * ome
    betal = 1 + el2 * (-0.5 - 0.125 * el2)
    ipl = inv_am * (1 + el2 + el2 * el2)
    tq = esine * (0.5 + el2 * (0.125 + 0.0625 * el2))
    sqvk = irs * vkm * iome
    rdv, rvdv = sqvk * esine, sqvk * betal
    sinu = (se - aynl - axnl * tq) * iome
    cosu = (ce - axnl + aynl * tq) * iome
    sin2u = 2 * sinu * cosu
    cos2u = 1 - 2 * sinu * sinu
    ipl2 = ipl * ipl
    mr = rl * (re + ipl2 * R["K41R"] * betal) + ipl * R["KXR"] * cos2u
    t2s = ipl2 * sin2u
    dsu = t2s * R["QX"]
    xnode = nodem + t2s * R["C15CO"]
    dinc = ipl2 * cos2u * R["C15CS"]
    nmt = nmx * ipl
    mv = rdv - nmt * R["X1V"] * sin2u
    rv = rvdv + nmt * (cos2u * R["X1V"] + R["C41V"])
    d2_ = dsu * dsu
    sdd = dsu - dsu * d2_ / 6
    cdd = 1 - 0.5 * d2_
    sinsu, cossu = sinu * cdd + cosu * sdd, cosu * cdd - sinu * sdd
    snod, cnod = trig(xnode)
    di2 = dinc * dinc
    sdi = dinc - dinc * di2 / 6
    cdi = 1 - 0.5 * di2
    sini = R["SINIO"] * cdi + R["COSIO"] * sdi
    cosi = R["COSIO"] * cdi - R["SINIO"] * sdi
    xmx, xmy = -snod * cosi, cnod * cosi
    ra, rb = mr * sinsu, mr * cossu
    r = np.stack([xmx * ra + cnod * rb, xmy * ra + snod * rb, sini * ra])
    va = mv * sinsu + rv * cossu
    vb = mv * cossu - rv * sinsu
    v = np.stack([xmx * va + cnod * vb, xmy * va + snod * vb, sini * va])
    EXTRA.update(dsu=dsu, dinc=dinc)
    return r, v


def main():
    g = oracle.wgs72()
    for name, cols, times in (("ISS", iss_columns(), np.linspace(0, 1440, 1000)),
                              ("starlink 500", starlink_like(500), np.linspace(0, 1440, 200)),
                              ("starlink 14d", starlink_like(200), np.linspace(0, 20160, 300))):
        s = oracle.init_columns(cols, 64)
        ref, codes = oracle.grid(s, times)
        R, re, vkm = record(s, g)
        r, v = cell_c1(R, times[None, :], re, vkm)
        dr = np.linalg.norm(r - ref[:3], axis=0)
        dv = np.linalg.norm(v - ref[3:], axis=0)
        print(f"{name}: max|dr| {dr.max():.3e} km  max|dv| {dv.max():.3e} km/s  "
              f"max|dsu| {np.abs(EXTRA['dsu']).max():.2e} max|dinc| {np.abs(EXTRA['dinc']).max():.2e}")


if __name__ == "__main__":
    main()
