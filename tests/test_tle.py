"""TLE/OMM ingest: known answers from the reference's tests (pkg/tests/
test_tle.py) and field-by-field equality with the reference's own decode of
both corpora (tests/golden/ref_parse.npz)."""

import math

import numpy as np
import pytest

from paper_2603_27830_b200 import (
    ChecksumError,
    TleError,
    checksum,
    decode_alpha5,
    parse_catalog_columns,
    parse_omm_kvp,
    parse_tle,
    read_tle_file,
    tle_to_elements,
)
from paper_2603_27830_b200.tle import (
    ELEMENT_COLUMNS,
    _implied_exponent,
    _split_epoch,
    elements_to_columns,
)
from tests.conftest import GOLDEN

PARSE_FIELDS = ("catalog_number", "epoch_year", "epoch_day_int", "epoch_day_frac",
                "ndot", "nddot", "bstar", "element_set_number", "inclination_deg",
                "raan_deg", "eccentricity", "argp_deg", "mean_anomaly_deg",
                "mean_motion_revday", "rev_number", "checksum1", "checksum2")


@pytest.fixture(scope="module")
def ref_parse():
    return dict(np.load(GOLDEN / "ref_parse.npz"))


@pytest.fixture(scope="module")
def all_pairs(corpus_lines, real_records):
    return list(corpus_lines) + list(real_records.values())


def test_every_field_equals_reference(all_pairs, ref_parse):
    recs = [parse_tle(a, b, strict=True) for a, b in all_pairs]
    for f in PARSE_FIELDS:
        got = np.array([getattr(r, f) for r in recs])
        assert np.array_equal(got, ref_parse[f]), f
    cols = elements_to_columns([tle_to_elements(r) for r in recs])
    for i, f in enumerate(ELEMENT_COLUMNS):
        assert np.array_equal(cols[i], ref_parse["el_" + f]), f


def test_vectorised_columns_equal_record_route(all_pairs, ref_parse):
    cols = parse_catalog_columns([a for a, _ in all_pairs], [b for _, b in all_pairs])
    for i, f in enumerate(ELEMENT_COLUMNS):
        assert np.array_equal(cols[i], ref_parse["el_" + f]), f


@pytest.mark.parametrize("field", [" 12345-3", "-11606-4", " 00000-0", " 00000+0", " 12345+1",
                                   "+12345-9", " 1-5", "-9+9", "      ", " 12345", "-00001-1",
                                   " 99999-9"])
def test_implied_exponent_columns_match_scalar(field):
    """The vectorised B* decoder (every shape the scalar decoder accepts)
    equals _implied_exponent bit for bit (tle.py:_implied_exponent)."""
    from paper_2603_27830_b200.tle import _implied_exponent, _implied_exponent_columns
    raw = np.char.strip(np.array([field, " 12345-3", field], dtype="S8"))
    got = _implied_exponent_columns(raw)
    want = _implied_exponent(field, "bstar")
    assert got[0] == want and got[2] == want and got[1] == _implied_exponent(" 12345-3", "b")
    assert np.signbit(got[0]) == np.signbit(want)


def test_checksum_rules(real_records):
    l1, _ = real_records["ISS"]
    assert checksum(l1) == int(l1[68])
    assert checksum(" " * 68) == 0
    assert checksum("-" + " " * 67) == 1
    assert checksum("A" * 68) == 0
    with pytest.raises(TleError):
        checksum("1 25544")


@pytest.mark.parametrize("field,value", [("25544", 25544), ("    7", 7), ("A0000", 100000),
                                         ("J0001", 180001), ("Z9999", 339999)])
def test_alpha5_known(field, value):
    assert decode_alpha5(field) == value


@pytest.mark.parametrize("bad", ["I0000", "O1234", "A12B4", "123456"])
def test_alpha5_rejects(bad):
    with pytest.raises(TleError):
        decode_alpha5(bad)


@pytest.mark.parametrize("field,value", [(" 10270-3", 0.10270e-3), ("-11606-4", -0.11606e-4),
                                         (" 00000-0", 0.0), (" 00000+0", 0.0),
                                         ("        ", 0.0), (" 13844-3", 0.13844e-3)])
def test_implied_exponent(field, value):
    assert _implied_exponent(field, "t") == value


def test_implied_exponent_garbage():
    with pytest.raises(TleError):
        _implied_exponent("1.2e-3x", "t")


def test_epoch_split():
    assert _split_epoch("57001.00000000")[0] == 1957
    assert _split_epoch("56001.00000000")[0] == 2056
    year, day, frac = _split_epoch("20344.91667824")
    assert (year, day, frac) == (2020, 344, 0.91667824)
    for bad in ("20367.00000000", "20000.50000000"):
        with pytest.raises(TleError):
            _split_epoch(bad)


def test_checksum_modes(real_records):
    l1, l2 = real_records["ISS"]
    bad = l1[:68] + str((int(l1[68]) + 1) % 10)
    assert any("checksum" in w for w in parse_tle(bad, l2).warnings)
    with pytest.raises(ChecksumError):
        parse_tle(bad, l2, strict=True)
    with pytest.raises(TleError):
        parse_tle(l2, l1)
    with pytest.raises(TleError):
        parse_tle(l1, "2 00001" + l2[7:])
    with pytest.raises(TleError):
        parse_tle(l1[:60], l2, lenient_length=False)


def test_units(real_records):
    el = tle_to_elements(parse_tle(*real_records["ISS"]))
    assert el.no_kozai == pytest.approx(15.49309239 * 2.0 * math.pi / 1440.0, rel=1e-15)
    for a in (el.nodeo, el.argpo, el.mo):
        assert 0.0 <= a < 2.0 * math.pi


OMM = """\
COMMENT generated for parser agreement
OBJECT_NAME = ISS (ZARYA)
EPOCH = 2020-12-09T22:00:00.999936
MEAN_MOTION = 15.49309239
ECCENTRICITY = 0.0001882
INCLINATION = 51.6442
RA_OF_ASC_NODE = 21.0
ARG_OF_PERICENTER = 345.0
MEAN_ANOMALY = 15.0
BSTAR = 0.00010270
"""


def test_omm_matches_tle_route(real_records):
    a = tle_to_elements(parse_tle(*real_records["ISS"]))
    b = parse_omm_kvp(OMM)
    for f in ELEMENT_COLUMNS:
        assert getattr(a, f) == getattr(b, f), f
    assert (b.epoch_year, b.epoch_day_int) == (2020, 344)
    assert b.epoch_day_frac == pytest.approx(a.epoch_day_frac, abs=1e-8)
    with pytest.raises(TleError, match="BSTAR"):
        parse_omm_kvp(OMM.replace("BSTAR = 0.00010270\n", ""))
    with pytest.raises(TleError):
        parse_omm_kvp(OMM.replace("2020-12-09T22:00:00.999936", "yesterday"))


def test_read_tle_file(tmp_path, real_records):
    recs = real_records
    path = tmp_path / "mixed.tle"
    names = list(recs)
    text = []
    for name in names[:3]:
        text += [name, *recs[name]]
    text += list(recs[names[3]])
    path.write_text("\n".join(text) + "\n")
    assert [r.catalog_number for r in read_tle_file(path)] == [25544, 44713, 43013, 20813]
    broken = tmp_path / "broken.tle"
    broken.write_text(recs["ISS"][0] + "\n")
    with pytest.raises(TleError):
        read_tle_file(broken)
    partial = tmp_path / "partial.tle"
    b1, b2 = recs["STARLINK-1007"]
    partial.write_text("\n".join([*recs["ISS"], b1, "2 !" + b2[3:]]) + "\n")
    with pytest.raises(TleError, match="record 1 at line 3"):
        read_tle_file(partial)
