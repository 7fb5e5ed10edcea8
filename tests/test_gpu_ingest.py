"""GPU catalogue ingest (ingest.read_catalog_columns / sgp4b_tle_columns)
against the host decoder parse_catalog_columns, which is itself pinned to
the reference's per-record parse (test_tle.py): bit for bit on real,
synthetic and edge-case catalogues, and the host path's errors."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


def _host(text: str):
    from paper_2603_27830_b200.ingest import _host_lines
    from paper_2603_27830_b200.tle import parse_catalog_columns
    l1, l2 = _host_lines(np.frombuffer(text.encode(), dtype=np.uint8))
    return parse_catalog_columns(l1, l2)


def _gpu(text: str):
    from paper_2603_27830_b200 import read_catalog_columns
    return read_catalog_columns(text.encode()).cpu().numpy()


def _same(a, b):
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("name", ["leo_corpus.tle", "real_tles.tle"])
def test_golden_catalogues_bitwise(name):
    text = (GOLDEN / name).read_text()
    _same(_gpu(text), _host(text))


def test_synthetic_catalogue_bitwise_and_file_path(tmp_path):
    from paper_2603_27830_b200 import read_catalog_columns
    from paper_2603_27830_b200.catalog import starlink_like_lines
    lines = starlink_like_lines(20000)
    text = "".join(f"STARLINK-{i}\n{a}\n{b}\n" for i, (a, b) in enumerate(lines))
    host = _host(text)
    _same(_gpu(text), host)
    path = tmp_path / "cat.tle"
    path.write_text(text.replace("\n", "\r\n"))                 # CRLF file
    _same(read_catalog_columns(path).cpu().numpy(), host)


def test_field_edge_cases_bitwise():
    """Signs, empty and short fields, B* without exponent or sign, exponent
    '+', and records routed to the host decoder (non-ASCII names, a field
    with an exponent form, a tab)."""
    base1 = "1 25544U 98067A   24001.50000000  .00016717  00000-0  10270-3 0  9990"
    base2 = "2 25544  51.6416 247.4627 0006703 130.5360 325.0288 15.49815367 12345"
    variants = [
        (base1, base2),
        (base1[:53] + "-11606-4" + base1[61:], base2),
        (base1[:53] + " 12345+1" + base1[61:], base2),
        (base1[:53] + "  12345 " + base1[61:], base2),
        (base1[:53] + "        " + base1[61:], base2),
        (base1[:53] + "+00000+0" + base1[61:], base2),
        (base1, base2[:8] + "   51.64" + base2[16:]),
        (base1, base2[:8] + "+51.6416" + base2[16:]),
        (base1, base2[:26] + "   6703" + base2[33:]),
        (base1, base2[:26] + "       " + base2[33:]),
        (base1, base2[:52] + "  15.49815" + base2[62:]),
        (base1, base2[:17] + "    360." + base2[25:]),
        (base1, base2[:43] + "     -0." + base2[51:]),
        (base1, base2[:34] + "1.305e02" + base2[42:]),          # host path (exponent form)
        (base1, base2[:8] + "\t51.6416" + base2[16:]),           # host path (tab)
        (base1.rstrip(), base2.rstrip() + "   "),
    ]
    text = "".join(f"SAT {k} é\n{a}\n{b}\n" for k, (a, b) in enumerate(variants))
    _same(_gpu(text), _host(text))
    # a non-ASCII byte inside a record line goes to the host decoder, which
    # rejects it (byte and str columns would differ)
    bad = "NÄME\n" + base1.replace("25544U", "2554éU")[:69] + "\n" + base2 + "\n"
    for fn in (_host, _gpu):
        with pytest.raises(UnicodeEncodeError):
            fn(bad)


def test_layouts_and_errors():
    from paper_2603_27830_b200 import read_catalog_columns
    from paper_2603_27830_b200.tle import TleError
    a = "1 25544U 98067A   24001.50000000  .00016717  00000-0  10270-3 0  9990"
    b = "2 25544  51.6416 247.4627 0006703 130.5360 325.0288 15.49815367 12345"
    # blank line between line 1 and 2 (host path), bare CR endings, no final newline
    for text in (f"{a}\n\n{b}\n", f"{a}\r{b}\r", f"{a}\n{b}", f"X\n{b}\n{a}\n{b}\n"):
        _same(_gpu(text), _host(text))
    assert _gpu("just a name\n").shape == (7, 0)
    with pytest.raises(TleError):
        read_catalog_columns(f"{a}\n{a}\n{b}\n".encode())
    with pytest.raises(ValueError):
        read_catalog_columns(f"{a}\n{b[:26]}  -6703{b[33:]}\n".encode())


def test_ingest_feeds_init_batch():
    """Device columns go straight into init_batch; the batch equals the one
    built from the host columns."""
    import torch
    import paper_2603_27830_b200 as pkg
    text = (GOLDEN / "leo_corpus.tle").read_text()
    dev_cols = pkg.read_catalog_columns(text.encode())
    times = np.linspace(0.0, 1440.0, 33)
    a = pkg.propagate_batch(pkg.init_batch(dev_cols, precision=32), times)
    b = pkg.propagate_batch(pkg.init_batch(_host(text), precision=32), times)
    assert np.array_equal(a.planes, b.planes) and np.array_equal(a.error, b.error)
