"""The sgp4kit CLI contract (reference cli.py; tests pkg/tests/test_cli.py)
on the drop-in, against the reference CLI's own output for the same
command line (tests/golden/ref_cli_batch_*, made by make_golden.py)."""

from __future__ import annotations

import io

import numpy as np
import pytest

from paper_2603_27830_b200 import read_grid_binary
from paper_2603_27830_b200.cli import EXIT_OK, EXIT_PARSE, EXIT_USAGE, main

from .conftest import GOLDEN

REAL = str(GOLDEN / "real_tles.tle")


def read_csv_rows(text: str):
    lines = text.strip().splitlines()
    return lines[0], [ln.split(",") for ln in lines[1:]]


# ---- CPU: argument handling and exit codes (nothing reaches the GPU) -------

def test_unknown_subcommand_is_usage_error():
    assert main(["orbit"]) == EXIT_USAGE


@pytest.mark.parametrize("argv", [
    ["propagate", REAL],                                               # no time flag
    ["propagate", REAL, "--tsince", "0:60:10", "--tsince-list", "0"],  # two flags
    ["propagate", REAL, "--tsince", "0:60"],
    ["propagate", REAL, "--tsince", "0:60:-5"],
    ["batch", REAL, "--tsince-list", "0", "--format", "csvx"],
    ["batch", REAL, "--tsince-list", "0", "--precision", "16"],
])
def test_usage_errors(argv, capsys):
    assert main(argv) == EXIT_USAGE
    assert "usage error" in capsys.readouterr().err


def test_jacobian_is_out_of_scope_usage_error(capsys):
    assert main(["jacobian", REAL, "--tsince", "60"]) == EXIT_USAGE
    assert "not part of this GPU drop-in" in capsys.readouterr().err


def test_parse_errors(tmp_path, capsys):
    bad = tmp_path / "bad.tle"
    bad.write_text("1 25544U\n2 99999\n")
    assert main(["propagate", str(bad), "--tsince-list", "0"]) == EXIT_PARSE
    assert "parse error" in capsys.readouterr().err
    empty = tmp_path / "empty.tle"
    empty.write_text("\n")
    assert main(["propagate", str(empty), "--tsince-list", "0"]) == EXIT_PARSE


def test_strict_checksum_is_parse_error(tmp_path):
    rows = [ln for ln in (GOLDEN / "real_tles.tle").read_text().splitlines() if ln]
    l1, l2 = rows[1], rows[2]
    bad = l1[:68] + str((int(l1[68]) + 1) % 10)
    path = tmp_path / "c.tle"
    path.write_text(bad + "\n" + l2 + "\n")
    assert main(["propagate", str(path), "--tsince-list", "0", "--strict"]) == EXIT_PARSE


# ---- GPU: the outputs -------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("precision", [32, 64])
def test_batch_binary_matches_reference_cli(tmp_path, precision):
    """`batch --format binary` from the device: same header and length as
    the reference CLI's file, identical code plane, planes within the bar."""
    out = tmp_path / "g.bin"
    assert main(["batch", REAL, "--tsince", "0:1500:300", "--precision", str(precision),
                 "--format", "binary", "--out", str(out)]) == EXIT_OK
    raw = out.read_bytes()
    ref_raw = (GOLDEN / f"ref_cli_batch_{precision}.bin").read_bytes()
    assert raw[:32] == ref_raw[:32] and len(raw) == len(ref_raw)
    got = read_grid_binary(io.BytesIO(raw))
    ref = read_grid_binary(io.BytesIO(ref_raw))
    ref64 = read_grid_binary(io.BytesIO((GOLDEN / "ref_cli_batch_64.bin").read_bytes()))
    assert np.array_equal(got.error, ref.error)
    ok = ref.error == 0
    tol = 1e-6 if precision == 64 else 0.1
    assert np.abs(got.planes[:, ok].astype(np.float64) - ref64.planes[:, ok]).max() <= tol


@pytest.mark.gpu
def test_batch_csv_matches_reference_cli(tmp_path):
    out = tmp_path / "b.csv"
    assert main(["batch", REAL, "--tsince-list", "0,90.5,1440,-60", "--out", str(out)]) == EXIT_OK
    head, rows = read_csv_rows(out.read_text())
    ref_head, ref_rows = read_csv_rows((GOLDEN / "ref_cli_batch_64.csv").read_text())
    assert head == ref_head and len(rows) == len(ref_rows)
    for a, b in zip(rows, ref_rows):
        assert a[0] == b[0] and a[7] == b[7]                      # time text, code
        if b[7] == "0":
            assert max(abs(float(x) - float(y)) for x, y in zip(a[1:4], b[1:4])) < 1e-6
            assert max(abs(float(x) - float(y)) for x, y in zip(a[4:7], b[4:7])) < 1e-9


@pytest.mark.gpu
def test_propagate_is_first_record_of_batch_and_stdout_is_csv(tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert main(["batch", REAL, "--tsince", "0:120:60", "--out", str(out)]) == EXIT_OK
    _, batch_rows = read_csv_rows(out.read_text())
    assert main(["propagate", REAL, "--tsince", "0:120:60"]) == EXIT_OK
    head, single_rows = read_csv_rows(capsys.readouterr().out)
    assert head == "tsince_min,rx,ry,rz,vx,vy,vz,error_code"
    assert batch_rows[:2] == single_rows


@pytest.mark.gpu
def test_utc_list_resolves_against_epoch(tmp_path):
    out = tmp_path / "p.csv"
    assert main(["propagate", REAL, "--utc-list", "2020-12-10T22:00:01",
                 "--out", str(out)]) == EXIT_OK
    _, rows = read_csv_rows(out.read_text())
    assert float(rows[0][0]) == pytest.approx(1440.0, abs=0.1)


@pytest.mark.gpu
def test_precision_report_shape(tmp_path):
    out = tmp_path / "d.csv"
    assert main(["precision-report", REAL, "--horizon-days", "1", "--step-minutes", "360",
                 "--out", str(out)]) == EXIT_OK
    head, rows = read_csv_rows(out.read_text())
    assert head.split(",")[0] == "day" and len(rows) == 5


@pytest.mark.gpu
def test_bench_command_emits_records(tmp_path):
    out = tmp_path / "bench.csv"
    assert main(["bench", REAL, "--axis", "satellites", "--sizes", "1,2", "--fixed", "4",
                 "--propagate-only", "--out", str(out)]) == EXIT_OK
    head, rows = read_csv_rows(out.read_text())
    assert head.split(",")[0] == "label" and len(rows) == 2
