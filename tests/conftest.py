"""Shared fixtures: the reference's own corpora (committed as golden TLE
files by tests/golden/make_golden.py), the CPU oracle, and GPU gating."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def read_tle_pairs(path: Path):
    rows = [ln for ln in path.read_text().splitlines() if ln.strip()]
    pairs, names, i = [], [], 0
    while i < len(rows):
        if rows[i].startswith("1 ") and i + 1 < len(rows) and rows[i + 1].startswith("2 "):
            names.append(rows[i - 1] if i > 0 and not rows[i - 1].startswith(("1 ", "2 ")) else "")
            pairs.append((rows[i], rows[i + 1]))
            i += 2
        else:
            i += 1
    return names, pairs


@pytest.fixture(scope="session")
def corpus_lines():
    """The reference's 1,200-record synthetic LEO catalogue (seed 20230101,
    pkg/tests/conftest.py:111-139)."""
    return read_tle_pairs(GOLDEN / "leo_corpus.tle")[1]


@pytest.fixture(scope="session")
def real_records():
    """name -> (line1, line2) for the reference's five real records
    (pkg/tests/conftest.py:73-92)."""
    names, pairs = read_tle_pairs(GOLDEN / "real_tles.tle")
    return dict(zip(names, pairs))


@pytest.fixture(scope="session")
def corpus_columns(corpus_lines):
    from paper_2603_27830_b200.tle import parse_catalog_columns
    return parse_catalog_columns([a for a, _ in corpus_lines], [b for _, b in corpus_lines])


@pytest.fixture(scope="session")
def real_elements(real_records):
    """Canonical elements of the near-Earth real records (ECCENTRIC excluded
    as in the reference fixture)."""
    from paper_2603_27830_b200 import parse_tle, tle_to_elements
    return {name: tle_to_elements(parse_tle(*pair)) for name, pair in real_records.items()
            if name != "ECCENTRIC"}


@pytest.fixture(scope="session")
def golden_states():
    """Reference propagate_batch output at both precisions for
    [ISS, STARLINK-1007, SSO, LOWPERIGEE] + the first 120 corpus records."""
    return {p: dict(np.load(GOLDEN / f"ref_states_{p}.npz")) for p in (32, 64)}


@pytest.fixture(scope="session")
def golden_columns(corpus_columns, real_records):
    from paper_2603_27830_b200 import parse_tle, tle_to_elements
    from paper_2603_27830_b200.tle import elements_to_columns
    near = [tle_to_elements(parse_tle(*real_records[k]))
            for k in ("ISS", "STARLINK-1007", "SSO", "LOWPERIGEE")]
    return np.concatenate([elements_to_columns(near), corpus_columns[:, :120]], axis=1)


@pytest.fixture(scope="session")
def failure_table():
    return json.loads((GOLDEN / "ref_failure_codes.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import sgp4_oracle
    return sgp4_oracle
