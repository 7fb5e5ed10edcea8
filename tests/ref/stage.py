"""Stage the reference package's own test modules next to this directory's
conftest so they run, unmodified, against the drop-in (
SURVEY.md §8(b) "callers to re-point: the tests").

The files are copied from /root/reference/pkg/tests at build time (this
container; ``__graft_entry__.build()`` calls ``stage()``) into tests/ref/,
where .gitignore keeps them out of history — they are the reference's
sources, not this repo's — while the gpurun/driver snapshot carries them to
the GPU box, like oracle/_ref.  ``tests/ref/conftest.py`` (this repo's)
aliases ``sgp4kit`` to ``paper_2603_27830_b200`` and provides the fixtures
the reference conftest would.

Staged: the modules whose subject is on the hot path or its §8(f) callers.
Not staged (out of scope): test_dmath (the NumPy arithmetic
layer the CUDA kernels replace), test_jacobian / test_estimator (Dual
autodiff, sklearn wrapper), test_bench (the CPU benchmark harness).
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

REF_TESTS = Path("/root/reference/pkg/tests")
HERE = Path(__file__).resolve().parent
STAGED = ("test_batch.py", "test_kernel.py", "test_acceptance.py", "test_drift.py",
          "test_cli.py", "test_tle.py")


def stage(quiet: bool = True) -> list[Path]:
    """Copy the staged modules if the reference is mounted; returns the
    files present afterwards (an empty list on the GPU box is fine: the
    snapshot already carries them)."""
    if REF_TESTS.is_dir():
        for name in STAGED:
            src = REF_TESTS / name
            if src.exists():
                shutil.copyfile(src, HERE / name)
    present = [HERE / n for n in STAGED if (HERE / n).exists()]
    if not quiet:
        print(f"staged {len(present)} reference test modules into {HERE}", file=sys.stderr)
    return present


if __name__ == "__main__":
    stage(quiet=False)
