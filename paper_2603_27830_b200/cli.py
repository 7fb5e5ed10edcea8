"""Command-line front end with the reference's contract (sgp4kit cli.py).

Same subcommands, flags, stdout formats and exit codes as ``sgp4kit``
(cli.py:1-8, 40-88): stdout carries only CSV or SGB1 bytes, diagnostics go
to stderr, exit 0 ok / 1 usage / 2 TLE parse / 3 runtime; per-cell error
codes never change the exit code.

What differs is where the bytes come from.  ``batch --format binary`` keeps
the grid in HBM and streams it to the output through pinned staging blocks
(``write_grid_binary`` on a device result, batch.py:244-251 semantics): the
process never holds the N x M grid on the host.  ``jacobian`` (forward-mode
``Dual`` autodiff) is outside this drop-in's scope and exits
with a usage error naming the reference command to use instead.
"""

from __future__ import annotations

import argparse
import os
import sys
from typing import Callable

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_PARSE, EXIT_RUNTIME = 0, 1, 2, 3

CSV_HEADER = "tsince_min,rx,ry,rz,vx,vy,vz,error_code\n"


class UsageError(Exception):
    """Bad command line: exit code 1."""


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):            # argparse would sys.exit(2)
        raise UsageError(message)


def _workers_default():
    return int(os.environ.get("SGP4_BATCH_WORKERS", 0)) or None


def _add_io(p: argparse.ArgumentParser, with_times: bool = True) -> None:
    p.add_argument("input", help="TLE file")
    p.add_argument("--precision", type=int, choices=(32, 64), default=64)
    p.add_argument("--workers", type=int, default=_workers_default(),
                   help="accepted for compatibility; the GPU needs no pool")
    p.add_argument("--strict", action="store_true", help="error on TLE checksum mismatches")
    p.add_argument("--out", default="-", help="output path, '-' for stdout")
    if with_times:
        p.add_argument("--tsince", metavar="START:STOP:STEP",
                       help="minutes since epoch, stop exclusive")
        p.add_argument("--tsince-list", metavar="V1,V2,...", help="explicit minutes since epoch")
        p.add_argument("--utc-list", metavar="ISO1,ISO2,...",
                       help="absolute UTC times against the first record's epoch")


def build_parser() -> _ArgParser:
    root = _ArgParser(prog="sgp4b", description=__doc__.splitlines()[0])
    sub = root.add_subparsers(dest="command", required=True)
    _add_io(sub.add_parser("propagate", help="one TLE to one or more times"))
    b = sub.add_parser("batch", help="TLE file x time grid")
    _add_io(b)
    b.add_argument("--format", choices=("csv", "binary"), default="csv")
    j = sub.add_parser("jacobian", help="not provided by this drop-in")
    _add_io(j, with_times=False)
    j.add_argument("--tsince", type=float, default=0.0)
    d = sub.add_parser("precision-report", help="FP32 vs FP64 drift CSV")
    _add_io(d, with_times=False)
    d.add_argument("--horizon-days", type=float, default=14.0)
    d.add_argument("--step-minutes", type=float, default=90.0)
    s = sub.add_parser("bench", help="timing sweep CSV")
    s.add_argument("input")
    s.add_argument("--axis", choices=("satellites", "times"), default="satellites")
    s.add_argument("--sizes", required=True, metavar="S1,S2,...")
    s.add_argument("--fixed", type=int, default=1)
    s.add_argument("--precision", type=int, choices=(32, 64), default=64)
    s.add_argument("--workers", type=int, default=_workers_default())
    s.add_argument("--propagate-only", action="store_true")
    s.add_argument("--out", default="-")
    return root


def parse_times(args, elements) -> np.ndarray:
    """Exactly one of --tsince / --tsince-list / --utc-list (cli.py:90-117)."""
    from .kernel import epoch_to_julian
    from .tle import _iso_epoch_to_split

    chosen = [flag for flag in ("tsince", "tsince_list", "utc_list")
              if getattr(args, flag) is not None]
    if len(chosen) != 1:
        raise UsageError("exactly one of --tsince, --tsince-list, --utc-list is required")
    flag = chosen[0]
    if flag == "tsince":
        fields = args.tsince.split(":")
        if len(fields) != 3:
            raise UsageError("--tsince wants START:STOP:STEP")
        start, stop, step = map(float, fields)
        if not step > 0:
            raise UsageError("--tsince step must be positive")
        return np.arange(start, stop, step)
    if flag == "tsince_list":
        return np.array([float(v) for v in args.tsince_list.split(",")])
    first = elements[0]
    jd0 = epoch_to_julian(first.epoch_year, first.epoch_day_int, first.epoch_day_frac)
    out = []
    for stamp in args.utc_list.split(","):
        jd = epoch_to_julian(*_iso_epoch_to_split(stamp))
        out.append((jd - jd0) * 1440.0)
    return np.array(out)


def write_state_csv(times, result, out) -> None:
    """One row per (satellite, time), satellites outer (cli.py:120-127):
    time at 9 significant digits, state at 17, int code."""
    planes = np.asarray(result.planes)
    error = np.asarray(result.error)
    out.write(CSV_HEADER)
    for i in range(result.n):
        block = planes[:, i, :].T.tolist()           # (m, 6) Python floats
        codes = error[i].tolist()
        out.write("".join(
            f"{times[j]:.9g}," + ",".join(format(x, ".17g") for x in block[j]) + f",{codes[j]}\n"
            for j in range(result.m)))


class _Output:
    """--out target: '-' is stdout (text or its binary buffer)."""

    def __init__(self, path: str, binary: bool = False):
        self.path, self.binary = path, binary

    def __enter__(self):
        if self.path == "-":
            self.fh, self.own = (sys.stdout.buffer if self.binary else sys.stdout), False
        else:
            self.fh, self.own = open(self.path, "wb" if self.binary else "w"), True
        return self.fh

    def __exit__(self, *exc):
        if self.own:
            self.fh.close()
        else:
            self.fh.flush()
        return False


def _load_elements(args):
    from .tle import TleError, read_tle_file, tle_to_elements

    records = read_tle_file(args.input, strict=args.strict)
    if not records:
        raise TleError(f"no TLE records found in {args.input}")
    for rec in records:
        for note in rec.warnings:
            print(f"warning: catalog {rec.catalog_number}: {note}", file=sys.stderr)
    return [tle_to_elements(rec) for rec in records]


def cmd_propagate(args) -> int:
    from .batch import init_batch, propagate_batch

    elements = _load_elements(args)
    times = parse_times(args, elements)
    result = propagate_batch(init_batch(elements[:1], precision=args.precision), times)
    with _Output(args.out) as fh:
        write_state_csv(times, result, fh)
    return EXIT_OK


def cmd_batch(args) -> int:
    from .batch import (init_batch, propagate_batch, propagate_batch_device,
                        write_grid_binary)

    elements = _load_elements(args)
    times = parse_times(args, elements)
    sats = init_batch(elements, precision=args.precision)
    if args.format == "binary":
        result = propagate_batch_device(sats, times)       # grid stays in HBM
        with _Output(args.out, binary=True) as fh:
            write_grid_binary(result, fh)
    else:
        result = propagate_batch(sats, times)
        with _Output(args.out) as fh:
            write_state_csv(times, result, fh)
    return EXIT_OK


def cmd_jacobian(args) -> int:
    raise UsageError("jacobian (Dual forward-mode autodiff) is not part of this GPU drop-in; "
                     "run it with the reference package (sgp4kit jacobian)")


def cmd_precision_report(args) -> int:
    from .drift import drift_report, emit_report_csv

    report = drift_report(_load_elements(args), args.horizon_days, args.step_minutes)
    with _Output(args.out) as fh:
        fh.write(emit_report_csv(report))
    return EXIT_OK


def cmd_bench(args) -> int:
    from .timing import emit_bench_csv, scaling_sweep
    from .tle import read_tle_file, tle_to_elements

    records = scaling_sweep(axis=args.axis, sizes=[int(s) for s in args.sizes.split(",")],
                            fixed_other=args.fixed,
                            elements=[tle_to_elements(t) for t in read_tle_file(args.input)],
                            precision=args.precision, workers=args.workers or 1,
                            full_pipeline=not args.propagate_only)
    with _Output(args.out) as fh:
        fh.write(emit_bench_csv(records))
    return EXIT_OK


COMMANDS: dict[str, Callable] = {
    "propagate": cmd_propagate,
    "batch": cmd_batch,
    "jacobian": cmd_jacobian,
    "precision-report": cmd_precision_report,
    "bench": cmd_bench,
}


def main(argv=None) -> int:
    from .tle import TleError

    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return COMMANDS[args.command](args)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        parser.print_usage(sys.stderr)
        return EXIT_USAGE
    except TleError as exc:
        print(f"parse error: {exc}", file=sys.stderr)
        return EXIT_PARSE
    except BrokenPipeError:
        return EXIT_RUNTIME
    except Exception as exc:            # runtime failure: message, exit 3
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
