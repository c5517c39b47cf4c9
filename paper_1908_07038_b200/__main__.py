"""Command line for the hot path: ``python -m paper_1908_07038_b200 remap ...`` — the
reference's ``spheregrid remap`` subcommand (cli.py:157-173, 213-219): distributed remap of
an analytic field on the GPU, field dump of the gathered result, optional error report.
The reference's other subcommands (info, grid, mesh/Gmsh, partition) are out of scope."""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .errors import SpheregridError
from .field import Kind, create_field, dump_field
from .grid import grid_from_name
from .pipeline import run_remap_pipeline


def cmd_remap(args) -> int:
    gathered, analytic, messages = run_remap_pipeline(args.source, args.target, args.parts, args.field,
                                                      method=args.method, partitioner=args.partitioner)
    target = grid_from_name(args.target)
    out = create_field("remap", (target.npts, 1), Kind.REAL64)
    out.host[:, 0] = gathered
    with open(args.out, "w") as f:
        dump_field(out, np.arange(target.npts), f)
    if args.report:
        err = np.abs(gathered - analytic)
        print(f"max_error: {err.max():.17g}")
        print(f"rms_error: {np.sqrt(np.mean(err ** 2)):.17g}")
        print(f"messages_during_interpolation: {sum(messages)}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1908_07038_b200")
    sub = p.add_subparsers(dest="command", required=True)
    r = sub.add_parser("remap", help="remap an analytic field between grids (on the GPU)")
    r.add_argument("--source", required=True)
    r.add_argument("--target", required=True)
    r.add_argument("--parts", type=int, default=1)
    r.add_argument("--field", required=True)
    r.add_argument("--out", required=True)
    r.add_argument("--report", action="store_true")
    r.add_argument("--method", default="finite-element", choices=["finite-element", "structured-bilinear"])
    r.add_argument("--partitioner", default="blocks", choices=["blocks", "equal_regions"])
    r.set_defaults(func=cmd_remap)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except SpheregridError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
