"""Command line: the spec'd `emit` and `eval` subcommands.

    python -m paper_2410_23745_b200 emit --op OP_DOC [--assign K=V,...] [--staged] [--output FILE]
    python -m paper_2410_23745_b200 eval --op OP_DOC --input X.tensor [--weights W.tensor ...]
                                         --output Y.tensor [--assign K=V,...] [--staged]
                                         [--upstream DY.tensor --grad-input DX.tensor
                                          --grad-weights DW.tensor ...]

OP_DOC is an operator document (pgraph.print_operator's format).  Tensors
use the reference's binary format (codegen.save_tensor).  `emit` is pure
host code; `eval` runs the B200 kernels in float64 (no CPU fallback).
Exit codes follow the spec: 0 success, 2 configuration / input error,
3 execution (device) error.
"""
from __future__ import annotations

import argparse
import sys


def _assignment(text):
    if not text:
        return None
    out = {}
    for item in text.replace(";", ",").split(","):
        if item.strip():
            k, _, v = item.partition("=")
            out[k.strip()] = int(v)
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2410_23745_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    e = sub.add_parser("emit", help="write the loop nest of an operator")
    e.add_argument("--op", required=True)
    e.add_argument("--assign", default="")
    e.add_argument("--staged", action="store_true")
    e.add_argument("--output", default="-")
    v = sub.add_parser("eval", help="run an operator on tensors")
    v.add_argument("--op", required=True)
    v.add_argument("--input", required=True)
    v.add_argument("--weights", nargs="*", default=[])
    v.add_argument("--output", required=True)
    v.add_argument("--assign", default="")
    v.add_argument("--staged", action="store_true")
    v.add_argument("--upstream")
    v.add_argument("--grad-input")
    v.add_argument("--grad-weights", nargs="*", default=[])
    args = ap.parse_args(argv)

    from . import codegen as C
    from .errors import DeviceError, GraphError, OperatorParseError, ShapeMismatch
    from .pgraph import parse_operator
    try:
        with open(args.op) as f:
            graph = parse_operator(f.read())
        assignment = _assignment(args.assign)
    except (OSError, OperatorParseError, GraphError, ValueError, KeyError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    if args.cmd == "emit":
        text = C.emit_loop_nest(graph, assignment, args.staged)
        if args.output == "-":
            sys.stdout.write(text)
        else:
            with open(args.output, "w") as f:
                f.write(text)
        return 0
    try:
        x = C.load_tensor(args.input)
        ws = [C.load_tensor(p) for p in args.weights]
        dy = C.load_tensor(args.upstream) if args.upstream else None
    except (OSError, ShapeMismatch) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    try:
        C.save_tensor(args.output, C.interpret(graph, x, ws, assignment, args.staged))
        if dy is not None:
            dx, dws = C.gradients(graph, x, dy, ws, assignment)
            if args.grad_input:
                C.save_tensor(args.grad_input, dx)
            for path, g in zip(args.grad_weights, dws):
                C.save_tensor(path, g)
    except ShapeMismatch as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (DeviceError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
