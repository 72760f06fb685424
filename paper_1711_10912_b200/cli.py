"""Command-line front end for the hot path: ``hopm`` on a tensor JSON file.

Mirrors the reference's ``tensorlib hopm`` subcommand (cli.py:139-164): the
tensor file is the reference's JSON interchange format (tensor.py:252-271),
the run is the device HOPM, and the exit status is 0 when converged, 2 when
the sweep limit was reached, 3 on degenerate input, 1 on unreadable input
and 64 on usage errors (cli.py:26-30).

    python -m paper_1711_10912_b200 hopm --in t.json [--sweeps 50] [--tol 1e-10] [--json]
"""

from __future__ import annotations

import argparse
import json
import sys

EXIT_OK, EXIT_FAIL, EXIT_NOT_CONVERGED, EXIT_DEGENERATE, EXIT_USAGE = 0, 1, 2, 3, 64


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


def _parser() -> _Parser:
    p = _Parser(prog="paper_1711_10912_b200", description=__doc__)
    sub = p.add_subparsers(dest="command", required=True)
    h = sub.add_parser("hopm", help="best rank-one approximation on the GPU")
    h.add_argument("--in", dest="input", required=True, help="tensor JSON file")
    h.add_argument("--sweeps", type=int, default=50)
    h.add_argument("--tol", type=float, default=1e-10)
    h.add_argument("--json", action="store_true")
    return p


def _load(path):
    from .tensor import DenseTensor

    try:
        with open(path) as fh:
            obj = json.load(fh)
    except OSError as exc:
        print(f"paper_1711_10912_b200: cannot read {path}: {exc}", file=sys.stderr)
        raise SystemExit(EXIT_FAIL)
    except json.JSONDecodeError as exc:
        print(f"paper_1711_10912_b200: parse error in {path}: line {exc.lineno} column {exc.colno}: {exc.msg}",
              file=sys.stderr)
        raise SystemExit(EXIT_FAIL)
    try:
        t = DenseTensor.from_dict(obj)
    except ValueError as exc:
        print(f"paper_1711_10912_b200: invalid tensor in {path}: {exc}", file=sys.stderr)
        raise SystemExit(EXIT_FAIL)
    return t if t.dtype.is_floating_point else t.to("float64")


def _cmd_hopm(args) -> int:
    from .hopm import DegenerateInputError, hopm, residual

    t = _load(args.input)
    try:
        state = hopm(t, max_sweeps=args.sweeps, tol=args.tol)
    except DegenerateInputError as exc:
        print(f"paper_1711_10912_b200: degenerate input: {exc}", file=sys.stderr)
        return EXIT_DEGENERATE
    res = residual(t, state)
    if args.json:
        print(json.dumps({"converged": state.converged, "sweeps": state.sweeps, "scale": state.scale,
                          "lambda_history": state.lambda_history, "residual": res,
                          "vectors": [u.data for u in state.u]}, indent=2))
    else:
        for k, lam in enumerate(state.lambda_history, start=1):
            print(f"sweep {k}: lambda = {lam!r}")
        print(f"converged: {'yes' if state.converged else 'no'}")
        print(f"residual: {res!r}")
        for r, u in enumerate(state.u, start=1):
            print(f"u{r} = {u.data!r}")
    return EXIT_OK if state.converged else EXIT_NOT_CONVERGED


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    if args.command == "hopm":
        return _cmd_hopm(args)
    return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
