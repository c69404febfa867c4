"""Command line front end for the B200 path.

``python -m paper_2105_12026_b200 summarize data.csv -k K`` is the reference's
``ebcsum summarize`` (cli.py:229-327) with the ``b200`` backend: the same CSV
contract (rectangular, finite cells, optional header, optional population
z-score per column), the same e0 kinds, greedy or sieve optimizer, and the same
JSON document.  ``surrogate`` writes the injection-molding case-study matrix
(cli.py:111-173 contract) so C4-shaped inputs can be produced without the
reference.  Exit codes follow the reference's scripting contract (cli.py:1-6):
0 ok, 1 usage error, 2 data/configuration error, 3 internal error.  ``bench``
is the reference's N / l / k sweep (cli.py:252-267, 330-342; ``sweep.py``) with
the ``b200`` backend.  The reference's ``layout-audit`` (device-model
simulator) is out of scope.
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import sys
from typing import List, Optional

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_INTERNAL = 0, 1, 2, 3


class CsvParseError(ValueError):
    """A CSV cell or row that cannot be turned into finite numbers."""


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse exits 2; the contract says usage errors are 1
        raise _UsageError(message)


def load_csv(path: str, has_header: bool = False, normalize: bool = False):
    """Numeric matrix from CSV (reference load_csv contract, cli.py:59-108):
    blank lines skipped, rectangular rows, every cell a finite float; errors
    name the 1-based row (and column).  normalize: z-score with the population
    standard deviation, constant columns left at 0.  Returns (fp64 array, header)."""
    rows: List[List[float]] = []
    header: Optional[List[str]] = None
    width: Optional[int] = None
    with open(path, newline="") as fh:
        for line_no, row in enumerate(csv.reader(fh), start=1):
            if not row:
                continue
            if has_header and header is None:
                header = [tok.strip() for tok in row]
                continue
            if width is None:
                width = len(row)
            elif len(row) != width:
                raise CsvParseError(f"row {line_no}: expected {width} columns, got {len(row)}")
            vals = []
            for col_no, tok in enumerate(row, start=1):
                try:
                    x = float(tok)
                except ValueError:
                    raise CsvParseError(f"row {line_no}, column {col_no}: not a number: {tok.strip()!r}") from None
                if not math.isfinite(x):
                    raise CsvParseError(f"row {line_no}, column {col_no}: non-finite value {tok.strip()!r}")
                vals.append(x)
            rows.append(vals)
    if not rows:
        raise CsvParseError(f"{path}: no data rows")
    data = np.array(rows, dtype=np.float64)
    if normalize:
        mu, sd = data.mean(axis=0), data.std(axis=0)
        out = np.zeros_like(data)
        live = sd > 0
        out[:, live] = (data[:, live] - mu[live]) / sd[live]
        data = out
    return data, header


def _positive_int(text: str) -> int:
    v = int(text)
    if v < 1:
        raise argparse.ArgumentTypeError(f"expected an integer >= 1, got {text}")
    return v


def _int_list(text: str) -> List[int]:
    try:
        vals = [int(tok) for tok in text.split(",") if tok.strip()]
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}") from None
    if not vals:
        raise argparse.ArgumentTypeError("empty value list")
    return vals


def build_parser() -> argparse.ArgumentParser:
    from .core import Precision

    parser = _Parser(prog="paper_2105_12026_b200", description="Exemplar-based summarization on B200")
    sub = parser.add_subparsers(dest="command", required=True, parser_class=_Parser)
    p = sub.add_parser("summarize", help="select k representatives from a CSV")
    p.add_argument("input")
    p.add_argument("-k", type=_positive_int, required=True)
    p.add_argument("--optimizer", choices=("greedy", "sieve"), default="greedy")
    p.add_argument("--backend", choices=("b200",), default="b200")
    p.add_argument("--precision", choices=[m.value for m in Precision], default="fp64")
    p.add_argument("--e0-kind", choices=("zero", "mean"), default="zero")
    p.add_argument("--epsilon", type=float, default=0.1)
    p.add_argument("--seed", type=int, default=0, help="stream order seed (sieve)")
    # accepted for scripts written against the reference (cli.py:247); the device
    # evaluator has no host thread pool, so the value (and $EBCSUM_THREADS) is ignored
    p.add_argument("--threads", type=_positive_int, default=None, help="ignored by the b200 backend")
    p.add_argument("--header", action="store_true")
    p.add_argument("--normalize", action="store_true")
    p.add_argument("--output", default=None)
    p.set_defaults(func=cmd_summarize)
    p = sub.add_parser("bench", help="sweep one axis and report runtimes/speedups")
    p.add_argument("--axis", choices=("N", "l", "k"), default="N")
    p.add_argument("--values", type=_int_list, default=None, help="comma-separated axis values (defaults per axis)")
    p.add_argument("--n", type=_positive_int, default=50000)
    p.add_argument("--l", type=_positive_int, default=5000)
    p.add_argument("-k", type=_positive_int, default=10)
    p.add_argument("--dims", type=_positive_int, default=100)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--precision", choices=[m.value for m in Precision], default="fp32")
    p.add_argument("--backends", default="b200", help="comma list of name[:threads]")
    p.add_argument("--repeats", type=_positive_int, default=15)
    p.add_argument("--format", choices=("csv", "markdown"), default="csv")
    p.add_argument("--output", default=None)
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("surrogate", help="write the injection-molding surrogate as CSV")
    p.add_argument("--cycles", type=_positive_int, default=1000)
    p.add_argument("--dims", type=_positive_int, default=100)
    p.add_argument("--regimes", type=_positive_int, default=5)
    p.add_argument("--cycles-per-regime", type=_positive_int, default=200)
    p.add_argument("--noise", type=float, default=0.01)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--output", required=True)
    p.set_defaults(func=cmd_surrogate)
    return parser


def cmd_summarize(args) -> int:
    from .core import GroundMatrix, Precision, make_auxiliary_vector
    from .ebc import EbcFunction
    from .optimize import OptimizerBudget, greedy_maximize, sieve_stream_maximize

    data, _ = load_csv(args.input, has_header=args.header, normalize=args.normalize)
    precision = Precision.parse(args.precision)
    ground = GroundMatrix(data, precision)
    if args.k > ground.n:
        raise ValueError(f"k={args.k} exceeds the {ground.n} rows of {args.input}")
    e0 = make_auxiliary_vector(ground.dims, args.e0_kind, ground)
    f = EbcFunction(ground, e0)
    if args.optimizer == "greedy":
        summary = greedy_maximize(f, OptimizerBudget(k=args.k, backend=args.backend))
    else:
        stream = np.random.default_rng(args.seed).permutation(ground.n)
        summary = sieve_stream_maximize(stream, f, args.k, epsilon=args.epsilon)
    doc = {"k": args.k, "selected_indices": [int(i) for i in summary.selected],
           "function_value": summary.value, "gains": [float(g) for g in summary.gains],
           "backend": args.backend, "precision": precision.value, "runtime_seconds": summary.runtime_seconds}
    text = json.dumps(doc, indent=2) + "\n"
    if args.output:
        with open(args.output, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return EXIT_OK


def cmd_surrogate(args) -> int:
    from . import surrogate

    data_path, lp = surrogate.write(args.output, args.cycles, args.dims, args.regimes, args.cycles_per_regime,
                                    args.noise, args.seed)
    print(f"wrote {args.cycles}x{args.dims} surrogate to {data_path}")
    print(f"wrote regime labels to {lp}")
    return EXIT_OK


def cmd_bench(args) -> int:
    from .core import Precision
    from .sweep import DEFAULT_AXIS_VALUES, ProblemSpec, emit_report, run_sweep

    values = args.values if args.values else DEFAULT_AXIS_VALUES[args.axis]
    base = ProblemSpec(n=args.n, l=args.l, k=args.k, dims=args.dims, seed=args.seed,
                       precision=Precision.parse(args.precision))
    backends = [tok.strip() for tok in args.backends.split(",") if tok.strip()]
    report = run_sweep(args.axis, values, base, backends, repeats=args.repeats)
    text = emit_report(report, format=args.format)
    if args.output:
        with open(args.output, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return EXIT_OK


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except _UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except SystemExit as exc:  # --help
        return int(exc.code or 0)
    try:
        return args.func(args)
    except (ValueError, IndexError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DATA
    except Exception as exc:  # pragma: no cover - defensive
        print(f"internal error: {exc!r}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
