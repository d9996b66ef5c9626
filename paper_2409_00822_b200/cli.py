"""The `run` and `gen` commands of the reference CLI
(/root/reference/pkg/src/rowtopk/cli.py:53-72,125-146,244-257) over the
GPU path: `run` streams an RTKM matrix file through the native file job
(io.topk_file: pread -> pinned -> device -> RTKR file) instead of
load_matrix -> batch_topk -> save_result, with the same result bytes.
Same arguments, messages and exit codes (0 ok, 1 validation, 3 i/o).  The
run manifest (manifest.py) and the analysis commands are outside the hot
path and not provided.

    python -m paper_2409_00822_b200 gen --rows 1048576 --cols 256 --out x.rtkm
    python -m paper_2409_00822_b200 run --matrix x.rtkm --k 32 --out r.rtkr
"""

from __future__ import annotations

import argparse
import os
import sys

from .batch import BatchConfig, _DeviceMatrix, resolve_workers
from .errors import BadMagicError, KOutOfRangeError, NaNInputError, RowTopKError, TruncatedFileError
from .experiments import DataGenSpec, generate_matrix
from .io import _read_header, load_matrix, save_matrix, topk_file
from .select import DEFAULT_HARD_CAP, SearchConfig

EXIT_OK = 0
EXIT_VALIDATION = 1
EXIT_IO = 3


class CliError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    # argparse exits with status 2 on bad flags; the reference reserves 2 for
    # verification failures and reports parse errors as validation errors
    # (cli.py:35-39).
    def error(self, message):
        raise CliError(message)


def _workers(text: str):
    return text if text == "auto" else int(text)


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="python -m paper_2409_00822_b200",
                description="row-wise top-k by binary threshold search (B200)")
    sub = p.add_subparsers(dest="command", required=True)
    g = sub.add_parser("gen", help="write a seeded std-normal matrix file")
    g.add_argument("--rows", type=int, required=True)
    g.add_argument("--cols", type=int, required=True)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--dist", choices=["std-normal"], default="std-normal")
    g.add_argument("--out", required=True)
    r = sub.add_parser("run", help="run batch top-k over a matrix file")
    r.add_argument("--matrix", required=True)
    r.add_argument("--k", type=int, required=True)
    r.add_argument("--mode", choices=["exact", "early-stop"], default="exact")
    r.add_argument("--epsilon-rel", type=float, default=0.0)
    r.add_argument("--max-iter", type=int, default=4)
    r.add_argument("--hard-cap", type=int, default=DEFAULT_HARD_CAP)
    r.add_argument("--workers", type=_workers, default="auto",
                   help="validated like the reference; the GPU path ignores the value")
    r.add_argument("--out", required=True)
    return p


def _cmd_gen(args) -> int:
    save_matrix(generate_matrix(DataGenSpec(args.rows, args.cols, seed=args.seed)), args.out)
    print(f"wrote {args.rows}x{args.cols} matrix to {args.out}")
    return EXIT_OK


def _cmd_run(args) -> int:
    # the reference's order (cli.py:136-146): the matrix file is opened and its
    # header checked first (i/o errors), then the search is configured, then
    # batch_topk validates NaN -> k -> workers (batch.py:106-112)
    with open(args.matrix, "rb") as fh:
        n_rows, n_cols = _read_header(fh, b"RTKM", args.matrix)
        if os.fstat(fh.fileno()).st_size < 24 + 4 * n_rows * n_cols:
            raise TruncatedFileError("unexpected end of file while reading matrix payload")
    if args.mode == "exact":
        search = SearchConfig.exact(epsilon_rel=args.epsilon_rel, hard_cap=args.hard_cap)
    else:
        search = SearchConfig.early_stop(max_iter=args.max_iter)
    try:
        resolve_workers(args.workers)
    except ValueError:
        # rare path: the workers error comes after the NaN and k checks
        x = load_matrix(args.matrix)
        r = _DeviceMatrix(x).first_nan_row()
        if r >= 0:
            raise NaNInputError(f"matrix contains NaN (first offending row: {r})") from None
        if not 1 <= args.k <= x.shape[1]:
            raise KOutOfRangeError(f"k must be in [1, {x.shape[1]}], got {args.k}") from None
        raise
    n, m = topk_file(args.matrix, args.out, BatchConfig(k=args.k, search=search))
    print(f"selected top-{args.k} of {n}x{m} -> {args.out}")
    return EXIT_OK


_COMMANDS = {"gen": _cmd_gen, "run": _cmd_run}


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return _COMMANDS[args.command](args)
    except CliError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except (BadMagicError, TruncatedFileError, OSError) as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (RowTopKError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION


def entry() -> None:
    sys.exit(main())
