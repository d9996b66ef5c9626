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
import sys

from .batch import BatchConfig
from .errors import BadMagicError, RowTopKError, TruncatedFileError
from .experiments import DataGenSpec, generate_matrix
from .io import save_matrix, topk_file
from .select import DEFAULT_HARD_CAP, SearchConfig

EXIT_OK = 0
EXIT_VALIDATION = 1
EXIT_IO = 3


def _workers(text: str):
    return text if text == "auto" else int(text)


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2409_00822_b200",
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
    r.add_argument("--workers", type=_workers, default="auto", help="accepted for compatibility (GPU path)")
    r.add_argument("--out", required=True)
    return p


def _cmd_gen(args) -> int:
    save_matrix(generate_matrix(DataGenSpec(args.rows, args.cols, seed=args.seed)), args.out)
    print(f"wrote {args.rows}x{args.cols} matrix to {args.out}")
    return EXIT_OK


def _cmd_run(args) -> int:
    if args.mode == "exact":
        search = SearchConfig.exact(epsilon_rel=args.epsilon_rel, hard_cap=args.hard_cap)
    else:
        search = SearchConfig.early_stop(max_iter=args.max_iter)
    n, m = topk_file(args.matrix, args.out, BatchConfig(k=args.k, search=search))
    print(f"selected top-{args.k} of {n}x{m} -> {args.out}")
    return EXIT_OK


_COMMANDS = {"gen": _cmd_gen, "run": _cmd_run}


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return _COMMANDS[args.command](args)
    except (BadMagicError, TruncatedFileError, OSError) as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (RowTopKError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION


def entry() -> None:
    sys.exit(main())
