"""``elastik``-compatible command line on the GPU path.

Same subcommands, flags, output formats and exit codes as the reference CLI
(pkg/src/elastik/cli.py:116-340): ``dist`` prints one JSON object (exit 2 when the
result is abandoned), ``nn`` prints one JSON line per query and a JSON summary,
``subseq`` one JSON object, ``bench`` a CSV table across engine variants, ``gen`` a
synthetic dataset.  Usage and configuration errors exit 1.

Differences, all additive: ``--backend`` also takes ``cuda`` (the only backend
here), and ``--precision float32`` selects the optional FP32 engines for ``dist``
/ ``nn`` / ``bench``.  Every query of ``nn`` / ``bench`` goes to the GPU in one
batched call (``classify_1nn``), so ``--threads`` / ``ELASTIK_THREADS`` are
accepted and echoed but have no effect; per-query ``wall_s`` is the batch time
divided by the number of queries.

    python -m paper_2102_05221_b200.cli nn --kind cdtw --window 51 --train TRAIN.tsv --test TEST.tsv
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import os
import sys
import time

import numpy as np

from . import _backend, ingest
from ._lib import PRECISIONS
from .engines import VARIANTS, distance_batch
from .errors import ElastikError
from .kernels import KINDS, DistanceSpec, make_recurrence
from .search import LB_MODES, SearchConfig, classify_1nn, subsequence_search
from .series import LabeledDataset, gen_random_walk, load_tsv, write_tsv, znormalize


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage problems exit 1 (argparse would exit 2)
        self.print_usage(sys.stderr)
        self.exit(1, f"{self.prog}: error: {message}\n")


# ------------------------------------------------------------------ shared flags

_SPEC_FLAGS = (  # flag, DistanceSpec field, type
    ("--window", "window", int), ("--wdtw-g", "wdtw_g", float), ("--erp-gap", "erp_gap", float),
    ("--msm-c", "msm_c", float), ("--twe-nu", "twe_nu", float), ("--twe-lambda", "twe_lambda", float),
)


def _add_spec(p):
    g = p.add_argument_group("distance")
    g.add_argument("--kind", required=True, choices=KINDS)
    g.add_argument("--cost", choices=("squared", "absolute"), default="squared")
    for flag, _, typ in _SPEC_FLAGS:
        g.add_argument(flag, type=typ, default=None)
    p.add_argument("--delimiter", choices=("tab", "comma"), default="tab")
    p.add_argument("--backend", choices=("auto", "cuda", "compiled", "python"), default=None)


def _spec(args) -> DistanceSpec:
    return DistanceSpec(kind=args.kind, cost_mode=args.cost,
                        **{field: getattr(args, field) for _, field, _ in _SPEC_FLAGS})


def _echo(spec: DistanceSpec, args) -> dict:
    out = {"kind": spec.kind, "cost": spec.cost_mode, "window": spec.window}
    out.update({f: getattr(spec, f) for _, f, _ in _SPEC_FLAGS[1:] if getattr(spec, f) is not None})
    out.update(variant=getattr(args, "variant", None), lb=getattr(args, "lb", None),
               backend=_backend.resolve(args.backend))
    if getattr(args, "precision", "float64") != "float64":
        out["precision"] = args.precision
    return out


def _threads(value):
    if value is not None:
        return value
    env = os.environ.get("ELASTIK_THREADS")
    return int(env) if env else 1


def _load(path, args, znorm=False):
    """A dataset file into a page-locked packed batch (ingest.load_tsv_packed); --znorm runs
    series.znormalize on the device (DeviceSeries.znormalize, bit-identical)."""
    ds = ingest.load_tsv_packed(path, delimiter=args.delimiter)
    if znorm:
        if np.any(ds.lengths < 2):  # the reference's error, from its own check
            znormalize(ds.series(int(np.argmin(ds.lengths))))
        with ingest.DeviceSeries.upload(ds) as d, d.znormalize() as z:
            ds = ingest.pack(z.to_host(), ds.labels, ds.name)
    return ds


def _side(args, side):
    """--a "1,2,3" or --a-file F [--a-row k] (cli.py:77-89)."""
    inline, path, row = getattr(args, side), getattr(args, f"{side}_file"), getattr(args, f"{side}_row")
    if inline is not None:
        return [float(tok) for tok in inline.split(",") if tok.strip()]
    if path is None:
        raise ElastikError(f"provide --{side} or --{side}-file")
    ds = load_tsv(path, delimiter=args.delimiter)
    if row >= len(ds):
        raise ElastikError(f"--{side}-row {row} out of range for {path} ({len(ds)} rows)")
    return ds.entries[row][1]


# ------------------------------------------------------------------ commands

def cmd_dist(args) -> int:
    spec = _spec(args)
    rec = make_recurrence(spec, _side(args, "a"), _side(args, "b"))
    cutoff = math.inf if args.cutoff is None else args.cutoff
    # the distance() facade's window rule (engines.py:121-147): base without a window
    # runs the full matrix, every other variant the effective window
    if args.variant == "base" and spec.window is None:
        window = len(rec.lines)
    else:
        window = spec.window if args.variant == "base" else spec.effective_window(len(rec.lines))
    costs, cells = distance_batch(spec, args.variant, [(rec.lines, rec.cols)], cutoffs=[cutoff], windows=[window],
                                  backend=args.backend, precision=args.precision)
    cost = float(costs[0])
    abandoned = math.isinf(cost)
    print(json.dumps({"cost": "abandoned" if abandoned else cost, "cells_computed": int(cells[0]),
                      "config": _echo(spec, args)}))
    return 2 if abandoned else 0


def _classify(train, test, cfg):
    t0 = time.perf_counter()
    records = classify_1nn(train, test, cfg)
    wall = time.perf_counter() - t0
    n = len(records)
    summary = {
        "queries": n,
        "accuracy": sum(r.predicted == r.actual for r in records) / n if n else 0.0,
        "total_cells": sum(r.cells for r in records),
        "total_computed": sum(r.computed for r in records),
        "total_abandoned": sum(r.abandoned for r in records),
        "total_lb_skips": sum(r.lb_skips for r in records),
        "wall_s": wall,
    }
    return records, summary


def cmd_nn(args) -> int:
    spec = _spec(args)
    cfg = SearchConfig(spec=spec, variant=args.variant, lb=args.lb, backend=args.backend, precision=args.precision)
    train, test = _load(args.train, args, args.znorm), _load(args.test, args, args.znorm)
    t0 = time.perf_counter()
    records, summary = _classify(train, test, cfg)
    keys = ("query_index", "actual", "predicted", "nn_index", "nn_distance", "computed", "abandoned", "lb_skips",
            "cells", "wall_time")
    names = ("query",) + keys[1:-1] + ("wall_s",)
    for r in records:
        print(json.dumps({n: getattr(r, k) for n, k in zip(names, keys)}))
    summary.update(command="nn", train=args.train, test=args.test, seed=None, config=_echo(spec, args),
                   threads=_threads(args.threads), znorm=args.znorm, total_wall_s=time.perf_counter() - t0)
    print(json.dumps(summary))
    return 0


def cmd_subseq(args) -> int:
    spec = _spec(args)
    cfg = SearchConfig(spec=spec, variant=args.variant, lb=args.lb, normalize=args.normalize, backend=args.backend)
    query = load_tsv(args.query, delimiter=args.delimiter).entries[args.query_row][1]
    reference = load_tsv(args.reference, delimiter=args.delimiter).entries[args.reference_row][1]
    offset, dist, stats = subsequence_search(query, reference, cfg)
    print(json.dumps({
        "command": "subseq", "offset": offset, "distance": "abandoned" if math.isinf(dist) else dist,
        "windows": len(reference) - len(query) + 1, "computed": stats.computed, "abandoned": stats.abandoned,
        "lb_skips": stats.lb_skips, "cells": stats.cells, "wall_s": stats.wall_time, "config": _echo(spec, args),
    }))
    return 0


def cmd_bench(args) -> int:
    spec = _spec(args)
    if args.train and args.test:
        train, test = _load(args.train, args), _load(args.test, args)
    else:
        train = gen_random_walk(args.gen_train, args.gen_length, args.gen_classes, args.seed, name="bench-train")
        test = gen_random_walk(args.gen_test, args.gen_length, args.gen_classes, args.seed + 1, name="bench-test")
    variants = [v.strip() for v in args.variants.split(",") if v.strip()]
    bad = [v for v in variants if v not in VARIANTS]
    if bad:
        raise ElastikError(f"unknown variant {bad[0]!r}; expected one of {VARIANTS}")
    out = csv.writer(sys.stdout)
    out.writerow(["variant", "rep", "cells", "computed", "abandoned", "lb_skips", "accuracy", "wall_s",
                  "speedup_vs_base"])
    base_wall = {}
    for rep in range(args.reps):
        for v in variants:
            cfg = SearchConfig(spec=spec, variant=v, lb=args.lb, backend=args.backend, precision=args.precision)
            t0 = time.perf_counter()
            _, s = _classify(train, test, cfg)
            wall = time.perf_counter() - t0
            if v == "base":
                base_wall[rep] = wall
            speed = f"{base_wall[rep] / wall:.3f}" if rep in base_wall else ""
            out.writerow([v, rep, s["total_cells"], s["total_computed"], s["total_abandoned"], s["total_lb_skips"],
                          f"{s['accuracy']:.6f}", f"{wall:.6f}", speed])
    return 0


def cmd_gen(args) -> int:
    train = gen_random_walk(args.gen_train, args.gen_length, args.gen_classes, args.seed, name="generated-train")
    test = gen_random_walk(args.gen_test, args.gen_length, args.gen_classes, args.seed + 1, name="generated-test")
    write_tsv(train, args.out_train, delimiter=args.delimiter)
    write_tsv(test, args.out_test, delimiter=args.delimiter)
    print(json.dumps({"command": "gen", "train": args.out_train, "test": args.out_test, "train_count": len(train),
                      "test_count": len(test), "length": args.gen_length, "classes": args.gen_classes,
                      "seed": args.seed}))
    return 0


# ------------------------------------------------------------------ parser

def _gen_flags(p):
    p.add_argument("--gen-train", type=int, default=50)
    p.add_argument("--gen-test", type=int, default=50)
    p.add_argument("--gen-length", type=int, default=128)
    p.add_argument("--gen-classes", type=int, default=2)
    p.add_argument("--seed", type=int, default=7)


def build_parser() -> _Parser:
    parser = _Parser(prog="elastik", description=__doc__.split("\n\n")[0])
    sub = parser.add_subparsers(dest="command", required=True)
    prec = dict(choices=PRECISIONS, default="float64", help="float32: the optional FP32 engines")

    p = sub.add_parser("dist", help="one distance between two series")
    _add_spec(p)
    p.add_argument("--variant", choices=VARIANTS, default="base")
    for side in ("a", "b"):
        p.add_argument(f"--{side}", help="comma-separated values")
        p.add_argument(f"--{side}-file")
        p.add_argument(f"--{side}-row", type=int, default=0)
    p.add_argument("--cutoff", type=float, default=None)
    p.add_argument("--precision", **prec)
    p.set_defaults(func=cmd_dist)

    p = sub.add_parser("nn", help="1-NN classification of a test set")
    _add_spec(p)
    p.add_argument("--train", required=True)
    p.add_argument("--test", required=True)
    p.add_argument("--variant", choices=VARIANTS, default="eapruned")
    p.add_argument("--lb", choices=LB_MODES, default="none")
    p.add_argument("--znorm", action="store_true", help="z-normalize every series after loading")
    p.add_argument("--threads", type=int, default=None)
    p.add_argument("--precision", **prec)
    p.set_defaults(func=cmd_nn)

    p = sub.add_parser("subseq", help="best window of a reference series")
    _add_spec(p)
    p.add_argument("--query", required=True)
    p.add_argument("--query-row", type=int, default=0)
    p.add_argument("--reference", required=True)
    p.add_argument("--reference-row", type=int, default=0)
    p.add_argument("--variant", choices=VARIANTS, default="eapruned")
    p.add_argument("--lb", choices=LB_MODES, default="none")
    p.add_argument("--normalize", action="store_true")
    p.set_defaults(func=cmd_subseq)

    p = sub.add_parser("bench", help="timing table across engine variants")
    _add_spec(p)
    p.add_argument("--train")
    p.add_argument("--test")
    _gen_flags(p)
    p.add_argument("--variants", default="base,ea,eapruned,pruned_only")
    p.add_argument("--lb", choices=LB_MODES, default="none")
    p.add_argument("--reps", type=int, default=1)
    p.add_argument("--threads", type=int, default=None)
    p.add_argument("--precision", **prec)
    p.set_defaults(func=cmd_bench)

    p = sub.add_parser("gen", help="write a synthetic random-walk dataset")
    _gen_flags(p)
    p.add_argument("--out-train", required=True)
    p.add_argument("--out-test", required=True)
    p.add_argument("--delimiter", choices=("tab", "comma"), default="tab")
    p.set_defaults(func=cmd_gen)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except (ElastikError, ValueError, OSError, RuntimeError) as exc:  # RuntimeError: no GPU / library
        print(f"elastik: error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
