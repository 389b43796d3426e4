"""``mlq`` command line: the reference's subcommands over the GPU engine.

Same contract as the reference CLI (pkg/src/mlq_sssp/cli.py): every subcommand prints one
JSON object; errors print ``{"error": {"type", "message"}}`` and exit 2 (cli.py:79-84,
576-579); ``verify`` exits 1 on a mismatch.  Config precedence for solve/verify is
explicit queue flags > trained selector (``--model`` / ``--auto`` with ``$MLQ_MODEL``) >
the rule list (cli.py:248-260).  Distances are inlined (``null`` = unreachable) up to
``--max-inline-distances`` vertices, otherwise written to a ``.distances.u64`` sidecar
(little-endian u64, all-ones = unreachable, engine.py:385-387).

B200 differences: ``--num-groups`` keeps the reference default ($MLQ_NUM_GROUPS or 4, one
warp per group) and also takes ``auto`` (every warp the device keeps resident, resolved to
an integer before any config is emitted, so the schemas stay valid); ``--device`` picks the
GPU; ``solve`` reports the device time next to the reference's metrics.

    python -m paper_2602_10080_b200.cli solve --gen rmat:16,16,1,255 --source 0
    python -m mlq_sssp.cli verify --gen grid2d:64x64,1,100 --l1 filter --l2 bucket
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import asdict
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import __version__
from .adaptive import (SelectorModel, benchmark_graphs, enumerate_candidates, read_records_csv,
                       select_config, select_rule_based, train_selector, write_records_csv)
from .core import L1_TYPES, L2_TYPES, EngineError, MlmqConfig
from .engine import (EngineConfig, compare_distances, dijkstra_oracle, distances_blob,
                     sssp_solve, unit_weight_view)
from .graph import CsrGraph, extract_features, generate_graph, load_graph, save_graph

ENV_NUM_GROUPS = "MLQ_NUM_GROUPS"
ENV_MODEL = "MLQ_MODEL"
EXIT_OK, EXIT_MISMATCH, EXIT_ERROR = 0, 1, 2
MAX_INLINE = 1_000_000

# flag name -> (config object path) for explicit queue configuration
_QUEUE_FLAGS = {
    "l1": ("l1_type",), "l2": ("l2_type",), "l0_capacity": ("l0_capacity",),
    "wb": ("l1_params", "wb"), "delta_nf": ("l1_params", "delta_nf"),
    "filter_f": ("l1_params", "filter_f"), "l1_capacity": ("l1_params", "capacity"),
    "delta": ("l2_params", "delta"), "block_size": ("l2_params", "block_size"),
    "block_num": ("l2_params", "block_num"), "bmax": ("l2_params", "bmax"),
    "bnum": ("l2_params", "bnum"), "node_batch": ("l2_params", "node_batch"),
    "pnum": ("l2_params", "pnum"),
}


def parse_gen_spec(spec: str) -> Tuple[str, dict]:
    """``path:N[,wmin,wmax]``, ``grid2d:RxC[,wmin,wmax]``, ``uniform:N,M[,wmin,wmax]``,
    ``rmat:SCALE[,EF[,wmin,wmax]]`` (cli.py:91-124 shorthand)."""
    kind, _, rest = spec.partition(":")
    kind = kind.strip()
    a = [x.strip() for x in rest.split(",")] if rest else []
    w = {}
    try:
        if kind == "path":
            p, tail = {"n": int(a[0])}, a[1:]
        elif kind == "grid2d":
            r, _, c = a[0].partition("x")
            p, tail = {"rows": int(r), "cols": int(c)}, a[1:]
        elif kind == "uniform":
            p, tail = {"n": int(a[0]), "m": int(a[1])}, a[2:]
        elif kind == "rmat":
            p = {"scale": int(a[0])}
            if len(a) >= 2:
                p["edge_factor"] = int(a[1])
            tail = a[2:]
        else:
            raise ValueError(f"unknown generator {kind!r}; expected path, grid2d, uniform or rmat")
        if len(tail) >= 2:
            w = {"wmin": int(tail[0]), "wmax": int(tail[1])}
    except (IndexError, ValueError) as exc:
        if "unknown generator" in str(exc):
            raise
        raise ValueError(f"bad generator spec {spec!r}: {exc}") from exc
    p.update(w)
    return kind, p


def _emit(obj: dict, out: Optional[str] = None) -> None:
    text = json.dumps(obj, indent=2)
    if not out:
        print(text)
        return
    with open(out, "w", encoding="utf-8") as fh:
        fh.write(text + "\n")
    brief = {k: obj[k] for k in ("subcommand", "graph") if k in obj}
    brief["out"] = out
    print(json.dumps(brief, indent=2))


def _load(args) -> Tuple[CsrGraph, dict]:
    if bool(args.graph) == bool(args.gen):
        raise ValueError("exactly one of --graph or --gen is required")
    if args.graph:
        g = load_graph(args.graph, fmt=args.format, weight_scale=args.weight_scale)
        origin = {"file": args.graph}
    else:
        kind, params = parse_gen_spec(args.gen)
        g = generate_graph(kind, seed=args.gen_seed, **params)
        origin = {"gen": args.gen, "gen_seed": args.gen_seed}
    origin.update(num_vertices=g.num_vertices, num_edges=g.num_edges)
    return g, origin


def _num_groups_arg(text: str):
    """--num-groups: a positive integer, or ``auto`` (every warp the device keeps resident)."""
    if str(text).strip().lower() == "auto":
        return "auto"
    return int(text)


def _groups(args, default=None):
    """cli.py:195-201: explicit flag, else $MLQ_NUM_GROUPS, else the reference's 4.
    ``auto`` becomes None here and is resolved to an integer against the device."""
    v = args.num_groups
    if v is None:
        v = os.environ.get(ENV_NUM_GROUPS) or (4 if default is None else default)
    return None if str(v).strip().lower() == "auto" else int(v)


def _concrete(cfg: MlmqConfig, g: CsrGraph, feats, args) -> MlmqConfig:
    """Resolve ``auto`` groups to the device's integer so emitted configs stay
    schema-valid (common.schema.json:63,73 require an integer)."""
    if cfg.num_groups is not None:
        return cfg
    from .engine import prepare
    resolved, _, _, _ = prepare(g, 0, cfg, EngineConfig(device=getattr(args, "device", 0)), features=feats)
    return resolved


def _explicit(args) -> Optional[MlmqConfig]:
    if all(getattr(args, f) is None for f in _QUEUE_FLAGS):
        return None
    cfg = MlmqConfig(num_groups=_groups(args))
    for flag, path in _QUEUE_FLAGS.items():
        v = getattr(args, flag)
        if v is None:
            continue
        obj = cfg
        for part in path[:-1]:
            obj = getattr(obj, part)
        setattr(obj, path[-1], v)
    return cfg


def _model_path(args) -> Optional[str]:
    return args.model or (os.environ.get(ENV_MODEL) if args.auto else None)


def _pick(args, feats) -> Tuple[MlmqConfig, str]:
    cfg = _explicit(args)
    if cfg is not None:
        return cfg, "explicit"
    path = _model_path(args)
    if path:
        ranked = select_config(feats, enumerate_candidates(), SelectorModel.load(path))
        return ranked[0][0].bind(feats, num_groups=_groups(args)), "model"
    return select_rule_based(feats).bind(feats, num_groups=_groups(args)), "rule_based"


def _engine(args) -> EngineConfig:
    return EngineConfig(num_groups=_groups(args), lanes_per_group=args.lanes, th_v=args.th_v,
                        duplicate_elimination=not args.no_dup_elim, seed=args.seed,
                        device=args.device)


def _run(args):
    g, origin = _load(args)
    feats = extract_features(g)
    cfg, src = _pick(args, feats)
    res = sssp_solve(g, args.source, cfg, _engine(args), features=feats,
                     unit_weights=args.unit_weights, watchdog_s=args.watchdog)
    eng = asdict(res.engine_used)
    out = {"version": __version__, "graph": origin, "source": args.source, "config_source": src,
           "config": res.config_used.to_json_dict(), "engine": eng,
           "unit_weights": args.unit_weights, "metrics": res.metrics.to_json_dict()}
    return g, res, out


def cmd_gen(args) -> int:
    kind, params = parse_gen_spec(args.spec)
    g = generate_graph(kind, seed=args.gen_seed, **params)
    save_graph(g, args.out, fmt=args.format)
    _emit({"subcommand": "gen", "spec": args.spec, "gen_seed": args.gen_seed, "path": args.out,
           "num_vertices": g.num_vertices, "num_edges": g.num_edges})
    return EXIT_OK


def cmd_features(args) -> int:
    g, origin = _load(args)
    _emit({"subcommand": "features", "graph": origin,
           "features": extract_features(g).to_json_dict()}, args.out)
    return EXIT_OK


def cmd_solve(args) -> int:
    g, res, out = _run(args)
    out["subcommand"] = "solve"
    d = res.dist_array
    reach = int(np.count_nonzero(np.isfinite(d))) if d.dtype == np.float32 else \
        int(np.count_nonzero(d != np.uint64(0xFFFFFFFFFFFFFFFF)))
    if args.report_device:  # timing varies run to run: opt-in (test_cli.py:171-179)
        out["device"] = {"kernel_ms": res.kernel_ms, "num_groups": res.native["num_groups"],
                         "dist_bits": res.native["dist_bits"], "reached_vertices": reach}
    if g.num_vertices <= args.max_inline_distances:
        out["distances"] = _inline(d)
    else:
        base = os.path.splitext(args.out)[0] if args.out else f"solve.s{args.source}"
        side = base + ".distances.u64"
        with open(side, "wb") as fh:
            fh.write(distances_blob(d) if d.dtype != np.float32 else d.astype("<f4").tobytes())
        out["distances_file"] = side
        out["distances_format"] = ("uint64 little-endian, all-ones is unreachable" if d.dtype != np.float32
                                   else "float32 little-endian, +inf is unreachable")
    _emit(out, args.out)
    return EXIT_OK


def _inline(d: np.ndarray) -> List[Optional[float]]:
    if d.dtype == np.float32:
        return [None if not np.isfinite(x) else float(x) for x in d]
    return [None if x == 0xFFFFFFFFFFFFFFFF else int(x) for x in d.tolist()]


def cmd_verify(args) -> int:
    g, res, out = _run(args)
    out["subcommand"] = "verify"
    want = dijkstra_oracle(unit_weight_view(g) if args.unit_weights else g, args.source)
    got = res.dist_array.tolist() if res.dist_array.dtype != np.float32 else list(res.dist_array)
    mm = compare_distances(got, want)
    out["match"] = mm is None
    if mm is not None:
        out["mismatch"] = {"vertex": mm[0], "engine": mm[1], "oracle": mm[2]}
    _emit(out, args.out)
    return EXIT_OK if mm is None else EXIT_MISMATCH


def cmd_select(args) -> int:
    g, origin = _load(args)
    feats = extract_features(g)
    path = _model_path(args)
    model = SelectorModel.load(path) if path else None
    ranked = select_config(feats, enumerate_candidates(), model)
    top = ranked[:args.top] if args.top else ranked
    out = {"subcommand": "select", "graph": origin, "features": feats.to_json_dict(),
           "selector": "model" if model is not None else "rule_based",
           "ranking": [{"rank": i + 1, "candidate": asdict(c), "score": s, "label": c.label()}
                       for i, (c, s) in enumerate(top)],
           "bound_config": _concrete(ranked[0][0].bind(feats, num_groups=_groups(args)), g, feats,
                                     args).to_json_dict()}
    if model is not None:
        out["model"] = {"path": path, "corpus_hash": model.corpus_hash, "trees": len(model.trees)}
    _emit(out, args.out)
    return EXIT_OK


def _csv_list(text, conv=str):
    return None if text is None else [conv(x.strip()) for x in text.split(",") if x.strip()]


def cmd_bench(args) -> int:
    """cli.py:457-534: time a candidate grid over --graph/--gen inputs into a records CSV.
    The GPU engine records the device time of each solve (``timing``)."""
    graphs = [(path, load_graph(path, fmt=args.format, weight_scale=args.weight_scale))
              for path in (args.graph or [])]
    for spec in args.gen or []:
        kind, params = parse_gen_spec(spec)
        graphs.append((f"{spec}@{args.gen_seed}", generate_graph(kind, seed=args.gen_seed, **params)))
    if not graphs:
        raise ValueError("bench needs at least one --graph or --gen")
    grid = {k: v for k, v in (("l1", _csv_list(args.grid_l1)), ("l2", _csv_list(args.grid_l2)),
                              ("delta_scale", _csv_list(args.delta_scales, float)),
                              ("wb", _csv_list(args.wb_list, int))) if v}
    cands = enumerate_candidates(grid or None)
    if not cands:
        raise ValueError("the candidate grid is empty")
    groups = _groups(args, default=1)
    recs = benchmark_graphs(graphs, cands, source=args.source, reps=args.reps, num_groups=groups,
                            watchdog_s=args.watchdog, timing=args.timing)
    write_records_csv(recs, args.out)
    best = {}
    for r in recs:
        if r.graph_id not in best or r.wall_time_us < best[r.graph_id]["wall_time_us"]:
            best[r.graph_id] = {"label": r.label(), "wall_time_us": r.wall_time_us}
    # figures need matplotlib (absent in this image); the record CSV carries the data
    _emit({"subcommand": "bench", "records": args.out, "rows": len(recs), "graphs": len(graphs),
           "candidates": len(cands), "reps": args.reps, "source": args.source,
           "num_groups": groups if groups is not None else
           _concrete(cands[0].bind(extract_features(graphs[0][1]), num_groups=None), graphs[0][1],
                     extract_features(graphs[0][1]), args).num_groups,
           "figures": [], "best_per_graph": best, "timing": args.timing})
    return EXIT_OK


def cmd_train(args) -> int:
    recs = read_records_csv(args.records)
    model = train_selector(recs, seed=args.seed, n_trees=args.trees, max_depth=args.depth,
                           min_leaf=args.min_leaf)
    model.save(args.out)
    _emit({"subcommand": "train", "records": args.records, "rows": len(recs),
           "graphs": len({r.graph_id for r in recs}),
           "configs": len({tuple(r.encoding) for r in recs}), "model": args.out,
           "trees": len(model.trees), "seed": args.seed, "corpus_hash": model.corpus_hash})
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    """The reference's subcommands and flags (cli.py:541-611), plus ``--device`` and
    ``--num-groups auto``."""
    ap = argparse.ArgumentParser(prog="mlq", description="MLMQ SSSP on B200 (reference-compatible CLI)")
    ap.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = ap.add_subparsers(dest="subcommand", required=True)

    def inputs(p):
        p.add_argument("--graph", help="graph file (.gr DIMACS or .mtx Matrix Market)")
        p.add_argument("--format", choices=("dimacs", "mm"))
        p.add_argument("--gen", help="generator spec, e.g. path:1000 or grid2d:30x40,1,100")
        p.add_argument("--gen-seed", type=int, default=0)
        p.add_argument("--weight-scale", type=int, default=1000)
        p.add_argument("--device", type=int, default=0, help="CUDA device (B200 extension)")

    def queue(p):
        p.add_argument("--l1", choices=L1_TYPES)
        p.add_argument("--l2", choices=L2_TYPES)
        for f in ("wb", "delta", "delta-nf", "filter-f", "l1-capacity", "l0-capacity", "block-size",
                  "block-num", "bmax", "bnum", "node-batch", "pnum"):
            p.add_argument("--" + f, type=int)
        p.add_argument("--auto", action="store_true", help=f"rank the grid with ${ENV_MODEL}'s model")
        p.add_argument("--model")
        p.add_argument("--num-groups", type=_num_groups_arg,
                       help=f"worker groups (warps) or 'auto'; default ${ENV_NUM_GROUPS} or 4")
        p.add_argument("--lanes", type=int)
        p.add_argument("--th-v", type=int)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--no-dup-elim", action="store_true")
        p.add_argument("--watchdog", type=float, default=60.0)

    p = sub.add_parser("gen", help="generate a graph file")
    p.add_argument("spec")
    p.add_argument("--gen-seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p.add_argument("--format", choices=("dimacs", "mm"))
    p.set_defaults(fn=cmd_gen)

    p = sub.add_parser("features", help="print the eight selector features")
    inputs(p)
    p.add_argument("--out")
    p.set_defaults(fn=cmd_features)

    for name, fn in (("solve", cmd_solve), ("verify", cmd_verify)):
        p = sub.add_parser(name)
        inputs(p)
        queue(p)
        p.add_argument("--source", type=int, default=0)
        p.add_argument("--unit-weights", action="store_true")
        if name == "solve":
            p.add_argument("--max-inline-distances", type=int, default=MAX_INLINE)
            p.add_argument("--report-device", action="store_true",
                           help="add the device time / group count / distance width (B200 extension)")
        p.add_argument("--out")
        p.set_defaults(fn=fn)

    p = sub.add_parser("select", help="rank queue configs for an input")
    inputs(p)
    p.add_argument("--model")
    p.add_argument("--auto", action="store_true")
    p.add_argument("--num-groups", type=_num_groups_arg)
    p.add_argument("--top", type=int, default=3)
    p.add_argument("--out")
    p.set_defaults(fn=cmd_select)

    p = sub.add_parser("train", help="fit the selector on benchmark records")
    p.add_argument("--records", required=True)
    p.add_argument("--out", required=True, help="model file to write")
    p.add_argument("--trees", type=int, default=64)
    p.add_argument("--depth", type=int, default=6)
    p.add_argument("--min-leaf", type=int, default=2)
    p.add_argument("--seed", type=int, default=0)
    p.set_defaults(fn=cmd_train)

    p = sub.add_parser("bench", help="time a config grid over a graph corpus")
    p.add_argument("--graph", action="append")
    p.add_argument("--format", choices=("dimacs", "mm"))
    p.add_argument("--gen", action="append")
    p.add_argument("--gen-seed", type=int, default=0)
    p.add_argument("--weight-scale", type=int, default=1000)
    p.add_argument("--grid-l1")
    p.add_argument("--grid-l2")
    p.add_argument("--delta-scales")
    p.add_argument("--wb-list")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--source", type=int, default=0)
    p.add_argument("--num-groups", type=_num_groups_arg, help="worker groups while timing (default 1)")
    p.add_argument("--watchdog", type=float, default=60.0)
    p.add_argument("--no-figures", action="store_true")
    p.add_argument("--timing", choices=("wall", "kernel"), default="kernel",
                   help="record device time (default) or host wall time")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--out", required=True, help="records CSV to write")
    p.set_defaults(fn=cmd_bench)
    return ap


def main(argv: Optional[Sequence[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (EngineError, ValueError, OSError) as exc:  # cli.py:576-579
        print(json.dumps({"error": {"type": type(exc).__name__, "message": str(exc)}}, indent=2))
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
