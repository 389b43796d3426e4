"""Config-5 sweep + selector retraining on GPU timings (BASELINE config 5).

    python tools/selector_sweep.py OUT_DIR

1. Times the reference's default 12-candidate grid (adaptive.py:153-157) plus the
   priority/multi L2 variants on a corpus of graphs with the GPU engine
   (``benchmark_graphs``, device time), the config-5 graph (power-law RMAT s24, f32
   U[0,1)) included.  Every solve is exact by construction; the records carry work
   counters too.
2. Writes the records CSV (adaptive.py:257-305 format).
3. Leave-one-graph-out evaluation of the selector (bagged trees, adaptive.py:527-577)
   trained on the GPU records, against the best fixed configuration and the reference's
   rule-based pick: mean relative performance (rp = best time / chosen time) and the
   share of graphs with rp >= 0.9 (the paper's coverage metric).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_10080_b200 import (ConfigCandidate, benchmark_graphs, enumerate_candidates,  # noqa: E402
                                   generate_graph, select_config, select_rule_based, train_selector,
                                   write_records_csv)
from paper_2602_10080_b200.graph import generate_grid2d, with_f32_weights  # noqa: E402


def corpus():
    g = []
    for s in (14, 16, 18, 20):
        g.append((f"rmat-s{s}", generate_graph("rmat", seed=1, scale=s, edge_factor=16, wmin=1, wmax=255)))
    for s in (16, 20):
        g.append((f"rmat-s{s}-f32", with_f32_weights(generate_graph("rmat", seed=2, scale=s, edge_factor=16), seed=3)))
    for side in (128, 512, 1024):
        g.append((f"grid-{side}", generate_grid2d(side, side, 1, 100, seed=1)))
    g.append(("grid-1024-road", generate_grid2d(1024, 1024, 10, 1000, seed=1)))
    g.append(("uniform-1M", generate_graph("uniform", seed=1, n=1 << 20, m=8 << 20, wmin=1, wmax=100)))
    g.append(("path-20k", generate_graph("path", seed=1, n=20000, wmin=1, wmax=9)))
    g.append(("C5-rmat-s24-f32", with_f32_weights(generate_graph("rmat", seed=1, scale=24, edge_factor=16), seed=1)))
    if os.environ.get("SWEEP_WIDE") == "1":  # round 2: large high-diameter meshes, road-like weights
        for side in (2048, 3000):
            g.append((f"grid-{side}", generate_grid2d(side, side, 1, 100, seed=2)))
            g.append((f"grid-{side}-road", generate_grid2d(side, side, 10, 1000, seed=2)))
        g.append(("grid-4096x256", generate_grid2d(4096, 256, 1, 100, seed=3)))
        g.append(("uniform-4M-deg4", generate_graph("uniform", seed=2, n=1 << 22, m=16 << 20, wmin=1, wmax=100)))
    return g


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    os.makedirs(out, exist_ok=True)
    cands = enumerate_candidates() + [ConfigCandidate(a, b) for a in ("vector", "slf")
                                      for b in ("priority", "multi")]
    graphs = corpus()
    recs = []
    t0 = time.time()
    for gid, g in graphs:
        cs = cands if g.num_edges <= (4 << 20) else enumerate_candidates()  # heaps on small graphs only
        try:
            r = benchmark_graphs([(gid, g)], cs, reps=3, num_groups=None, timing="kernel", watchdog_s=120)
        except Exception as e:  # noqa: BLE001
            print(f"{gid}: {type(e).__name__}: {e}", flush=True)
            continue
        recs.extend(r)
        best = min(r, key=lambda x: x.wall_time_us)
        print(f"{gid:18s} n={g.num_vertices:9d} m={g.num_edges:10d} best={best.label():24s} "
              f"{best.wall_time_us/1e3:9.3f} ms  ({time.time()-t0:.0f}s)", flush=True)
        for x in sorted(r, key=lambda x: x.wall_time_us):
            print(f"    {x.label():26s} {x.wall_time_us/1e3:9.3f} ms  rp={x.relative_performance:.3f} "
                  f"relax={x.relaxations}", flush=True)
    write_records_csv(recs, os.path.join(out, "selector_records.csv"))

    # leave-one-graph-out evaluation
    gids = sorted({r.graph_id for r in recs})
    summary = {"graphs": len(gids), "records": len(recs), "per_graph": {}}
    sel_rp, fix_rp, rule_rp = [], [], []
    for held in gids:
        train = [r for r in recs if r.graph_id != held]
        test = [r for r in recs if r.graph_id == held]
        model = train_selector(train, seed=0)
        feats = test[0].features
        test_cands = [r.candidate for r in test]
        rp = {r.candidate.label(): r.relative_performance for r in test}
        pick = select_config(feats, test_cands, model)[0][0].label()
        # best fixed config on the training graphs (mean rp)
        by = {}
        for r in train:
            by.setdefault(r.candidate.label(), []).append(r.relative_performance)
        fixed = max((k for k in by if k in rp), key=lambda k: float(np.mean(by[k])))
        rule = select_rule_based(feats).label()
        sel_rp.append(rp[pick])
        fix_rp.append(rp[fixed])
        rule_rp.append(rp.get(rule, 0.0))
        summary["per_graph"][held] = {"selected": pick, "rp_selected": rp[pick], "best_fixed": fixed,
                                      "rp_fixed": rp[fixed], "rule": rule, "rp_rule": rp.get(rule)}
        print(f"LOGO {held:18s} selected={pick:24s} rp={rp[pick]:.3f}  fixed={fixed:24s} rp={rp[fixed]:.3f}  "
              f"rule={rule} rp={rp.get(rule, 0):.3f}", flush=True)
    for name, v in (("selector", sel_rp), ("best_fixed", fix_rp), ("rule_based", rule_rp)):
        summary[name] = {"mean_rp": float(np.mean(v)), "coverage_rp_ge_0.9": float(np.mean(np.array(v) >= 0.9))}
    print(json.dumps({k: summary[k] for k in ("selector", "best_fixed", "rule_based")}), flush=True)
    with open(os.path.join(out, "selector_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
