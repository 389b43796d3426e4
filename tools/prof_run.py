"""Solve one bench workload a few times and print device time, work inflation and
(under MLMQ_DEBUG=1 MLMQ_PROFILE=1, the profile library) the per-phase split and the
managed-floor epoch log.

    MLMQ_DEBUG=1 MLMQ_PROFILE=1 python tools/prof_run.py c3 [--reps 2] [--set k=v ...]
    MLMQ_LIB=paper_2602_10080_b200/libmlmq_exp.so python tools/prof_run.py c2

``--set`` overrides EngineConfig fields (ints) or ``cfg.<field>`` / ``l1.<field>`` /
``l2.<field>`` of the bench's MlmqConfig.
"""
import argparse
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from bench import build_graph, solve_config, solve_engine  # noqa: E402
from paper_2602_10080_b200 import EngineConfig, extract_features  # noqa: E402
from paper_2602_10080_b200.engine import prepare  # noqa: E402


def _num(v):
    try:
        return int(v)
    except ValueError:
        try:
            return float(v)
        except ValueError:
            return v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--source", type=int, default=0)
    ap.add_argument("--set", nargs="*", default=[])
    ap.add_argument("--check", action="store_true", help="compare with the C oracle")
    ap.add_argument("--golden", action="store_true",
                    help="compare the distance hash with the committed golden hash (c2, c4, c5)")
    a = ap.parse_args()
    t = time.perf_counter()
    g = build_graph(a.config)
    print(f"graph {a.config} n={g.num_vertices} m={g.num_edges} gen {time.perf_counter() - t:.1f}s", flush=True)
    f = extract_features(g)
    cfg = solve_config(a.config, g, f)
    eng = solve_engine(a.config)
    for kv in a.set:
        k, v = kv.split("=", 1)
        v = _num(v)
        if k.startswith("cfg."):
            setattr(cfg, k[4:], v if v != "None" else None)
        elif k.startswith("l1."):
            setattr(cfg.l1_params, k[3:], v)
        elif k.startswith("l2."):
            setattr(cfg.l2_params, k[3:], v)
        else:
            eng = dataclasses.replace(eng, **{k: v})
    cfg_r, eng_r, dg, ncfg = prepare(g, a.source, cfg, eng, features=f)
    ms = []
    for i in range(a.reps):
        tw = time.perf_counter()
        m = dg.sssp_device(a.source, ncfg)
        tw = time.perf_counter() - tw
        if i == 0:
            print(f"first solve wall {tw * 1e3:.1f} ms (includes one-time device layout work)", flush=True)
        ms.append(m.kernel_ms)
        v, e = dg.reach()
        print(f"rep {i}: {m.kernel_ms:.3f} ms  {e / m.kernel_ms / 1e6:.2f} GTEPS  relax {m.relaxations} "
              f"infl {m.relaxations / max(1, e):.3f} groups {cfg_r.num_groups}", flush=True)
    print(f"best {min(ms):.3f} ms median {float(np.median(ms)):.3f} ms  "
          f"{cfg_r.l1_type}+{cfg_r.l2_type} delta={cfg_r.l2_params.delta}", flush=True)
    if a.golden:
        import hashlib
        import json
        from oracle import oracle
        big = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                          "tests", "golden", "big_configs.json")))
        got = dg.last_dist()
        if a.config == "c5":
            ok = hashlib.sha256(got.tobytes()).hexdigest() == big["c5"]["dist_f32_sha256"]
        elif a.config == "c4":
            ok = oracle.dist_sha256(got) == big["c4"]["dist_sha256"]
        else:
            ok = oracle.dist_sha256(got) == "f6d20099af4ad32ebcc888faa9f557f17b69be966c4c0808093799b5f3840788"
        print("golden match:", ok, flush=True)
    if a.check:
        from oracle import oracle
        got = dg.last_dist()
        if np.asarray(g.weights).dtype.kind == "f":
            want = oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, a.source)
        else:
            want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, a.source)
        print("oracle match:", bool(np.array_equal(got, want)), flush=True)


if __name__ == "__main__":
    main()
