"""Sweep engine configurations on one workload; prints kernel ms, GTEPS, work inflation.

    python tools/tune.py --config c2 [--quick]
"""
import argparse
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import CONFIGS, build_graph  # noqa: E402
from paper_2602_10080_b200 import EngineConfig, L1Params, L2Params, MlmqConfig, extract_features  # noqa: E402
from paper_2602_10080_b200.engine import prepare  # noqa: E402

SHA = {"c1": "f40804d404084c2be8d587d8f58312b83e33fc1b109d927ad0e26c201d760e45",
       "c2": "f6d20099af4ad32ebcc888faa9f557f17b69be966c4c0808093799b5f3840788",
       "c3": "2bf8e0cf2ab0c6ab8b906952288c22c564fbda5404ab78d48e8c90590c3bde41"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--grid", default="default")
    ap.add_argument("--source", type=int, default=0)
    args = ap.parse_args()
    t = time.time()
    g = build_graph(args.config)
    f = extract_features(g)
    print(f"# {args.config} n={g.num_vertices} m={g.num_edges} gen {time.time()-t:.1f}s "
          f"avg_w={f.avg_weight:.2f}", flush=True)
    aw = f.avg_weight if f.float_weights else max(1, round(f.avg_weight))
    l1s = ["vector", "near_far", "filter", "slf"]
    caps = [64, 256, 1024]
    dscales = [1, 4, 16]
    combos = []
    for l1, cap, l2, ds, hub in itertools.product(l1s, caps, ["fifo", "bucket"], dscales, [0]):
        if l2 == "fifo" and ds != 1:
            continue
        combos.append((l1, cap, l2, ds, hub))
    if args.grid == "small":
        combos = [c for c in combos if c[1] == 256]
    elif args.grid == "fifo":
        combos = [c for c in combos if c[2] == "fifo"]
    e_reach = None
    for l1, cap, l2, ds, hub in combos:
        cfg = MlmqConfig(l1_type=l1, l2_type=l2,
                         l1_params=L1Params(capacity=cap, wb=8, filter_f=4 * aw,
                                            delta_nf=ds * aw),
                         l2_params=L2Params(delta=ds * aw if l2 == "bucket" else None),
                         num_groups=None)
        try:
            cfg2, eng, dg, ncfg = prepare(g, args.source, cfg, EngineConfig(hub_chunk=hub),
                                          features=f)
            ms = []
            for _ in range(args.reps):
                m = dg.sssp_device(args.source, ncfg)
                ms.append(m.kernel_ms)
            if e_reach is None:
                e_reach = dg.reach()[1]
            ok = ""
            if args.config in SHA and not f.float_weights:
                import hashlib
                d = dg.last_dist()
                ok = "ok" if hashlib.sha256(d.astype("<u8").tobytes()).hexdigest() == SHA[args.config] else "MISMATCH"
            best = min(ms)
            print(f"{l1:8s} cap={cap:5d} {l2:6s} d={ds:3g} hub={hub} G={cfg2.num_groups:5d} "
                  f"ms={best:8.3f} med={np.median(ms):8.3f} GTEPS={e_reach/best/1e6:7.3f} "
                  f"infl={m.relaxations/e_reach:6.2f} hubitems={m.hub_items} {ok}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{l1} {cap} {l2} {ds}: {type(e).__name__}: {e}", flush=True)


if __name__ == "__main__":
    main()
