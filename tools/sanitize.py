"""compute-sanitizer driver (SURVEY §4.4 #3 evidence): small solves over every L1 x L2
combination, the managed bucket floor, the u64 and f32 distance kinds, the hub tier and
the queue harness, each checked against the oracle.  Run under a sanitizer tool:

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --quick
    compute-sanitizer --tool synccheck python tools/sanitize.py --quick

Small graphs and a few dozen groups keep the instrumented persistent kernel inside a few
minutes; the summaries go to profiles/r2_sanitizer.md.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2602_10080_b200 import (EngineConfig, L1Params, L2Params, MlmqConfig,  # noqa: E402
                                   extract_features, generate_graph, sssp_solve)
from paper_2602_10080_b200.graph import with_f32_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="fewer combinations (racecheck/synccheck are slow)")
    a = ap.parse_args()
    graphs = [("rmat10", generate_graph("rmat", seed=1, scale=10, edge_factor=16, wmin=1, wmax=255)),
              ("grid24", generate_graph("grid2d", seed=2, rows=24, cols=24, wmin=1, wmax=100))]
    l1s = ["vector", "near_far", "filter", "slf"]
    l2s = ["fifo", "bucket", "priority", "multi"]
    if a.quick:
        l1s, l2s = ["vector", "slf"], ["fifo", "bucket", "multi"]
    runs = bad = 0
    for name, g in graphs:
        f = extract_features(g)
        want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
        for l1 in l1s:
            for l2 in l2s:
                for groups, win in ((3, 0), (24, 1)):
                    cfg = MlmqConfig(l1_type=l1, l2_type=l2, l1_params=L1Params(capacity=64, wb=4),
                                     l2_params=L2Params(block_size=16, bmax=16), num_groups=groups)
                    r = sssp_solve(g, 0, cfg, EngineConfig(bucket_window=win, hub_chunk=64, hub_threshold=128,
                                                           spin_timeout_s=60), features=f, watchdog_s=600)
                    runs += 1
                    ok = np.array_equal(r.dist_array, want)
                    bad += not ok
                    print(f"{name} {l1}+{l2} groups={groups} window={win}: {'ok' if ok else 'MISMATCH'}", flush=True)
        r = sssp_solve(g, 0, MlmqConfig(num_groups=16), EngineConfig(dist_mode="u64"), features=f)
        runs += 1
        bad += not np.array_equal(r.dist_array, want)
    gf = with_f32_weights(graphs[0][1], seed=3)
    r = sssp_solve(gf, 0, MlmqConfig(num_groups=16))
    runs += 1
    bad += not np.array_equal(r.dist_array, oracle.dijkstra_f32(gf.row_offsets, gf.col_indices, gf.weights, 0))
    from paper_2602_10080_b200 import _native
    for kind in (0, 1, 2, 3):  # queue harness: a small concurrent stress per L2 family
        q = _native.DeviceQueue(kind, block_size=16, block_num=512, delta=64, bmax=16, bnum=2, node_batch=8,
                                pnum=2, num_groups=8, heap_nodes=4096)
        pairs, n, _, _ = q.stress(4, 4, 2000, 0, 2000, 8000, 8000 + 4 * 64)
        runs += 1
        bad += n != 8000
    print(f"SANITIZE-RUNS {runs} mismatches {bad}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
