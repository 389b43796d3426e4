"""Per-superstep profile of the 1D-partitioned solve on one GPU (logical shards).

    python tools/shard_profile.py c2 8
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import build_graph, solve_config  # noqa: E402
from paper_2602_10080_b200 import EngineConfig, MlmqConfig, extract_features  # noqa: E402
from paper_2602_10080_b200.sharded import GpuShard, solve_logical  # noqa: E402

name, P = sys.argv[1], int(sys.argv[2])
g = build_graph(name)
f = extract_features(g)
cfg = solve_config(name, g, f)
bks = [GpuShard(g, P, r, cfg, EngineConfig()) for r in range(P)]
for rep in range(2):
    res = solve_logical(bks, 0)
print(f"{name} P={P}: steps {res.steps} sent {res.sent} kernel_ms(sum) {res.kernel_ms:.2f} exchange_ms {res.exchange_ms:.2f}")
for s in range(res.steps):
    row = [(b.metrics[s].kernel_ms, b.metrics[s].relaxations) for b in bks]
    km = sum(k for k, _ in row)
    rl = sum(r for _, r in row)
    print(f"  step {s:2d}: kernel ms sum {km:7.3f} max {max(k for k, _ in row):6.3f}  relaxations {rl:>11d}")
tot_rel = sum(m.relaxations for b in bks for m in b.metrics)
print(f"total relaxations {tot_rel} ({tot_rel / g.num_edges:.2f} x m)")
