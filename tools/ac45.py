"""Reference acceptance criteria 4 and 5 (pkg/tests/test_acceptance.py:308-371) on the GPU
engine, printing the per-trial relaxation ratios (diagnostic for the staged suite)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10080_b200 import (EngineConfig, L1Params, MlmqConfig, extract_features,  # noqa: E402
                                   generate_graph, sssp_solve)

eng = EngineConfig(bucket_window=int(sys.argv[1])) if len(sys.argv) > 1 else None
trials = [("path", dict(n=2000 + 400 * i, wmin=1, wmax=50), i) for i in range(6)]
trials += [("grid2d", dict(rows=40 + 2 * i, cols=60, wmin=1, wmax=100), 20 + i) for i in range(14)]
wins, ratios = 0, []
for kind, params, seed in trials:
    g = generate_graph(kind, seed=seed, **params)
    f = extract_features(g)
    base = dict(l1_type="vector", l2_type="bucket", num_groups=2, lanes_per_group=4, l0_capacity=1)
    on = sssp_solve(g, 0, MlmqConfig(l1_params=L1Params(wb=8), **base), eng, features=f)
    off = sssp_solve(g, 0, MlmqConfig(l1_params=L1Params(wb=0), **base), eng, features=f)
    wins += on.metrics.relaxations <= off.metrics.relaxations
    ratios.append(on.metrics.relaxations / off.metrics.relaxations)
print(f"AC4: wins {wins}/20 (need 16), median ratio {statistics.median(ratios):.3f}", [round(r, 3) for r in ratios])
trials = [(dict(rows=100, cols=100, wmin=1, wmax=100), i) for i in range(10)]
trials += [(dict(rows=125, cols=80, wmin=10, wmax=1000), 10 + i) for i in range(10)]
wins, ratios = 0, []
for params, seed in trials:
    g = generate_graph("grid2d", seed=seed, **params)
    f = extract_features(g)
    kw = dict(num_groups=1, lanes_per_group=4, l0_capacity=1, l1_params=L1Params(wb=8))
    rb = sssp_solve(g, 0, MlmqConfig(l1_type="vector", l2_type="bucket", **kw), eng, features=f)
    rf = sssp_solve(g, 0, MlmqConfig(l1_type="vector", l2_type="fifo", **kw), eng, features=f)
    wins += rb.metrics.relaxations < rf.metrics.relaxations
    ratios.append(rb.metrics.relaxations / rf.metrics.relaxations)
print(f"AC5: wins {wins}/20 (need 16), median ratio {statistics.median(ratios):.3f}")
