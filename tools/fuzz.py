"""GPU fuzz: random graphs x random engine knobs vs the CPU oracle (stress for rare races).

    python tools/fuzz.py TRIALS SEED
"""
import os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle
from paper_2602_10080_b200 import EngineConfig, L1Params, L2Params, MlmqConfig, generate_graph, sssp_solve
from paper_2602_10080_b200.graph import generate_grid2d, generate_random_uniform

trials, seed = int(sys.argv[1]), int(sys.argv[2])
rng = random.Random(seed)
bad = 0
t0 = time.time()
for t in range(trials):
    kind = rng.choice(["grid2d", "rmat", "uniform", "path", "rmat-big"])
    if kind == "grid2d":
        g = generate_grid2d(rng.randint(1, 120), rng.randint(1, 120), 0, rng.choice([1, 5, 100, 1000]), seed=t)
    elif kind == "rmat":
        g = generate_graph("rmat", seed=t, scale=rng.randint(2, 14), edge_factor=rng.randint(1, 16), wmin=0, wmax=rng.choice([1, 255]))
    elif kind == "rmat-big":
        g = generate_graph("rmat", seed=t, scale=rng.randint(15, 17), edge_factor=16, wmin=1, wmax=255)
    elif kind == "uniform":
        n = rng.randint(1, 5000)
        g = generate_random_uniform(n, rng.randint(0, 8 * n), 0, 50, seed=t)
    else:
        g = generate_graph("path", seed=t, n=rng.randint(1, 3000), wmin=0, wmax=9)
    l2 = rng.choice(["fifo", "bucket", "priority", "multi", "fifo", "bucket"])
    cfg = MlmqConfig(l1_type=rng.choice(["vector", "near_far", "filter", "slf"]), l2_type=l2,
                     l0_capacity=rng.choice([1, 2, 4, 7, 16]),
                     l1_params=L1Params(capacity=rng.choice([1, 8, 64, 512, 1024]), wb=rng.choice([0, 1, 8])),
                     l2_params=L2Params(block_size=rng.choice([1, 7, 16, 64]), bmax=rng.choice([1, 3, 4, 64]),
                                        bnum=1, node_batch=rng.choice([1, 5, 32])),
                     num_groups=rng.choice([1, 3, 17, 300, None]), lanes_per_group=rng.choice([1, 2, 5, 8, 32]))
    eng = EngineConfig(duplicate_elimination=rng.random() < 0.8, bucket_window=rng.choice([0, 1, 2]),
                       read_batch=rng.choice([0, 32, 64]), hub_chunk=rng.choice([0, 64, 1024]),
                       hub_threshold=rng.choice([0, 100, 5000]), spin_timeout_s=20)
    s = rng.randrange(g.num_vertices)
    try:
        r = sssp_solve(g, s, cfg, eng, watchdog_s=60)
        want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, s)
        m = r.metrics
        ok = np.array_equal(r.dist_array, want) and m.l0_enqueues == m.l0_dequeues and \
            m.l1_enqueues == m.l1_dequeues and m.l2_enqueues == m.l2_dequeues
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", t, kind, type(e).__name__, e, flush=True)
    if not ok:
        bad += 1
        print("BAD", t, kind, g.num_vertices, g.num_edges, s, cfg, eng, flush=True)
print(f"trials {trials} bad {bad} in {time.time()-t0:.0f}s", flush=True)
