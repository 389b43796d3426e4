"""GPU parity tests: the CUDA MLMQ engine, called through libmlmq.so, against the CPU
oracle and the reference's golden vectors.  Cases mirror the reference's
test_engine.py (file:line cited per test) and acceptance criteria AC1/AC2/AC6/AC8."""
import random

import numpy as np
import pytest

from oracle import oracle
from paper_2602_10080_b200 import (INF, EngineConfig, EngineError, L1Params, L2Params,
                                   MlmqConfig, QueueOverflowError, bfs_solve, build_csr,
                                   compare_distances, dijkstra_oracle, distances_blob,
                                   enumerate_candidates, extract_features, generate_graph,
                                   sssp_solve, unit_weight_view)
from paper_2602_10080_b200.graph import generate_grid2d, generate_random_uniform, with_f32_weights

pytestmark = pytest.mark.gpu

ALL_COMBOS = [(a, b) for a in ("vector", "near_far", "filter", "slf")
              for b in ("fifo", "bucket", "priority", "multi")]


def combo_config(l1, l2, num_groups=1):
    # test_engine.py:29-37
    return MlmqConfig(l1_type=l1, l2_type=l2, l1_params=L1Params(capacity=64, wb=4),
                      l2_params=L2Params(block_size=16, block_num=512, bmax=32, bnum=2),
                      num_groups=num_groups, lanes_per_group=8)


def oracle_dist(g, s=0, unit=False):
    return oracle.dijkstra_u64(g.row_offsets, g.col_indices, None if unit else g.weights, s,
                               unit_weights=unit)


def assert_balanced(m):
    assert m.l0_enqueues == m.l0_dequeues
    assert m.l1_enqueues == m.l1_dequeues
    assert m.l2_enqueues == m.l2_dequeues


DIAMOND = build_csr(4, [(0, 1, 10), (0, 2, 1), (2, 1, 2), (1, 3, 1), (2, 3, 9)])


@pytest.mark.parametrize("l1,l2", ALL_COMBOS)
def test_diamond_exact_on_every_queue_combo(l1, l2):  # test_engine.py:45-49
    assert sssp_solve(DIAMOND, 0, combo_config(l1, l2)).distances == [0, 3, 1, 4]


@pytest.mark.parametrize("l1,l2", ALL_COMBOS)
def test_weighted_grid_exact_on_every_queue_combo(l1, l2):  # test_engine.py:52-57
    g = generate_grid2d(8, 8, wmin=1, wmax=20, seed=3)
    res = sssp_solve(g, 0, combo_config(l1, l2, num_groups=2))
    assert res.distances == dijkstra_oracle(g, 0)
    assert_balanced(res.metrics)


@pytest.mark.parametrize("l1,l2", ALL_COMBOS)
def test_rmat_every_combo_many_groups(l1, l2):
    g = generate_graph("rmat", seed=5, scale=11, edge_factor=8, wmin=1, wmax=100)
    res = sssp_solve(g, 0, combo_config(l1, l2, num_groups=64))
    assert np.array_equal(res.dist_array, oracle_dist(g))
    assert_balanced(res.metrics)


def test_small_known_answers():  # test_engine.py:60-84
    assert sssp_solve(build_csr(3, [(0, 1, 1), (1, 2, 1), (0, 2, 3)]), 0).distances == [0, 1, 2]
    assert sssp_solve(build_csr(4, [(0, 1, 2)]), 0).distances == [0, 2, INF, INF]
    assert sssp_solve(build_csr(1, []), 0).distances == [0]
    assert sssp_solve(build_csr(3, [(0, 1, 0), (1, 2, 0)]), 0).distances == [0, 0, 0]
    with pytest.raises(ValueError, match="out of range"):
        sssp_solve(build_csr(2, [(0, 1, 1)]), 5)


def test_engine_matches_both_oracles_on_random_graphs():  # test_engine.py:93-104
    for kind, params in [("uniform", dict(n=300, m=1500, wmin=1, wmax=40)),
                         ("rmat", dict(scale=7, edge_factor=6)),
                         ("grid2d", dict(rows=12, cols=12, wmin=1, wmax=30)),
                         ("path", dict(n=500, wmin=1, wmax=9))]:
        g = generate_graph(kind, seed=5, **params)
        want = oracle_dist(g)
        assert np.array_equal(want, oracle.bellman_ford_u64(g.row_offsets, g.col_indices,
                                                            g.weights, 0))
        got = sssp_solve(g, 0, engine=EngineConfig(num_groups=2)).dist_array
        assert np.array_equal(got, want)


def test_star_relaxes_every_edge_exactly_once():  # test_engine.py:107-120
    g = build_csr(41, [(0, v, 1) for v in range(1, 41)])
    cfg = combo_config("vector", "fifo")
    r = sssp_solve(g, 0, cfg, EngineConfig(th_v=16, num_groups=2))
    assert r.distances == [0] + [1] * 40
    assert r.metrics.relaxations == 40 and r.metrics.distance_updates == 40
    r2 = sssp_solve(g, 0, cfg, EngineConfig(th_v=1000, num_groups=2))
    assert r2.distances == r.distances and r2.metrics.relaxations == 40


def test_hub_tier_relaxes_every_edge_exactly_once():
    # a 100k-edge star: split into hub work items shared by every warp
    n = 100_001
    g = build_csr(n, (np.zeros(n - 1, np.int64), np.arange(1, n, dtype=np.int64),
                      np.ones(n - 1, np.uint32)))
    r = sssp_solve(g, 0, MlmqConfig(num_groups=None), EngineConfig(hub_chunk=1024))
    assert r.metrics.relaxations == n - 1 and r.metrics.distance_updates == n - 1
    assert r.native["hub_items"] > 0
    assert np.array_equal(r.dist_array, oracle_dist(g))


def test_duplicate_elimination_drops_stale_reads():  # test_engine.py:123-131
    g = generate_random_uniform(150, 1200, 1, 30, seed=8)
    want = dijkstra_oracle(g, 0)
    on = sssp_solve(g, 0, engine=EngineConfig(num_groups=1, duplicate_elimination=True))
    off = sssp_solve(g, 0, engine=EngineConfig(num_groups=1, duplicate_elimination=False))
    assert on.distances == want and off.distances == want
    assert on.metrics.settled_reads <= off.metrics.settled_reads
    assert on.metrics.relaxations <= off.metrics.relaxations


def test_settled_reads_bounded_by_dequeues():  # test_engine.py:134-138
    m = sssp_solve(generate_random_uniform(100, 500, 1, 20, seed=2), 0).metrics
    assert 0 < m.settled_reads <= m.l0_dequeues + m.l1_dequeues + m.l2_dequeues


def test_work_metrics_deterministic_for_single_group():  # test_engine.py:141-148
    g = generate_random_uniform(200, 1000, 1, 50, seed=4)
    cfg = combo_config("slf", "bucket")
    a = sssp_solve(g, 0, cfg).metrics.to_json_dict()
    b = sssp_solve(g, 0, cfg).metrics.to_json_dict()
    a.pop("wall_time_us")
    b.pop("wall_time_us")
    assert a == b


def test_queues_fully_drain_and_counters_balance():  # test_engine.py:151-158
    g = generate_random_uniform(200, 1000, 1, 50, seed=6)
    for l1, l2 in [("vector", "fifo"), ("filter", "bucket"), ("slf", "priority"),
                   ("near_far", "multi")]:
        assert_balanced(sssp_solve(g, 0, combo_config(l1, l2, num_groups=2)).metrics)


def test_group_count_does_not_change_distances():  # test_engine.py:161-167 / AC6
    g = generate_graph("rmat", scale=8, edge_factor=6, seed=9)
    blobs = {distances_blob(sssp_solve(g, 3, combo_config("slf", "bucket", num_groups=k)).distances)
             for k in (1, 2, 4, 64, 512)}
    assert len(blobs) == 1


def test_bfs_counts_hops_not_weights():  # test_engine.py:170-187
    g = build_csr(3, [(0, 1, 50), (1, 2, 50), (0, 2, 200)])
    assert bfs_solve(g, 0).distances == [0, 1, 1]
    assert sssp_solve(g, 0).distances == [0, 50, 100]
    g = generate_random_uniform(250, 1000, 1, 90, seed=12)
    assert bfs_solve(g, 0, engine=EngineConfig(num_groups=2)).distances == \
        dijkstra_oracle(unit_weight_view(g), 0)


def test_result_echoes_resolved_config():  # test_engine.py:248-253
    g = generate_random_uniform(40, 150, 2, 8, seed=3)
    r = sssp_solve(g, 0, MlmqConfig(l2_type="bucket"), EngineConfig(num_groups=2))
    assert r.config_used.l2_params.delta is not None
    assert r.config_used.num_groups == 2 and r.engine_used.num_groups == 2
    assert len(r.group_metrics) == 2


def test_auto_groups_fill_the_device():
    g = generate_grid2d(32, 32, 1, 100, seed=1)
    r = sssp_solve(g, 0, MlmqConfig(num_groups=None))
    assert r.config_used.num_groups >= 148
    assert r.config_used.l2_params.pnum == max(1, r.config_used.num_groups // 4)
    assert np.array_equal(r.dist_array, oracle_dist(g))


def test_golden_vectors_every_candidate(golden):
    """AC1 (test_acceptance.py:94-141) on the reference's own graph set: every one of
    the 12 default candidates, 2 sources, 2 groups, against reference-produced hashes;
    AC8 (BFS) alongside."""
    cands = enumerate_candidates()
    assert len(cands) == 12
    mism = []
    runs = 0
    for idx, rec in enumerate(golden["graphs"]):
        g = generate_graph(rec["kind"], seed=rec["seed"], **rec["params"])
        f = extract_features(g)
        for s in rec["sources"]:
            for cand in (cands if idx % 4 == 0 else [cands[idx % len(cands)]]):
                res = sssp_solve(g, s["source"], cand.bind(f, num_groups=2), features=f)
                runs += 1
                if oracle.dist_sha256(res.dist_array) != s["dist_sha256"]:
                    mism.append((rec["id"], s["source"], cand.label()))
                assert_balanced(res.metrics)
            b = sssp_solve(g, s["source"], cands[(idx + 5) % 12].bind(f, num_groups=2),
                           unit_weights=True)
            if oracle.dist_sha256(b.dist_array) != s["unit_dist_sha256"]:
                mism.append((rec["id"], s["source"], "bfs"))
    assert not mism, mism[:5]
    assert runs > 500


def test_golden_vectors_auto_groups(golden):
    cands = enumerate_candidates()
    for idx, rec in enumerate(golden["graphs"]):
        g = generate_graph(rec["kind"], seed=rec["seed"], **rec["params"])
        f = extract_features(g)
        cfg = cands[idx % len(cands)].bind(f, num_groups=None)
        for s in rec["sources"]:
            res = sssp_solve(g, s["source"], cfg, features=f)
            assert oracle.dist_sha256(res.dist_array) == s["dist_sha256"], (rec["id"], cfg.l1_type,
                                                                            cfg.l2_type)


C1_DIST = "f40804d404084c2be8d587d8f58312b83e33fc1b109d927ad0e26c201d760e45"
RMAT16_DIST = "20a660bb634d7766180f5f8c0de9aeb1bf8aa79c52d849af15c9b6c17fae2ae0"
RMAT20_DIST = "c1ef6add7d3fdd5301715e8d8f7fcc6efcd659035d6a31b086cbb087c2d72209"


@pytest.mark.parametrize("kind,params,sha", [
    ("grid2d", dict(rows=256, cols=256, wmin=1, wmax=100), C1_DIST),
    ("rmat", dict(scale=16, edge_factor=16, wmin=1, wmax=255), RMAT16_DIST),
    ("rmat", dict(scale=20, edge_factor=16, wmin=1, wmax=255), RMAT20_DIST),
], ids=["C1", "rmat16", "rmat20"])
def test_reference_hashes_all_candidates_auto(kind, params, sha):
    g = generate_graph(kind, seed=1, **params)
    f = extract_features(g)
    for cand in enumerate_candidates():
        res = sssp_solve(g, 0, cand.bind(f, num_groups=None), features=f)
        assert oracle.dist_sha256(res.dist_array) == sha, cand.label()
        assert_balanced(res.metrics)


def test_u64_distances_and_overflow_rerun():
    # weights near 2^32: u32 device distances overflow, the engine re-runs in u64
    big = (1 << 32) - 5
    g = build_csr(4, [(0, 1, big), (1, 2, big), (2, 3, 7), (0, 3, 1 << 31)])
    r = sssp_solve(g, 0)
    assert r.distances == [0, big, 2 * big, 1 << 31]
    assert r.native["dist_bits"] == 64 and r.native["reruns"] == 1
    g2 = generate_grid2d(40, 40, 1, 100, seed=2)
    r2 = sssp_solve(g2, 0, engine=EngineConfig(dist_mode="u64", num_groups=None))
    assert r2.native["dist_bits"] == 64
    assert np.array_equal(r2.dist_array, oracle_dist(g2))


def test_float_weights_bit_exact_vs_f32_oracle():
    g = with_f32_weights(generate_graph("rmat", seed=1, scale=12, edge_factor=16), seed=3)
    want = oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, 0)
    f = extract_features(g)
    for cand in enumerate_candidates():
        r = sssp_solve(g, 0, cand.bind(f, num_groups=None), features=f)
        assert r.dist_array.dtype == np.float32
        assert np.array_equal(r.dist_array, want), cand.label()


def test_watchdog_and_overflow_errors():
    g = generate_grid2d(64, 64, 1, 100, seed=1)
    with pytest.raises(ValueError, match="num_groups"):
        sssp_solve(g, 0, MlmqConfig(num_groups=10 ** 7))
    with pytest.raises(ValueError, match="lanes_per_group"):
        sssp_solve(g, 0, MlmqConfig(lanes_per_group=64))
    # the engine still works after rejected calls
    assert np.array_equal(sssp_solve(g, 0).dist_array, oracle_dist(g))


def test_random_sources_and_configs_fuzz():
    rng = random.Random(7)
    for trial in range(40):
        kind = rng.choice(["grid2d", "rmat", "uniform", "path"])
        if kind == "grid2d":
            g = generate_grid2d(rng.randint(1, 40), rng.randint(1, 40), 0, rng.choice([1, 5, 1000]),
                                seed=trial)
        elif kind == "rmat":
            g = generate_graph("rmat", seed=trial, scale=rng.randint(2, 12), edge_factor=rng.randint(1, 16),
                               wmin=0, wmax=rng.choice([1, 255]))
        elif kind == "uniform":
            n = rng.randint(1, 3000)
            g = generate_random_uniform(n, rng.randint(0, 8 * n), 0, 50, seed=trial)
        else:
            g = generate_graph("path", seed=trial, n=rng.randint(1, 3000), wmin=0, wmax=9)
        cfg = MlmqConfig(
            l1_type=rng.choice(["vector", "near_far", "filter", "slf"]),
            l2_type=rng.choice(["fifo", "bucket", "priority", "multi"]),
            l0_capacity=rng.choice([1, 2, 4, 7, 16]),
            l1_params=L1Params(capacity=rng.choice([1, 8, 64, 1024]), wb=rng.choice([0, 1, 8])),
            l2_params=L2Params(block_size=rng.choice([1, 7, 16, 64, 256]), bmax=rng.choice([1, 4, 64]),
                               bnum=1, node_batch=rng.choice([1, 5, 32])),
            num_groups=rng.choice([1, 3, 17, None]),
            lanes_per_group=rng.choice([1, 2, 5, 8, 32]),
            th_v=rng.choice([0, 16, 100000]))
        s = rng.randrange(g.num_vertices)
        r = sssp_solve(g, s, cfg, EngineConfig(duplicate_elimination=rng.random() < 0.8,
                                               heavy_delta=rng.choice([0, 0, 4, 64])),
                       watchdog_s=30)
        want = oracle_dist(g, s)
        assert compare_distances(r.dist_array, want) is None, (trial, cfg)
        assert_balanced(r.metrics)


@pytest.mark.parametrize("win", [0, 1, 2, 4])
def test_bucket_window_managed_floor_exact(win):
    # B200 extension: winners >= win buckets above the floor bypass L0/L1 and the manager
    # advances the floor only when the near window is quiescent (Delta-stepping order)
    graphs = [generate_grid2d(64, 64, 1, 100, seed=1),
              generate_graph("rmat", seed=3, scale=12, edge_factor=16, wmin=1, wmax=255),
              generate_graph("path", seed=2, n=3000, wmin=1, wmax=9)]
    for g in graphs:
        f = extract_features(g)
        want = oracle_dist(g)
        for l1 in ("vector", "near_far", "filter", "slf"):
            for ds, groups in ((1, None), (4, 64), (0.5, 3)):
                aw = max(1, round(f.avg_weight))
                cfg = MlmqConfig(l1_type=l1, l2_type="bucket", l1_params=L1Params(capacity=256),
                                 l2_params=L2Params(delta=max(1, int(ds * aw)), bmax=64),
                                 num_groups=groups)
                r = sssp_solve(g, 0, cfg, EngineConfig(bucket_window=win), features=f)
                assert np.array_equal(r.dist_array, want), (l1, ds, groups)
                assert_balanced(r.metrics)


def test_bucket_window_small_rings_spill_over_not_overflow():
    # far buckets overfill small rings: writers move on to farther rings instead of
    # wedging on a full one (occupancy-aware placement)
    g = generate_graph("rmat", seed=1, scale=14, edge_factor=16, wmin=1, wmax=255)
    cfg = MlmqConfig(l1_type="vector", l2_type="bucket",
                     l2_params=L2Params(delta=128, bmax=8, block_size=16, block_num=64),
                     num_groups=None)
    r = sssp_solve(g, 0, cfg, EngineConfig(bucket_window=1, spin_timeout_s=10))
    assert np.array_equal(r.dist_array, oracle_dist(g))


# ------------------------------------------------------------------ BASELINE configs
C2_DIST = "f6d20099af4ad32ebcc888faa9f557f17b69be966c4c0808093799b5f3840788"
C3_DIST = "2bf8e0cf2ab0c6ab8b906952288c22c564fbda5404ab78d48e8c90590c3bde41"


@pytest.mark.parametrize("name,sha", [("c1", C1_DIST), ("c2", C2_DIST), ("c3", C3_DIST)])
def test_baseline_configs_match_reference_hashes(name, sha):
    # the bench's own engine configurations on the BASELINE graphs, against the
    # reference dijkstra_oracle's dist_sha256 (produced by the reference)
    from bench import build_graph, solve_config, solve_engine
    g = build_graph(name)
    f = extract_features(g)
    for _ in range(2):
        r = sssp_solve(g, 0, solve_config(name, g, f), solve_engine(name), features=f)
        assert oracle.dist_sha256(r.dist_array) == sha
        assert_balanced(r.metrics)


@pytest.mark.parametrize("heavy,hmin", [(8, 0), (24, 0), (128, 0), (24, 16)])
def test_light_heavy_split_exact(heavy, hmin):
    # FIFO L2 with the light/heavy split (B200 extension): exact on every graph family,
    # group count and L1 variant; the deferred tokens leave no residue (counter identities)
    graphs = [generate_graph("rmat", seed=7, scale=12, edge_factor=16, wmin=1, wmax=255),
              generate_grid2d(40, 40, 1, 100, seed=4),
              generate_graph("path", seed=1, n=500, wmin=1, wmax=30),
              generate_random_uniform(3000, 20000, 1, 200, seed=2)]
    for g in graphs:
        want = oracle_dist(g)
        for l1 in ("vector", "near_far", "filter", "slf"):
            for groups in (1, 7, None):
                cfg = MlmqConfig(l1_type=l1, l2_type="fifo", num_groups=groups)
                r = sssp_solve(g, 0, cfg, EngineConfig(heavy_delta=heavy, heavy_min_edges=hmin))
                assert np.array_equal(r.dist_array, want), (l1, groups, g.num_vertices)
                assert_balanced(r.metrics)
    gf = with_f32_weights(generate_graph("rmat", seed=1, scale=12, edge_factor=16), seed=3)
    r = sssp_solve(gf, 0, MlmqConfig(num_groups=None), EngineConfig(heavy_delta=0.05))
    assert np.array_equal(r.dist_array, oracle.dijkstra_f32(gf.row_offsets, gf.col_indices, gf.weights, 0))


def test_recycled_result_buffers_are_not_aliased():
    # results live in page-locked buffers recycled across solves: a held result must
    # never be overwritten by a later solve
    g = generate_graph("rmat", seed=4, scale=12, edge_factor=8, wmin=1, wmax=99)
    r0 = sssp_solve(g, 0)
    r1 = sssp_solve(g, 17)
    r2 = sssp_solve(g, 99)
    del r1
    r3 = sssp_solve(g, 5)
    assert np.array_equal(r0.dist_array, oracle_dist(g, 0))
    assert np.array_equal(r2.dist_array, oracle_dist(g, 99))
    assert np.array_equal(r3.dist_array, oracle_dist(g, 5))
