"""Vertex relabeling by in-degree class (the device graph layout of a skewed graph,
mlmq_api.cu ensure_relabel): distances come back in the caller's vertex order and equal
the CPU oracle for every queue family, distance width and weight kind.  MLMQ_RELABEL=1
forces the relabel on graphs below the auto threshold; =0 forces it off."""
import random

import numpy as np
import pytest

from oracle import oracle
from paper_2602_10080_b200 import (EngineConfig, MlmqConfig, bfs_solve, build_csr,
                                   generate_graph, sssp_solve)
from paper_2602_10080_b200.graph import generate_grid2d, with_f32_weights

pytestmark = pytest.mark.gpu


@pytest.fixture
def relabel(monkeypatch):
    monkeypatch.setenv("MLMQ_RELABEL", "1")


def oracle_dist(g, s=0, unit=False):
    return oracle.dijkstra_u64(g.row_offsets, g.col_indices, None if unit else g.weights, s,
                               unit_weights=unit)


def reached_sources(g, k, seed):
    deg = np.diff(np.asarray(g.row_offsets))
    cand = np.nonzero(deg > 0)[0]
    rng = random.Random(seed)
    return [int(cand[rng.randrange(len(cand))]) for _ in range(k)]


@pytest.mark.parametrize("l2", ["fifo", "bucket", "priority", "multi"])
def test_relabeled_rmat_every_l2_family(relabel, l2):
    g = generate_graph("rmat", seed=7, scale=13, edge_factor=16, wmin=1, wmax=255)
    for s in [0] + reached_sources(g, 2, seed=1):
        r = sssp_solve(g, s, MlmqConfig(l2_type=l2, num_groups=None))
        assert np.array_equal(r.dist_array, oracle_dist(g, s)), (l2, s)
        m = r.metrics
        assert m.l2_enqueues == m.l2_dequeues


def test_relabeled_matches_caller_order_solve(monkeypatch):
    # the same graph solved with and without relabeling: identical distances and reach
    g = generate_graph("rmat", seed=3, scale=14, edge_factor=16, wmin=1, wmax=255)
    monkeypatch.setenv("MLMQ_RELABEL", "0")
    a = sssp_solve(g, 0)
    g2 = generate_graph("rmat", seed=3, scale=14, edge_factor=16, wmin=1, wmax=255)
    monkeypatch.setenv("MLMQ_RELABEL", "1")
    b = sssp_solve(g2, 0)
    assert np.array_equal(a.dist_array, b.dist_array)
    assert np.array_equal(b.dist_array, oracle_dist(g2))
    # relaxations count edges out of reached vertices: order-independent bound
    assert b.metrics.relaxations >= int(np.diff(np.asarray(g2.row_offsets))[b.dist_array != np.iinfo(np.uint64).max].sum())


def test_relabeled_f32_weights_bit_exact(relabel):
    g = with_f32_weights(generate_graph("rmat", seed=1, scale=13, edge_factor=16), seed=3)
    for s in [0] + reached_sources(g, 1, seed=2):
        r = sssp_solve(g, s)
        want = oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, s)
        assert r.dist_array.dtype == np.float32
        assert np.array_equal(r.dist_array.view(np.uint32), want.view(np.uint32)), s


def test_relabeled_u64_and_bfs(relabel):
    g = generate_graph("rmat", seed=11, scale=12, edge_factor=8, wmin=1, wmax=100)
    r = sssp_solve(g, 0, engine=EngineConfig(dist_mode="u64", num_groups=None))
    assert r.native["dist_bits"] == 64
    assert np.array_equal(r.dist_array, oracle_dist(g))
    g2 = generate_graph("rmat", seed=11, scale=12, edge_factor=8, wmin=1, wmax=100)
    b = bfs_solve(g2, 0)
    assert np.array_equal(b.dist_array, oracle_dist(g2, unit=True))


def test_relabeled_hub_star_and_isolated_vertices(relabel):
    n = 50_001
    src = np.zeros(n - 1, np.int64)
    dst = np.arange(1, n, dtype=np.int64)[::-1].copy()  # hub targets in reverse id order
    g = build_csr(n + 10, (src, dst, np.arange(1, n, dtype=np.uint32) % 7 + 1))  # 10 isolated vertices
    r = sssp_solve(g, 0, MlmqConfig(num_groups=None), EngineConfig(hub_chunk=1024))
    assert r.metrics.relaxations == n - 1
    assert np.array_equal(r.dist_array, oracle_dist(g))
    # a source that is not the hub, and one that is isolated
    r2 = sssp_solve(g, n + 3)
    assert r2.distances[n + 3] == 0 and sum(d == 0 for d in r2.distances) == 1


def test_relabeled_grid_forced(relabel):
    # a grid is not skewed (the auto policy keeps it in caller order); forced, it must
    # still be exact
    g = generate_grid2d(64, 64, 1, 100, seed=4)
    r = sssp_solve(g, 100, MlmqConfig(l2_type="bucket", num_groups=None))
    assert np.array_equal(r.dist_array, oracle_dist(g, 100))
