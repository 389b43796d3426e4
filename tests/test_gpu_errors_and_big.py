"""GPU tests for the failure paths (engine.py:127-133, 229-242, 267-279; l2.py:116-135) and
for the two BASELINE configs the reference cannot run itself (C4 Kronecker s26, C5 f32),
checked against the committed golden hashes (tests/golden/big_configs.json, made by
tests/golden/make_big_hashes.py from the reference-pinned generator and oracle)."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2602_10080_b200 import (CsrGraph, EngineConfig, EngineError, L1Params, L2Params,
                                   MlmqConfig, QueueOverflowError, build_csr, extract_features,
                                   generate_graph, sssp_solve)
from paper_2602_10080_b200.graph import generate_grid2d

pytestmark = pytest.mark.gpu

BIG = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "big_configs.json")))
C2_DIST = "f6d20099af4ad32ebcc888faa9f557f17b69be966c4c0808093799b5f3840788"


def _oracle(g, s=0):
    return oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, s)


# ------------------------------------------------------------------ invalid input
def test_bad_csr_is_rejected_at_the_abi():
    # a column >= n would index past dist on the device; the reference raises at the
    # Python level, the ABI validates on upload and reports ValueError
    g = CsrGraph(3, 2, [0, 1, 2, 2], [1, 7], [1, 1])
    with pytest.raises(ValueError, match="column indices lie outside"):
        sssp_solve(g, 0)
    g = CsrGraph(3, 2, [0, 2, 1, 2], [1, 2], [1, 1])
    with pytest.raises(ValueError, match="non-decreasing"):
        sssp_solve(g, 0)


# ------------------------------------------------------------------ watchdog
def test_watchdog_expiry_raises_engine_error_and_recovers():
    # engine.py:267-279: the manager is told to abort through the mapped host word and
    # the solve raises EngineError("watchdog expired after ...s")
    g = generate_grid2d(1500, 1500, 1, 100, seed=1)
    cfg = MlmqConfig(l1_type="vector", l2_type="bucket", l2_params=L2Params(delta=10), num_groups=64)
    with pytest.raises(EngineError, match=r"watchdog expired after 0\.02s"):
        sssp_solve(g, 0, cfg, watchdog_s=0.02)
    # the same device graph solves exactly afterwards (queues reset)
    r = sssp_solve(g, 0, MlmqConfig(l2_type="fifo", num_groups=None))
    assert np.array_equal(r.dist_array, _oracle(g))


# ------------------------------------------------------------------ queue overflow
def _assert_recovers(g):
    r = sssp_solve(g, 0, MlmqConfig(num_groups=None))
    assert np.array_equal(r.dist_array, _oracle(g))


def test_ring_overflow_raises_queue_overflow_error_with_fields():
    # l2.py:116-135: a writer that cannot get a free slot within spin_timeout raises
    # QueueOverflowError("ring slot S stayed busy for Ts (block_num=B, write_ptr=W,
    # read_ptr=R); block_num is likely too small for this workload")
    g = generate_graph("rmat", seed=2, scale=14, edge_factor=16, wmin=1, wmax=255)
    cfg = MlmqConfig(l1_type="vector", l2_type="fifo", l1_params=L1Params(capacity=32, wb=1),
                     l2_params=L2Params(block_size=8), num_groups=1)
    eng = EngineConfig(test_capacity=4, spin_timeout_s=0.3, share=False)
    with pytest.raises(QueueOverflowError) as ei:
        sssp_solve(g, 0, cfg, eng)
    msg = str(ei.value)
    for field in ("ring slot", "stayed busy for 0.3s", "block_num=4", "write_ptr=", "read_ptr=",
                  "block_num is likely too small"):
        assert field in msg, msg
    _assert_recovers(g)


def test_bucket_ring_overflow():
    g = generate_grid2d(300, 300, 1, 100, seed=4)
    cfg = MlmqConfig(l1_type="vector", l2_type="bucket", l1_params=L1Params(capacity=16, wb=1),
                     l2_params=L2Params(block_size=4, delta=50, bmax=8), num_groups=1)
    with pytest.raises(QueueOverflowError, match="ring slot"):
        sssp_solve(g, 0, cfg, EngineConfig(test_capacity=2, spin_timeout_s=0.3, bucket_window=0, share=False))
    _assert_recovers(g)


def test_heap_overflow():
    g = generate_graph("rmat", seed=3, scale=13, edge_factor=16, wmin=1, wmax=255)
    cfg = MlmqConfig(l1_type="vector", l2_type="priority", l1_params=L1Params(capacity=16, wb=1),
                     l2_params=L2Params(node_batch=4), num_groups=1)
    with pytest.raises(QueueOverflowError, match=r"batch heap 0 is full \(\d+ of 8 nodes\)"):
        sssp_solve(g, 0, cfg, EngineConfig(test_capacity=8, spin_timeout_s=0.3))
    _assert_recovers(g)


def test_hub_ring_overflow():
    # 40 hub lists in one batch, a hub ring of 2 descriptors and a single group: the third
    # publication waits on a slot only this group could free
    edges = [(0, i, 1) for i in range(1, 41)]
    for i in range(1, 41):
        edges += [(i, 41 + (i * 300 + k) % 9000, 5) for k in range(300)]
    g = build_csr(9100, edges)
    cfg = MlmqConfig(l1_type="vector", l2_type="fifo", num_groups=1)
    eng = EngineConfig(hub_chunk=64, hub_threshold=64, test_capacity=2, spin_timeout_s=0.3)
    with pytest.raises(QueueOverflowError, match="hub work ring slot"):
        sssp_solve(g, 0, cfg, eng)
    r = sssp_solve(g, 0, cfg, EngineConfig(hub_chunk=64, hub_threshold=64))
    assert np.array_equal(r.dist_array, _oracle(g))


# ------------------------------------------------------------------ C4 / C5 at full size
@pytest.fixture(scope="module")
def c4_graph():
    from bench import build_graph
    g = build_graph("c4")
    assert oracle.csr_sha256(g.row_offsets, g.col_indices, g.weights) == BIG["c4"]["csr_sha256"]
    return g


def test_c4_kronecker_s26_matches_golden_hash(c4_graph):
    # BASELINE.json configs[3] on one B200 (the whole 1.07 B-edge graph fits in HBM)
    from bench import solve_config, solve_engine
    f = extract_features(c4_graph)
    r = sssp_solve(c4_graph, 0, solve_config("c4", c4_graph, f), solve_engine("c4"), features=f)
    assert oracle.dist_sha256(r.dist_array) == BIG["c4"]["dist_sha256"]
    assert r.metrics.relaxations < 1.2 * BIG["c4"]["e_reach"]  # light/heavy split at work
    r = sssp_solve(c4_graph, 0, solve_config("c4", c4_graph, f), EngineConfig(bucket_window=1), features=f)
    assert oracle.dist_sha256(r.dist_array) == BIG["c4"]["dist_sha256"]
    m = r.metrics
    assert m.l0_enqueues == m.l0_dequeues and m.l2_enqueues == m.l2_dequeues


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_c4_sharded_matches_golden_hash(c4_graph, parts):
    # 1D-partitioned solve, P logical shards on one device, against the hash
    from paper_2602_10080_b200.sharded import sssp_solve_sharded
    res = sssp_solve_sharded(c4_graph, 0, parts, MlmqConfig(l2_type="fifo"))
    assert oracle.dist_sha256(res.local_dist) == BIG["c4"]["dist_sha256"], parts


def test_sharded_light_heavy_split_matches():
    # shards with the light/heavy split (heavy tokens drained inside each superstep)
    from paper_2602_10080_b200.sharded import sssp_solve_sharded
    g = generate_graph("rmat", seed=4, scale=12, edge_factor=16, wmin=1, wmax=255)
    want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    for P in (2, 4, 8):
        res = sssp_solve_sharded(g, 0, P, MlmqConfig(l2_type="fifo"), EngineConfig(heavy_delta=24))
        assert np.array_equal(res.local_dist, want), P
    from bench import build_graph
    c2 = build_graph("c2")
    for P in (2, 8):
        res = sssp_solve_sharded(c2, 0, P, MlmqConfig(l2_type="fifo"), EngineConfig(heavy_delta=24))
        assert oracle.dist_sha256(res.local_dist) == C2_DIST, P


def test_c2_sharded_matches_reference_hash():
    from bench import build_graph
    from paper_2602_10080_b200.sharded import sssp_solve_sharded
    g = build_graph("c2")
    for P in (2, 8):
        res = sssp_solve_sharded(g, 0, P, MlmqConfig(l2_type="fifo"))
        assert oracle.dist_sha256(res.local_dist) == C2_DIST, P


def test_c5_float_weights_match_golden_hash():
    from bench import build_graph, solve_config, solve_engine
    g = build_graph("c5")
    f = extract_features(g)
    for eng in (EngineConfig(), solve_engine("c5")):  # without and with the light/heavy split
        r = sssp_solve(g, 0, solve_config("c5", g, f), eng, features=f)
        d = np.ascontiguousarray(r.dist_array, dtype="<f4")
        assert hashlib.sha256(d.tobytes()).hexdigest() == BIG["c5"]["dist_f32_sha256"]
