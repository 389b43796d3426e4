"""The CPU oracle (oracle/) pinned against the reference's own outputs.

- every graph of tests/golden/reference_vectors.json (made by importing the reference:
  its generators, its dijkstra_oracle, its unit_weight_view) must reproduce the
  reference's dist_sha256 for both sources, weighted and unit-weight;
- the reference-produced hashes of SURVEY §8c / BASELINE.md §4 (C1, RMAT s16, s20; C2
  and C3 under MLMQ_SLOW=1);
- the known-answer cases of the reference's test_engine.py / test_cli.py.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_2602_10080_b200 import build_csr, generate_graph

INF = (1 << 64) - 1

# reference-produced hashes
BIG = [
    ("C1", "grid2d", dict(rows=256, cols=256, wmin=1, wmax=100),
     "fc3d4d1b2aed1a9c5f3c7eea4275aa0b4686ce7dce44852cd4b98a010dc2b119",
     "f40804d404084c2be8d587d8f58312b83e33fc1b109d927ad0e26c201d760e45"),
    ("rmat16", "rmat", dict(scale=16, edge_factor=16, wmin=1, wmax=255),
     "ebf60a9a266d20fba759e183f89ad16f2a701991e41af85fe69659c2a3c70d5a",
     "20a660bb634d7766180f5f8c0de9aeb1bf8aa79c52d849af15c9b6c17fae2ae0"),
    ("rmat20", "rmat", dict(scale=20, edge_factor=16, wmin=1, wmax=255),
     "9591d2bffa1a717c173a9f89a9e7a0bf3daa07961e5d11da97c41ce5427e9daf",
     "c1ef6add7d3fdd5301715e8d8f7fcc6efcd659035d6a31b086cbb087c2d72209"),
]
BIG_SLOW = [
    ("C2", "rmat", dict(scale=22, edge_factor=16, wmin=1, wmax=255),
     "fa759aa4567d9509fe6010c989efa9f31370d0130789e9473a79341d10d8f95e",
     "f6d20099af4ad32ebcc888faa9f557f17b69be966c4c0808093799b5f3840788"),
    ("C3", "grid2d", dict(rows=4900, cols=4900, wmin=1, wmax=100),
     "b2617a4e6e2578ff1bc69965fdea67c7a40ccc5400481ba5ac535a21d1806dc1",
     "2bf8e0cf2ab0c6ab8b906952288c22c564fbda5404ab78d48e8c90590c3bde41"),
]


def _check_big(kind, params, csr_sha, dist_sha):
    g = generate_graph(kind, seed=1, **params)
    assert oracle.csr_sha256(g.row_offsets, g.col_indices, g.weights) == csr_sha
    d = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    assert oracle.dist_sha256(d) == dist_sha


@pytest.mark.parametrize("name,kind,params,csr_sha,dist_sha", BIG, ids=[b[0] for b in BIG])
def test_oracle_reproduces_reference_hashes(name, kind, params, csr_sha, dist_sha):
    _check_big(kind, params, csr_sha, dist_sha)


@pytest.mark.slow
@pytest.mark.parametrize("name,kind,params,csr_sha,dist_sha", BIG_SLOW, ids=[b[0] for b in BIG_SLOW])
def test_oracle_reproduces_reference_hashes_large(name, kind, params, csr_sha, dist_sha):
    _check_big(kind, params, csr_sha, dist_sha)


def test_oracle_matches_reference_golden_vectors(golden):
    checked = 0
    for rec in golden["graphs"]:
        g = generate_graph(rec["kind"], seed=rec["seed"], **rec["params"])
        assert oracle.csr_sha256(g.row_offsets, g.col_indices, g.weights) == rec["csr_sha256"], rec["id"]
        for s in rec["sources"]:
            d = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, s["source"])
            assert oracle.dist_sha256(d) == s["dist_sha256"], (rec["id"], s["source"])
            du = oracle.dijkstra_u64(g.row_offsets, g.col_indices, None, s["source"], unit_weights=True)
            assert oracle.dist_sha256(du) == s["unit_dist_sha256"], (rec["id"], s["source"])
            if "dist" in s:
                assert [None if x == INF else int(x) for x in d] == s["dist"]
            checked += 1
    assert checked == 2 * len(golden["graphs"]) >= 200


def test_bellman_ford_agrees_with_dijkstra(golden):
    for rec in golden["graphs"][::7]:
        g = generate_graph(rec["kind"], seed=rec["seed"], **rec["params"])
        for s in rec["sources"]:
            a = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, s["source"])
            b = oracle.bellman_ford_u64(g.row_offsets, g.col_indices, g.weights, s["source"])
            assert np.array_equal(a, b), rec["id"]


KNOWN = [
    # test_engine.py:42-49 DIAMOND
    (4, [(0, 1, 10), (0, 2, 1), (2, 1, 2), (1, 3, 1), (2, 3, 9)], 0, [0, 3, 1, 4]),
    # test_engine.py:60-62 triangle
    (3, [(0, 1, 1), (1, 2, 1), (0, 2, 3)], 0, [0, 1, 2]),
    # test_engine.py:65-68 unreachable
    (4, [(0, 1, 2)], 0, [0, 2, INF, INF]),
    # test_engine.py:71-73 single vertex
    (1, [], 0, [0]),
    # test_engine.py:76-78 zero weights
    (3, [(0, 1, 0), (1, 2, 0)], 0, [0, 0, 0]),
    # tests/fixtures/tiny.gr (5 vertices, 7 arcs, 1-based in the file) -> test_cli.py:99-106
    (5, [(0, 1, 2), (1, 2, 2), (0, 2, 5), (2, 3, 1), (3, 4, 3), (1, 4, 9), (4, 0, 1)], 0,
     [0, 2, 4, 5, 8]),
]


@pytest.mark.parametrize("n,edges,src,want", KNOWN)
def test_oracle_known_answers(n, edges, src, want):
    g = build_csr(n, edges)
    d = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, src)
    assert [int(x) for x in d] == want


def test_oracle_unit_weights_known_answers():
    # test_engine.py:170-173 / test_cli.py:140-145
    g = build_csr(3, [(0, 1, 50), (1, 2, 50), (0, 2, 200)])
    assert list(oracle.dijkstra_u64(g.row_offsets, g.col_indices, None, 0, unit_weights=True)) == [0, 1, 1]
    tiny = build_csr(5, [(0, 1, 2), (1, 2, 2), (0, 2, 5), (2, 3, 1), (3, 4, 3), (1, 4, 9), (4, 0, 1)])
    du = oracle.dijkstra_u64(tiny.row_offsets, tiny.col_indices, None, 0, unit_weights=True)
    assert list(du) == [0, 1, 1, 2, 2]


def test_oracle_bad_source():
    g = build_csr(2, [(0, 1, 1)])
    with pytest.raises(ValueError, match="out of range"):
        oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 5)


def test_f32_oracle_is_exact_binary32_path_min():
    # on a DAG of doubled paths the f32 result must equal the min over paths of the
    # left-to-right binary32 sums, computed independently with numpy float32
    rng = np.random.default_rng(0)
    n = 40
    edges = []
    for u in range(n - 1):
        for v in (u + 1, min(n - 1, u + 2)):
            edges.append((u, v, float(np.float32(rng.random()))))
    g = build_csr(n, edges)
    d = oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, 0)
    best = np.full(n, np.inf, dtype=np.float32)
    best[0] = np.float32(0)
    for u in range(n):  # topological order
        for k in range(int(g.row_offsets[u]), int(g.row_offsets[u + 1])):
            v = int(g.col_indices[k])
            nd = np.float32(best[u] + g.weights[k])
            if nd < best[v]:
                best[v] = nd
    assert np.array_equal(d, best)
