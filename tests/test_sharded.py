"""Sharded (1D-partitioned) solve: the host-side driver on CPU (gloo,
world_size 2, and the single-process logical mode) with a host backend that restates the
shard kernel's superstep semantics, and -- under ``-m gpu`` -- the GPU shards through
libmlmq.so against the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2602_10080_b200 import generate_graph
from paper_2602_10080_b200.graph import generate_grid2d, with_f32_weights
from paper_2602_10080_b200.sharded import (local_count, merge_local, owner, shard_csr,
                                           solve_distributed, solve_logical)

U32_INF = 0xFFFFFFFF


class HostShard:
    """CPU restatement of one shard's superstep (mlmq_shard_step): apply the inbox,
    relax to local quiescence (FIFO worklist), prune remote relaxations against the
    ghost copy, emit improvements grouped by owner.  Test infrastructure only."""

    device = torch.device("cpu")

    def __init__(self, graph, nparts, rank):
        self.P, self.r, self.n = nparts, rank, graph.num_vertices
        self.row, self.col, self.w = shard_csr(graph, nparts, rank)
        self.shift = nparts.bit_length() - 1

    def begin(self):
        self.dist = np.full(self.row.size - 1, U32_INF, dtype=np.uint64)
        self.ghost = np.full(self.n, U32_INF, dtype=np.uint64)

    def empty_inbox(self):
        return torch.empty(0, dtype=torch.int32)

    def make_inbox(self, pairs):
        return torch.as_tensor(pairs.astype(np.uint32).view(np.int32).reshape(-1))

    def step(self, inbox):
        pairs = inbox.numpy().view(np.uint32).reshape(-1, 2)
        work = []
        for v, d in pairs:
            lv = int(v) >> self.shift
            assert owner(int(v), self.P) == self.r
            if d < self.dist[lv]:
                self.dist[lv] = d
                work.append(lv)
        out = []
        while work:
            u = work.pop(0)
            du = int(self.dist[u])
            for k in range(int(self.row[u]), int(self.row[u + 1])):
                v, nd = int(self.col[k]), du + int(self.w[k])
                if owner(v, self.P) == self.r:
                    lv = v >> self.shift
                    if nd < self.dist[lv]:
                        self.dist[lv] = nd
                        work.append(lv)
                elif nd < self.ghost[v]:
                    self.ghost[v] = nd
                    out.append((v, nd))
        out.sort(key=lambda x: owner(x[0], self.P))
        counts = [sum(1 for v, _ in out if owner(v, self.P) == q) for q in range(self.P)]
        arr = np.array(out, dtype=np.uint32).reshape(-1, 2)
        return torch.as_tensor(arr.view(np.int32).reshape(-1)), counts

    def local_dist(self):
        d = self.dist.copy()
        d[d == U32_INF] = np.uint64(0xFFFFFFFFFFFFFFFF)
        return d


def test_shard_csr_partition_covers_graph():
    g = generate_graph("rmat", seed=3, scale=9, edge_factor=8, wmin=1, wmax=50)
    for P in (1, 2, 4, 8):
        tot = 0
        for r in range(P):
            row, col, w = shard_csr(g, P, r)
            assert row.size - 1 == local_count(g.num_vertices, P, r)
            verts = np.arange(r, g.num_vertices, P)
            for i in (0, len(verts) // 2, len(verts) - 1):
                u = verts[i]
                lo, hi = g.row_offsets[u], g.row_offsets[u + 1]
                assert np.array_equal(col[row[i]:row[i + 1]], g.col_indices[lo:hi])
                assert np.array_equal(w[row[i]:row[i + 1]], g.weights[lo:hi])
            tot += col.size
        assert tot == g.num_edges
    with pytest.raises(ValueError):
        shard_csr(g, 3, 0)


def test_merge_local_interleaves():
    d = [np.array([0, 2, 4]), np.array([1, 3])]
    assert merge_local(d, 5).tolist() == [0, 1, 2, 3, 4]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_logical_superstep_protocol_matches_oracle(P):
    for g in (generate_graph("rmat", seed=5, scale=9, edge_factor=6, wmin=1, wmax=255),
              generate_grid2d(12, 17, 1, 100, seed=2)):
        for s in (0, g.num_vertices // 3):
            res = solve_logical([HostShard(g, P, r) for r in range(P)], s)
            want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, s)
            assert np.array_equal(res.local_dist, want)
            assert res.steps >= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "rmat":
            g = generate_graph("rmat", seed=7, scale=9, edge_factor=8, wmin=1, wmax=255)
        else:
            g = generate_grid2d(15, 11, 1, 60, seed=4)
        res = solve_distributed(HostShard(g, world, rank), 0)
        out = [None] * world
        dist.all_gather_object(out, (rank, res.local_dist, res.steps))
        if rank == 0:
            out.sort(key=lambda x: x[0])
            merged = merge_local([o[1] for o in out], g.num_vertices)
            want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
            q.put((bool(np.array_equal(merged, want)), out[0][2]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["rmat", "grid"])
def test_distributed_gloo_world2(kind):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok, steps = q.get(timeout=10)
    assert ok and steps >= 1


# --------------------------------------------------------------------------- GPU shards
@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_gpu_shards_match_oracle(P):
    from paper_2602_10080_b200 import MlmqConfig
    from paper_2602_10080_b200.sharded import sssp_solve_sharded
    for g in (generate_graph("rmat", seed=1, scale=14, edge_factor=16, wmin=1, wmax=255),
              generate_grid2d(64, 48, 1, 100, seed=3)):
        for s in (0, 777):
            res = sssp_solve_sharded(g, s, P, MlmqConfig(l2_type="fifo", num_groups=None))
            want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, s)
            assert np.array_equal(res.local_dist, want), (P, s)


@pytest.mark.gpu
def test_gpu_shards_float_weights_and_configs():
    from paper_2602_10080_b200 import L1Params, MlmqConfig
    from paper_2602_10080_b200.sharded import sssp_solve_sharded
    g = with_f32_weights(generate_graph("rmat", seed=2, scale=12, edge_factor=8), seed=5)
    want = oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, 0)
    for l1 in ("vector", "near_far", "filter", "slf"):
        res = sssp_solve_sharded(g, 0, 4, MlmqConfig(l1_type=l1, l2_type="fifo",
                                                     l1_params=L1Params(capacity=256), num_groups=64))
        assert np.array_equal(res.local_dist, want), l1
    with pytest.raises(ValueError):
        sssp_solve_sharded(g, 0, 2, MlmqConfig(l2_type="bucket"))
