"""1D-partitioned multi-GPU SSSP (BASELINE config C4).

The reference has no distributed path (PAPER.md:797 names a multi-GPU
"L3 queue" as future work).  This module is the B200 one, built on the shard entry points
of the C ABI (include/mlmq.h ``mlmq_shard_*``):

* **Partition.**  Shard ``r`` of ``P`` (a power of two) owns the vertices ``v`` with
  ``v mod P == r`` -- a cyclic owner spreads the RMAT/Kronecker hubs that cluster at low
  ids (graph.py:385-399) -- stored at local id ``v // P``; it holds those vertices'
  out-edges (columns keep global ids), their distances, its own MLMQ queues and a ghost
  copy of remote distances.
* **Supersteps.**  Each shard runs the persistent MLMQ kernel to local quiescence.  A
  relaxation of a remote edge is pruned against the ghost copy and otherwise appended to
  an outbox, grouped by owner after the step.  The outboxes are exchanged with one NCCL
  all-to-all-v (``torch.distributed.all_to_all_single``) and become the next step's
  inboxes; the solve ends when an all-reduce of the sent counts is zero.
* **Process model.**  One process per GPU (``torchrun``), or -- for tests and single-GPU
  boxes -- every shard in one process on one device (``solve_logical``), exchanging by
  slicing device tensors.  The exchange/termination driver is the same code in both, and
  takes any backend with ``begin() / step(inbox) / local_dist()``, so it is exercised on
  CPU with ``gloo`` and a host backend (tests/test_sharded.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .core import INF, MlmqConfig
from .engine import (DEFAULT_WATCHDOG_S, EngineConfig, _native_config, resolve_config)
from .graph import CsrGraph


def owner(v, nparts: int):
    return v & (nparts - 1)


def local_count(n: int, nparts: int, rank: int) -> int:
    """Vertices owned by ``rank``: ceil((n - rank) / nparts)."""
    return max(0, (n - rank + nparts - 1) // nparts)


def shard_csr(graph: CsrGraph, nparts: int, rank: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Rows of the vertices ``rank, rank + P, ...`` in local order; global column ids."""
    if nparts < 1 or nparts & (nparts - 1):
        raise ValueError(f"nparts must be a power of two (got {nparts})")
    off = graph.row_offsets
    verts = np.arange(rank, graph.num_vertices, nparts, dtype=np.int64)
    starts = off[verts].astype(np.int64)
    deg = off[verts + 1].astype(np.int64) - starts
    row = np.zeros(verts.size + 1, dtype=np.uint64)
    np.cumsum(deg, out=row[1:])
    total = int(row[-1])
    if total:
        # edge k of local row i sits at starts[i] + (k - row[i])
        idx = np.repeat(starts - row[:-1].astype(np.int64), deg) + np.arange(total, dtype=np.int64)
        col = graph.col_indices[idx]
        w = graph.weights[idx]
    else:
        col = np.zeros(0, dtype=np.uint32)
        w = np.zeros(0, dtype=graph.weights.dtype)
    return row, col, w


def merge_local(dists: Sequence[np.ndarray], n: int) -> np.ndarray:
    """Global distance array from per-shard arrays (shard r, local i -> v = i * P + r)."""
    P = len(dists)
    out = np.empty(n, dtype=dists[0].dtype)
    for r, d in enumerate(dists):
        out[r::P] = d
    return out


class GpuShard:
    """Backend: one shard on one GPU through libmlmq.so.

    ``graph`` may be None when ``shard=(row, col, w)`` and ``n_global`` are given (a rank
    that generated only its own slice, ``_native.generate_shard``); the Δ-type defaults
    then need ``features`` of the whole graph or explicit config values."""

    def __init__(self, graph: Optional[CsrGraph], nparts: int, rank: int, config: Optional[MlmqConfig] = None,
                 engine: Optional[EngineConfig] = None, *, device: int = 0,
                 watchdog_s: float = DEFAULT_WATCHDOG_S, send_cap: Optional[int] = None,
                 shard: Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]] = None,
                 n_global: Optional[int] = None, features=None):
        import torch
        self.torch = torch
        if graph is None and (shard is None or n_global is None):
            raise ValueError("without a graph, pass shard=(row, col, w) and n_global")
        self.nparts, self.rank = nparts, rank
        self.n_global = graph.num_vertices if graph is not None else int(n_global)
        cfg, eng = resolve_config(config or MlmqConfig(l2_type="fifo"), engine, graph, features)
        if cfg.l2_type != "fifo":
            raise ValueError("sharded solves run the FIFO L2 queue")
        row, col, w = shard if shard is not None else shard_csr(graph, nparts, rank)
        fw = graph.float_weights if graph is not None else np.asarray(w).dtype == np.float32
        kind = _native.W_F32 if fw else _native.W_U32
        self.dg = _native.DeviceShard(row, col, w, kind, self.n_global, rank, nparts, device)
        self.m_local = int(col.size)
        ncfg = _native_config(cfg, eng, False, watchdog_s)
        if cfg.num_groups is None:
            cfg.num_groups = self.dg.auto_groups(ncfg)
            ncfg = _native_config(cfg, eng, False, watchdog_s)
        self.cfg, self.ncfg = cfg, ncfg
        self.device = torch.device("cuda", device)
        # every remote relaxation can improve a ghost at most once per superstep and edge;
        # the kernel reports an overflow instead of writing past the buffer
        # (fire-and-forget ghost updates may send an improvement twice when two edges race,
        # and each group reserves outbox slots 512 at a time: leave room for both)
        cap = send_cap if send_cap is not None else max(1 << 16, 2 * self.m_local + self.dg.n + (1 << 21))
        self.send = torch.empty(2 * cap, dtype=torch.int32, device=self.device)
        self.send_cap = cap
        self.metrics: List[_native.Metrics] = []
        self.lib_stream = torch.cuda.ExternalStream(self.dg.stream_ptr(), device=self.device)

    def begin(self) -> None:
        self.dg.begin()
        self.metrics = []

    def step(self, inbox):
        """inbox: int32 device tensor of (global v, d) pairs.  Returns (send tensor of pairs
        grouped by owner, per-owner counts)."""
        n_in = int(inbox.numel() // 2)
        # the inbox was produced on torch's stream (all-to-all / slicing); the library
        # runs on its own stream: order them with an event (no host synchronisation)
        self.lib_stream.wait_stream(self.torch.cuda.current_stream(self.device))
        counts, m = self.dg.step(self.ncfg, inbox.data_ptr() if n_in else 0, n_in,
                                 self.send.data_ptr(), self.send_cap)
        self.metrics.append(m)
        tot = int(counts.sum())
        return self.send[: 2 * tot], [int(c) for c in counts]

    def empty_inbox(self):
        return self.torch.empty(0, dtype=self.torch.int32, device=self.device)

    def make_inbox(self, pairs: np.ndarray):
        return self.torch.as_tensor(pairs.astype(np.uint32).view(np.int32).reshape(-1), device=self.device)

    def local_dist(self) -> np.ndarray:
        return self.dg.last_dist()

    def reach(self) -> Tuple[int, int]:
        return self.dg.reach()

    def kernel_ms(self) -> float:
        return float(sum(m.kernel_ms for m in self.metrics))


def _source_inbox(backend, source: int, nparts: int, rank: int, zero_bits: int = 0):
    if owner(source, nparts) == rank:
        return backend.make_inbox(np.array([[source, zero_bits]], dtype=np.uint32))
    return backend.empty_inbox()


@dataclass
class ShardedResult:
    local_dist: np.ndarray
    steps: int
    sent: int
    kernel_ms: float = 0.0    # superstep kernels (library CUDA events), this rank / all shards
    exchange_ms: float = 0.0  # all-to-all + termination all-reduce (CUDA events on torch's stream)


def _backend_ms(backend) -> float:
    f = getattr(backend, "kernel_ms", None)
    return float(f()) if f else 0.0


class _Clock:
    """Accumulates device time of the exchange phases on torch's current stream."""

    def __init__(self, device):
        import torch
        self.on = device.type == "cuda"
        self.ms = 0.0
        if self.on:
            self.a, self.b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def start(self):
        if self.on:
            self.a.record()

    def stop(self):
        if self.on:
            self.b.record()
            self.b.synchronize()
            self.ms += self.a.elapsed_time(self.b)


def solve_distributed(backend, source: int, group=None, max_steps: int = 1 << 20) -> ShardedResult:
    """Superstep driver for one rank (torch.distributed initialised; NCCL on GPUs, gloo
    with a host backend).  Every rank calls it with the same source."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = backend.device
    backend.begin()
    inbox = _source_inbox(backend, source, P, r)
    steps = sent = 0
    clk = _Clock(dev)
    while steps < max_steps:
        send, counts = backend.step(inbox)
        steps += 1
        clk.start()
        # one collective + one host read per superstep: every rank gathers the whole
        # P x P count matrix, which gives both its receive sizes (its column) and the
        # global termination test (matrix sum == 0)
        c = torch.tensor(counts, dtype=torch.int64, device=dev)
        mat = torch.empty(P * P, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(mat, c, group=group)
        m = mat.view(P, P).tolist()
        if sum(map(sum, m)) == 0:
            clk.stop()
            break
        rcounts = [int(m[src][r]) for src in range(P)]
        recv = torch.empty(2 * sum(rcounts), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=[2 * x for x in rcounts],
                               input_split_sizes=[2 * x for x in counts], group=group)
        clk.stop()
        sent += sum(counts)
        inbox = recv
    return ShardedResult(backend.local_dist(), steps, sent, _backend_ms(backend), clk.ms)


def solve_logical(backends: Sequence, source: int, max_steps: int = 1 << 20) -> ShardedResult:
    """Every shard in this process (one device or several): the same superstep protocol
    with the all-to-all done by slicing.  Returns the merged global distances."""
    import torch
    P = len(backends)
    for b in backends:
        b.begin()
    inboxes = [_source_inbox(b, source, P, r) for r, b in enumerate(backends)]
    steps = sent = 0
    clk = _Clock(backends[0].device)
    while steps < max_steps:
        outs = [b.step(inboxes[r]) for r, b in enumerate(backends)]
        steps += 1
        total = sum(sum(c) for _, c in outs)
        if total == 0:
            break
        clk.start()
        sent += total
        nxt = []
        for dst in range(P):
            parts = []
            for src, (send, counts) in enumerate(outs):
                lo = 2 * sum(counts[:dst])
                parts.append(send[lo: lo + 2 * counts[dst]].to(backends[dst].device))
            nxt.append(torch.cat(parts) if parts else backends[dst].empty_inbox())
        inboxes = nxt
        clk.stop()
    dists = [b.local_dist() for b in backends]
    n = sum(d.size for d in dists)
    return ShardedResult(merge_local(dists, n), steps, sent, sum(_backend_ms(b) for b in backends), clk.ms)


def sssp_solve_sharded(graph: CsrGraph, source: int, nparts: int, config: Optional[MlmqConfig] = None,
                       engine: Optional[EngineConfig] = None, *, device: int = 0,
                       watchdog_s: float = DEFAULT_WATCHDOG_S) -> ShardedResult:
    """Convenience: ``nparts`` shards of ``graph`` on one device (logical partitions)."""
    if not (0 <= source < graph.num_vertices):
        raise ValueError(f"source {source} out of range for {graph.num_vertices} vertices")
    backends = [GpuShard(graph, nparts, r, config, engine, device=device, watchdog_s=watchdog_s)
                for r in range(nparts)]
    return solve_logical(backends, source)


__all__ = ["GpuShard", "ShardedResult", "local_count", "merge_local", "owner", "shard_csr",
           "solve_distributed", "solve_logical", "sssp_solve_sharded", "INF"]
