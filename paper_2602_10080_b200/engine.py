"""SSSP engine entry points: the drop-in for ``mlq_sssp.engine``.

``sssp_solve`` keeps the reference signature (pkg/src/mlq_sssp/engine.py:245-249)
and semantics (exact distances for any schedule, resolved config echoed, metric
identities, EngineError / QueueOverflowError / ValueError on the same
conditions), but the solve runs on the GPU: the CSR graph is uploaded once and
cached on the CsrGraph object, and one call of ``mlmq_sssp`` (libmlmq.so) runs
K3 init -> K1 persistent MLMQ kernel + K2 manager warp -> K5 audit.
There is no CPU fallback.
"""

from __future__ import annotations

import dataclasses
import heapq
import struct
from collections import deque
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _native
from .core import (INF, L1_TYPES, L2_TYPES, METRIC_FIELDS, EngineError, MlmqConfig,
                   RunMetrics)
from .graph import CsrGraph, GraphFeatures, extract_features

DEFAULT_WATCHDOG_S = 60.0


@dataclass
class EngineConfig:
    """Engine-side knobs; None fields fall back to the queue config (engine.py:37-45).

    ``dist_mode``: "auto" (u32 on device, re-run in u64 if a distance overflows),
    "u32" or "u64".  ``hub_chunk``: edges per hub work item (0 = library default).
    """

    num_groups: Optional[int] = None
    lanes_per_group: Optional[int] = None
    th_v: Optional[int] = None
    duplicate_elimination: bool = True
    seed: int = 0
    dist_mode: str = "auto"
    hub_chunk: int = 0
    spin_timeout_s: float = 15.0
    device: int = 0
    share: bool = True       # eager write-back to L2 while groups idle (B200 extension)
    fifo_park: bool = True   # FIFO readers park on unconditional tickets
    bucket_window: int = -1  # bucket L2: winners >= this many buckets above the floor skip L0/L1;
                             # -1 = auto: 1 (managed floor) with >= 64 groups, else 0 (the
                             # reference's floor rule, l2.py:282-287)
    read_batch: int = 64     # elements per L1 read (0 = lanes_per_group, the reference's want)
    hub_threshold: int = 0   # lists longer than this become hub descriptors (0 = 4 x hub_chunk)
    prefetch_targets: bool = False  # warm L2 with the row offsets of every improved target
    heavy_delta: float = 0.0  # FIFO L2: edges with w < heavy_delta are relaxed when a vertex is
                              # expanded, heavier ones later from a deferred token (0 = off)
    heavy_min_edges: int = 0  # defer only rows with at least this many heavy edges (0: every row;
                              # measured best on C2/C5: larger values re-expand the small rows)
    test_capacity: int = 0   # > 0: every queue store gets exactly this many entries (test hook
                             # that forces the QueueOverflowError paths, l2.py:116-135)


class SsspResult:
    """Result of one solve (engine.py:48-54).

    ``distances`` is a list (built lazily from ``dist_array``) so it compares
    ``==`` to lists exactly like the reference; ``dist_array`` is the numpy view
    (uint64 with INF = 2**64-1, or float32 with +inf on float graphs).
    """

    def __init__(self, dist_array: np.ndarray, metrics: RunMetrics, config_used: MlmqConfig,
                 engine_used: EngineConfig, group_shards: np.ndarray, native: dict):
        self.dist_array = dist_array
        self.metrics = metrics
        self.config_used = config_used
        self.engine_used = engine_used
        self._group_shards = group_shards
        self._group_metrics = None
        self._distances = None
        self.native = native

    @property
    def distances(self) -> List:
        if self._distances is None:
            self._distances = self.dist_array.tolist()
        return self._distances

    @property
    def group_metrics(self) -> List[RunMetrics]:
        if self._group_metrics is None:
            out = []
            for row in self._group_shards.tolist():
                out.append(RunMetrics(**dict(zip(METRIC_FIELDS, (int(x) for x in row)))))
            self._group_metrics = out
        return self._group_metrics

    @property
    def kernel_ms(self) -> float:
        return float(self.native.get("kernel_ms", 0.0))

    def __repr__(self) -> str:
        return (f"SsspResult(n={self.dist_array.size}, metrics={self.metrics}, "
                f"config_used={self.config_used})")


def resolve_config(config: MlmqConfig, engine: Optional[EngineConfig],
                   graph: Optional[CsrGraph] = None,
                   features: Optional[GraphFeatures] = None) -> Tuple[MlmqConfig, EngineConfig]:
    """Fill graph-dependent defaults and merge engine overrides (engine.py:57-103).

    Returns fresh objects; the caller's configs are never mutated.  On float-weight
    graphs the Δ-type defaults keep the unrounded average weight.
    ``num_groups=None`` ("auto") stays None here and is resolved against the device
    by ``sssp_solve``; ``pnum`` then follows the resolved group count.
    """
    cfg = dataclasses.replace(config, l1_params=dataclasses.replace(config.l1_params),
                              l2_params=dataclasses.replace(config.l2_params))
    eng = dataclasses.replace(engine) if engine is not None else EngineConfig()
    if eng.num_groups is not None:
        cfg.num_groups = eng.num_groups
    else:
        eng.num_groups = cfg.num_groups
    if eng.lanes_per_group is not None:
        cfg.lanes_per_group = eng.lanes_per_group
    else:
        eng.lanes_per_group = cfg.lanes_per_group
    if eng.th_v is not None:
        cfg.th_v = eng.th_v
    else:
        eng.th_v = cfg.th_v

    feats = features

    def avg_weight():
        nonlocal feats
        if feats is None:
            if graph is None:
                return 1
            feats = extract_features(graph)
        if feats.float_weights:
            return float(feats.avg_weight) if feats.avg_weight > 0 else 1.0
        return max(1, round(feats.avg_weight))

    l2p = cfg.l2_params
    if cfg.l2_type == "bucket" and l2p.delta is None:
        l2p.delta = avg_weight()
    if l2p.pnum is None and cfg.num_groups is not None:
        l2p.pnum = max(1, cfg.num_groups // 4)
    l1p = cfg.l1_params
    if cfg.l1_type == "near_far" and l1p.delta_nf is None:
        l1p.delta_nf = l2p.delta if cfg.l2_type == "bucket" else avg_weight()
    if cfg.l1_type == "filter" and l1p.filter_f is None:
        l1p.filter_f = 4 * avg_weight()
    cfg.validate()
    return cfg, eng


_DIST_MODES = {"auto": _native.DIST_AUTO, "u32": _native.DIST_U32, "u64": _native.DIST_U64}


def _native_config(cfg: MlmqConfig, eng: EngineConfig, unit_weights: bool,
                   watchdog_s: float) -> _native.Config:
    c = _native.Config()
    c.l1_type = L1_TYPES.index(cfg.l1_type)
    c.l2_type = L2_TYPES.index(cfg.l2_type)
    c.l0_capacity = cfg.l0_capacity
    c.l1_capacity = cfg.l1_params.capacity
    c.wb = cfg.l1_params.wb
    c.delta_nf = float(cfg.l1_params.delta_nf or 0)
    c.filter_f = float(cfg.l1_params.filter_f or 0)
    c.delta = float(cfg.l2_params.delta or 1)
    c.block_size = cfg.l2_params.block_size
    c.block_num = cfg.l2_params.block_num
    c.bmax = cfg.l2_params.bmax
    c.bnum = cfg.l2_params.bnum
    c.node_batch = cfg.l2_params.node_batch
    nq = cfg.num_groups or 1
    # a reader-less heap would strand work: clamp like l2.py:421
    c.pnum = max(1, min(cfg.l2_params.pnum or 1, nq))
    c.num_groups = cfg.num_groups or 0
    c.lanes_per_group = cfg.lanes_per_group
    c.th_v = cfg.th_v
    c.dup_elim = 1 if eng.duplicate_elimination else 0
    c.unit_weights = 1 if unit_weights else 0
    if eng.dist_mode not in _DIST_MODES:
        raise ValueError(f"unknown dist_mode {eng.dist_mode!r}")
    c.dist_mode = _DIST_MODES[eng.dist_mode]
    c.watchdog_s = float(watchdog_s or 0)
    c.spin_timeout_s = float(eng.spin_timeout_s)
    c.hub_chunk = int(eng.hub_chunk)
    c.share = 1 if eng.share else 0
    c.fifo_park = 1 if eng.fifo_park else 0
    bw = int(eng.bucket_window)
    if bw < 0:
        bw = 1 if (cfg.num_groups is None or cfg.num_groups >= 64) else 0
    c.bucket_window = bw
    c.read_batch = max(0, int(eng.read_batch))
    c.hub_threshold = max(0, int(eng.hub_threshold))
    c.test_capacity = max(0, int(eng.test_capacity))
    c.flags = (1 if eng.prefetch_targets else 0) | (max(0, min(0xFFFF, int(eng.heavy_min_edges))) << 8)
    hd = float(eng.heavy_delta or 0.0)
    c.heavy_delta = int(round(hd)) if hd >= 1 else 0
    c.heavy_delta_f = hd if hd > 0 else 0.0
    return c


def device_graph(graph: CsrGraph, device: int = 0) -> "_native.DeviceGraph":
    """Device copy of ``graph``, uploaded on first use and cached on the object."""
    cached = getattr(graph, "_mlmq_device", None)
    if cached is not None and cached[0] == device and cached[1].handle:
        return cached[1]
    if graph.float_weights:
        kind, w = _native.W_F32, graph.weights
    else:
        if graph.weights.dtype == np.uint64:
            raise ValueError("edge weights >= 2^32 are not supported by the GPU engine")
        kind, w = _native.W_U32, graph.weights
    dg = _native.DeviceGraph(graph.row_offsets, graph.col_indices, w, kind, device)
    object.__setattr__(graph, "_mlmq_device", (device, dg))
    return dg


def prepare(graph: CsrGraph, source: int, config: Optional[MlmqConfig] = None,
            engine: Optional[EngineConfig] = None, *, features: Optional[GraphFeatures] = None,
            unit_weights: bool = False, watchdog_s: float = DEFAULT_WATCHDOG_S):
    """Resolve a config against the device: returns (cfg, eng, DeviceGraph, native cfg)."""
    cfg, eng = resolve_config(config or MlmqConfig(), engine, graph, features)
    if not (0 <= source < graph.num_vertices):
        raise ValueError(f"source {source} out of range for {graph.num_vertices} vertices")
    dg = device_graph(graph, eng.device)
    ncfg = _native_config(cfg, eng, unit_weights, watchdog_s)
    if cfg.num_groups is None:
        g = dg.auto_groups(ncfg)
        cfg.num_groups = g
        eng.num_groups = g
        if cfg.l2_params.pnum is None:
            cfg.l2_params.pnum = max(1, g // 4)
        ncfg = _native_config(cfg, eng, unit_weights, watchdog_s)
    return cfg, eng, dg, ncfg


def sssp_solve(graph: CsrGraph, source: int, config: Optional[MlmqConfig] = None,
               engine: Optional[EngineConfig] = None, *,
               features: Optional[GraphFeatures] = None,
               unit_weights: bool = False,
               watchdog_s: float = DEFAULT_WATCHDOG_S) -> SsspResult:
    """Single-source shortest paths on the GPU MLMQ engine; exact for any schedule.

    Raises ValueError for a bad source or config, QueueOverflowError when a queue
    ring cannot absorb the workload, EngineError when the watchdog expires, the
    post-run audit fails or no device is available.
    """
    cfg, eng, dg, ncfg = prepare(graph, source, config, engine, features=features,
                                 unit_weights=unit_weights, watchdog_s=watchdog_s)
    dist, m, gm = dg.sssp(int(source), ncfg, want_groups=int(cfg.num_groups))
    metrics = RunMetrics(**{f: int(getattr(m, f)) for f in METRIC_FIELDS})
    metrics.wall_time_us = int(m.wall_time_us)
    native = {"kernel_ms": float(m.kernel_ms), "num_groups": int(m.num_groups),
              "hub_items": int(m.hub_items), "dist_bits": int(m.dist_bits),
              "reruns": int(m.reruns)}
    return SsspResult(dist, metrics, cfg, eng, gm, native)


def bfs_solve(graph: CsrGraph, source: int, config: Optional[MlmqConfig] = None,
              engine: Optional[EngineConfig] = None, *,
              watchdog_s: float = DEFAULT_WATCHDOG_S) -> SsspResult:
    """Hop distances: the same engine reading every weight as 1 (engine.py:300-305)."""
    return sssp_solve(graph, source, config, engine, unit_weights=True, watchdog_s=watchdog_s)


# ---------------------------------------------------------------------------
# Exact host-side reference solvers (API of engine.py:313-366).  These are the
# package's user-facing checkers for small graphs; the solve path never calls them.
# ---------------------------------------------------------------------------


def dijkstra_oracle(graph: CsrGraph, source: int) -> List[int]:
    """Binary-heap Dijkstra with stale-entry skipping, exact integers."""
    n = graph.num_vertices
    if not (0 <= source < n):
        raise ValueError(f"source {source} out of range for {n} vertices")
    off = graph.row_offsets.tolist()
    col = graph.col_indices.tolist()
    w = graph.weights.tolist()
    inf = float("inf") if graph.float_weights else INF
    dist = [inf] * n
    dist[source] = 0
    done = bytearray(n)
    pq = [(0, source)]
    while pq:
        d, u = heapq.heappop(pq)
        if done[u]:
            continue
        done[u] = 1
        for k in range(off[u], off[u + 1]):
            v = col[k]
            nd = d + w[k]
            if nd < dist[v]:
                dist[v] = nd
                heapq.heappush(pq, (nd, v))
    return dist


def bellman_ford_oracle(graph: CsrGraph, source: int) -> List[int]:
    """FIFO label-correcting solver; an independent cross-check."""
    n = graph.num_vertices
    if not (0 <= source < n):
        raise ValueError(f"source {source} out of range for {n} vertices")
    off = graph.row_offsets.tolist()
    col = graph.col_indices.tolist()
    w = graph.weights.tolist()
    dist = [INF] * n
    dist[source] = 0
    queued = bytearray(n)
    q = deque([source])
    queued[source] = 1
    while q:
        u = q.popleft()
        queued[u] = 0
        du = dist[u]
        for k in range(off[u], off[u + 1]):
            v = col[k]
            nd = du + w[k]
            if nd < dist[v]:
                dist[v] = nd
                if not queued[v]:
                    queued[v] = 1
                    q.append(v)
    return dist


def unit_weight_view(graph: CsrGraph) -> CsrGraph:
    """Same topology, every weight 1 (arrays shared)."""
    return CsrGraph(graph.num_vertices, graph.num_edges, graph.row_offsets, graph.col_indices,
                    np.ones(graph.num_edges, dtype=np.uint32))


def compare_distances(a, b) -> Optional[Tuple[int, int, int]]:
    """First (vertex, a_value, b_value) mismatch, or None when identical."""
    if len(a) != len(b):
        return (-1, len(a), len(b))
    aa = np.asarray(a)
    bb = np.asarray(b)
    if aa.dtype != object and bb.dtype != object:
        diff = np.nonzero(aa != bb)[0]
        if diff.size == 0:
            return None
        i = int(diff[0])
        return (i, a[i] if not isinstance(a, np.ndarray) else aa[i].item(),
                b[i] if not isinstance(b, np.ndarray) else bb[i].item())
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return (i, x, y)
    return None


def distances_blob(distances) -> bytes:
    """Little-endian uint64 packing, the byte-identity currency (engine.py:385-387)."""
    if isinstance(distances, np.ndarray) and distances.dtype == np.uint64:
        return distances.astype("<u8", copy=False).tobytes()
    return struct.pack(f"<{len(distances)}Q", *distances)
