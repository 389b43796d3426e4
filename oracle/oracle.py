"""ctypes wrapper over oracle/liboracle.so — TEST INFRASTRUCTURE ONLY.

Restates dijkstra_oracle (pkg/src/mlq_sssp/engine.py:313-338) and
bellman_ford_oracle (engine.py:341-366) in C; see sssp_oracle.c for the citations.
Inputs are numpy CSR arrays (row_offsets u64, col u32, weights u32 or f32).
ctypes releases the GIL during the call, so several solves can run on host threads
at once (bench.py's cpu_baseline uses that to occupy every host core).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

U64_INF = np.uint64(0xFFFFFFFFFFFFFFFF)


def build() -> str:
    """Compile liboracle.so in place (gcc, strict IEEE flags)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "sssp_oracle.c"))):
        try:
            build()
        except (OSError, subprocess.CalledProcessError):
            if not os.path.exists(_LIB_PATH):
                raise
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    U64 = ctypes.c_uint64
    lib.oracle_dijkstra_u64.argtypes = [U64, P, P, P, ctypes.c_int, U64, P]
    lib.oracle_dijkstra_u64.restype = ctypes.c_int
    lib.oracle_bellman_ford_u64.argtypes = [U64, P, P, P, ctypes.c_int, U64, P]
    lib.oracle_bellman_ford_u64.restype = ctypes.c_int
    lib.oracle_dijkstra_f32.argtypes = [U64, P, P, P, U64, P]
    lib.oracle_dijkstra_f32.restype = ctypes.c_int
    lib.oracle_reach_u64.argtypes = [U64, P, P, P, P]
    lib.oracle_reach_u64.restype = None
    lib.mlmq_gen_size.argtypes = [ctypes.c_int, P, P, P]
    lib.mlmq_gen_size.restype = ctypes.c_int
    lib.mlmq_gen_graph.argtypes = [ctypes.c_int, P, P, U64, P, P, P]
    lib.mlmq_gen_graph.restype = ctypes.c_int
    lib.mlmq_gen_f32_weights.argtypes = [U64, U64, P]
    lib.mlmq_gen_f32_weights.restype = ctypes.c_int
    lib.oracle_last_error.argtypes = []
    lib.oracle_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _arrays(row_offsets, col_indices, weights):
    off = np.ascontiguousarray(row_offsets, dtype=np.uint64)
    col = np.ascontiguousarray(col_indices, dtype=np.uint32)
    w = None if weights is None else np.ascontiguousarray(weights)
    return off, col, w


def _check(rc: int, source: int, n: int):
    if rc == 1:
        raise ValueError(f"source {source} out of range for {n} vertices")
    if rc != 0:
        raise MemoryError("oracle allocation failed")


def dijkstra_u64(row_offsets, col_indices, weights, source: int,
                 unit_weights: bool = False) -> np.ndarray:
    """Exact integer distances (u64, INF = 2**64-1); engine.py:313-338."""
    lib = _load()
    off, col, w = _arrays(row_offsets, col_indices, weights)
    n = off.size - 1
    if not unit_weights:
        w = np.ascontiguousarray(w, dtype=np.uint32)
    dist = np.empty(max(n, 0), dtype=np.uint64)
    rc = lib.oracle_dijkstra_u64(n, off.ctypes.data, col.ctypes.data,
                                 None if unit_weights else w.ctypes.data,
                                 int(bool(unit_weights)), source, dist.ctypes.data)
    _check(rc, source, n)
    return dist


def bellman_ford_u64(row_offsets, col_indices, weights, source: int,
                     unit_weights: bool = False) -> np.ndarray:
    """Queue-based label correcting; engine.py:341-366."""
    lib = _load()
    off, col, w = _arrays(row_offsets, col_indices, weights)
    n = off.size - 1
    if not unit_weights:
        w = np.ascontiguousarray(w, dtype=np.uint32)
    dist = np.empty(max(n, 0), dtype=np.uint64)
    rc = lib.oracle_bellman_ford_u64(n, off.ctypes.data, col.ctypes.data,
                                     None if unit_weights else w.ctypes.data,
                                     int(bool(unit_weights)), source, dist.ctypes.data)
    _check(rc, source, n)
    return dist


def dijkstra_f32(row_offsets, col_indices, weights, source: int) -> np.ndarray:
    """f32 Dijkstra with strict binary32 adds (extension for config 5)."""
    lib = _load()
    off, col, w = _arrays(row_offsets, col_indices, weights)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n = off.size - 1
    dist = np.empty(max(n, 0), dtype=np.float32)
    rc = lib.oracle_dijkstra_f32(n, off.ctypes.data, col.ctypes.data, w.ctypes.data,
                                 source, dist.ctypes.data)
    _check(rc, source, n)
    return dist


def reach(row_offsets, dist_u64: np.ndarray) -> Tuple[int, int]:
    """(V_reach, E_reach) of an integer distance vector."""
    lib = _load()
    off = np.ascontiguousarray(row_offsets, dtype=np.uint64)
    d = np.ascontiguousarray(dist_u64, dtype=np.uint64)
    v = ctypes.c_uint64()
    e = ctypes.c_uint64()
    lib.oracle_reach_u64(off.size - 1, off.ctypes.data, d.ctypes.data,
                         ctypes.byref(v), ctypes.byref(e))
    return int(v.value), int(e.value)


def dist_sha256(dist_u64: np.ndarray) -> str:
    """sha256 of distances_blob (engine.py:385-387): little-endian u64, INF all-ones."""
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(dist_u64, dtype="<u8").tobytes()).hexdigest()


class _GenParams(ctypes.Structure):
    """mlmq_gen_params_t (include/mlmq.h)"""
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("n", ctypes.c_int64),
                ("m", ctypes.c_int64), ("scale", ctypes.c_int64), ("edge_factor", ctypes.c_int64),
                ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
                ("d", ctypes.c_double), ("wmin", ctypes.c_int64), ("wmax", ctypes.c_int64)]


_GEN_KINDS = {"grid2d": 0, "path": 1, "uniform": 2, "rmat": 3}
_GEN_DEFAULTS = {"rmat": dict(edge_factor=8, a=0.57, b=0.19, c=0.19, d=0.05, wmin=1, wmax=100),
                 "grid2d": dict(wmin=1, wmax=1), "path": dict(wmin=1, wmax=1),
                 "uniform": dict(wmin=1, wmax=100)}


def generate(kind: str, seed: int = 0, **params):
    """The reference generators (graph.py:306-420; defaults graph.py:310-362) from the
    oracle library's own copy of the restatement -- for checkers and the bench's CPU
    reference arm, which must not load the product library.  Returns (off, col, w)."""
    lib = _load()
    gp = _GenParams()
    for k, v in {**_GEN_DEFAULTS[kind], **params}.items():
        setattr(gp, k, v)
    n, m = ctypes.c_uint64(), ctypes.c_uint64()
    if lib.mlmq_gen_size(_GEN_KINDS[kind], ctypes.byref(gp), ctypes.byref(n), ctypes.byref(m)):
        raise ValueError(lib.oracle_last_error().decode())
    off = np.empty(n.value + 1, dtype=np.uint64)
    col = np.empty(m.value, dtype=np.uint32)
    w = np.empty(m.value, dtype=np.uint32)
    s, limbs = abs(int(seed)), []
    while s:
        limbs.append(s & 0xFFFFFFFF)
        s >>= 32
    key = np.asarray(limbs or [0], dtype=np.uint32)
    if lib.mlmq_gen_graph(_GEN_KINDS[kind], ctypes.byref(gp), key.ctypes.data, key.size,
                          off.ctypes.data, col.ctypes.data, w.ctypes.data):
        raise ValueError(lib.oracle_last_error().decode())
    return off, col, w


def f32_weights(m: int, seed: int) -> np.ndarray:
    """Config-5 float weights U[0,1) (same counter-based stream as graph.with_f32_weights)."""
    out = np.empty(m, dtype=np.float32)
    _load().mlmq_gen_f32_weights(m, seed, out.ctypes.data)
    return out


def csr_sha256(row_offsets, col_indices, weights) -> str:
    """sha256(row_offsets <u8 || col <u4 || weights <u4) as in BASELINE.md §4."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(row_offsets, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(col_indices, dtype="<u4").tobytes())
    h.update(np.ascontiguousarray(weights, dtype="<u4").tobytes())
    return h.hexdigest()
