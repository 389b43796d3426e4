"""ctypes binding of libmlmq.so (include/mlmq.h).

The product path has no CPU fallback: if the library or a CUDA device is missing,
solves raise ``EngineError``.  Status codes map onto the reference's exception
types: EINVAL -> ValueError, EOVERFLOW -> QueueOverflowError,
everything else -> EngineError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional

import numpy as np

from .core import EngineError, QueueOverflowError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmlmq.so")
#: MLMQ_DEBUG=1 loads the debug build (make -C csrc debug): phase profile + wait states
DEBUG_LIB_PATH = os.path.join(_HERE, "libmlmq_debug.so")
#: MLMQ_DEBUG=1 MLMQ_PROFILE=1 loads the profile build (make -C csrc prof): the same hooks
#: without the per-line trace, so the phase split is representative
PROF_LIB_PATH = os.path.join(_HERE, "libmlmq_prof.so")

(MLMQ_OK, MLMQ_EINVAL, MLMQ_EOVERFLOW, MLMQ_EENGINE, MLMQ_ECUDA, MLMQ_ENOMEM, MLMQ_EFORMAT,
 MLMQ_ENEGATIVE, MLMQ_EIO, MLMQ_EFALLBACK) = range(10)
W_U32, W_F32, W_UNIT = 0, 1, 2
DIST_AUTO, DIST_U32, DIST_U64 = 0, 1, 2
GEN_KINDS = {"grid2d": 0, "path": 1, "uniform": 2, "rmat": 3}
GROUP_METRIC_FIELDS = 11


class Config(ctypes.Structure):
    """mlmq_config_t"""
    _fields_ = [
        ("l1_type", ctypes.c_int32), ("l2_type", ctypes.c_int32),
        ("l0_capacity", ctypes.c_int32), ("l1_capacity", ctypes.c_int32),
        ("wb", ctypes.c_int32),
        ("delta_nf", ctypes.c_double), ("filter_f", ctypes.c_double), ("delta", ctypes.c_double),
        ("block_size", ctypes.c_int32), ("block_num", ctypes.c_int64),
        ("bmax", ctypes.c_int32), ("bnum", ctypes.c_int32),
        ("node_batch", ctypes.c_int32), ("pnum", ctypes.c_int32),
        ("num_groups", ctypes.c_int32), ("lanes_per_group", ctypes.c_int32),
        ("th_v", ctypes.c_int32), ("dup_elim", ctypes.c_int32),
        ("unit_weights", ctypes.c_int32), ("dist_mode", ctypes.c_int32),
        ("watchdog_s", ctypes.c_double), ("spin_timeout_s", ctypes.c_double),
        ("hub_chunk", ctypes.c_int32), ("share", ctypes.c_int32), ("fifo_park", ctypes.c_int32),
        ("bucket_window", ctypes.c_int32), ("read_batch", ctypes.c_int32),
        ("hub_threshold", ctypes.c_int32), ("test_capacity", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("heavy_delta", ctypes.c_int32),
        ("heavy_delta_f", ctypes.c_float),
    ]


class Metrics(ctypes.Structure):
    """mlmq_metrics_t"""
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "relaxations", "distance_updates", "l0_enqueues", "l0_dequeues", "l1_enqueues",
        "l1_dequeues", "l2_enqueues", "l2_dequeues", "l2_atomic_ops", "flushes",
        "settled_reads", "wall_time_us")] + [
        ("kernel_ms", ctypes.c_double), ("num_groups", ctypes.c_uint64),
        ("hub_items", ctypes.c_uint64), ("dist_bits", ctypes.c_uint32),
        ("reruns", ctypes.c_uint32)]


class GenParams(ctypes.Structure):
    """mlmq_gen_params_t"""
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("n", ctypes.c_int64),
                ("m", ctypes.c_int64), ("scale", ctypes.c_int64), ("edge_factor", ctypes.c_int64),
                ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
                ("d", ctypes.c_double), ("wmin", ctypes.c_int64), ("wmax", ctypes.c_int64)]


#: every symbol include/mlmq.h declares (checked by tests/test_native_abi.py)
EXPORTED_SYMBOLS = (
    "mlmq_abi_version", "mlmq_last_error", "mlmq_device_count", "mlmq_device_info",
    "mlmq_graph_create", "mlmq_graph_destroy", "mlmq_graph_device_bytes", "mlmq_auto_groups",
    "mlmq_sssp", "mlmq_sssp_f32", "mlmq_sssp_device", "mlmq_last_dist", "mlmq_reach",
    "mlmq_feature_sums", "mlmq_gen_size", "mlmq_gen_graph", "mlmq_gen_shard", "mlmq_build_csr",
    "mlmq_gen_f32_weights", "mlmq_shard_create", "mlmq_shard_begin", "mlmq_shard_step", "mlmq_graph_stream",
    "mlmq_host_alloc", "mlmq_host_free", "mlmq_load_dimacs", "mlmq_load_matrix_market",
    "mlmq_csr_size", "mlmq_csr_copy", "mlmq_csr_free", "mlmq_queue_create", "mlmq_queue_destroy",
    "mlmq_queue_write", "mlmq_queue_read", "mlmq_queue_stats", "mlmq_queue_stress",
)

_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load libmlmq.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("MLMQ_LIB") or LIB_PATH  # experiment builds (make KSET=...)
        if os.environ.get("MLMQ_DEBUG") == "1" and not os.environ.get("MLMQ_LIB"):
            want = PROF_LIB_PATH if os.environ.get("MLMQ_PROFILE") == "1" else DEBUG_LIB_PATH
            if os.path.exists(want):
                path = want
        if not os.path.exists(path):
            raise EngineError(
                f"{path} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " or `make -C paper_2602_10080_b200/csrc`")
        L = ctypes.CDLL(path)
        P, U64, I32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        sig = {
            "mlmq_abi_version": ([], I32),
            "mlmq_last_error": ([], ctypes.c_char_p),
            "mlmq_device_count": ([P], I32),
            "mlmq_device_info": ([I32, P, P, P], I32),
            "mlmq_graph_create": ([P, P, P, I32, U64, U64, I32, P], I32),
            "mlmq_graph_destroy": ([P], None),
            "mlmq_graph_device_bytes": ([P, P], I32),
            "mlmq_auto_groups": ([P, P, P], I32),
            "mlmq_sssp": ([P, U64, P, P, P, P, U64], I32),
            "mlmq_sssp_f32": ([P, U64, P, P, P, P, U64], I32),
            "mlmq_sssp_device": ([P, U64, P, P], I32),
            "mlmq_last_dist": ([P, P], I32),
            "mlmq_reach": ([P, P, P], I32),
            "mlmq_feature_sums": ([P, P], I32),
            "mlmq_gen_size": ([I32, P, P, P], I32),
            "mlmq_gen_graph": ([I32, P, P, U64, P, P, P], I32),
            "mlmq_build_csr": ([U64, U64, P, P, P, P, P, P, P], I32),
            "mlmq_gen_f32_weights": ([U64, U64, P], I32),
            "mlmq_gen_shard": ([I32, P, P, U64, ctypes.c_uint32, ctypes.c_uint32, P, P, P, P], I32),
            "mlmq_shard_create": ([P, P, P, I32, U64, U64, U64, ctypes.c_uint32, ctypes.c_uint32, I32, P], I32),
            "mlmq_shard_begin": ([P], I32),
            "mlmq_graph_stream": ([P, P], I32),
            "mlmq_shard_step": ([P, P, P, U64, P, U64, P, P], I32),
            "mlmq_host_alloc": ([U64, P], I32),
            "mlmq_host_free": ([P], None),
            "mlmq_load_dimacs": ([ctypes.c_char_p, P], I32),
            "mlmq_load_matrix_market": ([ctypes.c_char_p, ctypes.c_int64, P], I32),
            "mlmq_csr_size": ([P, P, P], I32),
            "mlmq_csr_copy": ([P, P, P, P], I32),
            "mlmq_csr_free": ([P], None),
            "mlmq_queue_create": ([I32, P, P], I32),
            "mlmq_queue_destroy": ([P], None),
            "mlmq_queue_write": ([P, P, U64, ctypes.c_int32], I32),
            "mlmq_queue_read": ([P, ctypes.c_int32, P, U64, P], I32),
            "mlmq_queue_stats": ([P, P], I32),
            "mlmq_queue_stress": ([P, ctypes.c_int32, ctypes.c_int32, U64, U64, U64, U64, P, U64, P, P, U64,
                                   P, P], I32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.mlmq_abi_version() != 1:
            raise EngineError("libmlmq.so ABI version mismatch")
        _lib = L
        return L


def last_error() -> str:
    msg = lib().mlmq_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(status: int) -> None:
    if status == MLMQ_OK:
        return
    msg = last_error()
    if status == MLMQ_EINVAL:
        raise ValueError(msg)
    if status == MLMQ_EOVERFLOW:
        raise QueueOverflowError(msg)
    raise EngineError(msg or f"libmlmq error {status}")


def device_count() -> int:
    n = ctypes.c_int(0)
    lib().mlmq_device_count(ctypes.byref(n))
    return int(n.value)


class _PinnedBlock:
    """Owner of one page-locked host buffer; returns it to the pool when the last numpy
    array viewing it is garbage collected."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    def __del__(self):
        try:
            _pinned_release(self)
        except Exception:
            pass


_pool_lock = threading.Lock()
_pool: dict = {}
_POOL_MAX_PER_SIZE = 4


def _pinned_release(block: _PinnedBlock) -> None:
    with _pool_lock:
        free = _pool.setdefault(block.nbytes, [])
        if len(free) < _POOL_MAX_PER_SIZE:
            free.append(block.ptr)
            return
    lib().mlmq_host_free(block.ptr)


def pinned_empty(n: int, dtype) -> np.ndarray:
    """np.empty(n, dtype) in page-locked memory, recycled across solves (result buffers
    for device->host copies at full link speed)."""
    dt = np.dtype(dtype)
    nbytes = max(64, int(n) * dt.itemsize)
    ptr = None
    with _pool_lock:
        free = _pool.get(nbytes)
        if free:
            ptr = free.pop()
    if ptr is None:
        p = ctypes.c_void_p()
        check(lib().mlmq_host_alloc(nbytes, ctypes.byref(p)))
        ptr = p.value
    block = _PinnedBlock(ptr, nbytes)
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    buf._mlmq_block = block  # the ctypes buffer keeps the owner alive; numpy keeps the buffer
    return np.frombuffer(buf, dtype=dt, count=int(n))


def _note_no_device():
    """Test hook: tests/test_reference_suite.py runs the reference suites on a GPU-less host
    and needs to know which tests stopped at the missing device (MLMQ_NODEV_LOG)."""
    log = os.environ.get("MLMQ_NODEV_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write((os.environ.get("PYTEST_CURRENT_TEST") or "?").split(" ")[0] + "\n")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class DeviceGraph:
    """A CSR graph resident in device memory (owns an ``mlmq_graph*``)."""

    def __init__(self, row_offsets: np.ndarray, col: np.ndarray, weights: Optional[np.ndarray],
                 weight_kind: int, device: int = 0):
        L = lib()
        if device_count() < 1:
            _note_no_device()
            raise EngineError("no CUDA device is visible; the MLMQ engine has no CPU fallback")
        self._lib = L
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        self.col = np.ascontiguousarray(col, dtype=np.uint32)
        self.n = int(self.row_offsets.size - 1)
        self.m = int(self.col.size)
        self.weight_kind = weight_kind
        w = None
        if weight_kind == W_U32:
            w = np.ascontiguousarray(weights, dtype=np.uint32)
        elif weight_kind == W_F32:
            w = np.ascontiguousarray(weights, dtype=np.float32)
        h = ctypes.c_void_p()
        check(L.mlmq_graph_create(_ptr(self.row_offsets), _ptr(self.col), _ptr(w), weight_kind,
                                  self.n, self.m, device, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self._lib.mlmq_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def auto_groups(self, cfg: Config) -> int:
        out = ctypes.c_int32(0)
        check(self._lib.mlmq_auto_groups(self.handle, ctypes.byref(cfg), ctypes.byref(out)))
        return int(out.value)

    def sssp(self, source: int, cfg: Config, want_groups: int = 0):
        """Run one solve; returns (dist ndarray, Metrics, group metrics ndarray)."""
        m = Metrics()
        gm = np.zeros((max(want_groups, 1), GROUP_METRIC_FIELDS), dtype=np.uint64)
        if self.weight_kind == W_F32:
            dist = pinned_empty(self.n, np.float32)
            st = self._lib.mlmq_sssp_f32(self.handle, source, ctypes.byref(cfg), _ptr(dist),
                                         ctypes.byref(m), _ptr(gm), want_groups)
        else:
            dist = pinned_empty(self.n, np.uint64)
            st = self._lib.mlmq_sssp(self.handle, source, ctypes.byref(cfg), _ptr(dist),
                                     ctypes.byref(m), _ptr(gm), want_groups)
        check(st)
        return dist, m, gm

    def sssp_device(self, source: int, cfg: Config) -> Metrics:
        """Solve leaving distances on the device (benchmark path)."""
        m = Metrics()
        check(self._lib.mlmq_sssp_device(self.handle, source, ctypes.byref(cfg), ctypes.byref(m)))
        return m

    def last_dist(self) -> np.ndarray:
        dt = np.float32 if self.weight_kind == W_F32 else np.uint64
        out = np.empty(self.n, dtype=dt)
        check(self._lib.mlmq_last_dist(self.handle, _ptr(out)))
        return out

    def reach(self):
        v, e = ctypes.c_uint64(), ctypes.c_uint64()
        check(self._lib.mlmq_reach(self.handle, ctypes.byref(v), ctypes.byref(e)))
        return int(v.value), int(e.value)

    def feature_sums(self) -> np.ndarray:
        out = np.zeros(10, dtype=np.uint64)
        check(self._lib.mlmq_feature_sums(self.handle, _ptr(out)))
        return out

    def device_bytes(self) -> int:
        out = ctypes.c_uint64()
        check(self._lib.mlmq_graph_device_bytes(self.handle, ctypes.byref(out)))
        return int(out.value)


class DeviceShard(DeviceGraph):
    """One shard of a 1D-partitioned graph (include/mlmq.h mlmq_shard_*): owned rows in
    local order, GLOBAL column ids."""

    def __init__(self, row_offsets: np.ndarray, col: np.ndarray, weights: Optional[np.ndarray],
                 weight_kind: int, n_global: int, rank: int, nparts: int, device: int = 0):
        L = lib()
        if device_count() < 1:
            _note_no_device()
            raise EngineError("no CUDA device is visible; the MLMQ engine has no CPU fallback")
        self._lib = L
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        self.col = np.ascontiguousarray(col, dtype=np.uint32)
        self.n = int(self.row_offsets.size - 1)
        self.m = int(self.col.size)
        self.weight_kind = weight_kind
        self.n_global, self.rank, self.nparts = int(n_global), int(rank), int(nparts)
        w = None
        if weight_kind == W_U32:
            w = np.ascontiguousarray(weights, dtype=np.uint32)
        elif weight_kind == W_F32:
            w = np.ascontiguousarray(weights, dtype=np.float32)
        h = ctypes.c_void_p()
        check(L.mlmq_shard_create(_ptr(self.row_offsets), _ptr(self.col), _ptr(w), weight_kind, self.n,
                                  self.m, self.n_global, self.rank, self.nparts, device, ctypes.byref(h)))
        self.handle = h

    def begin(self) -> None:
        check(self._lib.mlmq_shard_begin(self.handle))

    def stream_ptr(self) -> int:
        """The library's CUDA stream for this shard (cudaStream_t as an int)."""
        p = ctypes.c_void_p()
        check(self._lib.mlmq_graph_stream(self.handle, ctypes.byref(p)))
        return int(p.value or 0)

    def step(self, cfg: Config, inbox_ptr: int, n_in: int, send_ptr: int, send_cap: int):
        """One superstep; inbox/send are DEVICE pointers to (v, d) u32 pairs.  Returns
        (per-owner send counts, Metrics)."""
        counts = np.zeros(self.nparts, dtype=np.uint64)
        m = Metrics()
        check(self._lib.mlmq_shard_step(self.handle, ctypes.byref(cfg), inbox_ptr or None, int(n_in),
                                        send_ptr, int(send_cap), _ptr(counts), ctypes.byref(m)))
        return counts, m


def seed_key(seed: int) -> np.ndarray:
    """CPython random_seed key: 32-bit little-endian limbs of |seed| ({0} for 0)."""
    s = abs(int(seed))
    limbs = []
    while s:
        limbs.append(s & 0xFFFFFFFF)
        s >>= 32
    return np.asarray(limbs or [0], dtype=np.uint32)


def generate(kind: str, seed: int, params: dict):
    """Native generator: returns (row_offsets u64, col u32, weights u32)."""
    L = lib()
    gp = GenParams()
    for k, v in params.items():
        setattr(gp, k, v)
    n, m = ctypes.c_uint64(), ctypes.c_uint64()
    check(L.mlmq_gen_size(GEN_KINDS[kind], ctypes.byref(gp), ctypes.byref(n), ctypes.byref(m)))
    off = np.empty(n.value + 1, dtype=np.uint64)
    col = np.empty(m.value, dtype=np.uint32)
    w = np.empty(m.value, dtype=np.uint32)
    key = seed_key(seed)
    check(L.mlmq_gen_graph(GEN_KINDS[kind], ctypes.byref(gp), _ptr(key), key.size,
                           _ptr(off), _ptr(col), _ptr(w)))
    return off, col, w


def load_csr(path: str, fmt: str, weight_scale: int = 1000):
    """Native DIMACS / Matrix Market reader: (row_offsets u64, col u32, w u32), or None when
    the file holds input only the Python reader restates exactly (MLMQ_EFALLBACK) or
    cannot be opened (the Python reader then raises the exact OSError)."""
    from .core import GraphFormatError, NegativeWeightError
    L = lib()
    h = ctypes.c_void_p()
    bpath = os.fsencode(path)
    st = (L.mlmq_load_dimacs(bpath, ctypes.byref(h)) if fmt == "dimacs"
          else L.mlmq_load_matrix_market(bpath, int(weight_scale), ctypes.byref(h)))
    if st in (MLMQ_EFALLBACK, MLMQ_EIO):
        return None
    if st == MLMQ_EFORMAT:
        raise GraphFormatError(last_error())
    if st == MLMQ_ENEGATIVE:
        raise NegativeWeightError(last_error())
    check(st)
    try:
        n, m = ctypes.c_uint64(), ctypes.c_uint64()
        check(L.mlmq_csr_size(h, ctypes.byref(n), ctypes.byref(m)))
        off = np.empty(n.value + 1, dtype=np.uint64)
        col = np.empty(m.value, dtype=np.uint32)
        w = np.empty(m.value, dtype=np.uint32)
        check(L.mlmq_csr_copy(h, _ptr(off), _ptr(col), _ptr(w)))
    finally:
        L.mlmq_csr_free(h)
    return off, col, w


def generate_shard(kind: str, seed: int, params: dict, nparts: int, rank: int):
    """Rank's slice of a generated graph (rows v % nparts == rank at local id v // nparts,
    global columns): (row_offsets u64, col u32, weights u32, n_global)."""
    L = lib()
    gp = GenParams()
    for k, v in params.items():
        setattr(gp, k, v)
    n, m = ctypes.c_uint64(), ctypes.c_uint64()
    check(L.mlmq_gen_size(GEN_KINDS[kind], ctypes.byref(gp), ctypes.byref(n), ctypes.byref(m)))
    n_loc = (int(n.value) - rank + nparts - 1) // nparts
    off = np.empty(n_loc + 1, dtype=np.uint64)
    key = seed_key(seed)
    mk = ctypes.c_uint64()
    check(L.mlmq_gen_shard(GEN_KINDS[kind], ctypes.byref(gp), _ptr(key), key.size, nparts, rank, _ptr(off),
                           None, None, ctypes.byref(mk)))
    col = np.empty(mk.value, dtype=np.uint32)
    w = np.empty(mk.value, dtype=np.uint32)
    check(L.mlmq_gen_shard(GEN_KINDS[kind], ctypes.byref(gp), _ptr(key), key.size, nparts, rank, _ptr(off),
                           _ptr(col), _ptr(w), ctypes.byref(mk)))
    return off, col, w, int(n.value)


def build_csr_native(n: int, src: np.ndarray, dst: np.ndarray, w: np.ndarray):
    L = lib()
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    w = np.ascontiguousarray(w, dtype=np.uint32)
    m = src.size
    off = np.empty(n + 1, dtype=np.uint64)
    col = np.empty(m, dtype=np.uint32)
    wo = np.empty(m, dtype=np.uint32)
    kept = ctypes.c_uint64()
    check(L.mlmq_build_csr(n, m, _ptr(src), _ptr(dst), _ptr(w), _ptr(off), _ptr(col), _ptr(wo),
                           ctypes.byref(kept)))
    k = int(kept.value)
    return off, col[:k].copy(), wo[:k].copy()


def f32_weights(m: int, seed: int) -> np.ndarray:
    out = np.empty(m, dtype=np.float32)
    check(lib().mlmq_gen_f32_weights(m, seed, _ptr(out)))
    return out


class QueueParams(ctypes.Structure):
    """mlmq_queue_params_t"""
    _fields_ = [("l2_type", ctypes.c_int32), ("block_size", ctypes.c_int32), ("block_num", ctypes.c_int64),
                ("delta", ctypes.c_double), ("bmax", ctypes.c_int32), ("bnum", ctypes.c_int32),
                ("node_batch", ctypes.c_int32), ("pnum", ctypes.c_int32), ("num_groups", ctypes.c_int32),
                ("reserved0", ctypes.c_int32), ("heap_nodes", ctypes.c_int64),
                ("spin_timeout_s", ctypes.c_double)]


class DeviceQueue:
    """One L2 queue in device memory driven by the solve kernel's own queue code
    (mlmq_queue_* in include/mlmq.h)."""

    STATS = 40

    def __init__(self, l2_type: int, *, block_size: int = 64, block_num: int = 4096, delta: float = 1.0,
                 bmax: int = 64, bnum: int = 1, node_batch: int = 32, pnum: int = 1, num_groups: int = 64,
                 heap_nodes: int = 0, spin_timeout_s: float = 15.0, device: int = 0):
        L = lib()
        if device_count() < 1:
            _note_no_device()
            raise EngineError("no CUDA device is visible; the MLMQ engine has no CPU fallback")
        qp = QueueParams(l2_type, block_size, block_num, float(delta), bmax, bnum, node_batch, pnum,
                         num_groups, 0, heap_nodes, float(spin_timeout_s))
        h = ctypes.c_void_p()
        check(L.mlmq_queue_create(device, ctypes.byref(qp), ctypes.byref(h)))
        self._lib, self.handle = L, h
        self.read_cap = max(block_size, 32)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.mlmq_queue_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def write(self, pairs: np.ndarray, group: int) -> None:
        a = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        check(self._lib.mlmq_queue_write(self.handle, _ptr(a), a.shape[0], group))

    def read(self, group: int) -> np.ndarray:
        out = np.empty((self.read_cap, 2), dtype=np.uint32)
        n = ctypes.c_uint64()
        check(self._lib.mlmq_queue_read(self.handle, group, _ptr(out), self.read_cap, ctypes.byref(n)))
        return out[: n.value]

    def stats(self) -> np.ndarray:
        out = np.zeros(self.STATS, dtype=np.uint64)
        check(self._lib.mlmq_queue_stats(self.handle, _ptr(out)))
        return out

    def stress(self, writers: int, readers: int, stride: int, begin: int, end: int, stop_at: int,
               cap: int, log_cap: int = 0):
        pairs = np.empty((max(cap, 1), 2), dtype=np.uint32)
        n = ctypes.c_uint64()
        ms = ctypes.c_double()
        logs = np.zeros((readers, max(log_cap, 1)), dtype=np.uint64) if log_cap else None
        logn = np.zeros(readers, dtype=np.uint64) if log_cap else None
        check(self._lib.mlmq_queue_stress(self.handle, writers, readers, stride, begin, end, stop_at,
                                          _ptr(pairs), cap, ctypes.byref(n), _ptr(logs), log_cap,
                                          _ptr(logn), ctypes.byref(ms)))
        k = min(int(n.value), cap)
        epochs = [logs[r, : int(logn[r])].tolist() for r in range(readers)] if log_cap else None
        return pairs[:k], int(n.value), epochs, float(ms.value)
