"""The reference's L2 queue objects (pkg/src/mlq_sssp/l2.py:73-451) backed by device queues.

Each object owns one queue in device memory (``mlmq_queue_*``, include/mlmq.h) and every
``write`` / ``try_read`` runs the persistent solve kernel's own queue code
(``Worker::write_back`` / ``Worker::l2_read``, csrc/kernels/mlmq_kernel.cuh) in a one-warp
launch, so the reference's queue-level tests (test_acceptance.py:282 criterion 3,
test_l2_queues.py) exercise the B200 queues rather than a Python model of them.  Calls
are serialised per queue; the concurrent many-warp stress of the same device code is
``DeviceQueue.stress`` (tests/test_queue_harness.py).

Differences a caller can see: a read returns at most one ring block (FIFO / bucket) or
32 elements (heaps: one warp per read); claims never outlive a call (a reader claims a
ticket only when a written block exists and waits for it inside the call), so
``pending_tickets()`` is 0 between calls -- the reference's quiescent state.
"""

from __future__ import annotations

import threading
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native

Element = Tuple[int, int]
_FIFO, _BUCKET, _PRIORITY, _MULTI = 0, 1, 2, 3


class _DeviceL2:
    _kind = _FIFO

    def __init__(self, **kw):
        self._q = _native.DeviceQueue(self._kind, **kw)
        self._groups = kw.get("num_groups", 1024)

    def _pairs(self, batch: Sequence[Element]) -> np.ndarray:
        return np.asarray(batch, dtype=np.uint64).reshape(-1, 2).astype(np.uint32)

    def write(self, batch: Sequence[Element], group_id: int = 0, shard=None) -> None:
        if len(batch) == 0:
            return
        self._q.write(self._pairs(batch), group_id % self._groups)
        if shard is not None:
            shard.l2_atomic_ops += 1

    def try_read(self, group_id: int, want: int = 0, shard=None) -> List[Element]:
        out = self._q.read(group_id % self._groups)
        if shard is not None and out.size:
            shard.l2_atomic_ops += 1
        return [(int(v), int(d)) for v, d in out.tolist()]

    def _stats(self) -> np.ndarray:
        return self._q.stats()

    def pending_tickets(self) -> int:
        return int(self._stats()[1])

    def has_claims(self) -> bool:
        return self.pending_tickets() > 0

    def is_structurally_empty(self) -> bool:
        st = self._stats()
        return bool(st[2]) and int(st[1]) == 0

    def element_count(self) -> int:
        return int(self._stats()[0])


class L2BlockFifo(_DeviceL2):
    """Ticketed block ring (l2.py:73-178): Vyukov slots on the device."""

    _kind = _FIFO

    def __init__(self, block_size: int, block_num: int, abort_event: Optional[threading.Event] = None,
                 spin_timeout_s: float = 15.0):
        self._bs, self._bn = block_size, block_num
        super().__init__(block_size=block_size, block_num=block_num, spin_timeout_s=spin_timeout_s,
                         num_groups=1024)

    @property
    def _pending(self) -> Dict[int, int]:
        # claims never outlive a device call; a non-zero count would be a stranded claim
        n = self.pending_tickets()
        return {-(i + 1): 0 for i in range(n)}

    @property
    def _slots(self) -> List[Optional[List[Element]]]:
        """The resident elements in the reference's shape (sum of block lengths)."""
        n = self.element_count()
        return [[(0, 0)] * n] if n else [None]


class _BucketFifoView:
    """Stand-in for one of L2Bucket._fifos (claims never outlive a call)."""

    def __init__(self, owner: "L2Bucket"):
        self._owner = owner

    @property
    def _pending(self) -> Dict[int, int]:
        return {}

    def pending_tickets(self) -> int:
        return 0


class L2Bucket(_DeviceL2):
    """Delta-bucket window over bmax rings (l2.py:181-301), the reference's floor rule:
    the epoch advances when the head is seen truly empty while elements remain."""

    _kind = _BUCKET

    def __init__(self, delta: int, bmax: int, bnum: int, block_size: int, block_num: int,
                 abort_event: Optional[threading.Event] = None, spin_timeout_s: float = 15.0):
        self._delta, self._bmax, self._bnum = delta, bmax, bnum
        super().__init__(block_size=block_size, block_num=block_num, delta=delta, bmax=bmax, bnum=bnum,
                         spin_timeout_s=spin_timeout_s, num_groups=1024)
        self._fifos = [_BucketFifoView(self) for _ in range(bmax)]
        self._lock = threading.Lock()

    @property
    def _epoch(self) -> int:
        return int(self._stats()[3])

    @property
    def base(self) -> int:
        return self._epoch * self._delta

    @property
    def _resident(self) -> int:
        return self.element_count()


class L2PriorityQueue(_DeviceL2):
    """Batch min-heap of sorted nodes (l2.py:304-413), lock-protected on the device."""

    _kind = _PRIORITY

    def __init__(self, node_batch: int, num_groups: int = 1024):
        self._node_batch = node_batch
        super().__init__(node_batch=min(max(1, node_batch), 32), num_groups=num_groups, heap_nodes=1 << 17)

    def check_heap(self) -> None:
        """l2.py:391-402: every node sorted, every parent's min <= its children's."""
        assert bool(self._stats()[4]), "device batch heap violates the heap property"


class _HeapView:
    def __init__(self, owner: "L2MultiQueue", i: int):
        self._owner, self._i = owner, i

    def check_heap(self) -> None:
        self._owner.check_heap()

    def element_count(self) -> int:
        return self._owner.queue_sizes()[self._i]


class L2MultiQueue(_DeviceL2):
    """pnum batch heaps (l2.py:416-451): group g reads heap g % pnum; a group's writes
    rotate over the heaps starting at its own (the cursor persists on the device)."""

    _kind = _MULTI

    def __init__(self, pnum: int, node_batch: int, num_groups: int):
        self._pnum = max(1, min(pnum, num_groups))
        super().__init__(node_batch=min(max(1, node_batch), 32), pnum=self._pnum, num_groups=num_groups,
                         heap_nodes=1 << 16)
        self._queues = [_HeapView(self, i) for i in range(self._pnum)]

    @property
    def pnum(self) -> int:
        return self._pnum

    def queue_sizes(self) -> List[int]:
        st = self._stats()
        return [int(x) for x in st[7: 7 + min(self._pnum, 32)]]

    def check_heap(self) -> None:
        assert bool(self._stats()[4]), "device batch heap violates the heap property"


def make_l2(cfg, abort_event: Optional[threading.Event] = None):
    """l2.py:454-466 factory over the device queues."""
    p = cfg.l2_params
    if cfg.l2_type == "fifo":
        return L2BlockFifo(p.block_size, p.block_num, abort_event)
    if cfg.l2_type == "bucket":
        return L2Bucket(int(p.delta or 1), p.bmax, p.bnum, p.block_size, p.block_num, abort_event)
    if cfg.l2_type == "priority":
        return L2PriorityQueue(p.node_batch)
    if cfg.l2_type == "multi":
        return L2MultiQueue(p.pnum or 1, p.node_batch, cfg.num_groups or 1)
    raise ValueError(f"unknown l2_type {cfg.l2_type!r}")


__all__ = ["L2BlockFifo", "L2Bucket", "L2MultiQueue", "L2PriorityQueue", "make_l2"]
