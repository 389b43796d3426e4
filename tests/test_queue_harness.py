"""Device-level L2 queue tests: the solve kernel's own queue code
(Worker::write_back / l2_read) driven by the queue harness (mlmq_queue_*, csrc/queue_harness.cu).

* concurrent W-writer x R-reader multiset conservation on every L2 family (the device
  analogue of the reference's acceptance criterion 3, test_acceptance.py:282-305), with
  the invariants checked at quiescence between the two phases: resident == written -
  consumed, no claimed-but-unconsumed tickets, heap property, bucket floor a multiple
  of Delta and never moving backwards as seen by any reader;
* single-group semantics of the reference queue objects (test_l2_queues.py): FIFO block
  order, bucket reads from the lowest non-empty bucket with the floor advancing only over
  an empty head, heap pops in key order, multi-queue write rotation.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOTAL, W, R, BS = 1_000_000, 8, 8, 64


def _dist(v):
    x = (np.asarray(v, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    x ^= x >> np.uint64(29)
    return (x & np.uint64((1 << 18) - 1)).astype(np.uint32)


def _queue(kind):
    from paper_2602_10080_b200 import _native
    if kind == "fifo":
        return _native.DeviceQueue(0, block_size=BS, block_num=20000, num_groups=W + R)
    if kind == "bucket":
        return _native.DeviceQueue(1, block_size=BS, block_num=8192, delta=4096, bmax=64, bnum=4, num_groups=W + R)
    if kind == "priority":
        return _native.DeviceQueue(2, node_batch=32, num_groups=W + R, heap_nodes=1 << 16)
    return _native.DeviceQueue(3, node_batch=32, pnum=R, num_groups=W + R, heap_nodes=1 << 15)


@pytest.mark.parametrize("kind", ["fifo", "bucket", "priority", "multi"])
def test_concurrent_writers_readers_conserve_the_multiset(kind):
    q = _queue(kind)
    per = TOTAL // W
    split = per * 3 // 5
    cap = TOTAL + R * 4096
    # phase 1: write 60 %, read >= 30 %, then check the invariants at quiescence
    p1, n1, ep1, ms1 = q.stress(W, R, per, 0, split, TOTAL * 3 // 10, cap, log_cap=4096)
    st = q.stats()
    assert n1 >= TOTAL * 3 // 10
    assert int(st[0]) == W * split - n1, (int(st[0]), W * split, n1)
    assert int(st[1]) == 0, "claimed tickets left unconsumed"
    assert int(st[4]) == 1, "heap property violated"
    # phase 2: write the rest and drain completely
    p2, n2, ep2, ms2 = q.stress(W, R, per, split, per, TOTAL - n1, cap, log_cap=4096)
    st = q.stats()
    assert n1 + n2 == TOTAL
    got = np.concatenate([p1, p2])
    ids = np.concatenate([np.arange(w * per, (w + 1) * per, dtype=np.uint64) for w in range(W)])
    want = np.sort((ids << np.uint64(32)) | _dist(ids).astype(np.uint64))
    have = np.sort((got[:, 0].astype(np.uint64) << np.uint64(32)) | got[:, 1].astype(np.uint64))
    assert np.array_equal(have, want), f"{kind}: read multiset differs from written"
    assert int(st[2]) == 1 and int(st[1]) == 0 and int(st[0]) == 0
    if kind == "bucket":
        for log in ep1 + ep2:  # per reader, in read order
            assert log == sorted(log), "floor moved backwards"
    print(f"{kind}: phase1 {ms1:.2f} ms, phase2 {ms2:.2f} ms for {TOTAL} elements")


def test_fifo_single_group_block_order():
    from paper_2602_10080_b200.l2 import L2BlockFifo
    q = L2BlockFifo(4, 64)
    q.write([(i, i) for i in range(10)], group_id=0)
    q.write([(100, 1)], group_id=1)
    got = []
    while True:
        b = q.try_read(0)
        if not b:
            break
        got.append(b)
    assert got == [[(0, 0), (1, 1), (2, 2), (3, 3)], [(4, 4), (5, 5), (6, 6), (7, 7)], [(8, 8), (9, 9)], [(100, 1)]]
    assert q.is_structurally_empty() and q.pending_tickets() == 0


def test_bucket_reads_lowest_bucket_and_floor_advances_over_empty_head():
    from paper_2602_10080_b200.l2 import L2Bucket
    q = L2Bucket(10, 8, 1, 16, 64)
    q.write([(1, 35), (2, 5), (3, 12), (4, 7)])
    assert q.base == 0
    assert sorted(q.try_read(0)) == [(2, 5), (4, 7)]  # bucket [0, 10)
    assert q.try_read(0) == [] and q.base == 10        # empty head: floor + delta
    assert q.try_read(0) == [(3, 12)]
    assert q.try_read(0) == [] and q.base == 20
    assert q.try_read(0) == [] and q.base == 30
    assert q.try_read(0) == [(1, 35)]
    assert q.is_structurally_empty()


def test_priority_pops_in_key_order():
    from paper_2602_10080_b200.l2 import L2PriorityQueue
    rng = np.random.default_rng(3)
    q = L2PriorityQueue(8)
    d = rng.integers(0, 10_000, size=500)
    for k in range(0, 500, 50):
        q.write([(int(i), int(d[i])) for i in range(k, k + 50)])
        q.check_heap()
    assert q.element_count() == 500
    out = []
    while True:
        b = q.try_read(0, 32)
        if not b:
            break
        out += b
    assert sorted(x for _, x in out) == [x for _, x in out] == sorted(d.tolist())
    assert q.is_structurally_empty()


def test_multi_queue_write_rotation():
    from paper_2602_10080_b200.l2 import L2MultiQueue
    q = L2MultiQueue(3, 8, 6)
    for k in range(6):  # group 1 writes to heaps 1, 2, 0, 1, 2, 0 (l2.py:430-436)
        q.write([(k, k)], group_id=1)
    assert q.queue_sizes() == [2, 2, 2]
    assert q.try_read(4, 8) == [(0, 0), (3, 3)]  # group 4 reads heap 4 % 3 = 1
