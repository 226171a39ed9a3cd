"""Standalone device WorkerCache (cache.hpp:73-240, libedx workercache.cu):
the reference's own cache KATs (tests/test_cache.cpp) and random traffic
against the oracle under both victim policies."""
import numpy as np
import pytest

from helpers import apply_cache_op, cache_footprint, cache_op_stream, device_cache_rows

pytestmark = pytest.mark.gpu


def test_first_insertion_and_retouch(gpu):
    """test_cache.cpp:58-76."""
    W = gpu.WorkerCache
    c = W(4)
    c.touch(3, True, 0)
    e = c.find(3)
    assert e is not None and e.mark == 1 and e.frequency == 1 and e.version_latest
    c = W(4)
    c.touch(3, True, 1)
    c.touch(3, True, 2)
    e = c.find(3)
    assert e.frequency == 2 and e.last_access == 2


def test_mark_advance_and_touch_full(gpu):
    """test_cache.cpp:78-98."""
    edx = gpu
    c = edx.WorkerCache(2)
    c.touch(1, True, 0)
    c.touch(2, True, 0)
    assert c.full() and c.current_mark() == 1
    ev = c.evict_for(1)
    assert c.current_mark() == 2 and len(ev) == 1
    c.touch(9, True, 1)
    assert c.find(9).mark == 2
    c = edx.WorkerCache(1)
    c.touch(1, True, 0)
    with pytest.raises(edx.LogicError, match="evict first"):
        c.touch(2, True, 0)
    c.touch(1, True, 1)


def test_victim_order_kats(gpu):
    """test_cache.cpp:100-142: version, then mark, then frequency."""
    W = gpu.WorkerCache
    c = W(2)
    c.touch(10, False, 0)
    c.touch(11, True, 0)
    assert c.select_victim() == 10
    c = W(2)
    c.touch(20, True, 0)
    c.touch(21, True, 0)
    c.evict_for(1)
    c.touch(22, True, 1)
    assert c.find(21).mark == 1 and c.find(22).mark == 2
    assert c.select_victim() == 21
    c = W(2)
    for _ in range(5):
        c.touch(30, True, 0)
    c.touch(31, True, 0)
    c.touch(31, True, 0)
    assert c.select_victim() == 31
    c = W(3)
    c.touch(1, True, 0)
    with pytest.raises(gpu.LogicError, match="requires a full cache"):
        c.select_victim()


def test_brute_force_victims(gpu):
    """test_cache.cpp:144-160 (500 trials, up to 5 entries) with a numpy
    restatement of the naive comparator."""
    rng = np.random.default_rng(1234)
    for trial in range(60):
        size = 2 + int(rng.integers(0, 4))
        c = gpu.WorkerCache(size)
        for i in range(size):
            latest = bool(rng.integers(0, 2))
            now = int(rng.integers(0, 4))
            for _ in range(1 + int(rng.integers(0, 3))):
                c.touch(100 + i, latest, now)
        es = c.entries()
        want = min(es.values(), key=lambda e: (e.version_latest, e.mark, e.frequency,
                                               e.last_access, e.id)).id
        assert c.select_victim() == want


def test_evict_for_kats(gpu):
    """test_cache.cpp:162-201: no-op with room, needs_push, pinned, capacity."""
    edx = gpu
    c = edx.WorkerCache(4)
    c.touch(1, True, 0)
    assert c.evict_for(2) == []
    for push in (True, False):
        c = edx.WorkerCache(2)
        c.touch(1, True, 0)
        c.touch(2, True, 1)
        ev = c.evict_for(1, (lambda i: i == 1) if push else (lambda i: False))
        assert ev == [(1, push)]
    c = edx.WorkerCache(2)
    c.touch(1, True, 0)
    c.touch(2, True, 1)
    assert c.evict_for(1, None, {1}) == [(2, False)]
    c.touch(2, True, 1)
    with pytest.raises(edx.LogicError, match="pinned"):
        c.evict_for(1, None, {1, 2})
    c = edx.WorkerCache(2)
    with pytest.raises(edx.InvalidArgument, match="capacity"):
        c.evict_for(3)


def test_priority_ratio_kat(gpu):
    """test_cache.cpp:217-233."""
    edx = gpu
    c = edx.WorkerCache(2, edx.VictimPolicy.PRIORITY_RATIO, lambda i: 8.0 if i == 1 else 1.0)
    c.touch(1, True, 0)
    c.touch(2, True, 0)
    c.touch(2, True, 0)
    assert c.select_victim() == 1
    u = edx.WorkerCache(2, edx.VictimPolicy.PRIORITY_RATIO)
    u.touch(5, False, 0)
    u.touch(6, True, 0)
    assert u.select_victim() == 5


def test_random_traffic_size_bound(gpu):
    """test_cache.cpp:203-215."""
    rng = np.random.default_rng(99)
    c = gpu.WorkerCache(8)
    for step in range(300):
        id_ = int(rng.integers(0, 32))
        if not c.resident(id_) and c.full():
            c.evict_for(1)
        c.touch(id_, bool(rng.integers(0, 2)), step)
        assert c.size() <= c.capacity()


@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("seed,capacity,id_range,ops", [(1, 1, 4, 150), (2, 3, 8, 250),
                                                        (3, 8, 32, 300), (4, 64, 200, 400)])
def test_device_cache_equals_oracle(gpu, oracle, policy, seed, capacity, id_range, ops):
    """Random traffic: every result, error message and the full state."""
    dev = gpu.WorkerCache(capacity, policy, cache_footprint)
    ref = oracle.cache(capacity, policy)
    for op in cache_op_stream(seed, capacity, ops, id_range):
        rd, rr = apply_cache_op(dev, op, True), apply_cache_op(ref, op, False)
        assert rd == rr, (op, rd, rr)
        assert (dev.size(), dev.current_mark()) == ref.info(), op
        assert device_cache_rows(dev) == ref.entries(), op


def test_large_cache_mass_eviction(gpu, oracle):
    """A 5000-entry cache (table rebuilds, long victim loops) against the oracle."""
    dev = gpu.WorkerCache(5000)
    ref = oracle.cache(5000)
    rng = np.random.default_rng(5)
    for now, id_ in enumerate(rng.integers(0, 20000, size=5000)):
        for c, d in ((dev, True), (ref, False)):
            r = apply_cache_op(c, ("touch", int(id_), True, now), d)
            assert r is None or r[0] != "raised"
    pins = [int(x) for x in rng.integers(0, 20000, size=300)]
    assert apply_cache_op(dev, ("evict_for", 1800, pins), True) == \
        apply_cache_op(ref, ("evict_for", 1800, pins), False)
    assert device_cache_rows(dev) == ref.entries()
