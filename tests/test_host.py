"""CPU tests (no GPU): the library loads and exports every declared symbol,
host-side validation and the input stream match the reference, and the
oracle restatement is pinned against the compiled reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from helpers import CONFIGS, canon_equal, offsets_for

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "edx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(edx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(edx):
    from paper_2512_21615_b200 import _lib
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(L, name), name
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound
    assert L.edx_abi_version() == 1


def test_validate_config_messages(edx):
    c = edx.ClusterConfig(n=65, m=1, bandwidths_bps=[1e9] * 65, cache_capacity=10)
    with pytest.raises(edx.InvalidArgument, match="at most 64 workers supported"):
        edx.validate(c, 1)
    c = edx.ClusterConfig(n=2, m=4, bandwidths_bps=[1e9], cache_capacity=10)
    with pytest.raises(edx.InvalidArgument, match="one bandwidth per worker"):
        edx.validate(c, 1)
    c = edx.ClusterConfig(n=2, m=4, bandwidths_bps=[1e9, 0.0], cache_capacity=10)
    with pytest.raises(edx.InvalidArgument, match="bandwidths must be positive"):
        edx.validate(c, 1)
    c = edx.ClusterConfig(n=2, m=256, bandwidths_bps=[1e9, 1e9], cache_capacity=5000)
    with pytest.raises(edx.InvalidArgument, match="cannot hold one micro-batch of 6656"):
        edx.validate(c, 26)
    c = edx.ClusterConfig(n=2, m=2, bandwidths_bps=[1e9, 1e9], cache_capacity=10, alpha=1.5)
    with pytest.raises(edx.InvalidArgument, match="alpha"):
        edx.validate(c, 1)
    edx.validate(edx.ClusterConfig(n=4, m=256, bandwidths_bps=[5e9] * 4, cache_capacity=10000), 26)


def test_unit_cost_known_answers(edx):
    """test_core.cpp:43-49."""
    c = edx.ClusterConfig(n=2, m=1, bandwidths_bps=[5e9, 5e8])
    assert edx.unit_cost(c, 0) == 3.2768e-6
    assert edx.unit_cost(c, 1) == 3.2768e-5
    with pytest.raises(edx.InvalidArgument):
        edx.unit_cost(c, 2)


def test_make_sample(edx):
    assert edx.make_sample([3, 1, 3, 2, 1]) == [3, 1, 2]
    with pytest.raises(edx.InvalidArgument):
        edx.make_sample([])


def test_expand_columns(edx):
    m = np.array([[1, 2], [3, 4], [5, 6]], float)
    sq = edx.expand_columns(m, [2, 0], 1)
    assert sq.values.tolist() == [[5, 6], [1, 2]]
    assert sq.col_to_worker.tolist() == [0, 1]
    with pytest.raises(edx.InvalidArgument):
        edx.expand_columns(m, [0], 1)


@pytest.mark.parametrize("name", ["C1", "P2", "C3"])
def test_zipf_stream_matches_oracle(edx, oracle, name):
    """The product's input stream (workload.cpp) == the reference's ZipfStream."""
    p = CONFIGS[name]
    R = p["n"] * p["m"]
    z = edx.ZipfStream(p["V"], p["L"], 1.05, 3, 42, R)
    for a, b in zip(z, oracle.zipf_batches(p["V"], p["L"], 1.05, 3, 42, R)):
        assert (a == b).all()


def test_oracle_port_kats(port, pyoracle):
    """The restatement reproduces the reference's own known answers."""
    c = pyoracle.Cfg(3, 1, [5e9, 5e9, 5e8])
    m = port.build_matrix_snapshot(c, {9: (4, 4, 4)}, np.array([9, 1, 2], np.uint32), [0, 1, 2, 3])
    assert m[0, 1] == 3.2768e-6 + 3.2768e-5
    cols, total = port.hungarian(np.array([[1, 2], [3, 1]], float))
    assert cols.tolist() == [0, 1] and total == 2.0
    rows, workers = port.greedy_dispatch(np.array([[0, 5], [0, 6], [1, 3], [2, 7]], float),
                                         [0, 1, 2, 3], [2, 2])
    assert workers.tolist() == [0, 0, 1, 1]
    s = port.sim(pyoracle.Cfg(3, 1, [5e9, 5e9, 5e8], cap=16))
    s.seed_entry(1, 0, True, False)
    s.seed_entry(9, 2, True, True)
    rep = s.step(np.array([1, 9, 8, 10, 11], np.uint32), [0, 1, 2, 5], [0, 1, 2])
    assert rep["miss_pull_w"] == [0, 1, 3] and rep["update_push_w"] == [0, 0, 1]
    assert rep["cost_w"] == [0.0, 3.2768e-6, 4 * 3.2768e-5]


@pytest.mark.parametrize("name,alpha,iters,seed", [("P2", 0.5, 50, 1234), ("P3", 1.0, 60, 7),
                                                   ("P8", 0.25, 30, 99), ("C1", 0.0, 6, 42)])
def test_oracle_port_equals_reference(port, ref, pyoracle, name, alpha, iters, seed):
    """Pins the plain-C oracle against the compiled, unmodified reference."""
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    cfg = pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha)
    a, b = port.sim(cfg), ref.sim(cfg)
    offs = offsets_for(R, L)
    for ids, ids2 in zip(port.zipf_batches(p["V"], L, 1.05, iters, seed, R),
                         ref.zipf_batches(p["V"], L, 1.05, iters, seed, R)):
        assert (ids == ids2).all()
        ma, mb = a.build_matrix(ids, offs), b.build_matrix(ids, offs)
        assert ma.tobytes() == mb.tobytes()
        da, db = port.ecomix(cfg, ma), ref.ecomix(cfg, mb)
        assert (da == db).all()
        assert a.step(ids, offs, da) == b.step(ids, offs, db)
    assert not canon_equal(a.canonical_state(), b.canonical_state())


def test_oracle_solver_equals_reference(port, ref):
    for k, maxv in [(5, 100), (40, 3), (128, 1000)]:
        sq = np.random.default_rng(k).integers(0, maxv + 1, (k, k)).astype(float)
        c1, t1 = port.hungarian(sq)
        c2, t2 = ref.hungarian(sq)
        assert (c1 == c2).all() and t1 == t2
    assert (port.bench_matrix(16) == ref.bench_matrix(16)).all()


@pytest.mark.parametrize("name", ["P2", "P3", "P8"])
def test_oracle_hitgreedy_equals_reference(port, ref, pyoracle, name):
    """baseline_hitgreedy restatement vs the compiled reference, driving both
    simulators with it (assign.hpp:346-392, sim.hpp:390-391)."""
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    cfg = pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.0)
    a, b = port.sim(cfg), ref.sim(cfg)
    offs = offsets_for(n * m, L)
    for ids in port.zipf_batches(p["V"], L, 1.05, 40, 11, n * m):
        da, db = a.hitgreedy(ids, offs), b.hitgreedy(ids, offs)
        assert (da == db).all()
        assert a.step(ids, offs, da) == b.step(ids, offs, db)
    assert not canon_equal(a.canonical_state(), b.canonical_state())


@pytest.mark.parametrize("V,L,R,iters", [(10_000_000, 26, 2048, 3), (10_000_000, 100, 1024, 2),
                                         (1000, 30, 64, 40)])
def test_zipf_stream_large_and_reset(edx, oracle, V, L, R, iters):
    """Guide-table mapping, chunked draws, hash dedup and the producer thread
    reproduce the reference's stream at the 10M-id vocabulary and with heavy
    rejection (L = 30 of 1,000 ids); reset() replays it."""
    z = edx.ZipfStream(V, L, 1.05, iters, 7, R)
    want = list(oracle.zipf_batches(V, L, 1.05, iters, 7, R))
    got = list(z)
    assert len(got) == iters and all((a == b).all() for a, b in zip(got, want))
    z.reset()
    assert (next(iter(z)) == want[0]).all()


def random_sized_case(seed, n, R=12, V=300):
    """A consistent random snapshot, ragged samples and per-id sizes."""
    rng = np.random.default_rng(seed)
    full = (1 << n) - 1

    def bits():
        return (int(rng.integers(0, 1 << 32)) << 32 | int(rng.integers(0, 1 << 32))) & full

    snap = {}
    for id_ in range(V):
        k = rng.integers(0, 4)
        if k == 0:
            continue
        res = bits()
        own = res & bits() if k == 3 else 0
        lat = own if own else res & bits()
        snap[id_] = (own, lat, res)
    size_of = {i: int(rng.choice([256, 1024, 2048, 4096, 3000, 777])) for i in range(V + 20)}
    samples = [list(rng.choice(V + 20, size=int(rng.integers(0, 25)), replace=False)) for _ in range(R)]
    ids = np.array([x for s in samples for x in s], np.uint32)
    offs = np.zeros(R + 1, np.uint64)
    offs[1:] = np.cumsum([len(s) for s in samples])
    sizes = np.array([size_of[int(x)] for x in ids], np.uint64)
    bw = rng.choice([5e9, 2e9, 5e8, 1e9, 3.3e9], size=n)
    return snap, samples, ids, offs, sizes, size_of, bw


def test_oracle_sized_kat(port, ref, pyoracle):
    """test_cost.cpp:241-249: non-uniform sizes flow through the cost hook."""
    cfg = pyoracle.Cfg(2, 1, [5e9, 5e9])
    ids = np.array([1, 2], np.uint32)
    offs = np.array([0, 2, 2], np.uint64)
    sizes = np.array([4096, 1024], np.uint64)
    for o in (port, ref):
        got = o.expected_costs_sized(cfg, {}, ids, offs, sizes)
        assert got[0, 0] == (4096.0 * 8 / 5e9) + (1024.0 * 8 / 5e9)


@pytest.mark.parametrize("n", [1, 3, 8, 33, 64])
def test_oracle_sized_equals_reference(port, ref, pyoracle, n):
    snap, _, ids, offs, sizes, _, bw = random_sized_case(50 + n, n)
    cfg = pyoracle.Cfg(n, 1, bw)
    a = port.expected_costs_sized(cfg, snap, ids, offs, sizes)
    b = ref.expected_costs_sized(cfg, snap, ids, offs, sizes)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("seed,capacity,id_range", [(1, 1, 4), (2, 3, 8), (3, 8, 32), (4, 16, 40)])
def test_oracle_cache_equals_reference(port, ref, policy, seed, capacity, id_range):
    """The restated standalone WorkerCache (both victim policies) against the
    reference class on random traffic: every result, error and state."""
    from helpers import apply_cache_op, cache_op_stream
    a, b = port.cache(capacity, policy), ref.cache(capacity, policy)
    for op in cache_op_stream(seed, capacity, 600, id_range):
        ra, rb = apply_cache_op(a, op, False), apply_cache_op(b, op, False)
        assert ra == rb, (op, ra, rb)
        assert a.info() == b.info(), op
        assert a.entries() == b.entries(), op
