"""GPU parity of the engine (SimState on device) against the oracle.

KATs from tests/test_sim.cpp, then multi-iteration runs over the reference's
own input stream comparing, after every iteration: every matrix cell
(bitwise), the decision, expected_cost_s, the IterationReport and the
canonical global + cache state."""
import numpy as np
import pytest

from helpers import CONFIGS, canon_equal, offsets_for

pytestmark = pytest.mark.gpu

U = 3.2768e-6


def make(edx, n, m, cap, bw=None, alpha=1.0, id_space=1 << 12, max_ids=1 << 12):
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=bw or [5e9] * n, d_tran_bytes=2048,
                          cache_capacity=cap, alpha=alpha)
    return c, edx.SimState(c, id_space=id_space, max_batch_ids=max_ids)


def test_walkthrough_fig2(gpu):
    """test_sim.cpp:50-83."""
    edx = gpu
    c, s = make(edx, 3, 1, 16, [5e9, 5e9, 5e8])
    s.seed_entry(1, 0, True, False)
    s.seed_entry(9, 2, True, True)
    rep = s.step([[1], [9], [8, 10, 11]], [0, 1, 2])
    assert rep.miss_pull_w == [0, 1, 3]
    assert rep.update_push_w == [0, 0, 1]
    assert rep.evict_push == 0 and rep.hits == 1 and rep.lookups == 5
    assert rep.cost_w == [0.0, U, 4 * 3.2768e-5]
    x9 = s.state_of(9)
    assert x9.owned_by(1) and not x9.owned_by(2) and not x9.latest_on(2) and x9.resident_on(2)
    ent = {int(r[0]): r for r in s.cache_entries(2)}
    assert 9 in ent and ent[9][1] == 0
    s.validate_consistency()


def test_owner_keeps_embedding(gpu):
    edx = gpu
    c, s = make(edx, 2, 1, 8)
    s.seed_entry(5, 0, True, True)
    rep = s.step([[5], [6]], [0, 1])
    assert rep.update_push == 0 and rep.miss_pull_w == [0, 1] and rep.hits == 1
    assert rep.cost_w[0] == 0.0
    rep = s.step([[7], [5]], [0, 1])
    assert rep.update_push_w == [1, 0] and rep.miss_pull_w == [1, 1]
    s.validate_consistency()


def test_mutual_pushes(gpu):
    edx = gpu
    c, s = make(edx, 2, 1, 8)
    rep = s.step([[3], [3]], [0, 1])
    assert rep.miss_pull == 2
    st = s.state_of(3)
    assert st.owned_by(0) and st.owned_by(1)
    rep = s.step([[3], [3]], [0, 1])
    assert rep.update_push == 2 and rep.miss_pull == 0 and rep.hits == 2
    s.validate_consistency()


def test_unbalanced_decision_rejected(gpu):
    edx = gpu
    c, s = make(edx, 2, 1, 8)
    with pytest.raises(edx.InvalidArgument):
        s.step([[1], [2]], [0, 0])
    with pytest.raises(edx.InvalidArgument):
        s.step([[1], [2]], [0])


def test_seed_full_cache(gpu):
    edx = gpu
    c, s = make(edx, 1, 1, 1)
    s.seed_entry(1, 0, True, False)
    with pytest.raises(edx.LogicError, match="full cache"):
        s.seed_entry(2, 0, True, False)
    s.seed_entry(1, 0, True, False)  # refresh is fine


def run_parity(edx, oracle, pyoracle, name, alpha, iters, seed=42, s=1.05, check_state_every=1,
               id_space=None):
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], d_tran_bytes=2048,
                          cache_capacity=p["cap"], alpha=alpha)
    eng = edx.SimState(c, id_space=id_space or p["V"], max_batch_ids=R * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha))
    offs = offsets_for(R, L)
    it = -1
    for it, ids in enumerate(oracle.zipf_batches(p["V"], L, s, iters, seed, R)):
        want_m = sim.build_matrix(ids, offs)
        eng.load((ids, offs))
        got_m = np.empty((R, n))
        eng.build(got_m)
        assert got_m.tobytes() == want_m.tobytes(), f"iter {it}: matrix differs"
        want_d = oracle.ecomix(pyoracle.Cfg(n, m, p["bw"], alpha=alpha), want_m)
        got_d, got_exp = eng.dispatch()
        assert (got_d == want_d).all(), f"iter {it}: decision differs"
        assert got_exp == oracle.decision_cost(want_m, want_d), f"iter {it}: expected cost"
        want_r = sim.step(ids, offs, want_d)
        got_r = eng.step().as_dict()
        assert got_r == want_r, f"iter {it}: report {got_r} vs {want_r}"
        if check_state_every and (it % check_state_every == 0 or it == iters - 1):
            msg = canon_equal(eng.canonical_state(), sim.canonical_state())
            assert not msg, f"iter {it}: {msg}"
    assert it == iters - 1
    eng.validate_consistency()
    return eng, sim


@pytest.mark.parametrize("alpha", [0.0, 0.5, 1.0])
def test_engine_eviction_pressure_p2(gpu, oracle, pyoracle, alpha):
    """test_sim.cpp:172-209 configuration (n=2, m=4, cap 12, V=60, L=3, 50 iters)."""
    run_parity(gpu, oracle, pyoracle, "P2", alpha, 50, seed=1234)


@pytest.mark.parametrize("alpha", [0.0, 0.25, 1.0])
def test_engine_eviction_pressure_p3(gpu, oracle, pyoracle, alpha):
    run_parity(gpu, oracle, pyoracle, "P3", alpha, 60, seed=7)


@pytest.mark.parametrize("alpha", [0.0, 0.5])
def test_engine_eviction_pressure_p8(gpu, oracle, pyoracle, alpha):
    run_parity(gpu, oracle, pyoracle, "P8", alpha, 40, seed=99)


@pytest.mark.parametrize("s", [0.6, 1.05])
def test_engine_mass_eviction(gpu, oracle, pyoracle, s):
    """Thousands of victims per worker per step (s = 0.6: > 4096, the full
    block sort; s = 1.05: the radix-select path), caches refilled every step."""
    run_parity(gpu, oracle, pyoracle, "PX", 0.0, 6, seed=11, s=s)


@pytest.mark.parametrize("name,alpha", [("P24", 0.5), ("P32", 1.0), ("P32", 0.25)])
def test_engine_wide_exact_block(gpu, oracle, pyoracle, name, alpha):
    """16 < n <= 32 engines through the hybrid dispatcher (two blocks per warp)."""
    run_parity(gpu, oracle, pyoracle, name, alpha, 15, seed=21)


@pytest.mark.parametrize("s", [0.6, 1.05])
def test_engine_mass_eviction_large_caches(gpu, oracle, pyoracle, s):
    """Caches of 13,000 entries (> the one-CTA selection size): victims through
    the device-wide candidate ranges, packing and sort, thousands per step."""
    run_parity(gpu, oracle, pyoracle, "PXL", 0.25, 7, seed=13, s=s)


def test_engine_c1(gpu, oracle, pyoracle):
    """C1: 4 workers, batch 1024, uniform, 10% cache, greedy only."""
    run_parity(gpu, oracle, pyoracle, "C1", 0.0, 30, check_state_every=10)


@pytest.mark.parametrize("alpha", [0.25, 0.5])
def test_engine_c2(gpu, oracle, pyoracle, alpha):
    """C2: 8 heterogeneous workers, hybrid."""
    run_parity(gpu, oracle, pyoracle, "C2", alpha, 12, check_state_every=4)


def test_iterate_equals_stepwise(gpu, oracle, pyoracle):
    """edx_engine_iterate (the fused run() body) gives the same results."""
    edx = gpu
    p = CONFIGS["P8"]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], cache_capacity=p["cap"], alpha=0.5)
    eng = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.5))
    offs = offsets_for(R, L)
    for ids in oracle.zipf_batches(p["V"], L, 1.05, 25, 5, R):
        dec, rep = eng.iterate(ids, offs)
        wdec, wexp, wrep, _ = sim.iteration(ids, offs)
        assert (dec == wdec).all()
        assert rep.as_dict() == wrep
        assert rep.expected_cost_s == wexp
    assert not canon_equal(eng.canonical_state(), sim.canonical_state())


@pytest.mark.parametrize("name,iters", [("P2", 50), ("P8", 40), ("C1", 15), ("C2", 10)])
def test_engine_hitgreedy_trajectory(gpu, oracle, pyoracle, name, iters):
    """run() with the hit-greedy mechanism: decisions on the live device state,
    then the step, equal to the reference simulator driven the same way."""
    edx = gpu
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], d_tran_bytes=2048,
                          cache_capacity=p["cap"], alpha=0.0)
    eng = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.0))
    offs = offsets_for(R, L)
    for it, ids in enumerate(oracle.zipf_batches(p["V"], L, 1.05, iters, 5, R)):
        want_d = sim.hitgreedy(ids, offs)
        eng.load((ids, offs))
        got_d = eng.dispatch_hitgreedy()
        assert (got_d == want_d).all(), f"iter {it}: decision differs"
        assert eng.step().as_dict() == sim.step(ids, offs, want_d), f"iter {it}: report"
    msg = canon_equal(eng.canonical_state(), sim.canonical_state())
    assert not msg, msg


def test_engine_64_workers(gpu, oracle, pyoracle):
    """n = 64 (the widest the reference accepts; the C5 sweep corner's worker
    count): full 64-bit masks through build, EcoMix, step and state."""
    edx = gpu
    n, m, L, V, cap = 64, 4, 5, 3000, 40
    bw = [5e9] * 32 + [5e8] * 32
    R = n * m
    for alpha in (0.0, 0.5):
        c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=bw, d_tran_bytes=2048,
                              cache_capacity=cap, alpha=alpha)
        eng = edx.SimState(c, id_space=V, max_batch_ids=R * L)
        sim = oracle.sim(pyoracle.Cfg(n, m, bw, cap=cap, alpha=alpha))
        offs = offsets_for(R, L)
        for it, ids in enumerate(oracle.zipf_batches(V, L, 1.05, 12, 3, R)):
            want_m = sim.build_matrix(ids, offs)
            eng.load((ids, offs))
            got_m = np.empty((R, n))
            eng.build(got_m)
            assert got_m.tobytes() == want_m.tobytes(), f"alpha {alpha} iter {it}: matrix"
            want_d = oracle.ecomix(pyoracle.Cfg(n, m, bw, alpha=alpha), want_m)
            got_d, _ = eng.dispatch()
            assert (got_d == want_d).all(), f"alpha {alpha} iter {it}: decision"
            assert eng.step().as_dict() == sim.step(ids, offs, want_d), f"alpha {alpha} iter {it}"
        msg = canon_equal(eng.canonical_state(), sim.canonical_state())
        assert not msg, msg


def test_device_batch_declared_total(gpu, oracle, pyoracle):
    """edx_engine_load_device_batch: a device-resident batch with its id count
    declared (no host round trip) gives the same iteration as a host load; a
    wrong count fails loudly at the next synchronising call."""
    import torch
    edx = gpu
    p = CONFIGS["P8"]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], cache_capacity=p["cap"], alpha=0.5)
    a = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    b = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    offs = offsets_for(R, L)
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    for ids in oracle.zipf_batches(p["V"], L, 1.05, 6, 3, R):
        d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
        torch.cuda.synchronize()
        a.load(None, on_device=True, ids_ptr=d_ids.data_ptr(), offsets_ptr=d_offs.data_ptr(), rows=R,
               total_ids=R * L)
        ma = np.empty((R, n))
        a.build(ma)
        da, _ = a.dispatch()
        ra = a.step().as_dict()
        b.load((ids, offs))
        mb = np.empty((R, n))
        b.build(mb)
        db, _ = b.dispatch()
        rb = b.step().as_dict()
        assert ma.tobytes() == mb.tobytes() and (da == db).all() and ra == rb
    torch.cuda.synchronize()
    a.load(None, on_device=True, ids_ptr=d_ids.data_ptr(), offsets_ptr=d_offs.data_ptr(), rows=R,
           total_ids=R * L - 1)
    with pytest.raises(edx.InvalidArgument, match="declared id count"):
        a.build(np.empty((R, n)))


@pytest.mark.parametrize("name,alpha", [("C2", 0.5), ("C1", 0.0), ("P8", 1.0)])
def test_iterate_device_graph_replay(gpu, oracle, pyoracle, name, alpha):
    """edx_engine_iterate_device: from the third iteration of a shape the
    iteration is a CUDA-graph replay; every decision, report and the final
    state equal the reference run() body, also across a shape change."""
    import torch
    edx = gpu
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], cache_capacity=p["cap"], alpha=alpha)
    eng = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha))
    offs = offsets_for(R, L)
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    batches = list(oracle.zipf_batches(p["V"], L, 1.05, 10, 17, R))
    for it, ids in enumerate(batches):
        if it == 6:  # a host-path iteration and a stepwise one in between (graph reuse)
            dec, rep = eng.iterate(ids, offs)
        else:
            d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
            torch.cuda.synchronize()
            dec, rep = eng.iterate_device(d_ids.data_ptr(), d_offs.data_ptr(), R, R * L)
        wdec, wexp, wrep, _ = sim.iteration(ids, offs)
        assert (dec == wdec).all(), f"iter {it}: decision"
        assert rep.as_dict() == wrep, f"iter {it}: report"
        assert rep.expected_cost_s == wexp, f"iter {it}: expected cost"
    msg = canon_equal(eng.canonical_state(), sim.canonical_state())
    assert not msg, msg


@pytest.mark.parametrize("name,alpha", [("C2", 0.5), ("C1", 0.0)])
def test_iterate_with_prefetch(gpu, oracle, pyoracle, name, alpha):
    """edx_engine_prefetch: batch i+1's host->device copy is issued before
    iteration i; every decision, report and the final state equal the
    reference run() body.  Also: a prefetched batch that is never consumed, a
    host batch that was not prefetched, and prefetch's offset validation."""
    import torch
    edx = gpu
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], cache_capacity=p["cap"], alpha=alpha)
    eng = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha))
    offs = torch.from_numpy(offsets_for(R, L).view(np.int64)).pin_memory().numpy().view(np.uint64)
    batches = [torch.from_numpy(b.view(np.int32)).pin_memory().numpy().view(np.uint32)
               for b in oracle.zipf_batches(p["V"], L, 1.05, 10, 23, R)]
    stray = batches[0].copy()
    eng.prefetch(batches[0], offs)
    for it, ids in enumerate(batches):
        if it == 4:
            eng.prefetch(stray, offs)  # never consumed: batch 5 is not prefetched
        elif it + 1 < len(batches) and it != 4:
            eng.prefetch(batches[it + 1], offs)
        dec, rep = eng.iterate(ids, offs)
        wdec, wexp, wrep, _ = sim.iteration(ids, offs)
        assert (dec == wdec).all(), f"iter {it}: decision"
        assert rep.as_dict() == wrep, f"iter {it}: report"
        assert rep.expected_cost_s == wexp, f"iter {it}: expected cost"
    msg = canon_equal(eng.canonical_state(), sim.canonical_state())
    assert not msg, msg
    bad = offs.copy()
    bad[1], bad[2] = bad[2], bad[1]
    with pytest.raises(edx.InvalidArgument, match="non-decreasing"):
        eng.prefetch(batches[0], bad)
    with pytest.raises(edx.InvalidArgument, match="no samples"):
        eng.prefetch(batches[0], offs[:1])


def test_iterate_prefetch_next(gpu, oracle, pyoracle):
    """edx_engine_iterate_prefetch: the loop bench.py's e2e leg runs (batch
    i+1 prefetched once iteration i is launched) equals the reference; a bad
    next batch is rejected before the iteration starts (clock unchanged)."""
    import torch
    edx = gpu
    p = CONFIGS["C2"]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], cache_capacity=p["cap"], alpha=0.5)
    eng = edx.SimState(c, id_space=p["V"], max_batch_ids=R * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.5))
    offs = torch.from_numpy(offsets_for(R, L).view(np.int64)).pin_memory().numpy().view(np.uint64)
    batches = [torch.from_numpy(b.view(np.int32)).pin_memory().numpy().view(np.uint32)
               for b in oracle.zipf_batches(p["V"], L, 1.05, 8, 29, R)]
    eng.prefetch(batches[0], offs)
    for it, ids in enumerate(batches):
        nxt = (batches[it + 1], offs) if it + 1 < len(batches) else None
        dec, rep = eng.iterate(ids, offs, prefetch_next=nxt)
        wdec, wexp, wrep, _ = sim.iteration(ids, offs)
        assert (dec == wdec).all(), f"iter {it}: decision"
        assert rep.as_dict() == wrep, f"iter {it}: report"
        assert rep.expected_cost_s == wexp, f"iter {it}: expected cost"
    bad = offs.copy()
    bad[1], bad[2] = bad[2], bad[1]
    clock = eng.clock()
    with pytest.raises(edx.InvalidArgument, match="non-decreasing"):
        eng.iterate(batches[0], offs, prefetch_next=(batches[1], bad))
    assert eng.clock() == clock
    msg = canon_equal(eng.canonical_state(), sim.canonical_state())
    assert not msg, msg
