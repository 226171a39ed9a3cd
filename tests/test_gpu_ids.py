"""Arbitrary 32-bit embedding ids (hashed engines: id_space = 0).

The reference keys its global state and every cache by uint32 id in
unordered_maps (sim.hpp:266, cache.hpp:238).  These tests run the engine with
no id bound -- the device id table (ids.cu) translating each batch -- on ids
spread over the whole [0, 2^32) range (a bijection of the reference's Zipf
ids), including table growth, imported states and VictimKeys wider than 64
bits, and compare every iteration with the compiled reference on the same ids."""
import numpy as np
import pytest

from helpers import CONFIGS, canon_equal, offsets_for
from scale_state import spread_id, spread_state, synthetic_full_state

pytestmark = pytest.mark.gpu


def _pair(edx, pyoracle, oracle, p, alpha, max_ids=None):
    n, m, L = p["n"], p["m"], p["L"]
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], d_tran_bytes=2048,
                          cache_capacity=p["cap"], alpha=alpha)
    eng = edx.SimState(c, id_space=0, max_batch_ids=max_ids or n * m * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha))
    return eng, sim


def _run(eng, sim, oracle, pyoracle, p, alpha, batches, state_every=1):
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    offs = offsets_for(R, L)
    for it, ids in enumerate(batches):
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
        assert eng.step().as_dict() == want_r, f"iter {it}: report differs"
        if state_every and (it % state_every == 0 or it == len(batches) - 1):
            msg = canon_equal(eng.canonical_state(), sim.canonical_state())
            assert not msg, f"iter {it}: {msg}"
    eng.validate_consistency()


def test_extreme_ids_kat(gpu, pyoracle, oracle):
    """Ids 0, 2^31, 2^32 - 2 and 2^32 - 1 through seed_entry, state_of and a step."""
    edx = gpu
    p = dict(n=3, m=1, bw=[5e9, 5e9, 5e8], cap=8, L=3)
    eng, sim = _pair(edx, pyoracle, oracle, p, 0.0, max_ids=16)
    big = [0, 1 << 31, 0xFFFFFFFE, 0xFFFFFFFF]
    for s in (eng, sim):
        s.seed_entry(big[3], 0, True, True)
        s.seed_entry(big[1], 2, True, False)
    assert eng.state_of(big[3]).owned_by(0)
    assert eng.state_of(123).owners == 0 and eng.state_of(0xFFFFFFFE).resident == 0
    samples = [[big[3], big[0]], [big[1]], [big[2], big[3], 7]]
    ids = np.array([x for smp in samples for x in smp], np.uint32)
    offs = np.array([0, 2, 3, 6], np.uint64)
    dec = [0, 1, 2]
    assert eng.step(samples, dec).as_dict() == sim.step(ids, offs, dec)
    assert not canon_equal(eng.canonical_state(), sim.canonical_state())
    eng.validate_consistency()


@pytest.mark.parametrize("name,alpha,iters,seed", [("P8", 0.5, 30, 99), ("C2", 0.5, 8, 42),
                                                   ("P24", 0.5, 10, 21)])
def test_spread_ids_trajectory(gpu, pyoracle, oracle, name, alpha, iters, seed):
    p = CONFIGS[name]
    eng, sim = _pair(gpu, pyoracle, oracle, p, alpha)
    batches = [spread_id(b) for b in oracle.zipf_batches(p["V"], p["L"], 1.05, iters, seed,
                                                         p["n"] * p["m"])]
    _run(eng, sim, oracle, pyoracle, p, alpha, batches, state_every=5)


@pytest.mark.parametrize("name", ["PX", "PXL"])
def test_spread_ids_table_growth(gpu, pyoracle, oracle, name):
    """500K-id vocabularies through a table that starts at 16 batches (102,400 slots):
    several growths, with thousands of evictions per worker per step."""
    p = CONFIGS[name]
    eng, sim = _pair(gpu, pyoracle, oracle, p, 0.25 if name == "PXL" else 0.0)
    batches = [spread_id(b) for b in oracle.zipf_batches(p["V"], p["L"], 0.6, 8, 13,
                                                         p["n"] * p["m"])]
    _run(eng, sim, oracle, pyoracle, p, 0.25 if name == "PXL" else 0.0, batches, state_every=4)


def test_spread_ids_wide_victim_keys(gpu, pyoracle, oracle):
    """An imported full state whose VictimKeys need ~95 bits (frequencies and
    access times up to 2^30, ids over 32 bits): the selection's 128-bit path."""
    p = dict(n=4, m=64, bw=[5e9, 5e9, 5e8, 5e8], cap=3000, V=200_000, L=26)
    eng, sim = _pair(gpu, pyoracle, oracle, p, 0.25)
    clock = 1 << 30
    state = spread_state(synthetic_full_state(p["n"], p["cap"], p["V"], clock, 5,
                                              freq_hi=1 << 30))
    eng.import_state(state, clock)
    sim.import_state(state, clock)
    assert not canon_equal(eng.canonical_state(), state)
    batches = [spread_id(b) for b in oracle.zipf_batches(p["V"], p["L"], 1.05, 4, 5,
                                                         p["n"] * p["m"])]
    _run(eng, sim, oracle, pyoracle, p, 0.25, batches, state_every=1)


def test_dense_wide_victim_keys(gpu, pyoracle, oracle):
    """The same wide keys on a dense-id engine (id field < 2^18, freq and
    last access over 30 bits each)."""
    p = dict(n=4, m=64, bw=[5e9, 5e9, 5e8, 5e8], cap=3000, V=200_000, L=26)
    n, m, L = p["n"], p["m"], p["L"]
    c = gpu.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], d_tran_bytes=2048,
                          cache_capacity=p["cap"], alpha=0.0)
    eng = gpu.SimState(c, id_space=p["V"], max_batch_ids=n * m * L)
    sim = oracle.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.0))
    clock = 1 << 30
    state = synthetic_full_state(n, p["cap"], p["V"], clock, 6, freq_hi=1 << 30)
    eng.import_state(state, clock)
    sim.import_state(state, clock)
    batches = list(oracle.zipf_batches(p["V"], L, 1.05, 4, 6, n * m))
    _run(eng, sim, oracle, pyoracle, p, 0.0, batches, state_every=1)
