"""Engine parity at the BASELINE.json shapes.

C3 and C4 start both sides from one imported, *evicting* steady state (every
cache at its 800,000-entry capacity; tests/scale_state.py) and then compare,
after every iteration, every matrix cell (bitwise), the decision, the
expected cost and the IterationReport against the compiled reference
(oracle/_ref), and the full canonical state after the last iteration.  The
C5 corner (n = 64, batch 65,536) and C2 at alpha = 1 (k = 1024) run from an
empty state over the reference's own input stream."""
import numpy as np
import pytest

from helpers import CONFIGS, canon_equal, offsets_for
from scale_state import synthetic_full_state

pytestmark = pytest.mark.gpu


def _engine(edx, pyoracle, ref, p, alpha):
    n, m, L = p["n"], p["m"], p["L"]
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], d_tran_bytes=2048,
                          cache_capacity=p["cap"], alpha=alpha)
    eng = edx.SimState(c, id_space=p["V"], max_batch_ids=n * m * L)
    sim = ref.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha))
    return eng, sim


def _iterate_and_compare(eng, sim, ref, pyoracle, p, alpha, batches, check_state_at=()):
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    offs = offsets_for(R, L)
    for it, ids in enumerate(batches):
        want_m = sim.build_matrix(ids, offs)
        eng.load((ids, offs))
        got_m = np.empty((R, n))
        eng.build(got_m)
        assert got_m.tobytes() == want_m.tobytes(), f"iter {it}: matrix differs"
        want_d = ref.ecomix(pyoracle.Cfg(n, m, p["bw"], alpha=alpha), want_m)
        got_d, got_exp = eng.dispatch()
        assert (got_d == want_d).all(), f"iter {it}: decision differs"
        assert got_exp == ref.decision_cost(want_m, want_d), f"iter {it}: expected cost"
        want_r = sim.step(ids, offs, want_d)
        got_r = eng.step().as_dict()
        assert got_r == want_r, f"iter {it}: report differs"
        if it in check_state_at:
            msg = canon_equal(eng.canonical_state(), sim.canonical_state())
            assert not msg, f"iter {it}: {msg}"


_STATES = {}
CLOCK = 400


def _state(name, seed):
    """One synthetic full state per config, shared by its parametrizations."""
    if name not in _STATES:
        p = CONFIGS[name]
        _STATES.clear()
        _STATES[name] = (synthetic_full_state(p["n"], p["cap"], p["V"], CLOCK, seed), [False])
    return _STATES[name]


def _evicting(edx, pyoracle, ref, name, alpha, iters, seed):
    p = CONFIGS[name]
    eng, sim = _engine(edx, pyoracle, ref, p, alpha)
    state, checked = _state(name, seed)
    eng.import_state(state, CLOCK)
    sim.import_state(state, CLOCK)
    if not checked[0]:  # the import round-trips (once per state)
        msg = canon_equal(eng.canonical_state(), state)
        assert not msg, f"imported state: {msg}"
        checked[0] = True
    sizes0 = [len(c[0]) for c in state[1]]
    assert sizes0 == [p["cap"]] * p["n"]
    batches = list(ref.zipf_batches(p["V"], p["L"], 1.05, iters, seed, p["n"] * p["m"]))
    _iterate_and_compare(eng, sim, ref, pyoracle, p, alpha, batches, check_state_at={iters - 1})
    # every cache stayed full: each insert evicted one entry
    assert [len(eng.cache_entries(j)) for j in range(p["n"])] == sizes0
    eng.validate_consistency()
    return eng, sim


@pytest.mark.parametrize("alpha", [0.125, 0.25])
def test_c3_evicting_steady_state(gpu, pyoracle, ref, alpha):
    """C3: 16 workers, batch 8192, 10M ids, full 800K caches; k = 1024 / 2048."""
    _evicting(gpu, pyoracle, ref, "C3", alpha, 3, seed=31)


@pytest.mark.parametrize("alpha", [0.0, 0.0625])
def test_c4_evicting_steady_state(gpu, pyoracle, ref, alpha):
    """C4: 32 workers, batch 16384, 100 ids/sample, full 800K caches; k = 0 / 1024."""
    _evicting(gpu, pyoracle, ref, "C4", alpha, 3, seed=41)


def test_c5_corner(gpu, pyoracle, ref):
    """C5 corner: 64 workers, batch 65,536, greedy, from empty (3 iterations)."""
    p = dict(n=64, m=1024, bw=[5e9] * 32 + [5e8] * 32, cap=800_000, V=10_000_000, L=26)
    eng, sim = _engine(gpu, pyoracle, ref, p, 0.0)
    batches = list(ref.zipf_batches(p["V"], p["L"], 1.05, 3, 42, p["n"] * p["m"]))
    _iterate_and_compare(eng, sim, ref, pyoracle, p, 0.0, batches, check_state_at={2})


def test_c2_alpha_one(gpu, pyoracle, ref):
    """C2 at alpha = 1: the whole batch through the exact solver (k = 1024)."""
    p = CONFIGS["C2"]
    eng, sim = _engine(gpu, pyoracle, ref, p, 1.0)
    batches = list(ref.zipf_batches(p["V"], p["L"], 1.05, 10, 42, p["n"] * p["m"]))
    _iterate_and_compare(eng, sim, ref, pyoracle, p, 1.0, batches, check_state_at={4, 9})
