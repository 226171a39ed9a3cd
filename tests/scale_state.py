"""Synthetic evicting steady states for the scale parity tests.

A full SimState (every worker's cache at capacity) in canonical_state()
format, built directly rather than by thousands of prefill iterations: both
sides import it (edx_engine_import_state / orc_sim_import_state) and then run
the same batches, so the next iterations evict from the first insert.  The
state satisfies every invariant SimState::validate_consistency checks
(sim.hpp:222-248): resident bits = cache membership, owners ⊆ latest ⊆
resident, owners != 0 ⇒ latest == owners, version flag = the worker's latest
bit, at_current_mark = #entries at the worker's current mark.  Cache contents
lean towards small ids, which ZipfStream draws most often (P(id) ∝
(id+1)^-s, workload.hpp:54-79), so the batches hit, miss and evict.  Some
workers hold every entry at the current mark, so their epoch advances at the
first eviction (cache.hpp:187-192)."""
import numpy as np


def synthetic_full_state(n, cap, V, clock, seed, all_current_every=4, freq_hi=60):
    rng = np.random.default_rng(seed)
    per_worker = []
    for j in range(n):
        # a hot prefix of small ids (each kept with probability 0.9) plus
        # distinct cold ids drawn uniformly above it
        h = int(rng.integers(cap // 4, cap // 2 + 1))
        hot = np.flatnonzero(rng.random(h) < 0.9).astype(np.uint32)
        need = cap - len(hot)
        cold = np.zeros(0, np.uint32)
        while len(cold) < need:
            draw = rng.integers(h, V, int((need - len(cold)) * 1.1) + 64).astype(np.uint32)
            cold = np.unique(np.concatenate([cold, draw]))
        cold = rng.permutation(cold)[:need]
        per_worker.append(np.sort(np.concatenate([hot, cold])))
    pairs_id = np.concatenate(per_worker)
    pairs_w = np.concatenate([np.full(len(x), j, np.uint64) for j, x in enumerate(per_worker)])
    order = np.argsort(pairs_id, kind="stable")
    sid = pairs_id[order]
    starts = np.flatnonzero(np.concatenate([[True], sid[1:] != sid[:-1]]))
    uniq = sid[starts]
    resident = np.bitwise_or.reduceat(np.left_shift(np.uint64(1), pairs_w[order]), starts)
    rnd = (rng.integers(0, 1 << 32, len(uniq), dtype=np.uint64) << np.uint64(32)) | \
        rng.integers(0, 1 << 32, len(uniq), dtype=np.uint64)
    latest = resident & rnd
    owned = (latest != 0) & (rng.random(len(uniq)) < 0.5)
    owners = np.where(owned, latest, np.uint64(0))
    glob = np.stack([uniq.astype(np.uint64), owners, latest, resident], 1)
    caches = []
    for j, ids in enumerate(per_worker):
        pos = np.searchsorted(uniq, ids)
        ver = (latest[pos] >> np.uint64(j)) & np.uint64(1)
        cur = int(rng.integers(1, 6))
        if all_current_every and j % all_current_every == 0:
            mark = np.full(len(ids), cur, np.uint64)  # the epoch advances at the first eviction
        else:
            mark = np.uint64(cur) - rng.integers(0, min(3, cur), len(ids)).astype(np.uint64)
        freq = rng.integers(1, freq_hi, len(ids)).astype(np.uint64)
        last = rng.integers(0, clock, len(ids)).astype(np.uint64)
        ent = np.stack([ids.astype(np.uint64), ver, mark, freq, last], 1)
        caches.append((ent, cur, int((mark == cur).sum())))
    return glob, caches


def spread_id(ids):
    """A bijection of uint32 (odd multiplier mod 2^32): maps the dense Zipf ids
    onto the whole [0, 2^32) range, order scrambled."""
    x = np.asarray(ids, np.uint64)
    return ((x * np.uint64(0x9E3779B1) + np.uint64(0x7F4A7C15)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def spread_state(state):
    """synthetic_full_state() output with every id mapped through spread_id,
    rows re-sorted by the new ids (canonical order)."""
    glob, caches = state
    g = glob.copy()
    g[:, 0] = spread_id(g[:, 0])
    g = g[np.argsort(g[:, 0], kind="stable")]
    out = []
    for ent, cur, at in caches:
        e = ent.copy()
        e[:, 0] = spread_id(e[:, 0])
        out.append((e[np.argsort(e[:, 0], kind="stable")], cur, at))
    return g, out
