"""Shared builders for the parity tests (configs follow SURVEY §8(d))."""
import numpy as np

HET = lambda n: [5e9] * (n // 2) + [5e8] * (n - n // 2)  # config.hpp:153 half fast, half slow

# (n, m, bandwidths, cache, V, L, iterations, zipf seed) — SURVEY §8(d)
CONFIGS = {
    "C1": dict(n=4, m=256, bw=[5e9] * 4, cap=10_000, V=100_000, L=26),
    "C2": dict(n=8, m=128, bw=HET(8), cap=10_000, V=100_000, L=26),
    "C3": dict(n=16, m=512, bw=HET(16), cap=800_000, V=10_000_000, L=26),
    "C4": dict(n=32, m=512, bw=HET(32), cap=800_000, V=10_000_000, L=100),
    # eviction pressure (test_sim.cpp:172-209)
    "P2": dict(n=2, m=4, bw=[5e9, 5e8], cap=12, V=60, L=3),
    "P3": dict(n=3, m=4, bw=[5e9, 5e9, 5e8], cap=14, V=80, L=3),
    "P8": dict(n=8, m=16, bw=HET(8), cap=120, V=400, L=6),
    # 16 < n <= 32: the two-blocks-per-warp exact solver
    "P24": dict(n=24, m=16, bw=HET(24), cap=160, V=1500, L=5),
    "P32": dict(n=32, m=12, bw=HET(32), cap=120, V=2000, L=4),
    # mass eviction: > 4096 victims per worker per step (the full-sort victim path)
    "PX": dict(n=2, m=64, bw=[5e9, 5e8], cap=12_000, V=500_000, L=100),
    # caches above the one-CTA selection size: host-sized device-wide victim path
    "PXL": dict(n=3, m=64, bw=[5e9, 5e9, 5e8], cap=13_000, V=500_000, L=100),
}


def offsets_for(R, L):
    return np.arange(R + 1, dtype=np.uint64) * np.uint64(L)


def canon_equal(a, b):
    """Compare (global, caches) canonical states; returns '' or a diff message."""
    ga, ca = a
    gb, cb = b
    if ga.shape != gb.shape or not (ga == gb).all():
        if ga.shape != gb.shape:
            return f"global count {ga.shape[0]} vs {gb.shape[0]}"
        bad = np.nonzero((ga != gb).any(1))[0][:5]
        return f"global rows differ at {bad.tolist()}: {ga[bad].tolist()} vs {gb[bad].tolist()}"
    for j, ((ea, ma, xa), (eb, mb, xb)) in enumerate(zip(ca, cb)):
        if ea.shape != eb.shape:
            return f"worker {j}: cache size {ea.shape[0]} vs {eb.shape[0]}"
        if not (ea == eb).all():
            bad = np.nonzero((ea != eb).any(1))[0][:5]
            return f"worker {j}: entries differ {ea[bad].tolist()} vs {eb[bad].tolist()}"
        if ma != mb or xa != xb:
            return f"worker {j}: marks ({ma},{xa}) vs ({mb},{xb})"
    return ""


def random_int_matrix(rows, cols, seed, max_value=100):
    """oracles::random_int_matrix (tests/oracles.hpp:80-95) semantics, numpy RNG."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, max_value + 1, size=(rows, cols)).astype(np.float64)


# ------------------------------------------------ standalone WorkerCache ops
def cache_footprint(id_):
    """A pure FootprintFn for the kPriorityRatio parity runs."""
    return 1.0 + float((id_ * 7) % 5) * 0.75


def cache_op_stream(seed, capacity, n_ops, id_range):
    """Random WorkerCache traffic: mostly touches (the reference's own random
    test, test_cache.cpp:181-191), set_version, erase, select_victim and
    evict_for with pinned sets -- errors included."""
    rng = np.random.default_rng(seed)
    for step in range(n_ops):
        k = rng.random()
        id_ = int(rng.integers(0, id_range))
        if k < 0.55:
            yield ("touch", id_, bool(rng.integers(0, 2)), int(rng.integers(0, max(step, 1) + 1)))
        elif k < 0.65:
            yield ("set_version", id_, bool(rng.integers(0, 2)))
        elif k < 0.72:
            yield ("erase", id_)
        elif k < 0.80:
            yield ("select_victim",)
        else:
            needed = int(rng.integers(0, capacity + 2))
            pins = [int(x) for x in rng.integers(0, id_range, size=int(rng.integers(0, capacity + 1)))]
            yield ("evict_for", needed, pins)


def _err_kind(e):
    n = type(e).__name__
    return ("logic" if "Logic" in n else "invalid" if "Invalid" in n else n, str(e))


def apply_cache_op(cache, op, device):
    """Run one op on a device WorkerCache (device=True) or an oracle Cache;
    returns its result or ('raised', kind, message)."""
    try:
        if op[0] == "touch":
            if device:
                return cache.touch(op[1], op[2], op[3])
            return cache.touch(op[1], op[2], op[3], cache_footprint(op[1]))
        if op[0] == "set_version":
            return cache.set_version(op[1], op[2])
        if op[0] == "erase":
            return cache.erase(op[1])
        if op[0] == "select_victim":
            return cache.select_victim()
        if op[0] == "evict_for":
            out = cache.evict_for(op[1], pinned=op[2]) if not device else \
                cache.evict_for(op[1], None, set(op[2]))
            return [v[0] for v in out] if device else out
    except Exception as e:  # noqa: BLE001 - compared against the other side
        return ("raised",) + _err_kind(e)
    raise AssertionError(op)


def device_cache_rows(cache):
    es = cache.entries()
    return [(e.id, int(e.version_latest), e.mark, e.frequency, e.last_access)
            for _, e in sorted(es.items())]
