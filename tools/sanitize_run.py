"""A small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of the path on reduced shapes --
C2-shaped iterations (K1 build, K3 sort, K6 exact solver, K4 greedy, K7 step
with the one-CTA victim selection), a cache above the one-CTA size (the
cooperative victim selection), a hashed-id engine (the device id table), the
dense K5 solver, hit-greedy and the standalone WorkerCache.  Run as
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("EDX_GRAPH", "0")


def run(edx, n, m, L, cap, V, alpha, iters, id_space, s=1.05, spread=False):
    R = n * m
    bw = [5e9] * (n // 2) + [5e8] * (n - n // 2)
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=bw, cache_capacity=cap, alpha=alpha)
    eng = edx.SimState(cfg, id_space=id_space, max_batch_ids=R * L)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    for ids in edx.ZipfStream(V, L, s, iters, 7, R):
        if spread:
            ids = ((ids.astype(np.uint64) * np.uint64(0x9E3779B1) + np.uint64(0x7F4A7C15))
                   & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        eng.iterate(ids, offs)
    eng.load((ids, offs))
    eng.dispatch_hitgreedy()
    eng.validate_consistency()
    return eng


def main():
    import paper_2512_21615_b200 as edx
    run(edx, 8, 32, 26, 600, 20_000, 0.5, 6, 20_000)                 # small caches, evicting
    run(edx, 3, 64, 100, 13_000, 500_000, 0.25, 4, 500_000, s=0.6)   # cooperative selection
    run(edx, 8, 32, 26, 600, 20_000, 0.25, 5, 0, spread=True)        # hashed ids
    rng = np.random.default_rng(3)
    edx.hungarian(rng.random((96, 96)))                               # K5 dense
    edx.hungarian(rng.random((1500, 1500)))                           # K5, two columns per thread
    c = edx.WorkerCache(16)
    for t in range(40):
        if c.full():
            c.evict_for(1)
        c.touch(int(rng.integers(0, 30)), True, t)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
