"""Per-iteration wall time of the fused iterate call over a long run (diagnostic)."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--device-path", action="store_true")
    a = ap.parse_args()
    import paper_2512_21615_b200 as edx
    w = dict(bench.WORKLOADS[a.config])
    n, m, L = w["n"], w["m"], w["L"]
    R = n * m
    w["R"] = R
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=w["bw"], cache_capacity=w["cap"], alpha=w["alpha"])
    eng = edx.SimState(cfg, id_space=w["V"], max_batch_ids=R * L)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    z = edx.ZipfStream(w["V"], L, bench.ZIPF_S, a.iters, bench.SEED, R)
    for it, ids in enumerate(z):
        t0 = time.perf_counter()
        dec, rep = eng.iterate(ids, offs)
        dt = time.perf_counter() - t0
        print(f"iter {it} {dt * 1e3:.2f} ms evict_push {rep.evict_push} miss {rep.miss_pull}", flush=True)


if __name__ == "__main__":
    main()
