"""Dump a steady-state EcoMix solve case (the C2 cost matrix after `prefill`
iterations) and time the product solver on it: used for ncu captures of the
exact solver (k_hungarian_blocks) in isolation."""
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
    ap.add_argument("--config", default="C2")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--prefill", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2512_21615_b200 as edx
    w = dict(bench.WORKLOADS[args.config])
    if args.alpha is not None:
        w["alpha"] = args.alpha
    n, m, L = w["n"], w["m"], w["L"]
    R = n * m
    host = bench.batches(dict(w, R=R), args.prefill + 1)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=w["bw"], cache_capacity=w["cap"],
                            alpha=w["alpha"])
    eng = edx.SimState(cfg, id_space=w["V"], max_batch_ids=R * L)
    for b in host[:args.prefill]:
        eng.iterate(b, offs, want_decision=False)
    eng.load((host[-1], offs))
    mat = np.empty((R, n))
    eng.build(mat)
    mult = edx.exact_multiplicity(m, w["alpha"])
    order = edx.rows_by_gap(mat)
    block = order[: n * mult]
    for r in range(args.reps):
        t0 = time.perf_counter()
        res = edx.hungarian_blocks(mat, block, mult)
        dt = time.perf_counter() - t0
        print(f"rep {r}: hungarian_blocks k={n * mult} {dt * 1e3:.2f} ms total={res.total_cost!r}")
        print("  stats", edx.solver_stats())
    np.save(os.path.join(ROOT, "gpurun_out", f"solver_{args.config}.npy"), mat)


if __name__ == "__main__":
    main()
