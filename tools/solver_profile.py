"""Exact-solver (K6) breakdown on a real EcoMix block: the `config`'s cost
matrix after `prefill` iterations (bench.py's stream), solved a few times with
per-phase cycle counters of k_hungarian_blocks_mw (edx_solver_stats):
steps, runs, cycles in the Dijkstra runs, in the row ends (potentials +
augment + re-sort checks).  Prints one JSON line per repetition."""
import argparse
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("EDX_SOLVER_TIMING", "1")  # the solver's per-phase cycle counters
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--prefill", type=int, default=3)
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
    block = edx.rows_by_gap(mat)[: n * mult]
    for r in range(args.reps):
        t0 = time.perf_counter()
        edx.hungarian_blocks(mat, block, mult)
        dt = time.perf_counter() - t0
        st = list(edx.solver_stats().values())
        steps, c_step, c_end, sorts, c_pot, runs, c_ref, total = st
        k = n * mult
        print(json.dumps({"config": args.config, "k": k, "ms": dt * 1e3, "steps": steps,
                          "runs": runs, "ns_per_step": dt * 1e9 / max(steps, 1),
                          "cyc_per_step_in_runs": c_step / max(steps, 1),
                          "cyc_per_run": c_step / max(runs, 1), "cyc_row_end": c_end / k,
                          "cyc_potentials": c_pot / k, "cyc_resort": c_ref / k,
                          "steps_per_row": steps / k, "runs_per_row": runs / k,
                          "total_cycles": total, "resorts": sorts,
                          "solver": os.environ.get("EDX_MW_BPW", "default")}))


if __name__ == "__main__":
    main()
