"""K1 work statistics at steady state: per id occurrence of the next batch,
whether every worker holds the latest copy (no cell adds), the owner count p
(the push-list length) and the active cells (workers lacking the latest copy).
Prints one JSON line per config: the reference's fp64 adds and the adds a
lockstep row-per-warp kernel issues with pushes padded to blocks of 1, 2, 8."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def popcount64(x):
    x = x.astype(np.uint64)
    c = np.zeros(x.shape, np.int64)
    for b in range(64):
        c += ((x >> np.uint64(b)) & np.uint64(1)).astype(np.int64)
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    args = ap.parse_args()
    import paper_2512_21615_b200 as edx
    w = dict(bench.WORKLOADS[args.config])
    n, m, L = w["n"], w["m"], w["L"]
    w["R"] = R = n * m
    host = bench.batches(w, w["prefill"] + 2)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=w["bw"], cache_capacity=w["cap"],
                            alpha=w["alpha"])
    eng = edx.SimState(cfg, id_space=w["V"], max_batch_ids=R * L)
    for b in host[:w["prefill"] + 1]:
        eng.iterate(b, offs, want_decision=False)
    gids, ow, la, _ = eng.global_masks()
    V = w["V"]
    OW = np.zeros(V, np.uint64)
    LA = np.zeros(V, np.uint64)
    OW[gids] = ow
    LA[gids] = la
    ids = host[-1].astype(np.int64)
    o, l = OW[ids], LA[ids]
    full = np.uint64((1 << n) - 1) if n < 64 else np.uint64(~0 & ((1 << 64) - 1))
    skip = (l & full) == full
    p = popcount64(o)
    act = n - popcount64(l & full)
    alg = int((act * (1 + p)).sum())
    lanes = 32 * ((n + 31) // 32)  # lanes per row (cells padded to the warp)
    res = {"config": args.config, "n": n, "occurrences": int(ids.size),
           "skip_frac": float(skip.mean()), "noowner_frac": float(((p == 0) & ~skip).mean()),
           "alg_adds": alg, "mean_active_of_kept": float(act[~skip].mean()),
           "p_hist_kept": np.bincount(p[~skip], minlength=n + 1).tolist()}
    kept = ~skip
    for blk in (1, 2, 8):
        pushes = ((p[kept] + blk - 1) // blk) * blk
        res[f"lockstep_adds_blk{blk}"] = int((lanes * (1 + pushes)).sum())
    res["lockstep_adds_noskip_blk2"] = int((lanes * (1 + ((p + 1) // 2) * 2)).sum())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
