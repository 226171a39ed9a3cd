"""One steady-state dispatch iteration inside an NVTX range "edx.iter", for
ncu launch lists of exactly that iteration:
  EDX_GRAPH=0 ncu --nvtx --nvtx-include "edx.iter/" --metrics gpu__time_duration.sum \\
      --csv --log-file out.csv python tools/one_iteration.py --config C5
The engine runs `prefill` eager iterations of bench.py's stream first."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--prefill", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None, help="C5 sweep point (bench.py --batch)")
    ap.add_argument("--workers", type=int, default=None, help="C5 sweep point (bench.py --workers)")
    args = ap.parse_args()
    import torch
    import paper_2512_21615_b200 as edx
    args.alpha, args.spread_ids = None, False
    w = bench.workload(args)  # the bench's own workload (C5 sweep overrides included)
    n, m, L = w["n"], w["m"], w["L"]
    R = w["R"]
    host = bench.batches(w, w["prefill"] + 2)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=w["bw"], cache_capacity=w["cap"],
                            alpha=w["alpha"])
    eng = edx.SimState(cfg, id_space=w["V"], max_batch_ids=R * L)
    for b in host[:w["prefill"] + 1]:
        eng.iterate(b, offs, want_decision=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("edx.iter")
    eng.iterate(host[-1], offs, want_decision=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
