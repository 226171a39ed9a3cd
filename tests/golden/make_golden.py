"""Generate tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref).

Run here, where /root/reference exists:  python tests/golden/make_golden.py
The fixtures pin the plain-C oracle (tests/test_golden.py, CPU) and the CUDA
path (tests/test_gpu_golden.py) on hosts without the reference sources.
Large arrays are stored as sha256 digests of their little-endian bytes.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import pyoracle  # noqa: E402
from helpers import CONFIGS, offsets_for, random_int_matrix  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def engine_trajectory(ref, name, alpha, iters, seed):
    p = CONFIGS[name]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    cfg = pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=alpha)
    sim = ref.sim(cfg)
    offs = offsets_for(R, L)
    steps = []
    for ids in ref.zipf_batches(p["V"], L, 1.05, iters, seed, R):
        mat = sim.build_matrix(ids, offs)
        dec = ref.ecomix(cfg, mat)
        exp = ref.decision_cost(mat, dec)
        rep = sim.step(ids, offs, dec)
        steps.append({"ids": digest(ids), "matrix": digest(mat), "decision": digest(dec),
                      "expected_cost_s": exp.hex(), "report": {k: (v.hex() if isinstance(v, float) else
                                                                 [x.hex() for x in v] if k == "cost_w" else v)
                                                             for k, v in rep.items()}})
    glob, caches = sim.canonical_state()
    state = {"global": digest(glob.astype(np.uint64)), "global_count": int(glob.shape[0]),
             "caches": [{"entries": digest(e.astype(np.uint64)), "size": int(e.shape[0]),
                         "current_mark": c, "at_current": a} for e, c, a in caches]}
    return {"config": name, "alpha": alpha, "iterations": iters, "seed": seed, "steps": steps,
            "final_state": state}


def matrix_cases(ref):
    cases = []
    for n, m, alpha, maxv, seed in [(2, 3, 1.0, 100, 1), (4, 8, 0.5, 3, 2), (8, 128, 0.5, 1000, 3),
                                    (8, 128, 1.0, 7, 4), (16, 64, 0.125, 50, 5), (5, 7, 0.3, 2, 6)]:
        mat = random_int_matrix(n * m, n, seed, maxv) * 3.2768e-6
        cfg = pyoracle.Cfg(n, m, [5e9] * n, alpha=alpha)
        dec = ref.ecomix(cfg, mat)
        cases.append({"n": n, "m": m, "alpha": alpha, "maxv": maxv, "seed": seed,
                      "order": digest(ref.rows_by_gap(mat).astype(np.uint64)),
                      "decision": dec.tolist(), "expected": ref.decision_cost(mat, dec).hex()})
    hung = []
    for k, maxv, seed in [(5, 100, 11), (8, 3, 12), (64, 1000, 13), (128, 5, 14)]:
        sq = random_int_matrix(k, k, seed, maxv)
        cols, total = ref.hungarian(sq)
        hung.append({"k": k, "maxv": maxv, "seed": seed, "col_of_row": cols.tolist(),
                     "total": total.hex()})
    bench = []
    for k in (32, 96):
        cols, total = ref.hungarian(ref.bench_matrix(k))
        bench.append({"k": k, "col_of_row": cols.tolist(), "total": total.hex()})
    return {"ecomix": cases, "hungarian": hung, "bench_matrix": bench}


def main():
    ref = pyoracle.Oracle("reference")
    json.dump(matrix_cases(ref), open(os.path.join(OUT, "matrix_cases.json"), "w"), indent=1)
    traj = [engine_trajectory(ref, "P2", 0.5, 50, 1234), engine_trajectory(ref, "P3", 1.0, 40, 7),
            engine_trajectory(ref, "P8", 0.25, 30, 99), engine_trajectory(ref, "C1", 0.0, 8, 42),
            engine_trajectory(ref, "C2", 0.5, 5, 42)]
    json.dump(traj, open(os.path.join(OUT, "engine_trajectories.json"), "w"), indent=1)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
