"""Replay of the committed reference fixtures (tests/golden/) against any
implementation exposing build / ecomix / decision_cost / step / state."""
import hashlib
import json
import os

import numpy as np

from helpers import CONFIGS, offsets_for, random_int_matrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return json.load(open(os.path.join(GOLDEN, name)))


def encode_report(rep):
    return {k: (v.hex() if isinstance(v, float) else [x.hex() for x in v] if k == "cost_w" else v)
            for k, v in rep.items()}


def check_trajectory(t, ids_source, run_iteration, final_state):
    """run_iteration(ids, offs) -> (matrix, decision, expected, report dict)."""
    p = CONFIGS[t["config"]]
    R, L = p["n"] * p["m"], p["L"]
    offs = offsets_for(R, L)
    for it, (ids, want) in enumerate(zip(ids_source(p["V"], L, 1.05, t["iterations"], t["seed"], R),
                                         t["steps"])):
        assert digest(ids) == want["ids"], f"iter {it}: input stream"
        mat, dec, exp, rep = run_iteration(ids, offs)
        assert digest(mat) == want["matrix"], f"iter {it}: matrix"
        assert digest(np.asarray(dec, np.int32)) == want["decision"], f"iter {it}: decision"
        assert exp.hex() == want["expected_cost_s"], f"iter {it}: expected cost"
        assert encode_report(rep) == want["report"], f"iter {it}: report"
    glob, caches = final_state()
    fs = t["final_state"]
    assert int(glob.shape[0]) == fs["global_count"]
    assert digest(glob.astype(np.uint64)) == fs["global"]
    for (e, c, a), w in zip(caches, fs["caches"]):
        assert digest(e.astype(np.uint64)) == w["entries"] and c == w["current_mark"] and a == w["at_current"]


def ecomix_case_inputs(case):
    mat = random_int_matrix(case["n"] * case["m"], case["n"], case["seed"], case["maxv"]) * 3.2768e-6
    return mat
