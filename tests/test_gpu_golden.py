"""GPU: the CUDA path reproduces the fixtures generated from the compiled
reference (no reference sources needed on the GPU box)."""
import numpy as np
import pytest

from golden_check import check_trajectory, digest, ecomix_case_inputs, load
from helpers import CONFIGS, random_int_matrix

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("idx", range(5))
def test_engine_trajectories(gpu, idx):
    edx = gpu
    t = load("engine_trajectories.json")[idx]
    p = CONFIGS[t["config"]]
    R = p["n"] * p["m"]
    cfg = edx.ClusterConfig(n=p["n"], m=p["m"], bandwidths_bps=p["bw"], cache_capacity=p["cap"],
                            alpha=t["alpha"])
    eng = edx.SimState(cfg, id_space=p["V"], max_batch_ids=R * p["L"])

    def source(V, L, s, iters, seed, R_):
        z = edx.ZipfStream(V, L, s, iters, seed, R_)
        return iter(z)

    def it(ids, offs):
        eng.load((ids, offs))
        mat = np.empty((R, p["n"]))
        eng.build(mat)
        dec, exp = eng.dispatch()
        return mat, dec, exp, eng.step().as_dict()

    check_trajectory(t, source, it, eng.canonical_state)


def test_matrix_cases(gpu):
    edx = gpu
    g = load("matrix_cases.json")
    for c in g["ecomix"]:
        mat = ecomix_case_inputs(c)
        cfg = edx.ClusterConfig(n=c["n"], m=c["m"], bandwidths_bps=[5e9] * c["n"], alpha=c["alpha"])
        assert digest(edx.rows_by_gap(mat).astype(np.uint64)) == c["order"]
        dec = edx.ecomix(mat, cfg).worker_of_sample
        assert dec.tolist() == c["decision"]
        assert edx.decision_cost(mat, dec).hex() == c["expected"]
    for h in g["hungarian"]:
        r = edx.hungarian(random_int_matrix(h["k"], h["k"], h["seed"], h["maxv"]))
        assert r.col_of_row.tolist() == h["col_of_row"] and r.total_cost.hex() == h["total"]
