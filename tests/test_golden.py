"""CPU: the plain-C oracle reproduces the fixtures generated from the compiled
reference (pins the oracle where /root/reference is absent)."""
import numpy as np
import pytest

from golden_check import check_trajectory, digest, ecomix_case_inputs, load
from helpers import CONFIGS, random_int_matrix


@pytest.mark.parametrize("idx", range(5))
def test_port_oracle_engine_trajectories(port, pyoracle, idx):
    t = load("engine_trajectories.json")[idx]
    p = CONFIGS[t["config"]]
    cfg = pyoracle.Cfg(p["n"], p["m"], p["bw"], cap=p["cap"], alpha=t["alpha"])
    sim = port.sim(cfg)

    def it(ids, offs):
        mat = sim.build_matrix(ids, offs)
        dec = port.ecomix(cfg, mat)
        return mat, dec, port.decision_cost(mat, dec), sim.step(ids, offs, dec)

    check_trajectory(t, port.zipf_batches, it, sim.canonical_state)


def test_port_oracle_matrix_cases(port, pyoracle):
    g = load("matrix_cases.json")
    for c in g["ecomix"]:
        mat = ecomix_case_inputs(c)
        cfg = pyoracle.Cfg(c["n"], c["m"], [5e9] * c["n"], alpha=c["alpha"])
        assert digest(port.rows_by_gap(mat).astype(np.uint64)) == c["order"]
        dec = port.ecomix(cfg, mat)
        assert dec.tolist() == c["decision"]
        assert port.decision_cost(mat, dec).hex() == c["expected"]
    for h in g["hungarian"]:
        cols, total = port.hungarian(random_int_matrix(h["k"], h["k"], h["seed"], h["maxv"]))
        assert cols.tolist() == h["col_of_row"] and total.hex() == h["total"]
    for b in g["bench_matrix"]:
        cols, total = port.hungarian(port.bench_matrix(b["k"]))
        assert cols.tolist() == b["col_of_row"] and total.hex() == b["total"]
