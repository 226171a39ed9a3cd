"""Multi-GPU engine parity (needs >= 2 GPUs; skipped otherwise): the row-
sharded build + NCCL gather + rank-0 solve + decision broadcast + replicated
step gives the single-engine results on every rank."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["EDX_ROOT"]); sys.path.insert(0, os.path.join(os.environ["EDX_ROOT"], "tests"))
import paper_2512_21615_b200 as edx
from oracle import pyoracle
from helpers import CONFIGS, canon_equal, offsets_for
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
if rank == 0:
    buf.copy_(torch.frombuffer(bytearray(edx.nccl_unique_id()), dtype=torch.uint8))
dist.broadcast(buf, 0)
nid = bytes(buf.cpu().numpy().tobytes())
p = CONFIGS["P8"]; n, m, L = p["n"], p["m"], p["L"]; R = n * m
cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=p["bw"], cache_capacity=p["cap"], alpha=0.5)
eng = edx.SimState(cfg, id_space=p["V"], max_batch_ids=R * L, device=rank, rank=rank,
                   world_size=world, nccl_id=nid)
orc = pyoracle.Oracle("reference" if os.path.exists(pyoracle.REF_SO) else "port")
sim = orc.sim(pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.5))
offs = offsets_for(R, L)
for it, ids in enumerate(orc.zipf_batches(p["V"], L, 1.05, 25, 99, R)):
    dec, rep = eng.iterate(ids, offs)
    wdec, wexp, wrep, _ = sim.iteration(ids, offs)
    assert (dec == wdec).all(), (rank, it)
    assert rep.as_dict() == wrep, (rank, it)
    assert rep.expected_cost_s == wexp, (rank, it)
msg = canon_equal(eng.canonical_state(), sim.canonical_state())
assert not msg, msg
dist.barrier()
open(os.path.join(os.environ["EDX_MARKS"], f"rank{rank}.ok"), "w").close()
dist.destroy_process_group()
'''


def test_two_gpu_sharded_engine(tmp_path):
    import torch
    world = int(os.environ.get("EDX_TEST_WORLD", "2"))
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, EDX_ROOT=ROOT, EDX_MARKS=str(tmp_path))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29517",
                        str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    # each rank marks its own success (stdout of the two ranks interleaves)
    assert all((tmp_path / f"rank{r}.ok").exists() for r in range(world))
