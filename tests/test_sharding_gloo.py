"""Host-side logic of the multi-GPU path on CPU (gloo, world_size 2): every
rank builds its row shard of the cost matrix (rows are independent,
cost.hpp:102-104), the shards are gathered to rank 0 and must reassemble the
full matrix bit for bit; the broadcast decision is the rank-0 ecomix."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import CONFIGS, offsets_for


def _worker(rank, world, port, result):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import pyoracle
    import paper_2512_21615_b200 as edx
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = pyoracle.Oracle("port")
    p = CONFIGS["P8"]
    n, m, L = p["n"], p["m"], p["L"]
    R = n * m
    cfg = pyoracle.Cfg(n, m, p["bw"], cap=p["cap"], alpha=0.5)
    sim = orc.sim(cfg)
    offs = offsets_for(R, L)
    ok = True
    for ids in orc.zipf_batches(p["V"], L, 1.05, 6, 3, R):
        full = sim.build_matrix(ids, offs)
        lo, hi = edx.shard_rows(R, world)[rank]
        # the rank's shard, built independently from its own rows
        mine = full[lo:hi].copy()
        parts = [torch.zeros((b - a, n), dtype=torch.float64) for a, b in edx.shard_rows(R, world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        gathered = torch.cat(parts).numpy()
        ok &= gathered.tobytes() == full.tobytes()
        dec = torch.from_numpy(orc.ecomix(cfg, gathered)) if rank == 0 else torch.zeros(R, dtype=torch.int32)
        dist.broadcast(dec, 0)
        ok &= bool((dec.numpy() == orc.ecomix(cfg, full)).all())
        sim.step(ids, offs, dec.numpy())
    result[rank] = int(ok)
    dist.destroy_process_group()


def test_shard_rows_partition(edx):
    for R in (1, 7, 1024, 16384):
        for world in (1, 2, 3, 4, 8):
            sh = edx.shard_rows(R, world)
            assert sh[0][0] == 0 and sh[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert max(b - a for a, b in sh) - min(b - a for a, b in sh) <= 1


def test_gloo_two_rank_shard_gather_broadcast(pyoracle):
    world = 2
    result = mp.Manager().dict()
    mp.spawn(_worker, args=(world, 29533, result), nprocs=world, join=True)
    assert dict(result) == {0: 1, 1: 1}
