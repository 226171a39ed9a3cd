"""The multi-GPU path's exchange bookkeeping on CPU (gloo): the product's own
row split (edx_shard_rows), row gather (edx_exchange_gather_rows) and
decision broadcast (edx_exchange_broadcast_decision) -- the code the engine
runs over NCCL (engine.cu engine_build / engine_dispatch) -- driven through a
gloo-backed edx_transport.  Every rank holds only its own shard of the cost
matrix (rows are independent, cost.hpp:102-104; the matrix values come from
the oracle); after the gather rank 0 must hold the full matrix bit for bit,
and every rank must receive rank 0's decision."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import CONFIGS, offsets_for


def _gloo_transport(edx):
    def send(buf, peer):
        dist.send(torch.from_numpy(buf), dst=peer)

    def recv(buf, peer):
        dist.recv(torch.from_numpy(buf), src=peer)

    def bcast(buf, root):
        dist.broadcast(torch.from_numpy(buf), src=root)

    return edx.HostTransport(send, recv, bcast)


def _worker(rank, world, port, result, rows_override):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import pyoracle
    import paper_2512_21615_b200 as edx
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = _gloo_transport(edx)
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
        if rows_override is not None:  # fewer rows than ranks: empty shards
            full = np.ascontiguousarray(full[:rows_override])
        lo, hi = edx.shard_rows(full.shape[0], world)[rank]
        mine = np.zeros_like(full)  # this rank built its shard only
        mine[lo:hi] = full[lo:hi]
        edx.exchange_gather_rows(tr, mine, world, rank, root=0)
        if rank == 0:
            ok &= mine.tobytes() == full.tobytes()
        else:  # non-roots keep their own rows and receive nothing
            ok &= mine[lo:hi].tobytes() == full[lo:hi].tobytes()
            ok &= not np.any(np.delete(mine, np.s_[lo:hi], axis=0))
        if rows_override is not None:
            continue
        dec = orc.ecomix(cfg, mine).astype(np.int32) if rank == 0 else np.full(R, -7, np.int32)
        edx.exchange_broadcast_decision(tr, dec, root=0)
        ok &= bool((dec == orc.ecomix(cfg, full)).all())
        sim.step(ids, offs, dec)
    result[rank] = int(ok)
    dist.destroy_process_group()


def test_shard_rows_partition(edx):
    for R in (0, 1, 7, 1024, 16384):
        for world in (1, 2, 3, 4, 8):
            sh = edx.shard_rows(R, world)
            assert len(sh) == world and sh[0][0] == 0 and sh[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert max(b - a for a, b in sh) - min(b - a for a, b in sh) <= 1


def test_exchange_rejects_bad_groups(edx):
    tr = edx.HostTransport(lambda b, p: None, lambda b, p: None, lambda b, r: None)
    mat = np.zeros((4, 3))
    with pytest.raises(edx.InvalidArgument):
        edx.exchange_gather_rows(tr, mat, world=2, rank=2)
    with pytest.raises(edx.InvalidArgument):
        edx.exchange_gather_rows(tr, mat, world=2, rank=0, root=5)


def test_exchange_reports_transport_failure(edx):
    def boom(buf, peer):
        raise RuntimeError("link down")
    tr = edx.HostTransport(boom, boom, boom)
    with pytest.raises(edx.EdxError, match="transport"):
        edx.exchange_gather_rows(tr, np.zeros((4, 3)), world=2, rank=1)


@pytest.mark.parametrize("world,port,rows", [(2, 29533, None), (3, 29541, None), (4, 29549, 3)])
def test_gloo_shard_gather_broadcast(pyoracle, world, port, rows):
    result = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, result, rows), nprocs=world, join=True)
    assert dict(result) == {r: 1 for r in range(world)}
