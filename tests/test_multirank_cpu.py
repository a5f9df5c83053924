"""CPU (gloo, world_size 2): the host side of the multi-rank path.

bench.py's N>1 launch broadcasts the NCCL unique id from rank 0 with
torch.distributed and every rank derives the same contiguous shard of sink
groups; the device exchange then scatters each rank's fixed-size window back.
Here the same shard/window arithmetic (restated from Simulation::step and
ShardExchange / unpack_kernel, csrc/engine.cu + csrc/capi.cu) runs in two gloo
processes, exchanges real per-group payloads with all_gather, and checks the
reassembled result covers every group exactly once."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def shard(ng, rank, world):  # Simulation::step: contiguous equal shard of the groups
    return ng * rank // world, ng * (rank + 1) // world


def window(n, gs, world):  # ShardExchange::window
    ng_max = (n + gs - 1) // gs
    return ((ng_max + world - 1) // world) * gs


def _worker(rank, world, port, n, na, gs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        assert uid[0] == bytes(range(128))
        ng = (na + gs - 1) // gs
        lo, hi = shard(ng, rank, world)
        per = window(n, gs, world)
        accum = np.zeros((2 * n + 64 * gs, 4), np.float32)  # prepare(): 2n + 64 gs slots
        for s in range(lo * gs, min(hi * gs, na)):  # this rank's walk writes its own slots
            accum[s] = (s, rank, 1.0, 0.0)
        send = torch.from_numpy(accum[lo * gs: lo * gs + per].copy())
        out = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(out, send)
        gathered = torch.cat(out).numpy()
        result = np.zeros((na, 4), np.float32)
        for r in range(world):  # unpack_kernel
            rlo, rhi = shard(ng, r, world)
            a, b = rlo * gs, min(rhi * gs, na)
            result[a:b] = gathered[r * per: r * per + (b - a)]
        q.put((rank, result))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,na,gs", [(1000, 1000, 32), (1000, 777, 32), (4096, 33, 7), (100, 100, 1)])
def test_two_rank_shards_cover_all_groups(n, na, gs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (n + na + gs) % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, n, na, gs, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        out = res[r]
        assert np.array_equal(out[:, 0], np.arange(na, dtype=np.float32))  # every slot exactly once
        assert np.all(out[:, 2] == 1.0)
        ng = (na + gs - 1) // gs
        owners = np.repeat([0, 1], [min(shard(ng, 0, 2)[1] * gs, na), na - min(shard(ng, 0, 2)[1] * gs, na)])
        assert np.array_equal(out[:, 1], owners.astype(np.float32))
