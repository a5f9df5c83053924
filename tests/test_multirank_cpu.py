"""CPU (gloo, world_size 2): the host side of the multi-rank path, through the product library.

bench.py's N>1 launch broadcasts the NCCL unique id from rank 0 with
torch.distributed and every rank derives the same contiguous shard of sink
groups; the device exchange then scatters each rank's fixed-size window back,
and the whole-system groups' slices are dealt to the ranks.  Here the library's
own host arithmetic (g2_mesh_shard / g2_mesh_window / g2_slice_owner, the code
Simulation::step, ShardExchange, unpack_kernel and walk_init_kernel run) drives
two gloo processes that exchange real per-group payloads with all_gather; the
reassembled result must cover every group and every slice exactly once."""
import ctypes as C
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _lib():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1811_02761_b200.gravitree import lib
    L = lib()
    L.g2_mesh_window.restype = C.c_size_t
    L.g2_slice_owner.restype = C.c_uint
    return L


def shard(ng, rank, world):  # Simulation::step's contiguous equal shard (g2_mesh_shard)
    lo, hi = C.c_uint(), C.c_uint()
    _lib().g2_mesh_shard(C.c_uint(ng), C.c_int(rank), C.c_int(world), C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def window(n, gs, world):  # ShardExchange::window (g2_mesh_window)
    return _lib().g2_mesh_window(C.c_size_t(n), C.c_size_t(gs), C.c_int(world))


def slice_owner(w, j, nh, world):  # walk_init_kernel's deal (g2_slice_owner)
    a = np.ascontiguousarray(w, dtype=np.float32)
    return _lib().g2_slice_owner(a.ctypes.data_as(C.c_void_p), C.c_uint(len(a)), C.c_uint(j), C.c_uint(nh),
                                 C.c_int(world))


def test_mesh_arithmetic_matches_its_definition():
    for ng in (0, 1, 7, 1000, 262144):
        for world in (1, 2, 3, 8):
            bounds = [shard(ng, r, world) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == ng
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
            assert all(b - a in (ng // world, ng // world + 1) for a, b in bounds)
    assert window(1000, 32, 2) == 512 and window(100, 1, 3) == 34


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slice_deal_covers_and_balances(world):
    rng = np.random.default_rng(world)
    for nk in (2, 5, 8):
        w = rng.uniform(0.1, 1.0, nk)
        nh = 58
        owners = np.array([slice_owner(w, j, nh, world) for j in range(nh * nk)])
        assert owners.min() >= 0 and owners.max() < world
        load = np.bincount(owners, weights=np.tile(w, nh), minlength=world)
        assert load.max() - load.min() <= w.max() + 1e-9  # within one slice of the lightest rank


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
        # the whole-system groups' slices: each rank publishes the ones it owns, the union is every slice once
        w, nh = np.array([0.3, 0.9, 0.1, 0.5, 0.7, 0.2, 0.6, 0.4]), 13
        mine = [j for j in range(nh * len(w)) if slice_owner(w, j, nh, world) == rank]
        got = [None] * world
        dist.all_gather_object(got, mine)
        slices = sorted(j for part in got for j in part)
        q.put((rank, result, slices == list(range(nh * len(w)))))
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
    res = {}
    for _ in ps:
        r, out, ok = q.get(timeout=120)
        res[r] = out
        assert ok  # every slice dealt to exactly one rank
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        out = res[r]
        assert np.array_equal(out[:, 0], np.arange(na, dtype=np.float32))  # every slot exactly once
        assert np.all(out[:, 2] == 1.0)
        ng = (na + gs - 1) // gs
        owners = np.repeat([0, 1], [min(shard(ng, 0, 2)[1] * gs, na), na - min(shard(ng, 0, 2)[1] * gs, na)])
        assert np.array_equal(out[:, 1], owners.astype(np.float32))
