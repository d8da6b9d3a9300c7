"""Host logic of the row-sharded landscape (C3) and of the N>1 env sharding, on CPU:
shard/halo planning, and the torch.distributed halo exchange over gloo with world_size 2-3."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_06102_b200.sharded import exchange_halos, halo_copies, plan_shards


@pytest.mark.parametrize("h,g,k", [(100, 1, 8), (100, 2, 8), (101, 3, 4), (16384, 8, 8), (20, 5, 3)])
def test_plan_shards_cover_and_halos(h, g, k):
    sh = plan_shards(h, g, k)
    assert sh[0].band[0] == 0 and sh[-1].band[1] == h
    for a, b in zip(sh, sh[1:]):
        assert a.band[1] == b.band[0]
    for s in sh:
        assert s.rows[0] == max(0, s.band[0] - k) and s.rows[1] == min(h, s.band[1] + k)
    # every halo row is refreshed from its owner, and only halo rows are written
    written = {i: set() for i in range(g)}
    for d, drow, s, srow, n in halo_copies(sh):
        for i in range(n):
            grow = sh[d].rows[0] + drow + i
            assert sh[s].band[0] <= grow < sh[s].band[1]
            assert sh[s].rows[0] + srow + i == grow
            assert not (sh[d].band[0] <= grow < sh[d].band[1])
            written[d].add(grow)
    for i, s in enumerate(sh):
        halo_rows = set(range(s.rows[0], s.band[0])) | set(range(s.band[1], s.rows[1]))
        assert written[i] == halo_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, h, w, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shards = plan_shards(h, world, k)
    me = shards[rank]
    # layer: band rows carry their global row id, halo rows start as garbage (255)
    layer = torch.full((me.rows[1] - me.rows[0], w), 255, dtype=torch.uint8)
    for g in range(*me.band):
        layer[g - me.rows[0]] = g % 250
    exchange_halos(dist, rank, shards,
                   get_rows=lambda r0, n: layer[r0:r0 + n].clone(),
                   set_rows=lambda r0, t: layer.__setitem__(slice(r0, r0 + t.shape[0]), t),
                   make_buffer=lambda n: torch.empty((n, w), dtype=torch.uint8))
    want = torch.tensor([(g % 250) for g in range(*me.rows)], dtype=torch.uint8)[:, None].expand(-1, w)
    q.put((rank, bool(torch.equal(layer, want))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 37, 16, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


def _env_worker(rank, world, port, scaling, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    e0, n = bench.rank_envs("C1", rank, world, scaling)
    out = [None] * world
    dist.all_gather_object(out, list(range(e0, e0 + n)))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)   # bench.py's max-over-ranks timing
    q.put((rank, [i for part in out for i in part], float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling,world", [("weak", 2), ("strong", 2), ("strong", 3)])
def test_gloo_env_sharding(scaling, world):
    """bench.py at N>1: weak scaling -- rank r owns global env ids [r*1024, (r+1)*1024); strong --
    the 1024 ids split in contiguous ranges (streams = ids); the union over ranks is disjoint and
    dense, and the time is the max over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_env_worker, args=(r, world, port, scaling, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    total = world * 1024 if scaling == "weak" else 1024
    for rank, ids, tmax in res:
        assert ids == list(range(total)) and tmax == float(world)


def _grad_worker(rank, world, port, n_envs, q):
    from paper_2512_06102_b200.distributed import env_range, reduce_loss_grad
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rs = np.random.default_rng(7)
    loss_all = rs.random(n_envs)
    grad_all = rs.standard_normal((n_envs, 6))
    f, l = env_range(rank, world, n_envs)
    loss, grad = reduce_loss_grad(dist, loss_all[f:l], grad_all[f:l], n_envs)
    q.put((rank, loss, grad.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_envs", [(2, 7), (3, 10), (2, 1)])
def test_c4_gradient_allreduce_gloo(world, n_envs):
    """C4 env sharding: each rank's per-env loss/gradient rows are gathered and summed in global
    env order -- bit-identical to the one-process sum, for any rank count."""
    from paper_2512_06102_b200.distributed import env_range, sum_loss_grad
    rs = np.random.default_rng(7)
    loss_all = rs.random(n_envs)
    grad_all = rs.standard_normal((n_envs, 6))
    want_loss, want_grad = sum_loss_grad(loss_all, grad_all)
    covered = []
    for r in range(world):
        covered += list(range(*env_range(r, world, n_envs)))
    assert covered == list(range(n_envs))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, world, port, n_envs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for _, loss, grad in res:
        assert loss == want_loss and grad == want_grad.tolist()
