"""Host-side logic of the multi-GPU path (no GPU): the cost-weighted contiguous split of the
domain decomposition and the rank bootstrap over a world_size-2 gloo group."""
import os

import numpy as np
import pytest


def test_split_costs_properties():
    from paper_1007_4591_b200 import split_costs
    rng = np.random.default_rng(0)
    for n, parts in ((1000, 8), (17, 4), (5, 8), (1, 1), (0, 3)):
        c = rng.random(n) ** 4 * 100
        b = split_costs(c, parts)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        if n >= 100:
            pre = np.concatenate([[0], np.cumsum(c)])
            share = np.diff(pre[b])
            assert share.max() - share.min() <= 2 * c.max() + 1e-9  # balanced to one item
    # uniform costs split evenly
    assert list(split_costs(np.ones(16), 4)) == [0, 4, 8, 12, 16]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1007_4591_b200 import split_costs
    obj = [os.urandom(128) if rank == 0 else None]   # stands in for fmmbem_get_unique_id on rank 0
    dist.broadcast_object_list(obj, src=0)
    costs = np.random.default_rng(5).random(1000)    # every rank derives the same costs
    b = split_costs(costs, world)
    out = [None] * world
    dist.all_gather_object(out, (obj[0], b.tolist()))
    q.put((rank, out))
    dist.destroy_process_group()


def test_gloo_two_ranks_agree_on_id_and_partition():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
    for _, out in res:
        ids = {o[0] for o in out}
        bounds = {tuple(o[1]) for o in out}
        assert len(ids) == 1 and len(bounds) == 1
        (b,) = bounds
        assert b[0] == 0 and b[-1] == 1000
