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


# ---- the exchange plan (halo + local essential tree) of a real tree, brute-forced

def _morton(ix, iy, iz):
    k = np.zeros(ix.shape, np.uint64)
    for b in range(21):
        for d, v in enumerate((ix, iy, iz)):
            k |= ((v.astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + d)
    return k


def _demorton(k):
    out = [np.zeros(k.shape, np.int64) for _ in range(3)]
    for b in range(21):
        for d in range(3):
            out[d] |= ((k >> np.uint64(3 * b + d)) & np.uint64(1)).astype(np.int64) << b
    return out


def real_skeleton(leaf_points=24):
    """A real leaf skeleton: 2 x 2 x 1 copies of a coarse synthetic lysozyme, panel centroids and
    atoms keyed in the bounding cube (test-side, independent of the library's tree code)."""
    from synth import configs
    cfg = configs.array((2, 2, 1), base=configs.lysozyme(16, 60), spacing=60.0)
    v, t = cfg["vertices"], cfg["triangles"]
    cen = v[t].mean(1)
    pts = np.concatenate([cen, cfg["charge_xyz"]])
    lo, hi = pts.min(0), pts.max(0)
    W = (hi - lo).max() * (1 + 1e-6)
    x0 = 0.5 * (lo + hi) - 0.5 * W
    L = 0
    while True:  # depth rule of the library (A10): mean panels per occupied leaf <= leaf_points
        ijk = np.floor((cen - x0) / (W / 2 ** L)).astype(np.int64).clip(0, 2 ** L - 1)
        if len(cen) / len(np.unique(_morton(*ijk.T))) <= leaf_points:
            break
        L += 1
    h = W / 2 ** L
    kp = _morton(*np.floor((cen - x0) / h).astype(np.int64).clip(0, 2 ** L - 1).T)
    kc = _morton(*np.floor((cfg["charge_xyz"] - x0) / h).astype(np.int64).clip(0, 2 ** L - 1).T)
    keys = np.unique(np.concatenate([kp, kc]))
    npan = np.searchsorted(np.sort(kp), keys, "right") - np.searchsorted(np.sort(kp), keys, "left")
    nchg = np.searchsorted(np.sort(kc), keys, "right") - np.searchsorted(np.sort(kc), keys, "left")
    return keys, npan.astype(np.int32), nchg.astype(np.int32), L


def library_plan(keys, npan, nchg, L, world, rank):
    import ctypes as C
    from paper_1007_4591_b200 import _lib
    lib = _lib.load()
    k = np.ascontiguousarray(keys, np.uint64)
    h = C.c_void_p()
    assert lib.fmmbem_plan_create(k.ctypes.data_as(C.POINTER(C.c_uint64)), npan.ctypes.data_as(C.POINTER(C.c_int32)),
                                  nchg.ctypes.data_as(C.POINTER(C.c_int32)), len(k), L, 1, world, rank,
                                  C.byref(h)) == 0

    def lst(kind, peer=0):
        n = lib.fmmbem_plan_list(h, kind, peer, None)
        out = np.empty(max(n, 1), np.int64)
        lib.fmmbem_plan_list(h, kind, peer, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out[:n].tolist()

    res = {"bounds": lst(5), "cell_keys": lst(6), "lvl_off": lst(7), "shared": lst(4), "shared_chg": lst(12),
           "windows": lst(13), "extra": lst(14)}
    for kind, name in ((0, "halo_send"), (1, "halo_recv"), (2, "let_send"), (3, "let_recv"), (10, "let_send_chg"),
                       (11, "let_recv_chg")):
        res[name] = [lst(kind, p) for p in range(world)]
    lib.fmmbem_plan_destroy(h)
    return res


def _plan_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    keys, npan, nchg, L = real_skeleton()
    mine = library_plan(keys, npan, nchg, L, world, rank)
    out = [None] * world
    dist.all_gather_object(out, mine)
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def brute_force_check(plans, keys, npan, nchg, L):
    R = len(plans)
    nl = len(keys)
    b = plans[0]["bounds"]
    assert all(p["bounds"] == b for p in plans) and b[0] == 0 and b[-1] == nl and all(np.diff(b) >= 0)
    lrank = np.repeat(np.arange(R), np.diff(b))
    ijk = np.stack(_demorton(np.asarray(keys, np.uint64)), 1)
    adj = np.abs(ijk[:, None, :] - ijk[None, :, :]).max(2) <= 1  # leaf neighbours, brute force
    # near-field halo: consistency, completeness, minimality
    for r in range(R):
        for p in range(R):
            assert plans[r]["halo_recv"][p] == plans[p]["halo_send"][r]
        halo = set(k for p in range(R) for k in plans[r]["halo_recv"][p])
        own = set(np.nonzero(lrank == r)[0].tolist())
        need = set(np.nonzero(adj[lrank == r].any(0))[0].tolist()) - own
        assert halo == need, (r, sorted(halo ^ need)[:10])
    # local essential tree: every source cell in the interaction list of a cell holding targets of
    # rank r is complete on r (pure and owned by r, received from its owner, or shared)
    lvl_keys = {l: np.unique(np.asarray(keys, np.uint64) >> np.uint64(3 * (L - l))) for l in range(L + 1)}
    off = plans[0]["lvl_off"]
    ck = np.asarray(plans[0]["cell_keys"], np.uint64)
    assert all(np.array_equal(ck[off[l]:off[l + 1]], lvl_keys[l]) for l in range(L + 1))

    def leaves_below(l, k):
        sh = np.uint64(3 * (L - l))
        return np.nonzero((np.asarray(keys, np.uint64) >> sh) == k)[0]

    tgt = npan + nchg
    for r in range(R):
        got = set(plans[r]["shared"])      # panel multipoles complete on r besides its pure cells
        got_c = set(plans[r]["shared_chg"])  # charge multipoles (the charge-FMM's sources)
        for p in range(R):
            if p != r:
                assert plans[r]["let_recv"][p] == plans[p]["let_send"][r]
                assert plans[r]["let_recv_chg"][p] == plans[p]["let_send_chg"][r]
                got |= set(plans[r]["let_recv"][p])
                got_c |= set(plans[r]["let_recv_chg"][p])
        # expansion slots: the window of level l = exactly the cells holding a leaf of r (brute force)
        win = plans[r]["windows"]
        assert len(win) == 2 * (L + 1)
        in_win = set()
        for l in range(L + 1):
            mine = [off[l] + j for j, k in enumerate(lvl_keys[l]) if (lrank[leaves_below(l, k)] == r).any()]
            assert list(range(win[2 * l], win[2 * l + 1])) == mine, (r, l)
            in_win |= set(mine)
        extra = plans[r]["extra"]
        assert extra == sorted(extra) and not (set(extra) & in_win)
        assert set(extra) == (got | got_c) - in_win
        slots = in_win | set(extra)
        for l in range(2, L + 1):
            cells = lvl_keys[l]
            cx = np.stack(_demorton(cells), 1)
            par = cx >> 1
            for i, t in enumerate(cells):
                lt = leaves_below(l, t)
                has_t = (tgt[lt][lrank[lt] == r] > 0).any()
                has_p = (npan[lt][lrank[lt] == r] > 0).any()
                if not has_t:
                    continue  # no targets of rank r below t
                near_par = np.abs(par - par[i]).max(1) <= 1
                far = np.abs(cx - cx[i]).max(1) > 1
                for j in np.nonzero(near_par & far)[0]:  # interaction list, brute force
                    ls = leaves_below(l, cells[j])
                    gidx = off[l] + j
                    owners = set(lrank[ls].tolist())
                    if npan[ls].sum() > 0 or (has_p and nchg[ls].sum() > 0):
                        assert gidx in slots, (r, l, int(t), int(cells[j]))  # its M2L reads a slot
                    if owners == {r}:
                        continue  # pure, computed locally
                    if npan[ls].sum() > 0:
                        assert gidx in got, (r, l, int(t), int(cells[j]))
                    if has_p and nchg[ls].sum() > 0:  # charge sources serve the panels (E_n, psi)
                        assert gidx in got_c, (r, l, int(t), int(cells[j]))
    # shared = exactly the cells with sources (panels / charges) straddling ranks
    for l in range(2, L + 1):
        for j, k in enumerate(lvl_keys[l]):
            ls = leaves_below(l, k)
            straddle = len(set(lrank[ls].tolist())) > 1
            assert ((off[l] + j) in set(plans[0]["shared"])) == (straddle and npan[ls].sum() > 0)
            assert ((off[l] + j) in set(plans[0]["shared_chg"])) == (straddle and nchg[ls].sum() > 0)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_exchange_plan_brute_force_over_gloo(world):
    """fmmbem_plan (the host code fmmbem_create runs on every rank) on a real tree, one process per
    rank over gloo: halo and LET lists agree pairwise and equal the brute-force needs."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world + (os.getpid() % 500)
    ps = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    plans = q.get(timeout=300)
    for p in ps:
        p.join(60)
    keys, npan, nchg, L = real_skeleton()
    assert L >= 3 and len(keys) > 50
    brute_force_check(plans, keys, npan, nchg, L)


def test_tree_lists_dual_accounting():
    """SPEC S:164 / S:173 dual accounting, brute force on the library's host lists (plan.cu, the same
    definitions as tree.cu's kernels): for every leaf t, its neighbour leaves plus the leaves below
    every cell in the interaction lists of t and of each of its ancestors cover ALL leaves exactly
    once -- every source is counted once, by P2P or by exactly one M2L."""
    import ctypes as C
    from paper_1007_4591_b200 import _lib
    keys, npan, nchg, L = real_skeleton()
    lib = _lib.load()
    k = np.ascontiguousarray(keys, np.uint64)
    h = C.c_void_p()
    assert lib.fmmbem_plan_create(k.ctypes.data_as(C.POINTER(C.c_uint64)), npan.ctypes.data_as(C.POINTER(C.c_int32)),
                                  nchg.ctypes.data_as(C.POINTER(C.c_int32)), len(k), L, 1, 1, 0, C.byref(h)) == 0

    def lst(kind, peer):
        n = lib.fmmbem_plan_list(h, kind, peer, None)
        out = np.empty(max(n, 1), np.int64)
        lib.fmmbem_plan_list(h, kind, peer, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out[:n]

    off = lst(7, 0)
    ck = lst(6, 0).astype(np.uint64)
    nl = len(keys)
    leaf_keys = np.asarray(keys, np.uint64)
    ijk = np.stack(_demorton(leaf_keys), 1)
    for t in range(nl):
        count = np.zeros(nl, np.int64)
        nb = lst(8, t)
        # neighbours: exactly the leaves with max |d ijk| <= 1 (brute force), incl. t itself
        want = np.nonzero(np.abs(ijk - ijk[t]).max(1) <= 1)[0]
        assert sorted(nb.tolist()) == want.tolist()
        count[nb] += 1
        for l in range(2, L + 1):  # ancestor of t at level l and its interaction list
            a = int(np.searchsorted(ck[off[l]:off[l + 1]], leaf_keys[t] >> np.uint64(3 * (L - l)))) + off[l]
            for s in lst(9, a):
                ls_ = int(np.searchsorted(np.asarray(off), s, "right")) - 1
                below = (leaf_keys >> np.uint64(3 * (L - ls_))) == ck[s]
                count[below] += 1
        assert count.min() == 1 and count.max() == 1, (t, np.nonzero(count != 1)[0][:10])
    lib.fmmbem_plan_destroy(h)
