"""Multi-rank tile sharding (north_star (3)) on CPU with the gloo backend, world size 2 and 3:
the product's ShardedRenderer driver, the library's LPT owner map and its host untile are
exercised end to end; per-rank tile rendering is supplied by the fp64 oracle (test
infrastructure) since there is no GPU here.  The assembled image must equal the oracle's
single-process image exactly.  The second axis (sub-box sharding: ranges of the partition's
sub-boxes per rank, all-reduce MIN / MAX) is exercised the same way."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShardCtx:
    """Stands in for Context.as_render_shard / as_untile on a CPU-only box."""

    def __init__(self, w, oracle):
        self.w, self.oracle = w, oracle
        self.camera = w.camera
        self.device = None

    def n_tiles(self, tile):
        W, H = self.camera["W"], self.camera["H"]
        return (-(-W // tile)) * (-(-H // tile))

    def as_render_shard(self, tile, batch, rank, world, cap, lo_tm, hi_tm, stats=False):
        import paper_2503_00308_b200 as ap
        nt = self.n_tiles(tile)
        costs = np.array([self.oracle.render_tiles(self.w, [t], tile=tile)[2]["pairs"]
                          for t in range(nt)], np.int64)
        owner = ap.as_lpt_assign(costs, world, cap)
        mine = np.nonzero(owner == rank)[0]
        lo, hi, _ = self.oracle.render_tiles(self.w, mine, tile=tile)
        W, H = self.camera["W"], self.camera["H"]
        ntx = -(-W // tile)
        for k, t in enumerate(mine):
            tx, ty = t % ntx, t // ntx
            for ly in range(tile):
                for lx in range(tile):
                    py, px = ty * tile + ly, tx * tile + lx
                    if py < H and px < W:
                        lo_tm[k, ly * tile + lx] = torch.from_numpy(lo[py, px].astype(np.float32))
                        hi_tm[k, ly * tile + lx] = torch.from_numpy(hi[py, px].astype(np.float32))
        owned = np.full(cap, -1, np.int32)
        owned[:len(mine)] = mine
        return lo_tm, hi_tm, owned, len(mine), None

    def as_untile(self, tile, world, cap, owned, n_owned, g_lo, g_hi):
        import paper_2503_00308_b200 as ap
        return ap.as_untile(self.camera["W"], self.camera["H"], tile, world, cap, owned, n_owned,
                            g_lo, g_hi)


def _worker(rank, world, port, name, kw, tile, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2503_00308_b200.dist import ShardedRenderer
        from workloads import make_config
        w = make_config(name, **kw)
        ctx = OracleShardCtx(w, pyoracle)
        sr = ShardedRenderer(ctx, rank, world, tile=tile, device="cpu")
        lo, hi, _ = sr.step()
        if rank == 0:
            olo, ohi, _ = pyoracle.render_bounds(w, tile=tile)
            q.put((bool(np.array_equal(lo, olo.astype(np.float32))),
                   bool(np.array_equal(hi, ohi.astype(np.float32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,kw,tile", [(2, "C2", dict(N=1500, res=40), 16),
                                                (3, "C4", dict(N=1500, res=36), 8)])
def test_sharded_gloo(world, name, kw, tile):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, kw, tile, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    ok_lo, ok_hi = q.get(timeout=5)
    assert ok_lo and ok_hi


class OracleSubboxCtx:
    """Stands in for Context.as_subbox_count / as_render_subboxes on a CPU-only box."""

    def __init__(self, w, oracle):
        self.w, self.oracle = w, oracle
        self.camera = w.camera
        self.device = None

    def as_subbox_count(self):
        return self.w.n_sub

    def as_render_subboxes(self, b, e, tile, batch, lo, hi, stats=False):
        olo, ohi, st = self.oracle.render_subboxes(self.w, b, e, tile=tile)
        lo.copy_(torch.from_numpy(olo.astype(np.float32)))
        hi.copy_(torch.from_numpy(ohi.astype(np.float32)))
        return lo, hi, st


def _subbox_worker(rank, world, port, kw, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2503_00308_b200.dist import SubboxShardedRenderer, subbox_range
        from workloads import make_config
        w = make_config("C3", **kw)
        sr = SubboxShardedRenderer(OracleSubboxCtx(w, pyoracle), rank, world, tile=16,
                                   device="cpu")
        lo, hi, st = sr.step()
        olo, ohi, _ = pyoracle.render_bounds(w, tile=16)
        b, e = subbox_range(w.n_sub, rank, world)
        q.put((rank, e - b, bool(np.array_equal(lo.numpy(), olo.astype(np.float32))),
               bool(np.array_equal(hi.numpy(), ohi.astype(np.float32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [3, 10])
def test_subbox_sharded_gloo(world):
    """C3's 8 yaw parts over 3 ranks (3/3/2) and over 10 ranks (two ranks get an empty range
    and contribute the union's identities); every rank ends with the oracle's full image."""
    from paper_2503_00308_b200.dist import subbox_range
    assert [subbox_range(8, r, 3) for r in range(3)] == [(0, 3), (3, 6), (6, 8)]
    assert sum(e - b for b, e in (subbox_range(8, r, 10) for r in range(10))) == 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    kw = dict(N=400, res=24)
    procs = [ctx.Process(target=_subbox_worker, args=(r, world, port, kw, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert sum(r[1] for r in res) == 8
    assert all(r[2] and r[3] for r in res)


def _uid_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_00308_b200.dist import share_bytes
        payload = bytes(range(128)) if rank == 0 else None
        got = share_bytes(payload, rank)
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_nccl_id_distribution_gloo():
    """dist.init_comm's out-of-band step: rank 0's 128-byte NCCL id reaches every rank
    unchanged (world 2, gloo; the NCCL communicator itself needs GPUs)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == res[1] == bytes(range(128))
