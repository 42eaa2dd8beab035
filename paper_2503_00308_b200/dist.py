"""Sharding over GPUs (north_star (3)), one process per GPU, the scene
replicated on every rank.

* In the library (the product path): `init_comm` hands rank 0's NCCL unique id to every
  rank (torch.distributed is only the out-of-band channel for those 128 bytes) and joins the
  context's communicator (as_comm_init); from then on as_render_bounds shards the image
  tiles (or the sub-boxes) over the ranks and runs the one collective itself, on the
  context's stream, leaving the full bound images on every rank.
* The Python-side drivers below (ShardedRenderer / SubboxShardedRenderer) run the same
  decomposition with torch.distributed collectives on the library's per-rank outputs; they
  serve the gloo CPU tests and bench's --emulate-world timing.

* Tiles (ShardedRenderer): image tiles assigned by the library's deterministic LPT owner map,
  each rank rendering only its tiles into a compact tile-major buffer, then ONE all-gather of
  the bound tiles (NCCL over NVLink / NVSwitch) and an untile on the root.
* Sub-boxes (SubboxShardedRenderer, the second axis): each rank renders the union over a
  contiguous range of the partition's sub-boxes for the whole image, then ONE all-reduce MIN
  on lo and MAX on hi (step 22's union) gives every rank the full image.  No
  work is replicated (each sub-box has its own per-Gaussian setup), so this is the better
  axis when the partition has at least as many sub-boxes as ranks (C3: 8).

Gaussians are never split across ranks: blending order is not commutative.
"""
from __future__ import annotations

import numpy as np

from .api import Context, as_untile


def share_bytes(payload, rank: int, group=None, src: int = 0) -> bytes:
    """Broadcast `payload` (bytes, meaningful on rank `src`) to every rank of the default
    torch.distributed group (or `group`); returns the bytes on every rank."""
    import torch.distributed as dist
    obj = [payload if rank == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return bytes(obj[0])


def init_comm(ctx: Context, rank: int, world: int, group=None, axis: int = 0):
    """Join the library communicator of `ctx` (rank `rank` of `world`); axis as
    Context.as_set_shard_axis.  Collective over the torch.distributed group."""
    from .api import as_nccl_id
    uid = share_bytes(as_nccl_id() if rank == 0 else None, rank, group)
    ctx.as_comm_init(rank, world, uid)
    ctx.as_set_shard_axis(axis)
    return ctx


class ShardedRenderer:
    """Render the abstract image of the context's scene/camera/box across `world` ranks."""

    def __init__(self, ctx: Context, rank: int, world: int, group=None, tile: int = 16,
                 batch: int = 64, slack: float = 0.25, device=None):
        import torch
        self.ctx, self.rank, self.world, self.group = ctx, rank, world, group
        self.tile, self.batch = tile, batch
        nt = ctx.n_tiles(tile)
        base = -(-nt // world)
        self.cap = base + max(1, int(base * slack))
        dev = device if device is not None else f"cuda:{ctx.device}"
        shape = (self.cap, tile * tile, 3)
        self.lo_tm = torch.empty(shape, dtype=torch.float32, device=dev)
        self.hi_tm = torch.empty(shape, dtype=torch.float32, device=dev)
        # gathered buffers are flat along dim 0 (world * cap) as both NCCL and gloo accept
        self.g_lo = torch.empty((world * self.cap,) + shape[1:], dtype=torch.float32, device=dev)
        self.g_hi = torch.empty((world * self.cap,) + shape[1:], dtype=torch.float32, device=dev)
        self.meta = torch.empty((self.cap + 1,), dtype=torch.int32, device=dev)
        self.g_meta = torch.empty((world * (self.cap + 1),), dtype=torch.int32, device=dev)

    def step(self, stats: bool = False):
        """One sharded render.  Returns (lo, hi) on rank 0 (None elsewhere) and stats."""
        import torch
        import torch.distributed as dist
        lo_tm, hi_tm, owned, n_owned, st = self.ctx.as_render_shard(
            self.tile, self.batch, self.rank, self.world, self.cap, self.lo_tm, self.hi_tm,
            stats=stats)
        meta = np.concatenate([[n_owned], owned]).astype(np.int32)
        self.meta.copy_(torch.from_numpy(meta), non_blocking=False)
        if self.world > 1:
            dist.all_gather_into_tensor(self.g_lo, self.lo_tm, group=self.group)
            dist.all_gather_into_tensor(self.g_hi, self.hi_tm, group=self.group)
            dist.all_gather_into_tensor(self.g_meta, self.meta, group=self.group)
        else:
            self.g_lo.copy_(self.lo_tm)
            self.g_hi.copy_(self.hi_tm)
            self.g_meta.copy_(self.meta)
        if self.rank != 0:
            return None, None, st
        gm = self.g_meta.cpu().numpy().reshape(self.world, self.cap + 1)
        g_lo, g_hi = self.g_lo, self.g_hi
        if not g_lo.is_cuda:  # host assembly path (CPU / gloo)
            g_lo, g_hi = g_lo.numpy(), g_hi.numpy()
        lo, hi = self.ctx.as_untile(self.tile, self.world, self.cap, gm[:, 1:], gm[:, 0],
                                    g_lo, g_hi)
        return lo, hi, st


def subbox_range(n_sub: int, rank: int, world: int):
    """Contiguous balanced range [b, e) of the n_sub sub-boxes for `rank` (may be empty)."""
    q, r = divmod(n_sub, world)
    b = rank * q + min(rank, r)
    return b, b + q + (1 if rank < r else 0)


class SubboxShardedRenderer:
    """Union over the partition's sub-boxes, split across `world` ranks (all-reduce min/max)."""

    def __init__(self, ctx: Context, rank: int, world: int, group=None, tile: int = 16,
                 batch: int = 64, device=None):
        import torch
        self.ctx, self.rank, self.world, self.group = ctx, rank, world, group
        self.tile, self.batch = tile, batch
        self.n_sub = ctx.as_subbox_count()
        self.range = subbox_range(self.n_sub, rank, world)
        H, W = int(ctx.camera["H"]), int(ctx.camera["W"])
        dev = device if device is not None else f"cuda:{ctx.device}"
        self.lo = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        self.hi = torch.empty((H, W, 3), dtype=torch.float32, device=dev)

    def step(self, stats: bool = False):
        """One sharded render; every rank returns the full (lo, hi) and its own stats."""
        import torch.distributed as dist
        b, e = self.range
        lo, hi, st = self.ctx.as_render_subboxes(b, e, self.tile, self.batch, self.lo, self.hi,
                                                 stats=stats)
        if self.world > 1:
            dist.all_reduce(self.lo, op=dist.ReduceOp.MIN, group=self.group)
            dist.all_reduce(self.hi, op=dist.ReduceOp.MAX, group=self.group)
        return self.lo, self.hi, st


def assemble_host(W: int, H: int, tile: int, world: int, cap: int, owned, n_owned, lo_tm, hi_tm):
    """Host-side assembly (as_untile with host pointers; no GPU needed)."""
    return as_untile(W, H, tile, world, cap, owned, n_owned, lo_tm, hi_tm)
