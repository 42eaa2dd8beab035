"""The multi-GPU path inside the library (north_star (3)): NCCL
communicator, device LPT owner map, one all-gather of bound tiles (or all-reduce MIN / MAX of
sub-box unions) and the on-device untile.  gpurun gives one GPU, so the collective runs on a
single-rank communicator with the shard axis forced (the same code path as world > 1), and
the device owner map is compared with the host LPT of as_lpt_assign for world 2..8."""
import numpy as np
import pytest

import paper_2503_00308_b200 as ap
from workloads import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.mark.parametrize("name,kw,axis", [("C4", dict(N=6000, res=72), 1),
                                          ("C3", dict(N=5000, res=56), 1),
                                          ("C3", dict(N=5000, res=56), 2)])
def test_single_rank_collective_equals_plain(torch_cuda, name, kw, axis):
    torch = torch_cuda
    w = make_config(name, **kw)
    with ap.Context(0) as plain, ap.Context(0) as c:
        plain.load_workload(w)
        lo0, hi0, _ = plain.as_render_bounds(w.tile, w.batch)
        c.load_workload(w)
        c.as_comm_init(0, 1, ap.as_nccl_id())
        c.as_set_shard_axis(axis)
        lo, hi, st = c.as_render_bounds(w.tile, w.batch)
        assert torch.equal(lo, lo0) and torch.equal(hi, hi0)
        assert st["world"] == 1 and st["ms_gather"] > 0
        # again: the tile axis keeps its owner map (no cost pass), same images
        lo2, hi2, st2 = c.as_render_bounds(w.tile, w.batch)
        assert torch.equal(lo2, lo0) and torch.equal(hi2, hi0)
        assert st2["pairs"] == st["pairs"] and st2["active_pairs"] == st["active_pairs"]
        if axis == 1:
            assert st["n_owned"] == c.n_tiles(w.tile)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_device_lpt_equals_host_lpt(torch_cuda, world):
    w = make_config("C4", N=8000, res=96)
    with ap.Context(0) as c:
        c.load_workload(w)
        nt = c.n_tiles(16)
        cap = -(-nt // world) + 2
        owner, costs = c.as_tile_owners(16, world, cap)
        assert costs.sum() > 0
        assert np.array_equal(owner, ap.as_lpt_assign(costs, world, cap))
