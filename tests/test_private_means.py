"""NEXT-2: per-Gaussian private mean offsets (independent intervals on each
Gaussian's mean, three private variables per Gaussian after the shared ones).  Pins: zero-width
private boxes change nothing; a private box on one Gaussian equals the shared group shift of
that Gaussian alone; independent sampling of every Gaussian's offset is contained (Theorem 1),
including a pair whose depth order flips inside the box (which a shared treatment would miss)."""
import copy

import numpy as np
import pytest

from tests import helpers as H
from workloads import make_config


def with_private(w, lo, hi):
    v = copy.deepcopy(w)
    sb = dict(v.scene_box) if v.scene_box is not None else dict(
        n_groups=0, group_of=None, dir=None, shift_lo=None, shift_hi=None, parts=[1, 1, 1],
        col_lo=None, col_hi=None, op_lo=None, op_hi=None)
    sb["priv_lo"] = np.asarray(lo, np.float32).reshape(-1, 3)
    sb["priv_hi"] = np.asarray(hi, np.float32).reshape(-1, 3)
    v.scene_box = sb
    return v


def test_zero_width_private_box_changes_nothing(oracle):
    w = make_config("C1")
    z = np.zeros((w.N, 3), np.float32)
    a = oracle.render_bounds(w)
    b = oracle.render_bounds(with_private(w, z, z))
    assert b[2]["n_vars"] == a[2]["n_vars"] + 3
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_single_private_box_equals_group_shift(oracle):
    w = make_config("C1")
    i = 5
    lo = np.zeros((w.N, 3), np.float32)
    hi = np.zeros((w.N, 3), np.float32)
    hi[i, 1] = 0.0625  # exact in float32 (private bounds are float32 inputs)
    p = oracle.render_bounds(with_private(w, lo, hi))
    g = copy.deepcopy(w)
    gof = np.full(w.N, -1, np.int32)
    gof[i] = 0
    g.scene_box = dict(n_groups=1, group_of=gof, dir=np.array([[0.0, 1.0, 0.0]]),
                       shift_lo=np.array([0.0]), shift_hi=np.array([0.0625]), parts=[1, 1, 1],
                       col_lo=None, col_hi=None, op_lo=None, op_hi=None)
    q = oracle.render_bounds(g)
    assert max(np.abs(p[0] - q[0]).max(), np.abs(p[1] - q[1]).max()) <= 1e-12


def _sampled_containment(oracle, w, lo, hi, n, seed):
    v = with_private(w, lo, hi)
    blo, bhi, st = oracle.render_bounds(v)
    rng = np.random.default_rng(seed)
    worst = 0.0
    params = H.sample_params(w, rng, n_random=n, corners=True)
    for k, p in enumerate(params * 2):
        e, t, shifts = H.pose_of(w, p)
        c = copy.deepcopy(w)
        if k < len(params):  # random independent offsets
            d = rng.uniform(lo, hi)
        else:                # per-Gaussian vertices, chosen independently
            d = np.where(rng.uniform(size=lo.shape) < 0.5, lo, hi)
        c.mean = (w.mean + d).astype(np.float32)
        img = oracle.render_concrete(c, euler=e, t=t, shifts=shifts)
        worst = max(worst, (blo - img).max(), (img - bhi).max())
    return worst, st


def test_independent_offsets_contained(oracle):
    w = make_config("C1")
    lo = np.full((w.N, 3), -0.02, np.float32)
    hi = np.full((w.N, 3), 0.02, np.float32)
    worst, st = _sampled_containment(oracle, w, lo, hi, 60, 3)
    assert worst <= 1e-9, worst


def test_depth_flip_between_two_private_boxes(oracle):
    """Two overlapping Gaussians at the same nominal depth, each with its own +-5 cm depth
    interval: their order flips inside the box, so the pair must be uncertain."""
    w = make_config("C1", N=2, res=16)
    m = w.mean.copy()
    m[0] = [0.0, 0.0, 5.0]
    m[1] = [0.02, 0.0, 5.0]
    w.mean = m
    w.pose_box["eps_t"] = [0.0, 0.0, 0.0]
    lo = np.array([[0, 0, -0.05], [0, 0, -0.05]], np.float32)
    hi = np.array([[0, 0, 0.05], [0, 0, 0.05]], np.float32)
    worst, st = _sampled_containment(oracle, w, lo, hi, 20, 5)
    assert st["uncertain_pairs"] >= 1
    assert worst <= 1e-9, worst


# ------------------------------------------------------------------ GPU (through the C ABI)
@pytest.fixture(scope="module")
def gctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_00308_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _gpu_vs_oracle(gctx, oracle, v):
    gctx.load_workload(v)
    lo, hi, st = gctx.as_render_bounds(v.tile, v.batch)
    olo, ohi, ost = oracle.render_bounds(v)
    err = max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max())
    assert err <= 1e-4, err
    assert st["n_vars"] == ost["n_vars"]
    assert st["pairs"] == ost["pairs"] and st["uncertain_pairs"] == ost["uncertain_pairs"]
    assert st["order_violations"] == 0


@pytest.mark.gpu
def test_gpu_private_parity_c1(gctx, oracle):
    w = make_config("C1")
    _gpu_vs_oracle(gctx, oracle, with_private(w, np.full((w.N, 3), -0.02), np.full((w.N, 3), 0.02)))


@pytest.mark.gpu
def test_gpu_private_parity_c5_blade(gctx, oracle):
    """C5 (reduced) with independent +-2 cm mean boxes on the blade Gaussians on top of the
    shared blade shift, the colour box and the camera box (n = 2 shared + 3 private)."""
    w = make_config("C5", N=3000, res=48)
    blade = w.scene_box["group_of"] >= 0
    lo = np.zeros((w.N, 3), np.float32)
    hi = np.zeros((w.N, 3), np.float32)
    lo[blade] = -0.02
    hi[blade] = 0.02
    _gpu_vs_oracle(gctx, oracle, with_private(w, lo, hi))


@pytest.mark.gpu
def test_gpu_private_depth_flip(gctx, oracle):
    w = make_config("C1", N=2, res=16)
    m = w.mean.copy()
    m[0] = [0.0, 0.0, 5.0]
    m[1] = [0.02, 0.0, 5.0]
    w.mean = m
    w.pose_box["eps_t"] = [0.0, 0.0, 0.0]
    v = with_private(w, np.array([[0, 0, -0.05]] * 2), np.array([[0, 0, 0.05]] * 2))
    _gpu_vs_oracle(gctx, oracle, v)
    gctx.as_set_scene_box(None)
