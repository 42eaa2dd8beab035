"""NEXT-1: BlendInd evaluated with linear relations along the sorted fold
(Alg. 3; §3.3 (4)), on tile lists whose pairs are all certain, intersected
with the interval blend (oracle mode 2).  Pins: zero-width boxes reproduce the concrete render;
one Gaussian reproduces the interval blend (the Exp tangent / chord concretise to the interval
bounds); sampled and brute-force containment (Theorem 1); the result lies inside the interval
blend's and is strictly tighter on C1; on lists with uncertain pairs certain positions use the
fold and uncertain ones their interval terms (reading O20), sound and tighter.""" 
import copy

import numpy as np
import pytest

from tests import helpers as H
from workloads import make_config

TAU = 1e-12


def zero_box(w):
    w = copy.deepcopy(w)
    for k in ("eps_t", "eps_R", "t_off", "R_off"):
        w.pose_box[k] = [0.0, 0.0, 0.0]
    if w.scene_box is not None:
        w.scene_box = dict(w.scene_box, shift_hi=np.array(w.scene_box["shift_lo"], float))
    return w


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_zero_width_box_is_concrete(oracle, name):
    w = zero_box(make_config(name, **({} if name == "C1" else dict(N=1500, res=32))))
    lo, hi, st = oracle.render_bounds(w, mode=2)
    ref = oracle.render_concrete(w)
    slack = w.N * TAU + 1e-12
    assert np.abs(lo - ref).max() <= slack and np.abs(hi - ref).max() <= slack


def test_single_gaussian_equals_interval(oracle):
    w = make_config("C1", N=1, res=16)
    w.pose_box["eps_t"] = [0.05, 0.03, 0.0]
    a = oracle.render_bounds(w, mode=0)
    b = oracle.render_bounds(w, mode=2)
    assert max(np.abs(a[0] - b[0]).max(), np.abs(a[1] - b[1]).max()) <= 1e-12


@pytest.mark.parametrize("name,nrand", [("C1", 150), ("C2", 30), ("C5", 30)])
def test_containment_and_inside_interval(oracle, name, nrand):
    w = make_config(name, **({} if name == "C1" else dict(N=2000, res=40)))
    ilo, ihi, ist = oracle.render_bounds(w, mode=0)
    lo, hi, st = oracle.render_bounds(w, mode=2)
    assert np.all(lo >= ilo) and np.all(hi <= ihi) and np.all(lo <= hi)
    rng = np.random.default_rng(8)
    worst = 0.0
    for p in H.sample_params(w, rng, n_random=nrand, corners=True):
        e, t, shifts = H.pose_of(w, p)
        col = None
        if w.scene_box is not None and w.scene_box["col_lo"] is not None:
            a = rng.uniform(size=(w.N, 1))
            col = (w.scene_box["col_lo"] + a * (w.scene_box["col_hi"] - w.scene_box["col_lo"]))
            col = col.astype(np.float32)
        img = oracle.render_concrete(w, euler=e, t=t, shifts=shifts, color=col)
        worst = max(worst, (lo - img).max(), (img - hi).max())
    assert worst <= 1e-9, worst


def test_c1_brute_force_and_tighter(oracle):
    w = make_config("C1")
    lo, hi, _ = oracle.render_bounds(w, mode=2)
    ilo, ihi, _ = oracle.render_bounds(w, mode=0)
    env_lo = np.full_like(lo, np.inf)
    env_hi = np.full_like(hi, -np.inf)
    for tx in np.linspace(-0.01, 0.01, 4001):
        img = oracle.render_concrete(w, t=[tx, 0.0, 0.0])
        np.minimum(env_lo, img, out=env_lo)
        np.maximum(env_hi, img, out=env_hi)
    assert np.all(lo <= env_lo + 1e-12) and np.all(env_hi <= hi + 1e-12)
    assert H.mpg(lo, hi) < 0.9 * H.mpg(ilo, ihi)  # the fold keeps the pose correlations


def test_uncertain_tiles_mixed_rule(oracle):
    """Reading O20 on lists with uncertain pairs: certain positions contribute through the
    linear fold, uncertain ones their interval-blend terms.  The result lies inside the
    interval blend everywhere (the two are intersected), it is sound (concrete renders at
    sampled poses of a 6-DoF box inside), and on the uncertain tiles it can tighten too."""
    w = make_config("C4", N=2000, res=48)
    a = oracle.render_bounds(w, mode=0)
    b = oracle.render_bounds(w, mode=2)
    assert np.all(b[0] >= a[0]) and np.all(b[1] <= a[1])
    ts = w.tile
    ntx = -(-48 // ts)
    n_unc, tighter = 0, 0
    for t in range(ntx * ntx):
        unc = oracle.render_tiles(w, [t])[2]["uncertain_pairs"]
        if unc > 0:
            n_unc += 1
            ys = slice((t // ntx) * ts, (t // ntx + 1) * ts)
            xs = slice((t % ntx) * ts, (t % ntx + 1) * ts)
            tighter += int(np.any(b[1][ys, xs] < a[1][ys, xs] - 1e-12) or
                           np.any(b[0][ys, xs] > a[0][ys, xs] + 1e-12))
    assert n_unc > 0 and tighter > 0
    rng = np.random.default_rng(21)
    for p in H.sample_params(w, rng, n_random=40):
        e, t, sh = H.pose_of(w, p)
        img = oracle.render_concrete(w, euler=e, t=t, shifts=sh)
        assert np.all(b[0] <= img + 1e-9) and np.all(img <= b[1] + 1e-9)


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


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw,parts", [("C1", {}, 1), ("C2", dict(N=3000, res=48), 1),
                                           ("C2", dict(N=3000, res=48), 2),
                                           ("C5", dict(N=3000, res=48), 1),
                                           ("C3", dict(N=3000, res=48), 1),
                                           ("C4", dict(N=4000, res=48), 1)])
def test_gpu_linear_blend_parity(gctx, oracle, name, kw, parts):
    w = make_config(name, **kw)
    if parts > 1:
        w.pose_box["parts"] = [parts, 1, 1, 1, 1, 1]
    gctx.load_workload(w)
    gctx.as_set_blend(1)
    try:
        lo, hi, st = gctx.as_render_bounds(w.tile, w.batch)
    finally:
        gctx.as_set_blend(0)
    ilo, ihi, _ = gctx.as_render_bounds(w.tile, w.batch)
    lo, hi = lo.cpu().numpy().astype(np.float64), hi.cpu().numpy().astype(np.float64)
    olo, ohi, ost = oracle.render_bounds(w, mode=2)
    err = max(np.abs(lo - olo).max(), np.abs(hi - ohi).max())
    assert err <= 1e-4, err
    il, ih = ilo.cpu().numpy(), ihi.cpu().numpy()
    assert np.all(lo >= il) and np.all(hi <= ih)  # inside the interval bounds
    if name == "C1":
        assert H.mpg(lo, hi) < 0.9 * H.mpg(il, ih)


@pytest.mark.gpu
def test_gpu_linear_blend_limits(gctx):
    """The linear blend renders full images; tile sharding (compact tile-major outputs) is
    refused.  Unknown modes are refused."""
    from paper_2503_00308_b200 import AbsplatError
    w = make_config("C3", N=2000, res=32)  # n = 4
    gctx.load_workload(w)
    gctx.as_set_blend(1)
    try:
        with pytest.raises(AbsplatError):
            gctx.as_render_shard(16, 16, 0, 2, 4)
    finally:
        gctx.as_set_blend(0)
    with pytest.raises(AbsplatError):
        gctx.as_set_blend(2)
