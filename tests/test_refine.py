"""Adaptive refinement (PAPER.md:470 (2)): the product's host driver
`paper_2503_00308_b200.refine` bisects sub-boxes with MatrixInv failures.  On CPU the failure
counts come from the fp64 oracle (a stand-in context), so the policy and the explicit
partitions are exercised without a GPU; the GPU test checks the library's counts and render
against the oracle on the refined partition."""
import copy
import math

import numpy as np
import pytest

from paper_2503_00308_b200 import refine
from tests import helpers as H
from workloads import make_config

GF_FAIL, GF_DROP = 4, 1


def spiky(N=24, yaw_deg=1.0, squash=0.2):
    """Thin Gaussians under a yaw box: MatrixInv fails for some of them."""
    w = make_config("C1", N=N)
    ch = w.chol.copy()
    ch[:, 2] *= squash
    ch[:, 4] *= squash
    ch[:, 5] *= squash
    w.chol = ch
    w.pose_box["eps_R"] = [0.0, 0.0, math.radians(yaw_deg)]
    return w


class OracleFailCtx:
    """as_set_subboxes / as_subbox_fails backed by the oracle's per-Gaussian flags."""

    def __init__(self, w, oracle):
        self.w, self.oracle, self.parts = copy.deepcopy(w), oracle, None

    def as_set_subboxes(self, bounds):
        self.parts = np.asarray(bounds, float).reshape(-1, 9, 2)
        self.w.pose_box = dict(self.w.pose_box, parts=[1] * 6, subboxes=self.parts)

    def as_subbox_fails(self):
        out = []
        for s in range(len(self.parts)):
            f = self.oracle.gaussian_forms(self.w, sub=s)["flags"].astype(np.int64)
            out.append(int(np.sum(((f & GF_FAIL) != 0) & ((f & GF_DROP) == 0))))
        return np.array(out, np.int64)


def test_partition_helpers():
    w = make_config("C3", N=100, res=16)
    full = refine.box_bounds(w.pose_box, w.scene_box)
    parts = refine.uniform_partition(w.pose_box, w.scene_box)
    assert parts.shape == (8, 9, 2)
    # the parts tile the yaw axis and copy the other axes
    assert np.allclose(parts[:, 5, 0], full[5, 0] + np.arange(8) * (full[5, 1] - full[5, 0]) / 8)
    assert np.allclose(parts[:, :5], full[:5]) and np.allclose(parts[:, 6:], full[6:])
    a, b = refine.bisect(parts[0], full)
    # failures come from the rotation: the split is along yaw even though the translation
    # axes are relatively wider
    assert a[5, 1] == b[5, 0] == 0.5 * (parts[0, 5, 0] + parts[0, 5, 1])
    assert np.allclose(np.delete(a, 5, axis=0), np.delete(parts[0], 5, axis=0))
    t = refine.box_bounds(dict(w.pose_box, eps_R=[0.0, 0.0, 0.0]), None)
    a, b = refine.bisect(t, t)  # no rotation: widest axis overall (tx, lowest on ties)
    assert a[0, 1] == b[0, 0] == 0.0


def test_refinement_removes_failures_soundly(oracle):
    w = spiky()
    ctx = OracleFailCtx(w, oracle)
    parts, hist = refine.refine_fails(ctx, w.pose_box, w.scene_box, max_subboxes=64)
    assert hist[0].sum() > 0                      # the unrefined box fails
    assert hist[-1].sum() == 0 and len(parts) > 1  # refinement removes every failure
    # the partition covers the box: every sub-box inside, volumes add up on the split axis
    full = refine.box_bounds(w.pose_box, w.scene_box)
    assert np.all(parts[:, :, 0] >= full[:, 0] - 1e-15) and np.all(parts[:, :, 1] <= full[:, 1] + 1e-15)
    var = [a for a in range(9) if full[a, 1] > full[a, 0]]
    vol = np.prod([parts[:, a, 1] - parts[:, a, 0] for a in var], axis=0).sum()
    assert vol == pytest.approx(np.prod([full[a, 1] - full[a, 0] for a in var]), rel=1e-12)
    # the union over the refined partition is sound (Theorem 1) and tighter than the FAIL box
    lo, hi, st = oracle.render_bounds(ctx.w)
    assert st["n_sub"] == len(parts)
    ulo, uhi, ust = oracle.render_bounds(w)
    assert H.mpg(lo, hi) < H.mpg(ulo, uhi)
    rng = np.random.default_rng(4)
    for p in H.sample_params(w, rng, n_random=60):
        e, t, sh = H.pose_of(w, p)
        img = oracle.render_concrete(w, euler=e, t=t)
        assert np.all(lo <= img + 1e-9) and np.all(img <= hi + 1e-9)


def test_refinement_budget(oracle):
    w = spiky()
    ctx = OracleFailCtx(w, oracle)
    parts, hist = refine.refine_fails(ctx, w.pose_box, w.scene_box, max_subboxes=3)
    assert len(parts) <= 3


@pytest.mark.gpu
def test_gpu_refinement_matches_oracle(oracle):
    """The library's per-sub-box FAIL counts equal the oracle's on every round, so the product
    driver reaches the same partition on the GPU as with the oracle's counts; the render of
    that explicit partition matches the oracle within 1e-4."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_00308_b200 import Context
    w = spiky()
    ref_parts, ref_hist = refine.refine_fails(OracleFailCtx(w, oracle), w.pose_box, w.scene_box)
    with Context(0) as ctx:
        ctx.load_workload(w)
        parts, hist = refine.refine_fails(ctx, w.pose_box, w.scene_box)
        assert len(hist) == len(ref_hist)
        for h, r in zip(hist, ref_hist):
            assert np.array_equal(h, r)
        assert np.array_equal(parts, ref_parts)
        lo, hi, st = ctx.as_render_bounds(16, 16)
        assert st["n_sub"] == len(parts) and st["fails"] == 0
        ew = copy.deepcopy(w)
        ew.pose_box = dict(w.pose_box, parts=[1] * 6, subboxes=parts)
        olo, ohi, ost = oracle.render_bounds(ew)
        err = max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max())
        assert err <= 1e-4, err
        # clearing the list restores the uniform partition
        ctx.as_set_subboxes(None)
        assert ctx.as_subbox_count() == 1
        with pytest.raises(Exception):
            bad = parts[:1].copy()
            bad[0, 5, 1] += 1.0
            ctx.as_set_subboxes(bad)


class OracleRenderCtx(OracleFailCtx):
    """as_set_subboxes / as_render_subboxes backed by the fp64 oracle (CPU stand-in)."""

    def as_render_subboxes(self, b, e, tile=16, batch=64):
        lo, hi, st = self.oracle.render_subboxes(self.w, b, e, tile=tile)
        return lo, hi, {"ms_total": 0.0}


def test_width_refinement_tightens_soundly(oracle):
    """Width-driven bisection (NEXT-3's second half): the union over the refined partition
    is sound (Theorem 1) and its MPG falls from the unrefined box's; on a 6-DoF box the first
    splits cut MPG substantially (partitions are the paper's main lever)."""
    w = make_config("C4", N=60, res=32)
    w.pose_box = dict(w.pose_box, eps_t=[0.05] * 3, eps_R=[math.radians(1.0)] * 3)
    ctx = OracleRenderCtx(w, oracle)
    parts, hist = refine.refine_width(ctx, w.pose_box, w.scene_box, max_subboxes=6)
    assert len(parts) == 6 and [h[0] for h in hist] == [1, 2, 3, 4, 5, 6]
    assert hist[-1][1] < 0.95 * hist[0][1]
    assert all(b[1] <= a[1] + 1e-12 for a, b in zip(hist, hist[1:]))  # never looser here
    ulo, uhi, _ = oracle.render_bounds(w)
    assert abs(hist[0][1] - H.mpg(ulo, uhi)) < 1e-9  # one sub-box = the plain render
    ew = copy.deepcopy(w)
    ew.pose_box = dict(w.pose_box, parts=[1] * 6, subboxes=parts)
    lo, hi, st = oracle.render_bounds(ew)
    assert st["n_sub"] == 6 and abs(H.mpg(lo, hi) - hist[-1][1]) < 1e-9
    rng = np.random.default_rng(5)
    for p in H.sample_params(w, rng, n_random=40, corners=False):
        e, t, sh = H.pose_of(w, p)
        img = oracle.render_concrete(w, euler=e, t=t)
        assert np.all(lo <= img + 1e-9) and np.all(img <= hi + 1e-9)
