"""Pins of the oracle's whole pipeline against what the paper
fixes: zero-width box == concrete render, Theorem 1 containment at sampled poses,
brute-force pose enumeration on C1, per-line soundness of every Alg. 1 intermediate,
the d^4 identity (l.9-10), the colour-box closed form, Lemma 2 via windowed == direct.
CPU only."""
import copy
import math

import numpy as np
import pytest

from tests import helpers as H
from workloads import make_config

TAU = 1e-12


def small(name, **kw):
    defaults = {"C1": {}, "C2": dict(N=2000, res=40), "C3": dict(N=3000, res=40),
                "C4": dict(N=3000, res=40), "C5": dict(N=2000, res=40)}
    args = dict(defaults[name])
    args.update(kw)
    return make_config(name, **args)


def zero_box(w):
    w = copy.deepcopy(w)
    for k in ("eps_t", "eps_R", "t_off", "R_off"):
        w.pose_box[k] = [0.0, 0.0, 0.0]
    w.pose_box["parts"] = [1] * 6
    if w.scene_box is not None:
        sb = w.scene_box
        sb["shift_hi"] = np.array(sb["shift_lo"], float)
        sb["col_hi"] = np.array(sb["col_lo"])
    return w


# ------------------------------------------------------------------ zero width == concrete
@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5"])
def test_zero_width_box_is_concrete_render(oracle, name):
    """A zero-width pose box reduces AbstractSplat to GaussianSplat (north_star):
    lo == hi == Alg. 1 + BlendSort, up to the culling slack N tau and rounding."""
    w = zero_box(small(name))
    lo, hi, st = oracle.render_bounds(w)
    assert st["n_vars"] == 0 and st["uncertain_pairs"] == 0
    cols = w.scene_box["col_lo"] if w.scene_box is not None else None
    img = oracle.render_concrete(w, color=cols, shifts=None if w.scene_box is None
                                 else np.array(w.scene_box["shift_lo"]))
    slack = 2 * w.N * TAU + 1e-12
    assert np.abs(hi - lo).max() <= slack
    assert np.all(lo <= img + 1e-12) and np.all(img <= hi + 1e-12)
    assert np.abs(img - 0.5 * (lo + hi)).max() <= slack
    assert img.max() > 0.05  # the scene is visible


# ------------------------------------------------------------------ Theorem 1 containment
@pytest.mark.parametrize("name,nrand", [("C1", 200), ("C2", 40), ("C3", 30), ("C4", 40),
                                        ("C5", 40)])
def test_containment_sampled_poses(oracle, name, nrand):
    """Theorem 1: every concrete render with parameters in the box lies in
    [lo, hi]; sampled at all 2^n corners, the centre and random points."""
    w = small(name)
    lo, hi, st = oracle.render_bounds(w)
    assert np.all(lo <= hi) and lo.min() >= 0 and hi.max() <= 1
    assert st["order_violations"] == 0
    rng = np.random.default_rng(5)
    worst = 0.0
    params = H.sample_params(w, rng, n_random=nrand, corners=True)
    if name == "C4":
        params = params[:1] + params[1:65:4] + params[65:]  # 16 of the 64 corners
    for p in params:
        e, t, shifts = H.pose_of(w, p)
        col = None
        if w.scene_box is not None and w.scene_box["col_lo"] is not None:
            a = rng.uniform(size=(w.N, 1))
            col = (w.scene_box["col_lo"] + a * (w.scene_box["col_hi"] - w.scene_box["col_lo"]))
            col = col.astype(np.float32)
        img = oracle.render_concrete(w, euler=e, t=t, shifts=shifts, color=col)
        worst = max(worst, (lo - img).max(), (img - hi).max())
    assert worst <= 1e-9, worst


def test_c1_brute_force_pose_grid(oracle):
    """Brute-force enumeration of the 1-D C1 box (north_star): 20001 poses enclosed."""
    w = make_config("C1")
    lo, hi, _ = oracle.render_bounds(w)
    env_lo = np.full_like(lo, np.inf)
    env_hi = np.full_like(hi, -np.inf)
    for tx in np.linspace(-0.01, 0.01, 20001):
        img = oracle.render_concrete(w, t=[tx, 0.0, 0.0])
        np.minimum(env_lo, img, out=env_lo)
        np.maximum(env_hi, img, out=env_hi)
    assert np.all(lo <= env_lo + 1e-12) and np.all(env_hi <= hi + 1e-12)
    # and the abstract image is informative: gap within a small factor of the envelope
    assert H.mpg(lo, hi) < 5 * H.mpg(env_lo, env_hi) + 1e-3


# ------------------------------------------------------------------ blend structure
@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_windowed_blend_equals_direct(oracle, name):
    """The prefix-product/exception-window blend equals Alg. 3 evaluated pair by pair
    (step 13 order structure), on boxes that do have uncertain depth pairs."""
    w = small(name, res=24, N=1200 if name == "C3" else 2000)
    lo0, hi0, st0 = oracle.render_bounds(w, mode=0)
    lo1, hi1, st1 = oracle.render_bounds(w, mode=1)
    assert st0["uncertain_pairs"] > 0 and st0["order_violations"] == 0
    assert np.abs(lo0 - lo1).max() <= 1e-12 and np.abs(hi0 - hi1).max() <= 1e-12


def test_translation_box_has_no_uncertain_pairs(oracle):
    for name in ("C1", "C2"):
        w = small(name)
        _, _, st = oracle.render_bounds(w)
        assert st["uncertain_pairs"] == 0 and st["n_vars"] == 1


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_tile_size_is_a_performance_knob(oracle, name):
    """Reading O1: culling is per pixel, so TS only changes the work, never the result."""
    w = small(name, res=36)
    lo, hi, st = oracle.render_bounds(w, tile=16)
    for ts in (8, 32):
        l2, h2, s2 = oracle.render_bounds(w, tile=ts)
        assert np.array_equal(lo, l2) and np.array_equal(hi, h2)
        assert s2["active_pairs"] == st["active_pairs"]


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_tile_free_pixel_bounds(oracle, name):
    """or_pixel_bounds (no tiles, every Gaussian, direct Alg. 3) == the tiled render."""
    w = small(name, res=32)
    lo, hi, _ = oracle.render_bounds(w)
    rng = np.random.default_rng(1)
    px = rng.integers(0, 32, 25)
    py = rng.integers(0, 32, 25)
    l, h = oracle.pixel_bounds(w, px, py)
    assert np.abs(l - lo[py, px]).max() <= 1e-12 and np.abs(h - hi[py, px]).max() <= 1e-12


# ------------------------------------------------------------------ per-line soundness
def _check_forms_contain(oracle, w, n_gauss=200, n_xi=12, rtol=1e-9):
    gf = oracle.gaussian_forms(w)
    n = gf["n"]
    rng = np.random.default_rng(3)
    params = H.sample_params(w, rng, n_random=n_xi, corners=False)
    idx = np.arange(min(n_gauss, w.N))
    bad = []
    for p in params:
        xi = H.xi_of(w, p)
        e, t, shifts = H.pose_of(w, p)
        for i in idx:
            flags = int(gf["flags"][i])
            cc = H.concrete_intermediates(w, e, t, shifts, i)
            items = [("uc0", cc["uc"][0]), ("uc1", cc["uc"][1]), ("uc2", cc["uc"][2]),
                     ("d", cc["d"]), ("up0", cc["up"][0]), ("up1", cc["up"][1]),
                     ("X00", cc["X"][0, 0]), ("X01", cc["X"][0, 1]), ("X11", cc["X"][1, 1]),
                     ("D2", cc["D2"]), ("DU0", cc["DU"][0]), ("DU1", cc["DU"][1])]
            items += [(f"Mp{a}{c}", cc["Mp"][a, c]) for a in range(2) for c in range(3)]
            if not flags & 4:
                items += [(f"conic{a}{b}", cc["conic"][a, b]) for a in range(2) for b in range(2)]
                items += [(f"W{a}{c}", cc["W"][a, c]) for a in range(2) for c in range(3)]
            for name, v in items:
                lo, hi = H.eval_form(gf[name][i], n, xi)
                tol = rtol * (1 + abs(v) + abs(lo) + abs(hi))
                if not (lo - tol <= v <= hi + tol):
                    bad.append((name, i, lo, v, hi))
    return bad, gf


@pytest.mark.parametrize("name", ["C2", "C4", "C5"])
def test_every_alg1_line_is_sound(oracle, name):
    """Theorem 1's proof line by line: at sampled poses, every intermediate of
    Alg. 1 (uc, d, up, Mp, X = Mp Mp^T, Conic = X^{-1}, W = Conic Mp, d^2, d up) lies
    between the lower and upper affine forms evaluated at that pose."""
    bad, gf = _check_forms_contain(oracle, small(name))
    assert not bad, bad[:5]



def test_translation_forms_exact_at_vertices(oracle):
    """a1-a3 on translation-only boxes: uc, d, up are exactly affine (lower == upper) and
    equal the concrete values at the box vertices."""
    w = small("C2")
    gf = oracle.gaussian_forms(w)
    n = gf["n"]
    for name in ("uc0", "uc1", "uc2", "d", "up0", "up1"):
        f = gf[name]
        assert np.allclose(f[:, :n + 1], f[:, n + 1:], rtol=0, atol=1e-12)
    for s in (-1.0, 1.0):
        p = np.zeros(9)
        p[0] = w.pose_box["t_off"][0] + s * w.pose_box["eps_t"][0]
        e, t, sh = H.pose_of(w, p)
        for i in range(50):
            cc = H.concrete_intermediates(w, e, t, sh, i)
            lo, hi = H.eval_form(gf["d"][i], n, np.array([s]))
            assert abs(lo - cc["d"]) < 1e-12 and abs(hi - cc["d"]) < 1e-12


def test_d4_identity(oracle):
    """Alg. 1 l.9-10 equal the textbook 2-D Gaussian o exp(-1/2 (u-mu)^T S^-1 (u-mu)) with
    mu = (f x/z + c) and S = J_std Sigma_cam J_std^T, J_std = [[f/z,0,-f x/z^2],[0,f/z,-f y/z^2]]
    (the d^4 factors cancel).  Single-Gaussian scenes, pc = a c with c = (1,1,1)."""
    from workloads.synth import Workload
    rng = np.random.default_rng(11)
    worst = 0.0
    for trial in range(300):
        mean, chol, o, _ = __import__("workloads").random_scene(1000 + trial, 1)
        cam = dict(fx=rng.uniform(10, 800), fy=rng.uniform(10, 800), cx=8.0, cy=8.0, W=16, H=16,
                   euler=list(rng.uniform(-0.2, 0.2, 3)), t=list(rng.uniform(-0.3, 0.3, 3)))
        w = Workload("d4", mean.astype(np.float32), chol.astype(np.float32),
                     o.astype(np.float32), np.ones((1, 3), np.float32), cam,
                     dict(eps_t=[0] * 3, eps_R=[0] * 3, t_off=[0] * 3, R_off=[0] * 3, t_frame=0,
                          parts=[1] * 6), None)
        px = rng.integers(0, 16, 4)
        py = rng.integers(0, 16, 4)
        pc = oracle.render_concrete(w, px=px, py=py)
        R = H.rot_c2w(cam["euler"]).T
        c = w.chol[0].astype(float)
        Mw = np.array([[c[0], 0, 0], [c[1], c[2], 0], [c[3], c[4], c[5]]])
        uc = R @ (w.mean[0].astype(float) - np.array(cam["t"]))
        if uc[2] <= 0.01:
            continue
        Sc = R @ Mw @ Mw.T @ R.T
        x, y, z = uc
        Js = np.array([[cam["fx"] / z, 0, -cam["fx"] * x / z ** 2],
                       [0, cam["fy"] / z, -cam["fy"] * y / z ** 2]])
        S = Js @ Sc @ Js.T
        mu = np.array([cam["fx"] * x / z + cam["cx"], cam["fy"] * y / z + cam["cy"]])
        for k in range(4):
            dv = np.array([px[k] + 0.5, py[k] + 0.5]) - mu
            a = float(w.opacity[0]) * math.exp(-0.5 * dv @ np.linalg.solve(S, dv))
            worst = max(worst, abs(pc[k, 0] - a))
    assert worst <= 1e-12, worst


def test_colour_box_closed_form(oracle):
    """Colour intervals only (zero-width pose and shift): pc is linear in c with weights
    T a >= 0 (Alg. 3 l.3), so lo = render(c_lo), hi = render(c_hi) exactly."""
    w = small("C5")
    w.pose_box["eps_t"] = [0.0, 0.0, 0.0]
    w.scene_box["shift_hi"] = np.array(w.scene_box["shift_lo"], float)
    lo, hi, st = oracle.render_bounds(w)
    assert st["n_vars"] == 0
    r_lo = oracle.render_concrete(w, color=w.scene_box["col_lo"], shifts=np.zeros(1))
    r_hi = oracle.render_concrete(w, color=w.scene_box["col_hi"], shifts=np.zeros(1))
    slack = w.N * TAU + 1e-12
    assert np.abs(lo - r_lo).max() <= slack and np.abs(hi - r_hi).max() <= slack
    assert (hi - lo).max() > 0.1  # the red interval is visible


def test_opacity_box_single_gaussian_closed_form(oracle):
    """Opacity intervals only (zero-width pose), one Gaussian: pc = a c with a = o e^{-s/2}
    linear in o (Alg. 1 l.10), so lo = render(o_lo) and hi = render(o_hi) exactly."""
    from workloads import opacity_variant
    w = zero_box(make_config("C1", N=1, res=16))
    v = opacity_variant(w, np.ones(1, bool), scale=0.6, delta=0.3)
    lo, hi, st = oracle.render_bounds(v)
    assert st["n_vars"] == 0
    r_lo = oracle.render_concrete(v, opacity=v.scene_box["op_lo"])
    r_hi = oracle.render_concrete(v, opacity=v.scene_box["op_hi"])
    slack = v.N * TAU + 1e-12
    assert np.abs(lo - r_lo).max() <= slack and np.abs(hi - r_hi).max() <= slack
    assert (hi - lo).max() > 0.05


def test_opacity_box_contains_sampled_scenes(oracle):
    """The paper's opacity experiment (§4.6: opacities scaled by 0.1, +0.1 box) on the
    C5 blade group together with its pose, shift and colour boxes: Theorem 1 containment at
    sampled (pose, shift, colour, opacity) points, and looser than without the opacity box."""
    from workloads import opacity_variant
    w = small("C5")
    v = opacity_variant(w, w.scene_box["group_of"] >= 0)
    lo, hi, st = oracle.render_bounds(v)
    assert np.all(lo <= hi) and lo.min() >= 0 and hi.max() <= 1
    rng = np.random.default_rng(11)
    worst = 0.0
    sb = v.scene_box
    for p in H.sample_params(v, rng, n_random=30, corners=True):
        e, t, shifts = H.pose_of(v, p)
        a = rng.uniform(size=(v.N, 1))
        col = (sb["col_lo"] + a * (sb["col_hi"] - sb["col_lo"])).astype(np.float32)
        b = rng.uniform(size=v.N)
        op = (sb["op_lo"] + b * (sb["op_hi"] - sb["op_lo"])).astype(np.float32)
        img = oracle.render_concrete(v, euler=e, t=t, shifts=shifts, color=col, opacity=op)
        worst = max(worst, (lo - img).max(), (img - hi).max())
    assert worst <= 1e-9, worst
    # the same scene with the opacities fixed at their nominal (scaled) values is tighter
    fixed = copy.deepcopy(v)
    fixed.scene_box = dict(v.scene_box, op_lo=None, op_hi=None)
    flo, fhi, _ = oracle.render_bounds(fixed)
    assert H.mpg(lo, hi) > H.mpg(flo, fhi)
    assert np.all(lo <= flo + 1e-12) and np.all(hi >= fhi - 1e-12)


def test_partitioning_tightens(oracle):
    """Trend: partitioning C tightens the union of bounds."""
    w = small("C3", N=1500, res=24)
    w.pose_box["parts"] = [1, 1, 1, 1, 1, 1]
    lo1, hi1, _ = oracle.render_bounds(w)
    w.pose_box["parts"] = [1, 1, 1, 1, 1, 4]
    lo4, hi4, st = oracle.render_bounds(w)
    assert st["n_sub"] == 4
    assert H.mpg(lo4, hi4) < H.mpg(lo1, hi1)


# ------------------------------------------------------------------ edge cases
def test_edge_cases(oracle):
    from workloads.synth import Workload
    w = make_config("C1")
    empty = Workload("empty", w.mean[:0], w.chol[:0], w.opacity[:0], w.color[:0], w.camera,
                     w.pose_box, None)
    lo, hi, st = oracle.render_bounds(empty)
    assert np.all(lo == 0) and np.all(hi == 0) and st["pairs"] == 0
    behind = copy.deepcopy(w)
    behind.mean = behind.mean.copy()
    behind.mean[:, 2] = -behind.mean[:, 2]
    lo, hi, st = oracle.render_bounds(behind)
    assert np.all(hi <= 16 * TAU) and st["dropped"] == 16
    with pytest.raises(ValueError):
        bad = copy.deepcopy(w)
        bad.pose_box["parts"] = [1, 2, 1, 1, 1, 1]  # partitions on an unperturbed axis
        oracle.render_bounds(bad)


def test_spiky_gaussians_fail_soundly(oracle):
    """Near-singular covariances make MatrixInv's contraction fail under a
    rotation box; the fallback a in [0, o_hi] keeps the bounds sound."""
    w = make_config("C1", N=24)
    rng = np.random.default_rng(2)
    ch = w.chol.copy()
    ch[:, 2] *= 1e-3  # squash the y axis of the factor -> thin Gaussians
    ch[:, 4] *= 1e-3
    ch[:, 5] *= 1e-3
    w.chol = ch
    w.pose_box["eps_R"] = [0.0, 0.0, math.radians(3.0)]
    lo, hi, st = oracle.render_bounds(w)
    assert st["fails"] > 0
    for p in H.sample_params(w, rng, n_random=60):
        e, t, sh = H.pose_of(w, p)
        img = oracle.render_concrete(w, euler=e, t=t)
        assert np.all(lo <= img + 1e-9) and np.all(img <= hi + 1e-9)


def test_subbox_ranges_compose_to_the_union(oracle):
    """Step 22: the abstract image is the elementwise min / max union over sub-boxes,
    so renders of disjoint sub-box ranges combine exactly into the full render (sub-box
    sharding, §8(e)); an empty range is the union's identity (lo = 1, hi = 0); and a
    one-sub-box range equals the render of a box built directly as that sub-box (G18: uniform
    split, yaw part m of P covers [lo + 2 eps m / P, lo + 2 eps (m + 1) / P])."""
    w = make_config("C3", N=500, res=32)
    P = w.n_sub
    assert P == 8
    flo, fhi, fst = oracle.render_bounds(w)
    lo_a, hi_a, st_a = oracle.render_subboxes(w, 0, 3)
    lo_b, hi_b, st_b = oracle.render_subboxes(w, 3, P)
    assert st_a["n_sub"] == 3 and st_b["n_sub"] == P - 3
    assert np.array_equal(np.minimum(lo_a, lo_b), flo)
    assert np.array_equal(np.maximum(hi_a, hi_b), fhi)
    assert st_a["pairs"] + st_b["pairs"] == fst["pairs"]
    lo_e, hi_e, st_e = oracle.render_subboxes(w, 5, 5)
    assert np.all(lo_e == 1.0) and np.all(hi_e == 0.0) and st_e["pairs"] == 0
    m = 5
    one = copy.deepcopy(w)
    pb = copy.deepcopy(w.pose_box)
    eps = pb["eps_R"][2]
    lo_yaw = pb["R_off"][2] - eps
    pb["R_off"][2] = lo_yaw + 2 * eps * (2 * m + 1) / (2 * P)
    pb["eps_R"][2] = eps / P
    pb["parts"] = [1, 1, 1, 1, 1, 1]
    one.pose_box = pb
    s_lo, s_hi, _ = oracle.render_subboxes(w, m, m + 1)
    d_lo, d_hi, _ = oracle.render_bounds(one)
    assert max(np.abs(s_lo - d_lo).max(), np.abs(s_hi - d_hi).max()) <= 1e-12
    with pytest.raises(ValueError):
        oracle.render_subboxes(w, 0, P + 1)


def _uniform_as_explicit(w):
    """The uniform yaw partition of w written as an explicit sub-box list [P][9][2]."""
    pb = w.pose_box
    lo = [pb["t_off"][a] - pb["eps_t"][a] for a in range(3)] + \
         [pb["R_off"][a] - pb["eps_R"][a] for a in range(3)] + [0.0, 0.0, 0.0]
    hi = [pb["t_off"][a] + pb["eps_t"][a] for a in range(3)] + \
         [pb["R_off"][a] + pb["eps_R"][a] for a in range(3)] + [0.0, 0.0, 0.0]
    P = pb["parts"][5]
    out = np.zeros((P, 9, 2))
    for m in range(P):
        for a in range(9):
            out[m, a] = (lo[a], hi[a])
        wd = hi[5] - lo[5]
        out[m, 5] = (lo[5] + wd * m / P, lo[5] + wd * (m + 1) / P)
    return out


def test_explicit_partition_equals_uniform(oracle):
    """NEXT-3 (P:470 (2)): an explicit sub-box list describing the uniform partition
    renders the same union (up to the rounding of the sub-box centres), and a list with one
    box equal to the whole box renders the unpartitioned image."""
    w = make_config("C3", N=400, res=24)
    ulo, uhi, ust = oracle.render_bounds(w)
    e = copy.deepcopy(w)
    e.pose_box = dict(w.pose_box, parts=[1, 1, 1, 1, 1, 1], subboxes=_uniform_as_explicit(w))
    elo, ehi, est = oracle.render_bounds(e)
    assert est["n_sub"] == ust["n_sub"] == 8 and est["pairs"] == ust["pairs"]
    assert max(np.abs(elo - ulo).max(), np.abs(ehi - uhi).max()) <= 1e-12
    one = copy.deepcopy(w)
    one.pose_box = dict(w.pose_box, parts=[1, 1, 1, 1, 1, 1])
    olo, ohi, _ = oracle.render_bounds(one)
    whole = _uniform_as_explicit(w)[:1].copy()
    whole[0, 5] = (w.pose_box["R_off"][2] - w.pose_box["eps_R"][2],
                   w.pose_box["R_off"][2] + w.pose_box["eps_R"][2])
    one.pose_box = dict(one.pose_box, subboxes=whole)
    xlo, xhi, _ = oracle.render_bounds(one)
    assert max(np.abs(xlo - olo).max(), np.abs(xhi - ohi).max()) <= 1e-12
    bad = copy.deepcopy(one)
    wb = whole.copy()
    wb[0, 5, 1] += 0.1  # beyond the box
    bad.pose_box = dict(one.pose_box, subboxes=wb)
    with pytest.raises(ValueError):
        oracle.render_bounds(bad)
