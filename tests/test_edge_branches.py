"""Oracle pins for the method branches no C1-C5 workload reaches:

* the near plane (reading G8, d_min = 0.01): Gaussians whose depth interval over the box
  contains d_min ('straddle': a_lo = 0, footprint from max(d_lo, d_min), reading O4) and
  Gaussians dropped at d_hi <= d_min;
* exact depth ties (reading G6 / H4): duplicated Gaussians with identical depth forms, whose
  order is decided by the scene-index tie-break (translation boxes: certain pairs) or is
  uncertain (rotation boxes).

Pins are independent of oracle/: a textbook numpy 3DGS renderer (tests/helpers.py, EWA
projection rather than the paper's d^4 form) at zero width and at sampled poses (Theorem 1,
P:564-567), and closed forms (a lone straddling Gaussian has lo = 0 everywhere)."""
import copy

import numpy as np
import pytest

from tests import helpers as H
from workloads import nearplane_config, stacked_config, ties_config


def _containment(oracle, w, lo, hi, n_random=40, seed=0):
    rng = np.random.default_rng(seed)
    worst = 0.0
    for p in H.sample_params(w, rng, n_random=n_random):
        e, t, sh = H.pose_of(w, p)
        img = H.concrete_render_np(w, e, t, sh)
        worst = max(worst, float((lo - img).max()), float((img - hi).max()))
    return worst


@pytest.mark.parametrize("eps,rot", [(4e-4, 0.0), (1e-3, 0.0), (4e-4, 0.5)])
def test_nearplane_sound_and_straddles(oracle, eps, rot):
    w = nearplane_config(eps_tz=eps, rot_deg=rot)
    lo, hi, st = oracle.render_bounds(w)
    assert st["straddles"] > 0 and st["dropped"] > 0 and st["fails"] == 0
    assert np.all(lo <= hi) and lo.min() >= 0 and hi.max() <= 1
    assert _containment(oracle, w, lo, hi) <= 1e-9


def test_nearplane_zero_width_is_concrete(oracle):
    """A zero-width box has no straddles: every Gaussian is either dropped (d <= d_min, as the
    concrete renderer culls it) or ordinary, and lo = hi = the textbook render (+- N tau)."""
    w = nearplane_config(eps_tz=0.0)
    lo, hi, st = oracle.render_bounds(w)
    assert st["straddles"] == 0 and st["dropped"] > 0
    ref = H.concrete_render_np(w, w.camera["euler"], w.camera["t"])
    assert np.abs(lo - ref).max() <= 1e-9 and np.abs(hi - ref).max() <= 1e-9


def test_lone_straddling_gaussian_has_zero_lower_bound(oracle):
    """One Gaussian whose depth interval contains d_min: a_lo = 0 (G8) at every pixel, so the
    lower image is exactly 0 (after the -N tau and the clamp), while hi still covers the
    concrete renders at every sampled pose in front of the near plane."""
    w = nearplane_config(eps_tz=1e-3)
    eps = w.pose_box["eps_t"][2]
    z = w.mean[:, 2].astype(np.float64)  # identity camera: d = z - t_z, t_z in [-eps, eps]
    cand = [i for i in range(w.N) if z[i] - eps <= H.D_MIN < z[i] + eps]
    assert cand, "no straddling Gaussian"
    i = cand[0]
    v = copy.deepcopy(w)
    for f in ("mean", "chol", "opacity", "color"):
        setattr(v, f, getattr(w, f)[i:i + 1].copy())
    lo, hi, st = oracle.render_bounds(v)
    assert st["straddles"] == 1
    assert np.all(lo == 0.0) and hi.max() > 0.05
    assert _containment(oracle, v, lo, hi, n_random=100) <= 1e-9


def test_ties_translation_box_tiebreak(oracle):
    """Duplicated Gaussians under a translation-only box: d_i - d_j is exactly 0, so every
    duplicate pair is *certain* and ordered by the scene index (G6): no uncertain pairs, the
    zero-width render is the textbook BlendSort with ascending-index ties, which differs from
    the strict-Ind blend (tied Gaussians not occluding each other), and the box render
    contains the concrete renders."""
    w = ties_config()
    z = copy.deepcopy(w)
    z.pose_box = dict(z.pose_box, eps_t=[0.0, 0.0, 0.0])
    lo, hi, st = oracle.render_bounds(z)
    ref = H.concrete_render_np(z, z.camera["euler"], z.camera["t"])
    strict = H.concrete_render_np(z, z.camera["euler"], z.camera["t"], tiebreak=False)
    assert np.abs(lo - ref).max() <= 1e-9 and np.abs(hi - ref).max() <= 1e-9
    assert np.abs(strict - ref).max() > 1e-3  # the tie-break decides the image
    lo, hi, st = oracle.render_bounds(w)
    assert st["uncertain_pairs"] == 0 and st["order_violations"] == 0
    assert _containment(oracle, w, lo, hi) <= 1e-9


def test_ties_rotation_box_uncertain(oracle):
    """Under a yaw box the duplicates' identical depth forms have nonzero width: each duplicate
    pair is '?' (Ind relaxation, Table 2), the exception machinery handles them,
    and the bounds contain the concrete renders (which order ties by index)."""
    w = ties_config(rot_deg=1.0)
    lo, hi, st = oracle.render_bounds(w)
    assert st["uncertain_pairs"] > 0 and st["order_violations"] == 0
    assert _containment(oracle, w, lo, hi) <= 1e-9
    # the windowed blend (mode 0) equals the direct Alg. 3 evaluation (mode 1) on ties
    dlo, dhi, _ = oracle.render_bounds(w, mode=1)
    assert np.abs(lo - dlo).max() <= 1e-12 and np.abs(hi - dhi).max() <= 1e-12


@pytest.mark.parametrize("kw", [dict(N=150, rot_deg=2.0), dict(N=300, rot_deg=0.7, axis_frac=0.5)])
def test_stacked_long_windows(oracle, kw):
    """Near-opaque slab under a rotation box: exception windows past 128 positions, windows
    mixing certain and uncertain partners, transmittance far below 1e-25.  The windowed
    blend (prefix products + exception windows, step 13's order structure) equals the direct
    Alg. 3 evaluation, and the bounds contain the textbook renders."""
    w = stacked_config(**kw)
    lo, hi, st = oracle.render_bounds(w)
    dlo, dhi, _ = oracle.render_bounds(w, mode=1)
    assert st["uncertain_pairs"] > 1000 and st["order_violations"] == 0
    assert np.abs(lo - dlo).max() <= 1e-12 and np.abs(hi - dhi).max() <= 1e-12
    assert _containment(oracle, w, lo, hi, n_random=20) <= 1e-9
