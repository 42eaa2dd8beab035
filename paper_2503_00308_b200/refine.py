"""Adaptive refinement of the input box (PAPER.md:470 (2): "iteratively
divide the input range until the assertion at Line 2 [rho < 1] is satisfied").

MatrixInv (Alg. 4) fails for a Gaussian when its covariance relaxation is too wide (det <= 0 or
rho >= 1); the Gaussian then only contributes a in [0, o_hi] (reading G11).  Failures are a
property of the sub-box, so the host bisects every sub-box that has failing Gaussians, along
its widest axis relative to the full box, until no sub-box fails or the sub-box budget is
spent.  Counting failures needs only the per-Gaussian setup (`as_subbox_fails`), not a render;
the final partition is installed with `as_set_subboxes` and rendered as usual (the union over
sub-boxes).

Host logic only: every number of the method is computed by the library.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def box_bounds(pose_box: dict, scene_box) -> np.ndarray:
    """(lo, hi) of the 9 box axes [9, 2]: t offsets, Euler offsets, group shifts 0..2."""
    b = np.zeros((9, 2))
    for a in range(3):
        b[a] = (pose_box["t_off"][a] - pose_box["eps_t"][a], pose_box["t_off"][a] + pose_box["eps_t"][a])
        b[3 + a] = (pose_box["R_off"][a] - pose_box["eps_R"][a],
                    pose_box["R_off"][a] + pose_box["eps_R"][a])
    ng = int(scene_box["n_groups"]) if scene_box is not None else 0
    for g in range(ng):
        b[6 + g] = (float(scene_box["shift_lo"][g]), float(scene_box["shift_hi"][g]))
    return b


def uniform_partition(pose_box: dict, scene_box) -> np.ndarray:
    """The uniform grid of `parts` as an explicit list [P, 9, 2], in the library's sub-box order
    (multi-index over the axes, axis 0 fastest)."""
    full = box_bounds(pose_box, scene_box)
    parts = list(pose_box["parts"]) + (list(scene_box.get("parts", [1, 1, 1]))
                                       if scene_box is not None else [1, 1, 1])
    parts = [int(p) for p in parts[:9]]
    P = int(np.prod(parts))
    out = np.zeros((P, 9, 2))
    for s in range(P):
        rem = s
        for a in range(9):
            m = rem % parts[a]
            rem //= parts[a]
            lo, hi = full[a]
            w = hi - lo
            out[s, a] = (lo + w * m / parts[a], lo + w * (m + 1) / parts[a]) if w > 0 else (lo, hi)
    return out


def bisect(box: np.ndarray, full: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Split a sub-box [9, 2] in half along its widest axis relative to the full box (lowest
    axis on ties), among the Euler axes when the box perturbs any: only the rotation changes
    the projected covariance X = Mp Mp^T enough to break MatrixInv's contraction (translation
    enters through J only), so splitting translations or group shifts does not remove
    failures."""
    rel = np.full(9, -1.0)
    for a in range(9):
        fw = full[a, 1] - full[a, 0]
        if fw > 0:
            rel[a] = (box[a, 1] - box[a, 0]) / fw
    if np.any(rel[3:6] > 0):
        rel[:3] = -1.0
        rel[6:] = -1.0
    a = int(np.argmax(rel))
    mid = 0.5 * (box[a, 0] + box[a, 1])
    lo, hi = box.copy(), box.copy()
    lo[a, 1] = mid
    hi[a, 0] = mid
    return lo, hi


def refine_fails(ctx, pose_box: dict, scene_box, max_subboxes: int = 64,
                 max_rounds: int = 8) -> Tuple[np.ndarray, List[np.ndarray]]:
    """Bisect failing sub-boxes (in order, while the budget allows) until none fails.

    ctx: a Context (or anything with as_set_subboxes / as_subbox_fails) holding the scene,
    camera and box.  Returns the final partition [P, 9, 2] (installed in ctx) and the FAIL
    counts per sub-box of every round."""
    full = box_bounds(pose_box, scene_box)
    parts = uniform_partition(pose_box, scene_box)
    history = []
    for _ in range(max_rounds):
        ctx.as_set_subboxes(parts)
        fails = np.asarray(ctx.as_subbox_fails())
        history.append(fails)
        if not np.any(fails > 0):
            break
        new = []
        for i, b in enumerate(parts):
            remaining = len(parts) - i - 1
            if fails[i] > 0 and len(new) + 2 + remaining <= max_subboxes:
                new.extend(bisect(b, full))
            else:
                new.append(b)
        if len(new) == len(parts):  # budget spent
            break
        parts = np.asarray(new)
    ctx.as_set_subboxes(parts)
    return parts, history


def bisect_widest(box: np.ndarray, full: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Split a sub-box [9, 2] in half along its widest axis relative to the full box (lowest
    axis on ties), any axis: the width-driven rule (every perturbed axis widens the bound)."""
    rel = np.full(9, -1.0)
    for a in range(9):
        fw = full[a, 1] - full[a, 0]
        if fw > 0:
            rel[a] = (box[a, 1] - box[a, 0]) / fw
    a = int(np.argmax(rel))
    mid = 0.5 * (box[a, 0] + box[a, 1])
    lo, hi = box.copy(), box.copy()
    lo[a, 1] = mid
    hi[a, 0] = mid
    return lo, hi


def _mpg(lo, hi) -> float:
    """Mean Pixel Gap of bound images (torch or numpy [H, W, 3])."""
    if hasattr(lo, "cpu"):
        import torch
        return float(torch.linalg.vector_norm(hi - lo, dim=-1).mean())
    return float(np.linalg.norm(np.asarray(hi) - np.asarray(lo), axis=-1).mean())


def _union(images):
    lo = images[0][0]
    hi = images[0][1]
    if hasattr(lo, "cpu"):
        import torch
        for l, h in images[1:]:
            lo = torch.minimum(lo, l)
            hi = torch.maximum(hi, h)
        return lo, hi
    for l, h in images[1:]:
        lo = np.minimum(lo, l)
        hi = np.maximum(hi, h)
    return lo, hi


def refine_width(ctx, pose_box: dict, scene_box, tile: int = 16, batch: int = 64,
                 max_subboxes: int = 16):
    """Width-driven refinement ("split sub-boxes where ... width is
    large"; partitions are the paper's main tightness lever): starting from the
    box's uniform partition, repeatedly bisect the sub-box whose own bound image has the largest
    Mean Pixel Gap, along its widest relative axis, until `max_subboxes`.  Each sub-box is
    rendered once (its two halves when it is split) through as_set_subboxes +
    as_render_subboxes(s, s + 1); the union (step 22) is the elementwise min / max of the kept
    images.

    Returns (partition [P, 9, 2] installed in ctx, history): history[i] = (number of
    sub-boxes, MPG of the union, sum of the sub-box render times in ms)."""
    full = box_bounds(pose_box, scene_box)
    parts = [b for b in uniform_partition(pose_box, scene_box)]
    imgs, mpgs, ms = [], [], []

    def render_one(box):
        ctx.as_set_subboxes(np.asarray([box]))
        lo, hi, st = ctx.as_render_subboxes(0, 1, tile, batch)
        return lo, hi, _mpg(lo, hi), (st["ms_total"] if st else 0.0)

    for b in parts:
        lo, hi, m, t = render_one(b)
        imgs.append((lo, hi))
        mpgs.append(m)
        ms.append(t)
    history = [(len(parts), _mpg(*_union(imgs)), float(sum(ms)))]
    while len(parts) < max_subboxes:
        i = int(np.argmax(mpgs))
        a, b = bisect_widest(parts[i], full)
        la, ha, ma, ta = render_one(a)
        lb, hb, mb, tb = render_one(b)
        parts[i:i + 1] = [a, b]
        imgs[i:i + 1] = [(la, ha), (lb, hb)]
        mpgs[i:i + 1] = [ma, mb]
        ms[i:i + 1] = [ta, tb]
        history.append((len(parts), _mpg(*_union(imgs)), float(sum(ms))))
    out = np.asarray(parts)
    ctx.as_set_subboxes(out)
    return out, history
