"""Test-side helpers: pose sampling inside a box and plain numpy versions of the concrete
Alg. 1 intermediates, used to pin the oracle's abstract forms at sampled
poses.  Independent of oracle/ and of the CUDA package."""
import itertools
import math

import numpy as np


def rot_c2w(e):
    """Rz(e2) Ry(e1) Rx(e0) (XYZ Euler)."""
    c0, s0 = math.cos(e[0]), math.sin(e[0])
    c1, s1 = math.cos(e[1]), math.sin(e[1])
    c2, s2 = math.cos(e[2]), math.sin(e[2])
    Rx = np.array([[1, 0, 0], [0, c0, -s0], [0, s0, c0]])
    Ry = np.array([[c1, 0, s1], [0, 1, 0], [-s1, 0, c1]])
    Rz = np.array([[c2, -s2, 0], [s2, c2, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def box_axes(w):
    """The 9 (lo, hi) parameter ranges: t offsets, Euler offsets, group shifts."""
    b = w.pose_box
    ax = []
    for a in range(3):
        ax.append((b["t_off"][a] - b["eps_t"][a], b["t_off"][a] + b["eps_t"][a]))
    for a in range(3):
        ax.append((b["R_off"][a] - b["eps_R"][a], b["R_off"][a] + b["eps_R"][a]))
    sb = w.scene_box
    for g in range(3):
        if sb is not None and g < sb["n_groups"]:
            ax.append((float(sb["shift_lo"][g]), float(sb["shift_hi"][g])))
        else:
            ax.append((0.0, 0.0))
    return ax


def sample_params(w, rng, n_random=40, corners=True):
    """Parameter vectors (9,) inside the full box: all 2^n corners, centre, randoms."""
    ax = box_axes(w)
    var = [k for k in range(9) if ax[k][1] > ax[k][0]]
    out = []
    centre = np.array([(lo + hi) / 2 for lo, hi in ax])
    out.append(centre)
    if corners and len(var) <= 8:
        for signs in itertools.product((0, 1), repeat=len(var)):
            p = centre.copy()
            for k, s in zip(var, signs):
                p[k] = ax[k][s]
            out.append(p)
    for _ in range(n_random):
        p = centre.copy()
        for k in var:
            p[k] = rng.uniform(ax[k][0], ax[k][1])
        out.append(p)
    return out


def pose_of(w, p):
    """Camera (euler, t) and group shifts for parameter vector p (step 0-1 semantics)."""
    cam = w.camera
    e = [cam["euler"][k] + p[3 + k] for k in range(3)]
    off = np.array(p[:3])
    if w.pose_box["t_frame"] == 1:
        t = np.array(cam["t"]) + rot_c2w(cam["euler"]) @ off
    else:
        t = np.array(cam["t"]) + off
    ng = w.scene_box["n_groups"] if w.scene_box is not None else 0
    shifts = np.array(p[6:6 + ng], float)
    return e, t, shifts


def concrete_intermediates(w, e, t, shifts, idx):
    """uc, d, up, Mp, X, Conic, W = Conic Mp, D2, DU for Gaussian idx (Alg. 1 l.2-9)."""
    cam = w.camera
    R = rot_c2w(e).T
    uw = w.mean[idx].astype(np.float64).copy()
    if w.scene_box is not None and w.scene_box["n_groups"] > 0:
        g = w.scene_box["group_of"][idx]
        if g >= 0:
            uw = uw + shifts[g] * np.asarray(w.scene_box["dir"][g], float)
    c = w.chol[idx].astype(np.float64)
    Mw = np.array([[c[0], 0, 0], [c[1], c[2], 0], [c[3], c[4], c[5]]])
    uc = R @ (uw - t)
    Mc = R @ Mw
    fx, fy, cx, cy = cam["fx"], cam["fy"], cam["cx"], cam["cy"]
    J = np.array([[fx * uc[2], 0, -fx * uc[0]], [0, fy * uc[2], -fy * uc[1]]])
    up = np.array([fx * uc[0] + cx * uc[2], fy * uc[1] + cy * uc[2]])
    Mp = J @ Mc
    X = Mp @ Mp.T
    conic = np.linalg.inv(X)
    W = conic @ Mp
    d = uc[2]
    return dict(uc=uc, d=d, up=up, Mp=Mp, X=X, conic=conic, W=W, D2=d * d, DU=d * up)


def xi_of(w, p, sub_centres=None):
    """xi in [-1,1]^n of parameter vector p for a single-sub-box problem."""
    ax = box_axes(w)
    xi = []
    for k in range(9):
        lo, hi = ax[k]
        if hi > lo:
            xi.append((p[k] - (lo + hi) / 2) / ((hi - lo) / 2))
    return np.array(xi)


def eval_form(f, n, xi):
    return f[:n] @ xi + f[n], f[n + 1:2 * n + 1] @ xi + f[2 * n + 1]


def mpg(lo, hi):
    """Mean Pixel Gap."""
    return float(np.linalg.norm(hi - lo, axis=-1).mean())
