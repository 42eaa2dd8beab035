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


D_MIN = 0.01  # near plane (reading G8)


def concrete_render_np(w, e, t, shifts=None, tiebreak=True):
    """Textbook 3DGS render at one pose in plain numpy fp64, independent of oracle/:
    mu = K uc / d, Sigma_2D = Jc Sigma_c Jc^T with the EWA Jacobian Jc of the perspective map,
    a = o exp(-1/2 (u - mu)^T Sigma_2D^-1 (u - mu)) at pixel centres u = index + 1/2 (G7),
    Gaussians with d <= d_min culled (G8), front-to-back alpha blending in ascending depth
    with ascending scene index on exact ties (Alg. 2 BlendSort; tie-break G6), black
    background, no heuristics.  tiebreak=False blends equal depths with the
    paper's strict Ind instead: tied Gaussians do not occlude each other."""
    cam = w.camera
    R = rot_c2w(e).T
    uw = w.mean.astype(np.float64).copy()
    if shifts is not None and w.scene_box is not None and w.scene_box["n_groups"] > 0:
        g = w.scene_box["group_of"]
        for k in range(w.scene_box["n_groups"]):
            uw[g == k] += shifts[k] * np.asarray(w.scene_box["dir"][k], float)
    uc = (uw - np.asarray(t, float)) @ R.T
    d = uc[:, 2]
    keep = d > D_MIN
    c = w.chol.astype(np.float64)
    n = len(c)
    Mw = np.zeros((n, 3, 3))
    Mw[:, 0, 0], Mw[:, 1, 0], Mw[:, 1, 1] = c[:, 0], c[:, 1], c[:, 2]
    Mw[:, 2, 0], Mw[:, 2, 1], Mw[:, 2, 2] = c[:, 3], c[:, 4], c[:, 5]
    Sw = Mw @ np.transpose(Mw, (0, 2, 1))
    Sc = R[None] @ Sw @ R.T[None]
    fx, fy, cx, cy = cam["fx"], cam["fy"], cam["cx"], cam["cy"]
    ds = np.where(keep, d, 1.0)
    Jc = np.zeros((n, 2, 3))
    Jc[:, 0, 0] = fx / ds
    Jc[:, 0, 2] = -fx * uc[:, 0] / ds ** 2
    Jc[:, 1, 1] = fy / ds
    Jc[:, 1, 2] = -fy * uc[:, 1] / ds ** 2
    S2 = Jc @ Sc @ np.transpose(Jc, (0, 2, 1))
    mu = np.stack([fx * uc[:, 0] / ds + cx, fy * uc[:, 1] / ds + cy], axis=1)
    Si = np.linalg.inv(S2)
    H, W = cam["H"], cam["W"]
    ys, xs = np.mgrid[0:H, 0:W]
    u = np.stack([xs + 0.5, ys + 0.5], axis=-1).reshape(-1, 2)
    img = np.zeros((H * W, 3))
    T = np.ones(H * W)
    order = np.lexsort((np.arange(n), d))  # ascending depth, then index
    ids = [i for i in order if keep[i]]
    k = 0
    while k < len(ids):
        grp = [ids[k]]
        while (not tiebreak and k + len(grp) < len(ids) and d[ids[k + len(grp)]] == d[ids[k]]):
            grp.append(ids[k + len(grp)])
        alphas = []
        for i in grp:
            r = u - mu[i]
            s = np.einsum("pa,ab,pb->p", r, Si[i], r)
            alphas.append(w.opacity[i] * np.exp(-0.5 * s))
        for i, a in zip(grp, alphas):
            img += (T * a)[:, None] * w.color[i].astype(np.float64)[None]
        for a in alphas:
            T = T * (1.0 - a)
        k += len(grp)
    return img.reshape(H, W, 3)
