"""Synthetic, deterministic workloads C1-C5 (BASELINE.json configs).

Distributions mimic the paper's workload classes (P = /root/reference/PAPER.md):
  * a single object on an empty background (BullDozer, Fig. 1) -> C2, C5;
  * outdoor / large scenes (PineTree/OSM/Airport/Garden/Stump) -> C3, C4;
  * a tiny random scene the oracle finishes in milliseconds -> C1.
Gaussians are <uw, Mw, o, c> with Mw the lower Cholesky factor of Cov, stored
as float32 SoA arrays: mean [N,3], chol [N,6] (m00 m10 m11 m20 m21 m22), opacity [N],
color [N,3].  Cameras use XYZ Euler angles of camera->world, R_c2w = Rz Ry Rx,
camera looking along +z_cam, x right, y down.  Nothing here evaluates the method.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

CONFIGS = ("C1", "C2", "C3", "C4", "C5")


@dataclasses.dataclass
class Workload:
    name: str
    mean: np.ndarray      # [N,3] float32
    chol: np.ndarray      # [N,6] float32
    opacity: np.ndarray   # [N] float32
    color: np.ndarray     # [N,3] float32
    camera: dict          # fx, fy, cx, cy, W, H, euler[3], t[3]
    pose_box: dict        # eps_t[3], eps_R[3], t_off[3], R_off[3], t_frame, parts[6]
    scene_box: Optional[dict]  # group_of, dir, shift_lo, shift_hi, parts, col_lo/hi, op_lo/hi
    tile: int = 16
    batch: int = 64
    description: str = ""

    @property
    def N(self) -> int:
        return int(self.mean.shape[0])

    @property
    def n_sub(self) -> int:
        p = 1
        for a in range(6):
            p *= int(self.pose_box["parts"][a])
        if self.scene_box is not None:
            for g in range(int(self.scene_box["n_groups"])):
                p *= int(self.scene_box["parts"][g])
        return p


# ----------------------------------------------------------------------------- helpers
def look_at_euler(eye, target, up=(0.0, 0.0, 1.0)):
    """XYZ Euler angles (e0,e1,e2) with Rz(e2) Ry(e1) Rx(e0) = [x_cam y_cam z_cam] (columns),
    z_cam = viewing direction, x_cam = right, y_cam = down (image rows grow downwards)."""
    eye = np.asarray(eye, np.float64)
    z = np.asarray(target, np.float64) - eye
    z /= np.linalg.norm(z)
    x = np.cross(z, np.asarray(up, np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z], axis=1)
    e1 = -math.asin(max(-1.0, min(1.0, R[2, 0])))
    e0 = math.atan2(R[2, 1], R[2, 2])
    e2 = math.atan2(R[1, 0], R[0, 0])
    return [e0, e1, e2]


def _random_rotations(rng, n):
    """Uniform random rotation matrices via unit quaternions."""
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _frame_with_normal(rng, normals):
    """Rotations whose third column is the given unit normal, random in-plane angle."""
    n = normals.shape[0]
    a = np.where(np.abs(normals[:, :1]) < 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 1.0, 0]]))
    t1 = np.cross(normals, a)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(normals, t1)
    th = rng.uniform(0, 2 * math.pi, size=(n, 1))
    u = np.cos(th) * t1 + np.sin(th) * t2
    v = np.cross(normals, u)
    return np.stack([u, v, normals], axis=2)


def _chol_from(R, s):
    """Lower Cholesky factor of R diag(s^2) R^T, packed (m00 m10 m11 m20 m21 m22)."""
    cov = np.einsum("nij,nj,nkj->nik", R, s * s, R)
    L = np.linalg.cholesky(cov)
    return np.stack([L[:, 0, 0], L[:, 1, 0], L[:, 1, 1], L[:, 2, 0], L[:, 2, 1], L[:, 2, 2]],
                    axis=1)


def _loguniform(rng, lo, hi, size):
    return np.exp(rng.uniform(math.log(lo), math.log(hi), size=size))


def _camera(eye, target, fov_deg, W, H):
    f = (W / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return dict(fx=f, fy=f, cx=W / 2.0, cy=H / 2.0, W=int(W), H=int(H),
                euler=look_at_euler(eye, target), t=[float(v) for v in eye])


def _pose_box(eps_t=(0, 0, 0), eps_R=(0, 0, 0), t_off=(0, 0, 0), R_off=(0, 0, 0), t_frame=0,
              parts=(1, 1, 1, 1, 1, 1)):
    return dict(eps_t=[float(v) for v in eps_t], eps_R=[float(v) for v in eps_R],
                t_off=[float(v) for v in t_off], R_off=[float(v) for v in R_off],
                t_frame=int(t_frame), parts=[int(v) for v in parts])


def _pack(name, mean, chol, opacity, color, camera, pose_box, scene_box=None, tile=16,
          batch=16, description=""):
    return Workload(name=name,
                    mean=np.ascontiguousarray(mean, np.float32),
                    chol=np.ascontiguousarray(chol, np.float32),
                    opacity=np.ascontiguousarray(opacity, np.float32),
                    color=np.ascontiguousarray(np.clip(color, 0, 1), np.float32),
                    camera=camera, pose_box=pose_box, scene_box=scene_box, tile=tile,
                    batch=batch, description=description)


# ----------------------------------------------------------------------------- scenes
def random_scene(seed: int, N: int, depth=(4.0, 6.0), xy=1.0, scale=(0.05, 0.3),
                 opacity=(0.3, 0.99)):
    """C1-style: means U([-xy,xy]^2 x depth) in the camera frame of an identity pose."""
    rng = np.random.default_rng(seed)
    mean = np.stack([rng.uniform(-xy, xy, N), rng.uniform(-xy, xy, N),
                     rng.uniform(depth[0], depth[1], N)], axis=1)
    s = _loguniform(rng, scale[0], scale[1], (N, 3))
    chol = _chol_from(_random_rotations(rng, N), s)
    o = rng.uniform(opacity[0], opacity[1], N)
    c = rng.uniform(0, 1, (N, 3))
    return mean, chol, o, c


_BULLDOZER_PARTS = [
    # name, box min, box max, colour
    ("body", (-0.80, -0.60, 0.25), (0.90, 0.60, 0.80), (0.90, 0.72, 0.10)),
    ("cab", (-0.20, -0.50, 0.80), (0.60, 0.50, 1.25), (0.85, 0.68, 0.12)),
    ("blade", (-1.10, -0.80, 0.00), (-0.95, 0.80, 0.60), (0.55, 0.55, 0.55)),
    ("track_l", (-0.80, -0.80, 0.00), (1.20, -0.55, 0.30), (0.15, 0.15, 0.15)),
    ("track_r", (-0.80, 0.55, 0.00), (1.20, 0.80, 0.30), (0.15, 0.15, 0.15)),
]


def bulldozer_scene(seed: int, N: int):
    """C2: five surface-sampled boxes (body, cab, blade, two tracks) in about
    [-1.1,1.2] x [-0.8,0.8] x [0,1.25]; thin disks 4-30 mm, normal axis x0.2."""
    rng = np.random.default_rng(seed)
    faces = []  # (part index, origin, edge u, edge v, normal, area)
    for pi, (_, lo, hi, _) in enumerate(_BULLDOZER_PARTS):
        lo = np.array(lo, float)
        hi = np.array(hi, float)
        ext = hi - lo
        for ax in range(3):
            u_ax, v_ax = [a for a in range(3) if a != ax]
            for side in (0, 1):
                o = lo.copy()
                o[ax] = hi[ax] if side else lo[ax]
                eu = np.zeros(3)
                eu[u_ax] = ext[u_ax]
                ev = np.zeros(3)
                ev[v_ax] = ext[v_ax]
                nrm = np.zeros(3)
                nrm[ax] = 1.0 if side else -1.0
                faces.append((pi, o, eu, ev, nrm, ext[u_ax] * ext[v_ax]))
    area = np.array([f[5] for f in faces])
    fi = rng.choice(len(faces), size=N, p=area / area.sum())
    ab = rng.uniform(0, 1, (N, 2))
    orig = np.stack([faces[k][1] for k in fi])
    eu = np.stack([faces[k][2] for k in fi])
    ev = np.stack([faces[k][3] for k in fi])
    nrm = np.stack([faces[k][4] for k in fi])
    part = np.array([faces[k][0] for k in fi], np.int32)
    mean = orig + ab[:, :1] * eu + ab[:, 1:] * ev
    s12 = _loguniform(rng, 0.004, 0.030, (N, 2))
    s3 = 0.2 * np.sqrt(s12[:, 0] * s12[:, 1])
    s = np.concatenate([s12, s3[:, None]], axis=1)
    chol = _chol_from(_frame_with_normal(rng, nrm), s)
    base = np.array([p[3] for p in _BULLDOZER_PARTS])[part]
    color = base + rng.normal(0, 0.05, (N, 3))
    o = rng.uniform(0.5, 0.99, N)
    return mean, chol, o, color, part


def outdoor_scene(seed: int, N: int, n_trees: int = 60, extent: float = 30.0):
    """C3/C4: 60% ground-plane disks over a 30 x 30 m patch in front of the camera
    (scales 1-8 cm, flattened), 40% on 60 cone-shaped trees up to 4 m tall."""
    rng = np.random.default_rng(seed)
    n_ground = int(round(0.6 * N))
    n_tree = N - n_ground
    # ground patch x in [-15,15], y in [0,30]
    gx = rng.uniform(-extent / 2, extent / 2, n_ground)
    gy = rng.uniform(0.0, extent, n_ground)
    gz = rng.normal(0, 0.01, n_ground)
    g_mean = np.stack([gx, gy, gz], axis=1)
    gs12 = _loguniform(rng, 0.01, 0.08, (n_ground, 2))
    gs = np.concatenate([gs12, 0.2 * gs12.min(axis=1, keepdims=True)], axis=1)
    gn = np.tile(np.array([[0.0, 0.0, 1.0]]), (n_ground, 1))
    gn += rng.normal(0, 0.05, gn.shape)
    gn /= np.linalg.norm(gn, axis=1, keepdims=True)
    g_chol = _chol_from(_frame_with_normal(rng, gn), gs)
    g_col = np.array([0.36, 0.31, 0.20]) + rng.normal(0, 0.06, (n_ground, 3))
    g_col[rng.uniform(size=n_ground) < 0.5] = (np.array([0.22, 0.40, 0.15])
                                               + rng.normal(0, 0.05, (1, 3)))
    # trees
    tx = rng.uniform(-extent / 2 + 1, extent / 2 - 1, n_trees)
    ty = rng.uniform(2.0, extent - 1, n_trees)
    th = rng.uniform(2.0, 4.0, n_trees)
    tr = th * rng.uniform(0.2, 0.35, n_trees)
    which = rng.integers(0, n_trees, n_tree)
    hfrac = 1.0 - np.sqrt(rng.uniform(0, 1, n_tree))  # more mass near the base (cone area)
    ang = rng.uniform(0, 2 * math.pi, n_tree)
    rad = tr[which] * (1.0 - hfrac) * np.sqrt(rng.uniform(0.6, 1.0, n_tree))
    t_mean = np.stack([tx[which] + rad * np.cos(ang), ty[which] + rad * np.sin(ang),
                       0.3 + hfrac * th[which]], axis=1)
    ts = _loguniform(rng, 0.02, 0.10, (n_tree, 3))
    t_chol = _chol_from(_random_rotations(rng, n_tree), ts)
    t_col = np.array([0.10, 0.42, 0.14]) + rng.normal(0, 0.07, (n_tree, 3))
    mean = np.concatenate([g_mean, t_mean])
    chol = np.concatenate([g_chol, t_chol])
    color = np.concatenate([g_col, t_col])
    o = rng.uniform(0.4, 0.99, N)
    perm = rng.permutation(N)
    return mean[perm], chol[perm], o[perm], color[perm]


# ----------------------------------------------------------------------------- configs
def opacity_variant(w: Workload, member: np.ndarray, scale: float = 0.1,
                    delta: float = 0.1) -> Workload:
    """The paper's opacity experiment (§4.6): the member Gaussians' opacities are scaled
    by `scale` (capped at 1) and perturbed by +`delta`, i.e. o in [o', min(1, o' + delta)]
    with the nominal o' = min(1, scale * o).  Other scene-box entries of w are kept."""
    import copy
    v = copy.deepcopy(w)
    o = np.asarray(w.opacity, np.float32).copy()
    o[member] = np.minimum(np.float32(1.0), np.float32(scale) * o[member])
    hi = o.copy()
    hi[member] = np.minimum(np.float32(1.0), o[member] + np.float32(delta))
    v.opacity = o
    sb = dict(v.scene_box) if v.scene_box is not None else dict(
        n_groups=0, group_of=None, dir=None, shift_lo=None, shift_hi=None, parts=[1, 1, 1],
        col_lo=None, col_hi=None)
    sb["op_lo"] = o.copy()
    sb["op_hi"] = hi
    v.scene_box = sb
    v.name = w.name + "-opacity"
    return v


def make_config(name: str, N: Optional[int] = None, res: Optional[int] = None) -> Workload:
    """Build config C1..C5.  N / res override the Gaussian count and image edge (the
    focal length scales with res so the field of view is unchanged) for reduced-size
    parity cases; the defaults are the BASELINE.json configs."""
    name = name.upper()
    if name == "C1":
        n = 16 if N is None else N
        W = 16 if res is None else res
        mean, chol, o, c = random_scene(0, n)
        f = 16.0 * W / 16.0
        cam = dict(fx=f, fy=f, cx=W / 2.0, cy=W / 2.0, W=W, H=W, euler=[0.0, 0.0, 0.0],
                   t=[0.0, 0.0, 0.0])
        box = _pose_box(eps_t=(0.01, 0, 0))
        return _pack("C1", mean, chol, o, c, cam, box, tile=16, batch=16,
                     description="16 random Gaussians, 16x16, camera x-translation +-1 cm")
    if name in ("C2", "C5"):
        n = 100_000 if N is None else N
        W = 200 if res is None else res
        mean, chol, o, c, part = bulldozer_scene(2, n)
        cam = _camera((0.0, -4.0, 1.8), (0.0, 0.0, 0.5), 40.0, W, W)
        if name == "C2":
            # Fig. 1: "camera shifts horizontally by 10cm" -> camera-x in [0, +0.10] (G10)
            box = _pose_box(eps_t=(0.05, 0, 0), t_off=(0.05, 0, 0), t_frame=1)
            return _pack("C2", mean, chol, o, c, cam, box, tile=16, batch=24,
                         description="bulldozer-shaped ~100k, 200x200, 10 cm horizontal shift")
        # C5: scene-variation box: blade group moved along +y by [0, 0.05] m (one shared
        # variable), blade red channel [c_r, min(1, c_r + 0.5)], camera-x +-1 cm.
        blade = (part == 2)
        group_of = np.where(blade, 0, -1).astype(np.int32)
        cf = np.clip(c, 0, 1).astype(np.float32)
        col_lo = cf.copy()
        col_hi = cf.copy()
        col_hi[blade, 0] = np.minimum(1.0, cf[blade, 0] + 0.5)
        sbox = dict(n_groups=1, group_of=group_of, dir=np.array([[0.0, 1.0, 0.0]]),
                    shift_lo=np.array([0.0]), shift_hi=np.array([0.05]), parts=[1, 1, 1],
                    col_lo=col_lo, col_hi=col_hi, op_lo=None, op_hi=None)
        box = _pose_box(eps_t=(0.01, 0, 0), t_frame=1)
        return _pack("C5", mean, chol, o, c, cam, box, scene_box=sbox, tile=8, batch=32,
                     description="C2 scene + blade mean/colour box + camera-x +-1 cm")
    if name == "C3":
        n = 300_000 if N is None else N
        W = 400 if res is None else res
        mean, chol, o, c = outdoor_scene(3, n)
        cam = _camera((0.0, -2.0, 1.6), (0.0, 10.0, 1.0), 60.0, W, W)
        box = _pose_box(eps_t=(0.05, 0.05, 0.05), eps_R=(0, 0, math.radians(2.0)),
                        parts=(1, 1, 1, 1, 1, 8))
        return _pack("C3", mean, chol, o, c, cam, box, tile=16, batch=24,
                     description="outdoor ~300k, 400x400, yaw +-2 deg (8 parts) + t +-5 cm")
    if name == "C4":
        n = 750_000 if N is None else N
        W = 800 if res is None else res
        mean, chol, o, c = outdoor_scene(4, n)
        cam = _camera((0.0, -2.0, 1.6), (0.0, 10.0, 1.0), 60.0, W, W)
        box = _pose_box(eps_t=(0.01, 0.01, 0.01), eps_R=(math.radians(0.1),) * 3)
        return _pack("C4", mean, chol, o, c, cam, box, tile=16, batch=24,
                     description="outdoor 750k, 800x800, 6-DoF box (t +-1 cm, Euler +-0.1 deg)")
    raise ValueError(f"unknown config {name!r}")


# ----------------------------------------------------------------------------- edge-case scenes
def nearplane_config(N: int = 48, res: int = 32, seed: int = 11, eps_tz: float = 4e-4,
                     rot_deg: float = 0.0) -> Workload:
    """Near-plane case (reading G8, d_min = 0.01): a C1-style random scene shrunk by 1/500 so
    depths lie in [0.008, 0.012] m around d_min, with a camera-z translation box +-eps_tz
    (optionally also a yaw box).  Gaussians with d_hi <= d_min are dropped, those whose depth
    interval contains d_min 'straddle' (a_lo = 0, footprint from max(d_lo, d_min), O4), the
    rest are ordinary.  The projection is scale invariant, so the nominal image is the
    unshrunk scene's.  Nothing here evaluates the method."""
    mean, chol, o, c = random_scene(seed, N, depth=(4.0, 6.0), xy=0.8, scale=(0.03, 0.12))
    s = 1.0 / 500.0
    mean = mean * s
    chol = chol * s
    f = float(res)
    cam = dict(fx=f, fy=f, cx=res / 2.0, cy=res / 2.0, W=res, H=res, euler=[0.0, 0.0, 0.0],
               t=[0.0, 0.0, 0.0])
    box = _pose_box(eps_t=(0, 0, eps_tz), eps_R=(0, 0, math.radians(rot_deg)))
    return _pack("near", mean, chol, o, c, cam, box, tile=16, batch=16,
                 description=f"{N} Gaussians at depth 0.008-0.012 m, tz +-{eps_tz} m "
                             f"(near plane d_min = 0.01)")


def ties_config(N: int = 24, res: int = 32, seed: int = 12, rot_deg: float = 0.0,
                eps_t: float = 0.01) -> Workload:
    """Exact depth ties (reading G6, H4): a C1-style scene in which every Gaussian is
    duplicated (same mean and covariance, a different colour and opacity), so each
    duplicate pair has identical depth forms and an exact kappa tie, broken by the scene
    index.  Box: camera-x translation +-eps_t (ties stay certain: d_i - d_j = 0 exactly) and,
    with rot_deg > 0, a yaw box (identical non-constant forms: the pair is uncertain)."""
    mean, chol, o, c = random_scene(seed, N, depth=(3.0, 5.0), xy=0.8, scale=(0.08, 0.3))
    rng = np.random.default_rng(seed + 1000)
    o2 = rng.uniform(0.3, 0.99, N)
    c2 = rng.uniform(0, 1, (N, 3))
    # interleave: Gaussian 2k and 2k+1 are the duplicate pair (plus a few far-apart copies)
    perm = rng.permutation(N)
    mean = np.concatenate([mean, mean[perm]])
    chol = np.concatenate([chol, chol[perm]])
    o = np.concatenate([o, o2])
    c = np.concatenate([c, c2])
    f = float(res)
    cam = dict(fx=f, fy=f, cx=res / 2.0, cy=res / 2.0, W=res, H=res, euler=[0.0, 0.0, 0.0],
               t=[0.0, 0.0, 0.0])
    box = _pose_box(eps_t=(eps_t, 0, 0), eps_R=(0, 0, math.radians(rot_deg)))
    return _pack("ties", mean, chol, o, c, cam, box, tile=16, batch=16,
                 description=f"{N} duplicated Gaussian pairs (exact depth ties), tx +-{eps_t}"
                             + (f", yaw +-{rot_deg} deg" if rot_deg else ""))


def stacked_config(N: int = 200, res: int = 32, seed: int = 13, rot_deg: float = 0.5,
                   depth_spread: float = 0.005, opacity=(0.9, 0.99),
                   axis_frac: float = 0.0) -> Workload:
    """Exception-machinery stress case: N nearly opaque Gaussians stacked in a thin slab
    (depth 5 +- depth_spread m) in front of an identity camera, under a rotation box.  Almost every
    pair in a tile is uncertain (Table 2 Ind '?'), so exception windows span most of the list
    (long E_F / E_G lists, window lengths past the 128-position masks), and the transmittance
    deep in the stack underflows far below 1e-25 (the guarded-division paths).  Nothing here
    evaluates the method."""
    rng = np.random.default_rng(seed)
    mean = np.stack([rng.uniform(-0.15, 0.15, N), rng.uniform(-0.15, 0.15, N),
                     5.0 + rng.uniform(-depth_spread, depth_spread, N)], axis=1)
    # axis_frac of them on the optical axis column (|x| < 2 mm): their depth barely moves under
    # yaw, so pairs among them stay certain while pairs with off-axis ones are uncertain
    # (windows mixing kept and excepted positions)
    on = rng.uniform(size=N) < axis_frac
    mean[on, 0] = rng.uniform(-0.002, 0.002, int(on.sum()))
    s = _loguniform(rng, 0.05, 0.2, (N, 3))
    s[:, 2] *= 0.1
    chol = _chol_from(_frame_with_normal(rng, np.tile([[0.0, 0.0, 1.0]], (N, 1))), s)
    o = rng.uniform(opacity[0], opacity[1], N)
    c = rng.uniform(0, 1, (N, 3))
    f = 2.0 * res
    cam = dict(fx=f, fy=f, cx=res / 2.0, cy=res / 2.0, W=res, H=res, euler=[0.0, 0.0, 0.0],
               t=[0.0, 0.0, 0.0])
    # rotation about the camera's vertical axis (Euler e1): depth changes by about x * angle,
    # so the on-axis column's depths stay nearly fixed
    box = _pose_box(eps_t=(0.005, 0, 0), eps_R=(0, math.radians(rot_deg), 0))
    return _pack("stacked", mean, chol, o, c, cam, box, tile=16, batch=24,
                 description=f"{N} near-opaque Gaussians in a {2 * depth_spread} m slab, "
                             f"e1 +-{rot_deg} deg, on-axis fraction {axis_frac}")
