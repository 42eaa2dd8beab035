"""ctypes binding of the fp64 CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
NVMAX = 9


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2, no fast-math, OpenMP)."""
    stale = (not os.path.exists(_LIB)
             or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC", "-Wall",
               _SRC, "-o", _LIB + ".tmp"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("W", C.c_int32), ("H", C.c_int32), ("euler", C.c_double * 3),
                ("t", C.c_double * 3)]


class PoseBox(C.Structure):
    _fields_ = [("eps_t", C.c_double * 3), ("eps_R", C.c_double * 3), ("t_off", C.c_double * 3),
                ("R_off", C.c_double * 3), ("t_frame", C.c_int32), ("parts", C.c_int32 * 6),
                ("n_explicit", C.c_int32), ("explicit_bounds", C.c_void_p),
                ("k_tol", C.c_double), ("k_max", C.c_int32), ("inv_backward", C.c_int32)]


class SceneBox(C.Structure):
    _fields_ = [("n_groups", C.c_int32), ("group_of", C.c_void_p), ("dir", C.c_void_p),
                ("shift_lo", C.c_void_p), ("shift_hi", C.c_void_p), ("parts", C.c_int32 * 3),
                ("col_lo", C.c_void_p), ("col_hi", C.c_void_p), ("op_lo", C.c_void_p),
                ("op_hi", C.c_void_p), ("priv_lo", C.c_void_p), ("priv_hi", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("active_pairs", C.c_int64),
                ("uncertain_pairs", C.c_int64), ("fails", C.c_int64),
                ("straddles", C.c_int64), ("dropped", C.c_int64),
                ("order_violations", C.c_int64), ("kmax", C.c_int32), ("n_sub", C.c_int32),
                ("n_vars", C.c_int32), ("pad", C.c_int32)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        L = _lib
        L.or_render_bounds.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int32, C.c_int32,
                                       C.c_int32, P, P, P]
        L.or_pixel_bounds.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int32, C.c_int64, P,
                                      P, C.c_int32, P, P]
        L.or_render_tiles.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int32, C.c_int64, P,
                                      C.c_int32, P, P, P]
        L.or_render_subboxes.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int32, P, P, P]
        L.or_render_concrete.argtypes = [C.c_int64, P, P, P, P, P, C.c_int32, P, P, P,
                                         C.c_int32, C.c_int64, P, P, C.c_int32, P]
        L.or_blend_sort.argtypes = [C.c_int64, P, P, P, P]
        L.or_blend_ind.argtypes = [C.c_int64, P, P, P, C.c_int32, P]
        L.or_form_conc.argtypes = [C.c_int32, P, P, P]
        L.or_form_mul.argtypes = [C.c_int32, P, P, P]
        L.or_form_sq.argtypes = [C.c_int32, P, P]
        L.or_exp_relax.argtypes = [C.c_double, C.c_double, P, P, P, P]
        L.or_ind_relax.argtypes = [C.c_double, C.c_double]
        L.or_ind_relax.restype = C.c_int32
        L.or_matrix_inv.argtypes = [C.c_int32, P, C.c_int32, P, P, P]
        L.or_matrix_inv.restype = C.c_int32
        L.or_matrix_inv_bwd.argtypes = [C.c_int32, P, C.c_int32, P, P, P]
        L.or_matrix_inv_bwd.restype = C.c_int32
        L.or_pose_forms.argtypes = [P, P, P, C.c_int32, P, P, P]
        L.or_pose_forms.restype = C.c_int32
        L.or_gaussian_forms.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int32, P, P]
        L.or_gaussian_forms.restype = C.c_int32
        L.or_gaussian_forms_stride.argtypes = [C.c_int32]
        L.or_gaussian_forms_stride.restype = C.c_int32
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def camera_struct(cam: dict) -> Camera:
    c = Camera()
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    c.W, c.H = int(cam["W"]), int(cam["H"])
    for k in range(3):
        c.euler[k] = float(cam["euler"][k])
        c.t[k] = float(cam["t"][k])
    return c


def pose_box_struct(box: dict) -> PoseBox:
    b = PoseBox()
    for k in range(3):
        b.eps_t[k] = float(box["eps_t"][k])
        b.eps_R[k] = float(box["eps_R"][k])
        b.t_off[k] = float(box["t_off"][k])
        b.R_off[k] = float(box["R_off"][k])
    b.t_frame = int(box["t_frame"])
    for k in range(6):
        b.parts[k] = int(box["parts"][k])
    b.k_tol = float(box.get("k_tol", 0.0))
    b.k_max = int(box.get("k_max", 8))
    b.inv_backward = int(box.get("inv_backward", 0))
    sub = box.get("subboxes")
    if sub is not None and len(sub) > 0:
        arr = np.ascontiguousarray(sub, np.float64).reshape(-1, 9, 2)
        b._keep = arr  # keep alive with the struct
        b.n_explicit = arr.shape[0]
        b.explicit_bounds = arr.ctypes.data
    return b


class _SceneBoxHolder:
    """Keeps the numpy arrays referenced by a SceneBox alive."""

    def __init__(self, sbox: dict | None, N: int):
        self.s = None
        self.keep = []
        if sbox is None:
            return
        s = SceneBox()
        ng = int(sbox.get("n_groups", 0))
        s.n_groups = ng

        def arr(x, dt, shape=None):
            if x is None:
                return None
            a = np.ascontiguousarray(x, dtype=dt)
            if shape is not None:
                a = a.reshape(shape)
            self.keep.append(a)
            return a

        s.group_of = _ptr(arr(sbox.get("group_of"), np.int32)) if ng > 0 else None
        s.dir = _ptr(arr(sbox.get("dir"), np.float64, (-1,))) if ng > 0 else None
        s.shift_lo = _ptr(arr(sbox.get("shift_lo"), np.float64)) if ng > 0 else None
        s.shift_hi = _ptr(arr(sbox.get("shift_hi"), np.float64)) if ng > 0 else None
        parts = sbox.get("parts", [1, 1, 1])
        for g in range(3):
            s.parts[g] = int(parts[g]) if g < len(parts) else 1
        s.col_lo = _ptr(arr(sbox.get("col_lo"), np.float32))
        s.col_hi = _ptr(arr(sbox.get("col_hi"), np.float32))
        s.op_lo = _ptr(arr(sbox.get("op_lo"), np.float32))
        s.op_hi = _ptr(arr(sbox.get("op_hi"), np.float32))
        s.priv_lo = _ptr(arr(sbox.get("priv_lo"), np.float32))
        s.priv_hi = _ptr(arr(sbox.get("priv_hi"), np.float32))
        self.s = s

    def ref(self):
        return None if self.s is None else C.addressof(self.s)


def _scene(w):
    return (np.ascontiguousarray(w.mean, np.float32), np.ascontiguousarray(w.chol, np.float32),
            np.ascontiguousarray(w.opacity, np.float32), np.ascontiguousarray(w.color, np.float32))


def render_bounds(w, tile=None, mode=0, nthreads=0, camera=None, pose_box=None, scene_box="same"):
    """Full abstract image [H,W,3] lo/hi (fp64) and stats for a workloads.Workload."""
    tile = w.tile if tile is None else tile
    cam = camera_struct(camera or w.camera)
    box = pose_box_struct(pose_box or w.pose_box)
    sb = _SceneBoxHolder(w.scene_box if scene_box == "same" else scene_box, w.N)
    mean, chol, op, col = _scene(w)
    H, W = cam.H, cam.W
    lo = np.zeros((H, W, 3))
    hi = np.zeros((H, W, 3))
    st = Stats()
    rc = lib().or_render_bounds(w.N, _ptr(mean), _ptr(chol), _ptr(op), _ptr(col),
                                C.addressof(cam), C.addressof(box), sb.ref(), tile, mode,
                                nthreads, _ptr(lo), _ptr(hi), C.addressof(st))
    if rc != 0:
        raise ValueError(f"or_render_bounds failed ({rc})")
    return lo, hi, st.asdict()


def render_subboxes(w, sub_begin, sub_end, tile=None, nthreads=0):
    """Union over the sub-boxes [sub_begin, sub_end) only (empty: lo = 1, hi = 0)."""
    tile = w.tile if tile is None else tile
    cam = camera_struct(w.camera)
    box = pose_box_struct(w.pose_box)
    sb = _SceneBoxHolder(w.scene_box, w.N)
    mean, chol, op, col = _scene(w)
    lo = np.zeros((cam.H, cam.W, 3))
    hi = np.zeros((cam.H, cam.W, 3))
    st = Stats()
    rc = lib().or_render_subboxes(w.N, _ptr(mean), _ptr(chol), _ptr(op), _ptr(col),
                                  C.addressof(cam), C.addressof(box), sb.ref(), tile, sub_begin,
                                  sub_end, nthreads, _ptr(lo), _ptr(hi), C.addressof(st))
    if rc != 0:
        raise ValueError(f"or_render_subboxes failed ({rc})")
    return lo, hi, st.asdict()


def render_tiles(w, tiles, tile=None, nthreads=0):
    """Abstract bounds of the listed tile ids only (others left zero)."""
    tile = w.tile if tile is None else tile
    cam = camera_struct(w.camera)
    box = pose_box_struct(w.pose_box)
    sb = _SceneBoxHolder(w.scene_box, w.N)
    mean, chol, op, col = _scene(w)
    tl = np.ascontiguousarray(tiles, np.int32)
    lo = np.zeros((cam.H, cam.W, 3))
    hi = np.zeros((cam.H, cam.W, 3))
    st = Stats()
    rc = lib().or_render_tiles(w.N, _ptr(mean), _ptr(chol), _ptr(op), _ptr(col),
                               C.addressof(cam), C.addressof(box), sb.ref(), tile, len(tl),
                               _ptr(tl), nthreads, _ptr(lo), _ptr(hi), C.addressof(st))
    if rc != 0:
        raise ValueError(f"or_render_tiles failed ({rc})")
    return lo, hi, st.asdict()


def pixel_bounds(w, px, py, tile=None, nthreads=0):
    tile = w.tile if tile is None else tile
    cam = camera_struct(w.camera)
    box = pose_box_struct(w.pose_box)
    sb = _SceneBoxHolder(w.scene_box, w.N)
    mean, chol, op, col = _scene(w)
    px = np.ascontiguousarray(px, np.int32)
    py = np.ascontiguousarray(py, np.int32)
    lo = np.zeros((len(px), 3))
    hi = np.zeros((len(px), 3))
    rc = lib().or_pixel_bounds(w.N, _ptr(mean), _ptr(chol), _ptr(op), _ptr(col),
                               C.addressof(cam), C.addressof(box), sb.ref(), tile, len(px),
                               _ptr(px), _ptr(py), nthreads, _ptr(lo), _ptr(hi))
    if rc != 0:
        raise ValueError(f"or_pixel_bounds failed ({rc})")
    return lo, hi


def render_concrete(w, euler=None, t=None, shifts=None, color=None, opacity=None, blend=0,
                    px=None, py=None, nthreads=0):
    """Concrete Alg. 1 render at a pose (defaults: the nominal camera)."""
    cam_d = dict(w.camera)
    if euler is not None:
        cam_d["euler"] = list(euler)
    if t is not None:
        cam_d["t"] = list(t)
    cam = camera_struct(cam_d)
    mean, chol, op, col = _scene(w)
    if color is not None:
        col = np.ascontiguousarray(color, np.float32)
    if opacity is not None:
        op = np.ascontiguousarray(opacity, np.float32)
    sbox = w.scene_box
    ng = int(sbox["n_groups"]) if sbox is not None else 0
    keep = []
    gof = dirp = shp = None
    if ng > 0:
        g = np.ascontiguousarray(sbox["group_of"], np.int32)
        d = np.ascontiguousarray(sbox["dir"], np.float64).reshape(-1)
        s = np.ascontiguousarray(shifts if shifts is not None else np.zeros(ng), np.float64)
        keep += [g, d, s]
        gof, dirp, shp = _ptr(g), _ptr(d), _ptr(s)
    if px is None:
        img = np.zeros((cam.H, cam.W, 3))
        npix = 0
        pxp = pyp = None
    else:
        pxa = np.ascontiguousarray(px, np.int32)
        pya = np.ascontiguousarray(py, np.int32)
        keep += [pxa, pya]
        img = np.zeros((len(pxa), 3))
        npix = len(pxa)
        pxp, pyp = _ptr(pxa), _ptr(pya)
    rc = lib().or_render_concrete(w.N, _ptr(mean), _ptr(chol), _ptr(op), _ptr(col),
                                  C.addressof(cam), ng, gof, dirp, shp, blend, npix, pxp, pyp,
                                  nthreads, _ptr(img))
    if rc != 0:
        raise ValueError(f"or_render_concrete failed ({rc})")
    return img


def blend_sort(a, c, d):
    a = np.ascontiguousarray(a, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    pc = np.zeros(3)
    lib().or_blend_sort(len(a), _ptr(a), _ptr(c), _ptr(d), _ptr(pc))
    return pc


def blend_ind(a, c, d, tiebreak=True):
    a = np.ascontiguousarray(a, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    pc = np.zeros(3)
    lib().or_blend_ind(len(a), _ptr(a), _ptr(c), _ptr(d), int(bool(tiebreak)), _ptr(pc))
    return pc


# ----------------------------------------------------------------------------- forms
def form(lA, lb, uA, ub):
    return np.concatenate([np.asarray(lA, float), [lb], np.asarray(uA, float), [ub]])


def form_conc(f, n):
    f = np.ascontiguousarray(f, np.float64)
    lo = C.c_double()
    hi = C.c_double()
    lib().or_form_conc(n, _ptr(f), C.addressof(lo), C.addressof(hi))
    return lo.value, hi.value


def form_mul(f, g, n):
    f = np.ascontiguousarray(f, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    out = np.zeros(2 * (n + 1))
    lib().or_form_mul(n, _ptr(f), _ptr(g), _ptr(out))
    return out


def form_sq(f, n):
    f = np.ascontiguousarray(f, np.float64)
    out = np.zeros(2 * (n + 1))
    lib().or_form_sq(n, _ptr(f), _ptr(out))
    return out


def exp_relax(xl, xh):
    v = [C.c_double() for _ in range(4)]
    lib().or_exp_relax(xl, xh, *(C.addressof(x) for x in v))
    return tuple(x.value for x in v)


def ind_relax(xl, xh):
    return int(lib().or_ind_relax(xl, xh))


def matrix_inv(X, n, k=8, backward=False):
    """X: [4, 2(n+1)] forms.  Returns (status, conic [4,2(n+1)], eps, rho); backward=True
    bounds the conic by back-substitution (NEXT-4)."""
    X = np.ascontiguousarray(X, np.float64).reshape(-1)
    out = np.zeros(4 * 2 * (n + 1))
    eps = C.c_double()
    rho = C.c_double()
    fn = lib().or_matrix_inv_bwd if backward else lib().or_matrix_inv
    st = fn(n, _ptr(X), k, _ptr(out), C.addressof(eps), C.addressof(rho))
    return st, out.reshape(4, 2 * (n + 1)), eps.value, rho.value


def pose_forms(w, sub=0):
    cam = camera_struct(w.camera)
    box = pose_box_struct(w.pose_box)
    sb = _SceneBoxHolder(w.scene_box, w.N)
    R = np.zeros(9 * 2 * (NVMAX + 1))
    t = np.zeros(3 * 2 * (NVMAX + 1))
    nv = C.c_int32()
    nsub = lib().or_pose_forms(C.addressof(cam), C.addressof(box), sb.ref(), sub, _ptr(R),
                               _ptr(t), C.addressof(nv))
    if nsub < 0:
        raise ValueError("or_pose_forms failed")
    n = nv.value
    fs = 2 * (n + 1)
    return R[:9 * fs].reshape(9, fs), t[:3 * fs].reshape(3, fs), n, nsub


GFIELDS = (["uc0", "uc1", "uc2", "d", "up0", "up1"]
           + [f"Mp{a}{c}" for a in range(2) for c in range(3)]
           + ["X00", "X01", "X11", "conic00", "conic01", "conic10", "conic11"]
           + [f"W{a}{c}" for a in range(2) for c in range(3)]
           + ["D2", "DU0", "DU1"])
GSCALARS = ["flags", "eps", "rho", "kappa", "mu_lo0", "mu_lo1", "mu_hi0", "mu_hi1", "r2", "k"]


def gaussian_forms(w, sub=0):
    """Per-Gaussian forms of sub-box `sub`: dict name -> [N, 2(n+1)] plus scalars [N]."""
    cam = camera_struct(w.camera)
    box = pose_box_struct(w.pose_box)
    sb = _SceneBoxHolder(w.scene_box, w.N)
    mean, chol, op, col = _scene(w)
    # n is not known before the call: use the maximum stride
    stride_max = lib().or_gaussian_forms_stride(NVMAX)
    out = np.zeros(w.N * stride_max)
    nv = C.c_int32()
    rc = lib().or_gaussian_forms(w.N, _ptr(mean), _ptr(chol), _ptr(op), _ptr(col),
                                 C.addressof(cam), C.addressof(box), sb.ref(), sub, _ptr(out),
                                 C.addressof(nv))
    if rc < 0:
        raise ValueError("or_gaussian_forms failed")
    n = nv.value
    stride = lib().or_gaussian_forms_stride(n)
    o = out[:w.N * stride].reshape(w.N, stride)
    fs = 2 * (n + 1)
    res = {}
    for k, name in enumerate(GFIELDS):
        res[name] = o[:, k * fs:(k + 1) * fs]
    base = len(GFIELDS) * fs
    for k, name in enumerate(GSCALARS):
        res[name] = o[:, base + k]
    res["n"] = n
    return res
