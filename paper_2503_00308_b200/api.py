"""Thin Python binding of the C ABI (include/absplat.h), same names as the C entry points.

Argument marshalling only: every step of the path runs in libabsplat.so's CUDA kernels.
PyTorch is used for device memory (output tensors) and streams.  Accepts numpy arrays (host
pointers) or torch tensors (host or CUDA; CUDA tensors are passed as device pointers).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _abi

AS_PTR_DEVICE = _abi.AS_PTR_DEVICE
AS_ASYNC = _abi.AS_ASYNC


class AbsplatError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_abi.STATUS.get(status, status)}: {msg}")
        self.status = status


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x, dtype):
    """(pointer, is_device, keepalive) of a numpy array or torch tensor of dtype."""
    if x is None:
        return None, False, None
    if _is_torch(x):
        import torch
        tdt = {np.float32: torch.float32, np.int32: torch.int32, np.float64: torch.float64}[dtype]
        if x.dtype != tdt or not x.is_contiguous():
            x = x.to(tdt).contiguous()
        return x.data_ptr(), bool(x.is_cuda), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, False, a


def camera_struct(cam: dict) -> _abi.AsCamera:
    c = _abi.AsCamera()
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    c.W, c.H = int(cam["W"]), int(cam["H"])
    for k in range(3):
        c.euler[k] = float(cam["euler"][k])
        c.t[k] = float(cam["t"][k])
    return c


def pose_box_struct(box: dict) -> _abi.AsPoseBox:
    b = _abi.AsPoseBox()
    for k in range(3):
        b.eps_t[k] = float(box["eps_t"][k])
        b.eps_R[k] = float(box["eps_R"][k])
        b.t_off[k] = float(box.get("t_off", [0, 0, 0])[k])
        b.R_off[k] = float(box.get("R_off", [0, 0, 0])[k])
    b.t_frame = int(box.get("t_frame", 0))
    parts = box.get("parts", [1] * 6)
    for k in range(6):
        b.parts[k] = int(parts[k])
    return b


class Context:
    """One as_ctx on one CUDA device and stream."""

    def __init__(self, device: int = 0, stream=None):
        self._L = _abi.lib()
        self.device = int(device)
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(self.device)
            except Exception:  # pragma: no cover
                stream = None
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self.stream = stream
        out = C.c_void_p()
        st = self._L.as_create(C.byref(out), self.device, C.c_void_p(handle or 0))
        if st != 0:
            raise AbsplatError(st, f"as_create(device={device}) failed (is a CUDA GPU present?)")
        self._ctx = out
        self.camera: Optional[dict] = None
        self.N = 0

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_ctx", None):
            self._L.as_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st: int):
        if st != 0:
            msg = self._L.as_last_error(self._ctx)
            raise AbsplatError(st, msg.decode() if msg else "")

    # ------------------------------------------------------------------ memory
    def as_set_allocator(self, alloc=None, free=None):
        """Route the context's device memory through alloc(nbytes, stream) -> int pointer and
        free(ptr, nbytes, stream); both None restores cudaMalloc/cudaFree."""
        if (alloc is None) != (free is None):
            raise ValueError("alloc and free must both be given or both be None")
        if alloc is None:
            cbs = (_abi.ALLOC_FN(), _abi.FREE_FN())
        else:
            def _a(user, nbytes, stream):
                try:
                    return int(alloc(int(nbytes), int(stream or 0)))
                except Exception:  # reported as AS_E_OOM by the library
                    return None

            def _f(user, ptr, nbytes, stream):
                try:
                    free(int(ptr), int(nbytes), int(stream or 0))
                except Exception:
                    pass
            cbs = (_abi.ALLOC_FN(_a), _abi.FREE_FN(_f))
        self._check(self._L.as_set_allocator(self._ctx, cbs[0], cbs[1], None))
        # buffers keep the free callback they were allocated with: keep every set alive
        self._alloc_cbs = getattr(self, "_alloc_cbs", []) + [cbs]

    def use_torch_allocator(self):
        """Bind as_set_allocator to torch's CUDA caching allocator."""
        import torch
        dev = self.device
        self.as_set_allocator(
            lambda n, s: torch.cuda.caching_allocator_alloc(n, dev, s),
            lambda p, n, s: torch.cuda.caching_allocator_delete(p))

    # ------------------------------------------------------------------ inputs
    def as_load_scene(self, mean, chol, opacity, color):
        keep = [_ptr(a, np.float32) for a in (mean, chol, opacity, color)]
        devs = {k[1] for k in keep}
        if len(devs) != 1:
            raise ValueError("scene arrays must all be host or all be device")
        N = int(keep[2][2].shape[0])
        flags = AS_PTR_DEVICE if devs.pop() else 0
        self._check(self._L.as_load_scene(self._ctx, N, *(C.c_void_p(k[0]) for k in keep), flags))
        self.N = N

    def as_set_camera(self, cam: dict):
        c = camera_struct(cam)
        self._check(self._L.as_set_camera(self._ctx, C.byref(c)))
        self.camera = dict(cam)

    def as_set_pose_box(self, box: dict):
        b = pose_box_struct(box)
        self._check(self._L.as_set_pose_box(self._ctx, C.byref(b)))

    def as_set_scene_box(self, sbox: Optional[dict]):
        if sbox is None:
            self._check(self._L.as_set_scene_box(self._ctx, None))
            return
        s = _abi.AsSceneBox()
        keep = []

        def host(x, dt):
            if x is None:
                return None
            a = np.ascontiguousarray(x.cpu().numpy() if _is_torch(x) else x, dtype=dt)
            keep.append(a)
            return a.ctypes.data

        ng = int(sbox.get("n_groups", 0))
        s.n_groups = ng
        if ng > 0:
            s.group_of = host(sbox["group_of"], np.int32)
            s.dir = host(np.asarray(sbox["dir"], np.float64).reshape(-1), np.float64)
            s.shift_lo = host(sbox["shift_lo"], np.float64)
            s.shift_hi = host(sbox["shift_hi"], np.float64)
        parts = sbox.get("parts", [1, 1, 1])
        for g in range(3):
            s.parts[g] = int(parts[g]) if g < len(parts) else 1
        s.col_lo = host(sbox.get("col_lo"), np.float32)
        s.col_hi = host(sbox.get("col_hi"), np.float32)
        s.op_lo = host(sbox.get("op_lo"), np.float32)
        s.op_hi = host(sbox.get("op_hi"), np.float32)
        s.priv_lo = host(sbox.get("priv_lo"), np.float32)
        s.priv_hi = host(sbox.get("priv_hi"), np.float32)
        self._check(self._L.as_set_scene_box(self._ctx, C.byref(s)))

    def load_workload(self, w):
        """Scene + camera + pose box + scene box of a workloads.Workload."""
        self.as_load_scene(w.mean, w.chol, w.opacity, w.color)
        self.as_set_camera(w.camera)
        self.as_set_pose_box(w.pose_box)
        self.as_set_scene_box(w.scene_box)
        self.as_set_inverse_mode(0)
        self.as_set_matrixinv(w.pose_box.get("k_tol", 0.0), w.pose_box.get("k_max", 8))
        self.as_set_inverse_mode(w.pose_box.get("inv_backward", 0))
        if w.pose_box.get("subboxes") is not None:
            self.as_set_subboxes(w.pose_box["subboxes"])

    # ------------------------------------------------------------------ render
    def _image_out(self, lo, hi, shape):
        if lo is None:
            import torch
            lo = torch.empty(shape, dtype=torch.float32, device=f"cuda:{self.device}")
            hi = torch.empty(shape, dtype=torch.float32, device=f"cuda:{self.device}")
        pl, dl, _ = _ptr(lo, np.float32)
        ph, dh, _ = _ptr(hi, np.float32)
        if dl != dh:
            raise ValueError("lo and hi must both be host or both be device")
        if not _is_torch(lo) and not (lo.flags["C_CONTIGUOUS"] and lo.dtype == np.float32):
            raise ValueError("host outputs must be C-contiguous float32")
        return lo, hi, pl, ph, dl

    def as_render_bounds(self, tile: int = 16, batch: int = 64, lo=None, hi=None,
                         stats: bool = True, sync: bool = True):
        """Abstract render; returns (lo, hi, stats dict or None)."""
        H, W = int(self.camera["H"]), int(self.camera["W"])
        lo, hi, pl, ph, dev = self._image_out(lo, hi, (H, W, 3))
        flags = (AS_PTR_DEVICE if dev else 0) | (AS_ASYNC if (dev and not sync) else 0)
        st = _abi.AsStats() if stats else None
        self._check(self._L.as_render_bounds(self._ctx, tile, batch, C.c_void_p(pl), C.c_void_p(ph),
                                             flags, C.byref(st) if st is not None else None))
        return lo, hi, (st.asdict() if st is not None else None)

    def as_render_subboxes(self, sub_begin: int, sub_end: int, tile: int = 16, batch: int = 64,
                           lo=None, hi=None, stats: bool = True, sync: bool = True):
        """Union over sub-boxes [sub_begin, sub_end) only (empty range: lo = 1, hi = 0)."""
        H, W = int(self.camera["H"]), int(self.camera["W"])
        lo, hi, pl, ph, dev = self._image_out(lo, hi, (H, W, 3))
        flags = (AS_PTR_DEVICE if dev else 0) | (AS_ASYNC if (dev and not sync) else 0)
        st = _abi.AsStats() if stats else None
        self._check(self._L.as_render_subboxes(self._ctx, tile, batch, int(sub_begin),
                                               int(sub_end), C.c_void_p(pl), C.c_void_p(ph),
                                               flags, C.byref(st) if st is not None else None))
        return lo, hi, (st.asdict() if st is not None else None)

    def as_set_subboxes(self, bounds=None):
        """Explicit partition: bounds [n, 9, 2] (lo, hi per box axis); None / empty clears."""
        if bounds is None or len(bounds) == 0:
            self._check(self._L.as_set_subboxes(self._ctx, 0, None))
            return
        b = np.ascontiguousarray(bounds, np.float64).reshape(-1, 9, 2)
        self._check(self._L.as_set_subboxes(self._ctx, b.shape[0], C.c_void_p(b.ctypes.data)))

    def as_set_matrixinv(self, k_tol: float = 0.0, k_max: int = 8):
        """Adaptive MatrixInv order: smallest k >= 8 with Eps <= k_tol (<= k_max); 0 = fixed 8."""
        self._check(self._L.as_set_matrixinv(self._ctx, float(k_tol), int(k_max)))

    def as_set_chunk_target(self, target: int = 0):
        """Positions per (tile, chunk) work item; 0 = automatic (performance knob only)."""
        self._check(self._L.as_set_chunk_target(self._ctx, int(target)))

    def as_set_blend(self, mode: int = 0):
        """0: interval blend; 1: + linear-relation blend on exception-free tiles (n <= 3)."""
        self._check(self._L.as_set_blend(self._ctx, int(mode)))

    DEBUG_COUNTERS = ("thi_bits", "thi_div_unsafe", "thi_ovf", "thi_ovf_window", "fin_slow",
                      "fin_unstaged", "fin_ovf", "tmode3")

    def as_debug_counters(self, enable: int = -1):
        """Rare-path counters of the last render (dict) and, with enable 0 / 1, switch
        counting for later renders (include/absplat.h, as_debug_counters)."""
        out = np.zeros(len(self.DEBUG_COUNTERS), np.uint64)
        self._check(self._L.as_debug_counters(self._ctx, int(enable), out.ctypes.data))
        return {k: int(v) for k, v in zip(self.DEBUG_COUNTERS, out)}

    def as_comm_init(self, rank: int, world: int, uid: bytes):
        """Join rank `rank` of `world` with the 128-byte NCCL id from as_nccl_id (collective).
        Afterwards as_render_bounds / as_render_subboxes shard the work over the ranks and
        return the complete images on every rank (include/absplat.h)."""
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        self._check(self._L.as_comm_init(self._ctx, int(rank), int(world), buf))

    def as_set_shard_axis(self, axis: int = 0):
        """Multi-GPU axis: 0 auto, 1 image tiles (all-gather), 2 sub-boxes (all-reduce)."""
        self._check(self._L.as_set_shard_axis(self._ctx, int(axis)))

    def as_set_inverse_mode(self, backward: int = 0):
        """MatrixInv conic bounds: 0 forward forms, 1 back-substitution (NEXT-4)."""
        self._check(self._L.as_set_inverse_mode(self._ctx, int(backward)))

    def as_subbox_fails(self):
        """MatrixInv FAIL count per sub-box of the current partition (setup only)."""
        n = self.as_subbox_count()
        out = np.zeros(max(n, 1), np.int64)
        self._check(self._L.as_subbox_fails(self._ctx, n, C.c_void_p(out.ctypes.data)))
        return out[:n]

    def as_subbox_count(self) -> int:
        n = C.c_int32(0)
        self._check(self._L.as_subbox_count(self._ctx, C.byref(n)))
        return int(n.value)

    def n_tiles(self, tile: int) -> int:
        H, W = int(self.camera["H"]), int(self.camera["W"])
        return ((W + tile - 1) // tile) * ((H + tile - 1) // tile)

    def as_tile_owners(self, tile: int, world: int, max_tiles: int):
        n = self.n_tiles(tile)
        owner = np.zeros(n, np.int32)
        costs = np.zeros(n, np.int64)
        self._check(self._L.as_tile_owners(self._ctx, tile, world, max_tiles,
                                           C.c_void_p(owner.ctypes.data),
                                           C.c_void_p(costs.ctypes.data)))
        return owner, costs

    def as_render_shard(self, tile: int, batch: int, rank: int, world: int, max_tiles: int,
                        lo_tm=None, hi_tm=None, stats: bool = True):
        """Render the tiles this rank owns into compact tile-major buffers [max_tiles, tile*tile, 3].
        Returns (lo_tm, hi_tm, owned ids (np.int32[max_tiles], -1 padded), n_owned, stats)."""
        shape = (max_tiles, tile * tile, 3)
        lo_tm, hi_tm, pl, ph, dev = self._image_out(lo_tm, hi_tm, shape)
        owned = np.full(max_tiles, -1, np.int32)
        n_owned = C.c_int32(0)
        st = _abi.AsStats() if stats else None
        self._check(self._L.as_render_shard(self._ctx, tile, batch, rank, world, C.c_void_p(pl),
                                            C.c_void_p(ph), max_tiles,
                                            C.c_void_p(owned.ctypes.data), C.byref(n_owned),
                                            AS_PTR_DEVICE if dev else 0,
                                            C.byref(st) if st is not None else None))
        return lo_tm, hi_tm, owned, int(n_owned.value), (st.asdict() if st is not None else None)

    def as_untile(self, tile: int, world: int, max_tiles: int, owned, n_owned, lo_tm, hi_tm,
                  lo=None, hi=None):
        """Assemble gathered tile-major buffers [world, max_tiles, tile*tile, 3] into images."""
        H, W = int(self.camera["H"]), int(self.camera["W"])
        return as_untile(W, H, tile, world, max_tiles, owned, n_owned, lo_tm, hi_tm, lo, hi,
                         ctx=self)

    def as_render_concrete(self, xi, img=None):
        H, W = int(self.camera["H"]), int(self.camera["W"])
        x = np.ascontiguousarray(xi, np.float64).reshape(-1)
        if img is None:
            import torch
            img = torch.empty((H, W, 3), dtype=torch.float32, device=f"cuda:{self.device}")
        p, dev, _ = _ptr(img, np.float32)
        self._check(self._L.as_render_concrete(self._ctx, C.c_void_p(x.ctypes.data if x.size else 0),
                                               C.c_void_p(p), AS_PTR_DEVICE if dev else 0))
        return img


def as_lpt_assign(costs, world: int, cap: int):
    """Pure host LPT owner map (C ABI as_lpt_assign)."""
    L = _abi.lib()
    c = np.ascontiguousarray(costs, np.int64)
    owner = np.zeros(len(c), np.int32)
    st = L.as_lpt_assign(len(c), C.c_void_p(c.ctypes.data), world, cap,
                         C.c_void_p(owner.ctypes.data))
    if st != 0:
        raise AbsplatError(st, "as_lpt_assign failed")
    return owner


def as_untile(W: int, H: int, tile: int, world: int, max_tiles: int, owned, n_owned, lo_tm,
              hi_tm, lo=None, hi=None, ctx: Optional[Context] = None):
    """C ABI as_untile.  With numpy (host) buffers no context or GPU is needed."""
    L = _abi.lib()
    ptm_l, dtl, k1 = _ptr(lo_tm, np.float32)
    ptm_h, dth, k2 = _ptr(hi_tm, np.float32)
    if lo is None:
        if dtl:
            import torch
            lo = torch.empty((H, W, 3), dtype=torch.float32, device=lo_tm.device)
            hi = torch.empty((H, W, 3), dtype=torch.float32, device=lo_tm.device)
        else:
            lo = np.zeros((H, W, 3), np.float32)
            hi = np.zeros((H, W, 3), np.float32)
    pl, dl, _ = _ptr(lo, np.float32)
    ph, dh, _ = _ptr(hi, np.float32)
    if not (dl == dh == dtl == dth):
        raise ValueError("tile-major inputs and images must share one pointer space")
    if dl and ctx is None:
        raise ValueError("device buffers need a Context")
    ow = np.ascontiguousarray(owned, np.int32).reshape(-1)
    no = np.ascontiguousarray(n_owned, np.int32).reshape(-1)
    c = ctx._ctx if ctx is not None else None
    st = L.as_untile(c, W, H, tile, world, max_tiles, C.c_void_p(ow.ctypes.data),
                     C.c_void_p(no.ctypes.data), C.c_void_p(ptm_l), C.c_void_p(ptm_h),
                     C.c_void_p(pl), C.c_void_p(ph), AS_PTR_DEVICE if dl else 0)
    if st != 0:
        msg = L.as_last_error(c).decode() if c is not None else "as_untile failed"
        raise AbsplatError(st, msg)
    return lo, hi


def as_nccl_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for as_comm_init; AbsplatError(AS_E_COMM) when the
    process cannot load NCCL."""
    buf = (C.c_uint8 * 128)()
    st = _abi.lib().as_nccl_id(buf)
    if st != 0:
        raise AbsplatError(st, "as_nccl_id: NCCL unavailable")
    return bytes(buf)


def as_version() -> int:
    return int(_abi.lib().as_version())
