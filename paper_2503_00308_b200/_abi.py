"""ctypes view of include/absplat.h (argument marshalling only; no computation here).

Loading fails loudly when libabsplat.so is missing: there is no CPU or Python fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# ABSPLAT_LIB: an alternative in-tree build of the same library (A/B performance runs)
LIB_PATH = os.environ.get("ABSPLAT_LIB") or os.path.join(HERE, "libabsplat.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "absplat.h")

AS_PTR_DEVICE = 1
AS_ASYNC = 2
AS_MAX_VARS = 9

STATUS = {0: "AS_OK", 1: "AS_E_ARG", 2: "AS_E_SCENE", 3: "AS_E_NUMERIC", 4: "AS_E_CUDA",
          5: "AS_E_OOM", 6: "AS_E_STATE", 7: "AS_E_COMM"}


class AsCamera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("W", C.c_int32), ("H", C.c_int32), ("euler", C.c_double * 3),
                ("t", C.c_double * 3)]


class AsPoseBox(C.Structure):
    _fields_ = [("eps_t", C.c_double * 3), ("eps_R", C.c_double * 3), ("t_off", C.c_double * 3),
                ("R_off", C.c_double * 3), ("t_frame", C.c_int32), ("parts", C.c_int32 * 6)]


class AsSceneBox(C.Structure):
    _fields_ = [("n_groups", C.c_int32), ("group_of", C.c_void_p), ("dir", C.c_void_p),
                ("shift_lo", C.c_void_p), ("shift_hi", C.c_void_p), ("parts", C.c_int32 * 3),
                ("col_lo", C.c_void_p), ("col_hi", C.c_void_p), ("op_lo", C.c_void_p),
                ("op_hi", C.c_void_p), ("priv_lo", C.c_void_p), ("priv_hi", C.c_void_p)]


class AsStats(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("active_pairs", C.c_int64),
                ("uncertain_pairs", C.c_int64), ("fails", C.c_int64), ("straddles", C.c_int64),
                ("dropped", C.c_int64), ("order_violations", C.c_int64), ("launches", C.c_int64),
                ("kmax", C.c_int32), ("n_sub", C.c_int32), ("n_vars", C.c_int32),
                ("n_tiles", C.c_int32), ("ms_pose", C.c_double), ("ms_setup", C.c_double),
                ("ms_bin", C.c_double), ("ms_pairs", C.c_double), ("ms_tile", C.c_double),
                ("ms_total", C.c_double), ("tile_kernel_ms", C.c_double),
                ("device_bytes", C.c_size_t), ("n_items", C.c_int32), ("grid", C.c_int32),
                ("ring_len", C.c_int32), ("max_window", C.c_int32), ("ms_gather", C.c_double),
                ("world", C.c_int32), ("n_owned", C.c_int32), ("peak_bytes", C.c_size_t),
                ("host_syncs", C.c_int32), ("resized", C.c_int32), ("graph_replay", C.c_int32),
                ("ms_sort", C.c_double), ("ms_merge", C.c_double), ("kmean", C.c_double)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
# as_alloc_fn / as_free_fn (include/absplat.h)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def declared_functions():
    """Function names declared in include/absplat.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:as_status|const char\*|int32_t)\s+(as_\w+)\s*\(",
                                 txt, flags=re.M)))


def lib():
    """Load libabsplat.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                           "`python -m paper_2503_00308_b200.build` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i32, i64 = C.c_int32, C.c_int64
    sig = {
        "as_create": (i32, [C.POINTER(P), i32, P]),
        "as_destroy": (i32, [P]),
        "as_last_error": (C.c_char_p, [P]),
        "as_version": (i32, []),
        "as_load_scene": (i32, [P, i64, P, P, P, P, i32]),
        "as_set_camera": (i32, [P, P]),
        "as_set_pose_box": (i32, [P, P]),
        "as_set_scene_box": (i32, [P, P]),
        "as_render_bounds": (i32, [P, i32, i32, P, P, i32, P]),
        "as_render_shard": (i32, [P, i32, i32, i32, i32, P, P, i32, P, P, i32, P]),
        "as_untile": (i32, [P, i32, i32, i32, i32, i32, P, P, P, P, P, P, i32]),
        "as_tile_owners": (i32, [P, i32, i32, i32, P, P]),
        "as_lpt_assign": (i32, [i32, P, i32, i32, P]),
        "as_render_concrete": (i32, [P, P, P, i32]),
        "as_set_allocator": (i32, [P, ALLOC_FN, FREE_FN, P]),
        "as_render_subboxes": (i32, [P, i32, i32, i32, i32, P, P, i32, P]),
        "as_subbox_count": (i32, [P, P]),
        "as_set_subboxes": (i32, [P, i32, P]),
        "as_subbox_fails": (i32, [P, i32, P]),
        "as_set_matrixinv": (i32, [P, C.c_double, i32]),
        "as_set_chunk_target": (i32, [P, i32]),
        "as_set_blend": (i32, [P, i32]),
        "as_set_inverse_mode": (i32, [P, i32]),
        "as_debug_counters": (i32, [P, i32, P]),
        "as_nccl_id": (i32, [P]),
        "as_comm_init": (i32, [P, i32, i32, P]),
        "as_set_shard_axis": (i32, [P, i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
