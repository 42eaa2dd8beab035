"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, exports every symbol
include/absplat.h declares, fails loudly without a device, and its host-side sharding
logic (LPT owner map, tile-major assembly) is correct."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import paper_2503_00308_b200 as ap
from paper_2503_00308_b200 import _abi


def test_library_exports_every_declared_symbol():
    names = _abi.declared_functions()
    assert len(names) >= 14
    lib = ctypes.CDLL(_abi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_version_and_no_gpu_fails_loudly():
    assert ap.as_version() == 1
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ap.AbsplatError) as e:
        ap.Context(0)
    assert "AS_E_CUDA" in str(e.value)


def test_lpt_assign():
    rng = np.random.default_rng(0)
    costs = rng.integers(0, 1000, 300)
    for world in (1, 2, 3, 8):
        cap = -(-300 // world) + 5
        own = ap.as_lpt_assign(costs, world, cap)
        assert own.min() >= 0 and own.max() < world
        counts = np.bincount(own, minlength=world)
        assert counts.max() <= cap
        loads = np.bincount(own, weights=costs + 1, minlength=world)
        # LPT bound: max load <= (4/3 - 1/(3m)) OPT + slack; OPT >= max(mean, max item)
        opt = max(loads.sum() / world, (costs + 1).max())
        assert loads.max() <= (4 / 3) * opt + 1
    # deterministic and tie-broken by tile id then rank
    own = ap.as_lpt_assign([1, 1, 1, 1], 2, 2)
    assert list(own) == [0, 1, 0, 1]
    with pytest.raises(ap.AbsplatError):
        ap.as_lpt_assign([1, 1, 1], 1, 2)  # cap * world < n


@pytest.mark.parametrize("W,H,tile,world", [(40, 24, 16, 2), (200, 200, 16, 3), (33, 17, 8, 4)])
def test_host_untile_roundtrip(W, H, tile, world):
    """Tile-major shards -> row-major image (a11), pure host path of as_untile."""
    ntx, nty = -(-W // tile), -(-H // tile)
    nt = ntx * nty
    cap = -(-nt // world) + 1
    own = ap.as_lpt_assign(np.arange(nt)[::-1] % 7, world, cap)
    img = np.random.default_rng(1).uniform(size=(H, W, 3)).astype(np.float32)
    tm_lo = np.zeros((world, cap, tile * tile, 3), np.float32)
    tm_hi = np.zeros((world, cap, tile * tile, 3), np.float32)
    owned = np.full((world, cap), -1, np.int32)
    n_owned = np.zeros(world, np.int32)
    for t in range(nt):
        r = own[t]
        k = n_owned[r]
        owned[r, k] = t
        n_owned[r] += 1
        tx, ty = t % ntx, t // ntx
        for ly in range(tile):
            for lx in range(tile):
                py, px = ty * tile + ly, tx * tile + lx
                if py < H and px < W:
                    tm_lo[r, k, ly * tile + lx] = img[py, px]
                    tm_hi[r, k, ly * tile + lx] = 1 - img[py, px]
    lo, hi = ap.as_untile(W, H, tile, world, cap, owned, n_owned, tm_lo, tm_hi)
    assert np.array_equal(lo, img) and np.array_equal(hi, 1 - img)
    bad = owned.copy()
    bad[0, 0] = bad[world - 1, 0]  # a tile owned twice / one missing
    with pytest.raises(ap.AbsplatError):
        ap.as_untile(W, H, tile, world, cap, bad, n_owned, tm_lo, tm_hi)


def test_checked_build_is_the_same_abi():
    """The checked build (device bounds checks, tools/checked_run.sh) exports the same ABI."""
    from paper_2503_00308_b200 import build as b
    lib = b.LIB_CHECKED
    if not os.path.exists(lib):
        pytest.skip("checked build not present")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(_abi.declared_functions()) <= exported


def _header_struct_fields(name):
    """(ctype, field) pairs of a typedef struct in include/absplat.h (comments stripped;
    pointers map to c_void_p, arrays to ctype * n)."""
    import re
    base = {"int64_t": ctypes.c_int64, "int32_t": ctypes.c_int32, "double": ctypes.c_double,
            "size_t": ctypes.c_size_t, "float": ctypes.c_float}
    txt = open(_abi.HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    end = re.search(r"\}\s*" + name + ";", txt)
    assert end, name
    start = txt.rfind("typedef struct {", 0, end.start())
    body = txt[start + len("typedef struct {"):end.start()]
    out = []
    for decl in body.split(";"):
        decl = decl.replace("const ", "").strip()
        if not decl:
            continue
        ty, rest = decl.split(None, 1)
        ptr = ty.endswith("*")
        ty = ty.rstrip("*")
        for item in rest.split(","):
            item = item.strip()
            ptr_i = ptr or item.startswith("*")
            item = item.lstrip("*")
            m = re.match(r"(\w+)(?:\[(\d+)\])?$", item)
            assert m, item
            ct = ctypes.c_void_p if ptr_i else base[ty]
            if m.group(2):
                ct = ct * int(m.group(2))
            out.append((ct, m.group(1)))
    return out


@pytest.mark.parametrize("cname,pyname", [("as_stats", "AsStats"), ("as_camera", "AsCamera"),
                                           ("as_pose_box", "AsPoseBox"),
                                           ("as_scene_box", "AsSceneBox")])
def test_struct_mirrors_match_header(cname, pyname):
    """The ctypes mirrors have the header's fields, in order, with the same types and size."""
    hdr = _header_struct_fields(cname)
    py = getattr(_abi, pyname)._fields_
    assert [f for _, f in hdr] == [n for n, _ in py]
    for (ct, f), (n, t) in zip(hdr, py):
        assert ctypes.sizeof(ct) == ctypes.sizeof(t) and ctypes.alignment(ct) == ctypes.alignment(t), f
        if not issubclass(t, ctypes.Array):
            assert ct is t, (f, ct, t)
