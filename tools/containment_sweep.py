"""Randomized soundness sweep (Theorem 1 on the GPU output): random reduced workloads and pose
boxes; concrete renders (the library's fp64 concrete renderer) at random points of the box,
its corners and centre must lie inside the GPU's [lo, hi].  Reports the worst violation.
usage: python tools/containment_sweep.py [n] [seed0] [poses]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_2503_00308_b200 import Context  # noqa: E402
from tests import helpers as H  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
poses = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ctx = Context(0)
rows, t0 = [], time.time()
for seed in range(seed0, seed0 + n):
    w, tile, batch = _case(seed)
    ctx.load_workload(w)
    lo, hi, st = ctx.as_render_bounds(tile, batch)
    lo, hi = lo.cpu().numpy().astype(np.float64), hi.cpu().numpy().astype(np.float64)
    ax = H.box_axes(w)
    var = [k for k in range(9) if ax[k][1] > ax[k][0]]
    rng = np.random.default_rng(seed)
    worst = 0.0
    for t in range(poses):
        if t == 0:
            xi = np.zeros(len(var))
        elif t <= 2:
            xi = np.full(len(var), 1.0 if t == 1 else -1.0)
        else:
            xi = rng.uniform(-1, 1, len(var))
        img = ctx.as_render_concrete(xi).cpu().numpy().astype(np.float64)
        worst = max(worst, float((lo - img).max()), float((img - hi).max()))
    rows.append(dict(seed=seed, cfg=w.name, tile=tile, n_vars=st["n_vars"], worst=worst))
    print(json.dumps(rows[-1]), flush=True)
ctx.close()
v = np.array([r["worst"] for r in rows])
print(f"\n| cases | poses each | violations > 1e-6 | > 1e-5 | worst | wall s |")
print(f"|---|---|---|---|---|---|")
print(f"| {n} | {poses} | {(v > 1e-6).sum()} | {(v > 1e-5).sum()} | {v.max():.1e} | {time.time() - t0:.0f} |")
