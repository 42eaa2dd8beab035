"""Measure the bounds the GPU tests assert: TS / BS invariance of the bounds and containment
of GPU concrete renders (run on a B200: python tools/measure_tolerances.py)."""
import numpy as np, sys
sys.path.insert(0, '.')
from tests import helpers as H
from workloads import make_config
from paper_2503_00308_b200 import Context
SMALL = {"C2": dict(N=4000, res=72), "C3": dict(N=5000, res=56), "C4": dict(N=6000, res=72), "C5": dict(N=4000, res=72)}
ctx = Context(0)
def gr(w, t=None, b=None):
    ctx.load_workload(w)
    lo, hi, st = ctx.as_render_bounds(tile=t or w.tile, batch=b or w.batch)
    return lo.cpu().numpy().astype(np.float64), hi.cpu().numpy().astype(np.float64)
for name in ["C2", "C4"]:
    w = make_config(name, **SMALL[name])
    blo, bhi = gr(w, 16, 64)
    for t, b in ((8, 1), (8, 256), (16, 7), (32, 32), (32, 128)):
        lo, hi = gr(w, t, b)
        print("tsbs", name, t, b, max(np.abs(lo - blo).max(), np.abs(hi - bhi).max()))
for name in ["C2", "C4", "C5"]:
    w = make_config(name, **SMALL[name])
    lo, hi = gr(w)
    ax = H.box_axes(w)
    var = [k for k in range(9) if ax[k][1] > ax[k][0]]
    rng = np.random.default_rng(3)
    worst = -1.0
    for trial in range(64):
        xi = rng.uniform(-1, 1, len(var)) if trial else np.ones(len(var))
        img = ctx.as_render_concrete(xi).cpu().numpy().astype(np.float64)
        worst = max(worst, (lo - img).max(), (img - hi).max())
    print("contain", name, worst)
