"""Randomized sweep of explicit input partitions (as_set_subboxes: the refinement drivers' path):
each case cuts the box into a random set of axis-aligned sub-boxes by repeated random bisection
(any perturbed axis, group shifts included) and compares the union render with the oracle's on
the same explicit list (1e-4, integer statistics equal).  usage: python tools/partition_sweep.py [n] [seed0]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from oracle import pyoracle as oracle  # noqa: E402
from paper_2503_00308_b200 import Context  # noqa: E402
from tests import helpers as H  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 130000
ctx = Context(0)
rows, fails, t0 = [], [], time.time()
for seed in range(seed0, seed0 + n):
    w, tile, batch = _case(seed)
    rng = np.random.default_rng(seed + 3)
    ax = np.array(H.box_axes(w))  # [9, 2]
    var = [k for k in range(9) if ax[k, 1] > ax[k, 0]]
    parts = [ax.copy()]
    for _ in range(int(rng.integers(1, 9))):  # random bisections of random parts
        i = int(rng.integers(0, len(parts)))
        k = int(rng.choice(var))
        a = parts.pop(i)
        f = float(rng.uniform(0.2, 0.8))
        m = a[k, 0] + f * (a[k, 1] - a[k, 0])
        lo_p, hi_p = a.copy(), a.copy()
        lo_p[k, 1] = m
        hi_p[k, 0] = m
        parts += [lo_p, hi_p]
    bounds = np.stack(parts)
    w.pose_box = dict(w.pose_box, parts=[1] * 6)
    ctx.load_workload(w)
    ctx.as_set_subboxes(bounds)
    lo, hi, st = ctx.as_render_bounds(tile, batch)
    ow = w
    ow.pose_box = dict(w.pose_box, subboxes=bounds)
    olo, ohi, ost = oracle.render_bounds(ow, tile=tile)
    err = float(max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max()))
    same = all(st[k] == ost[k] for k in ("pairs", "active_pairs", "uncertain_pairs", "fails", "dropped"))
    ok = err <= 1e-4 and same and st["n_sub"] == len(parts)
    rows.append(dict(seed=seed, cfg=w.name, parts=len(parts), tile=tile, err=err, stats_equal=same, ok=ok))
    print(json.dumps(rows[-1]), flush=True)
    if not ok:
        fails.append(seed)
ctx.close()
print(f"\n| cases | failed | max abs err | mean parts | wall s |\n|---|---|---|---|---|")
print(f"| {len(rows)} | {len(fails)} {fails[:10]} | {max(r['err'] for r in rows):.2e} | "
      f"{np.mean([r['parts'] for r in rows]):.1f} | {time.time() - t0:.0f} |")
