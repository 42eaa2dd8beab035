#!/usr/bin/env python
"""Width-driven refinement curve (NEXT-3, P:667 / P:710 trend): MPG of the union vs number of
sub-boxes on a workload, with the render time of each partition (GPU, through the C ABI).
usage: python tools/refine_curve.py [C4] [max_subboxes]  -> JSON lines + a markdown table"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_00308_b200 import Context, refine  # noqa: E402
from workloads import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 16
w = make_config(name)
with Context(0) as ctx:
    ctx.load_workload(w)
    t0 = time.time()
    parts, hist = refine.refine_width(ctx, w.pose_box, w.scene_box, tile=w.tile, batch=w.batch,
                                      max_subboxes=budget)
    wall = time.time() - t0
    # the final partition rendered as one call (union inside the library)
    lo, hi, st = ctx.as_render_bounds(w.tile, w.batch)
    final = refine._mpg(lo, hi)
print("| sub-boxes | MPG of the union | sum of sub-box render ms |")
print("|---|---|---|")
for n, m, ms in hist:
    print(f"| {n} | {m:.4f} | {ms:.1f} |")
print(json.dumps({"workload": name, "history": hist, "final_mpg_one_call": final,
                  "final_ms_one_call": st["ms_total"], "driver_wall_s": wall,
                  "axes_split": [int(a) for a in (parts[:, :, 1] - parts[:, :, 0] <
                                                  (refine.box_bounds(w.pose_box, w.scene_box)[:, 1]
                                                   - refine.box_bounds(w.pose_box, w.scene_box)[:, 0]) - 1e-15).sum(0)]}))
