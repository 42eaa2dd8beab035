#!/usr/bin/env python
"""Small renders for compute-sanitizer: C1, a reduced C4 (6-DoF box, uncertain
depth pairs, exception ring) and a reduced C5 (TS 8, scene box, long windows), plus the
stacked stress case.  usage (under gpurun, one tool per call):
  compute-sanitizer --tool memcheck  python tools/sanitize.py
  compute-sanitizer --tool racecheck python tools/sanitize.py
  compute-sanitizer --tool synccheck python tools/sanitize.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_00308_b200 import Context  # noqa: E402
from workloads import make_config, stacked_config  # noqa: E402

cases = [("C1", make_config("C1")), ("C4-small", make_config("C4", N=3000, res=48)),
         ("C5-small", make_config("C5", N=3000, res=48)),
         ("stacked", stacked_config(N=150, rot_deg=2.0))]
with Context(0) as ctx:
    for name, w in cases:
        ctx.load_workload(w)
        lo, hi, st = ctx.as_render_bounds(tile=w.tile, batch=w.batch)
        print(name, "pairs", st["pairs"], "uncertain", st["uncertain_pairs"], "hi max",
              float(hi.max()), flush=True)
print("sanitize run done")
