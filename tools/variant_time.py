#!/usr/bin/env python
"""Tile-kernel time and counts of C4 variants (what the exception machinery costs): the full
6-DoF box, translation only (no uncertain depth pairs), rotation only."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2503_00308_b200 import Context  # noqa: E402
from workloads import make_config  # noqa: E402

variants = {"6dof": None, "t_only": dict(eps_R=[0.0] * 3), "R_only": dict(eps_t=[0.0] * 3)}
with Context(0) as ctx:
    for name, ch in variants.items():
        w = make_config("C4")
        if ch:
            w.pose_box = dict(w.pose_box, **ch)
        ctx.load_workload(w)
        for _ in range(2):
            ctx.as_render_bounds(w.tile, w.batch)
        ts = []
        for _ in range(3):
            lo, hi, st = ctx.as_render_bounds(w.tile, w.batch)
            ts.append(st["tile_kernel_ms"])
        print(name, "tile ms %.2f" % min(ts), "active %.3e" % st["active_pairs"], "pairs", st["pairs"],
              "uncertain", st["uncertain_pairs"], "n", st["n_vars"],
              "ns/active-pair %.3f" % (min(ts) * 1e6 / st["active_pairs"]), flush=True)
