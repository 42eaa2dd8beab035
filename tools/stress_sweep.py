"""Randomized sweep of the exception-machinery stress workloads (workloads.stacked_config: near-
opaque Gaussians in a thin slab under a rotation box: long windows past the 128-bit masks, many
E_G operands, finalisation records past the staged ones, transmittance underflow) and of the
near-plane and exact-tie workloads, with random sizes, rotation widths, on-axis fractions, slab
depths, tile sizes and batches, against the fp64 oracle (1e-4, integer statistics equal).
usage: python tools/stress_sweep.py [n] [seed0]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from oracle import pyoracle as oracle  # noqa: E402
from paper_2503_00308_b200 import Context  # noqa: E402
from workloads import nearplane_config, stacked_config, ties_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 70000
ctx = Context(0)
ctx.as_debug_counters(1)
rows, fails, t0 = [], [], time.time()
fired = {}
for seed in range(seed0, seed0 + n):
    rng = np.random.default_rng(seed)
    kind = ["stacked", "stacked", "nearplane", "ties"][seed % 4]
    if kind == "stacked":
        w = stacked_config(N=int(rng.integers(50, 500)), res=int(rng.choice([24, 32, 40])),
                           seed=int(rng.integers(0, 1000)), rot_deg=float(rng.uniform(0.05, 2.5)),
                           depth_spread=float(10 ** rng.uniform(-3.5, -1.5)),
                           opacity=(float(rng.uniform(0.3, 0.9)), 0.99),
                           axis_frac=float(rng.choice([0.0, rng.uniform(0.2, 0.9)])))
    elif kind == "nearplane":
        w = nearplane_config(seed=int(rng.integers(0, 1000)), eps_tz=float(10 ** rng.uniform(-4, -2.5)),
                             rot_deg=float(rng.choice([0.0, rng.uniform(0, 1)])))
    else:
        w = ties_config(seed=int(rng.integers(0, 1000)), rot_deg=float(rng.choice([0.0, rng.uniform(0, 2)])))
    tile = int(rng.choice([8, 16, 32]))
    batch = int(rng.choice([1, 7, 16, 24, 64, 128]))
    ctx.load_workload(w)
    lo, hi, st = ctx.as_render_bounds(tile, batch)
    c = ctx.as_debug_counters()
    for k, v in c.items():
        fired[k] = fired.get(k, 0) + v
    olo, ohi, ost = oracle.render_bounds(w, tile=tile)
    err = float(max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max()))
    same = all(st[k] == ost[k] for k in ("pairs", "active_pairs", "uncertain_pairs", "fails",
                                            "dropped", "straddles"))
    ok = err <= 1e-4 and same and st["order_violations"] == 0
    rows.append(dict(seed=seed, kind=kind, tile=tile, batch=batch, err=err, stats_equal=same,
                     uncertain=st["uncertain_pairs"], max_window=st["max_window"],
                     straddles=st["straddles"], ok=ok))
    print(json.dumps(rows[-1]), flush=True)
    if not ok:
        fails.append(seed)
ctx.as_debug_counters(0)
ctx.close()
print("\nrare-path counters:", fired)
print(f"\n| cases | failed | max abs err | windows > 128 | straddling cases | wall s |")
print(f"|---|---|---|---|---|---|")
print(f"| {len(rows)} | {len(fails)} {fails[:10]} | {max(r['err'] for r in rows):.2e} | "
      f"{sum(r['max_window'] > 128 for r in rows)} | {sum(r['straddles'] > 0 for r in rows)} | {time.time() - t0:.0f} |")
