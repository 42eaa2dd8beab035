"""Randomized parity sweep over the optional method paths (on top of tools/parity_sweep.py's
random pose boxes): backward MatrixInv bounds (NEXT-4), adaptive Taylor order, the linear blend
(NEXT-1), private per-Gaussian mean intervals and opacity intervals (NEXT-2), each case against
the fp64 oracle in the same mode (1e-4, integer statistics equal).
usage: python tools/feature_sweep.py [n] [seed0]"""
import copy
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from oracle import pyoracle as oracle  # noqa: E402
from paper_2503_00308_b200 import Context  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
ctx = Context(0)
fails, rows, worst = [], [], 0.0
t0 = time.time()
for seed in range(seed0, seed0 + n):
    w, tile, batch = _case(seed)
    rng = np.random.default_rng(seed + 7)
    w = copy.deepcopy(w)
    feats = []
    if rng.uniform() < 0.3:
        w.pose_box = dict(w.pose_box, inv_backward=1)
        feats.append("backward")
    if rng.uniform() < 0.3:
        w.pose_box = dict(w.pose_box, k_tol=float(10 ** rng.uniform(-8, -4)), k_max=int(rng.choice([12, 24])))
        feats.append("adaptive_k")
    N = w.N
    if rng.uniform() < 0.3:  # private mean intervals on a random subset, opacity intervals
        sb = dict(w.scene_box) if w.scene_box is not None else dict(
            n_groups=0, group_of=None, dir=None, shift_lo=None, shift_hi=None, parts=[1, 1, 1],
            col_lo=None, col_hi=None, op_lo=None, op_hi=None)
        lo = np.zeros((N, 3), np.float32)
        hi = np.zeros((N, 3), np.float32)
        sel = rng.uniform(size=N) < 0.2
        hi[sel] = rng.uniform(0, 0.02, (int(sel.sum()), 3)).astype(np.float32)
        sb["priv_lo"], sb["priv_hi"] = lo, hi
        if rng.uniform() < 0.5:
            o = np.asarray(w.opacity, np.float32)
            sb["op_lo"] = np.clip(o - 0.1, 0, 1).astype(np.float32)
            sb["op_hi"] = o.copy()
        w.scene_box = sb
        feats.append("private")
    linear = rng.uniform() < 0.25 and "private" not in feats
    if linear:
        feats.append("linear")
    ctx.load_workload(w)
    if linear:
        ctx.as_set_blend(1)
    try:
        lo, hi, st = ctx.as_render_bounds(tile, batch)
    except Exception as ex:  # a mode a configuration does not support (e.g. n > 9 linear)
        ctx.as_set_blend(0)
        rows.append(dict(seed=seed, feats=feats, skipped=str(ex)[:80]))
        print(json.dumps(rows[-1]), flush=True)
        continue
    finally:
        if linear:
            ctx.as_set_blend(0)
    olo, ohi, ost = oracle.render_bounds(w, tile=tile, mode=2 if linear else 0)
    lo, hi = lo.cpu().numpy(), hi.cpu().numpy()
    err = float(max(np.abs(lo - olo).max(), np.abs(hi - ohi).max()))
    same = all(st[k] == ost[k] for k in ("pairs", "active_pairs", "uncertain_pairs", "fails",
                                            "dropped"))
    ok = err <= 1e-4 and same and st["order_violations"] == 0
    worst = max(worst, err)
    rows.append(dict(seed=seed, cfg=w.name, feats=feats, n_vars=st["n_vars"], tile=tile,
                     err=err, stats_equal=same, ok=ok))
    print(json.dumps(rows[-1]), flush=True)
    if not ok:
        fails.append(seed)
ctx.close()
done = [r for r in rows if "ok" in r]
print(f"\n| cases | skipped | failed | max abs err | backward | adaptive_k | private | linear | wall s |")
print(f"|---|---|---|---|---|---|---|---|---|")
cnt = {f: sum(1 for r in done if f in r["feats"]) for f in ("backward", "adaptive_k", "private", "linear")}
print(f"| {len(done)} | {len(rows) - len(done)} | {len(fails)} {fails[:10]} | {worst:.2e} | "
      f"{cnt['backward']} | {cnt['adaptive_k']} | {cnt['private']} | {cnt['linear']} | {time.time() - t0:.0f} |")
