"""Randomized sweep of the API paths around the render: sub-box range unions
(as_render_subboxes vs the oracle's), random chunk targets (vs the oracle), and tile sharding
(as_render_shard for every rank of a random world + as_untile, bit-identical to the full render).
usage: python tools/api_sweep.py [n] [seed0]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from oracle import pyoracle as oracle  # noqa: E402
from paper_2503_00308_b200 import Context  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 40000
ctx = Context(0)
fails, rows = [], []
t0 = time.time()
for seed in range(seed0, seed0 + n):
    w, tile, batch = _case(seed)
    rng = np.random.default_rng(seed + 11)
    ctx.load_workload(w)
    kind = ["subboxes", "chunks", "shard"][seed % 3]
    ok, err, info = True, 0.0, {}
    if kind == "subboxes":
        P = ctx.as_subbox_count()
        b = int(rng.integers(0, P + 1))
        e = int(rng.integers(b, P + 1))
        lo, hi, st = ctx.as_render_subboxes(b, e, tile, batch)
        olo, ohi, ost = oracle.render_subboxes(w, b, e, tile=tile)
        err = float(max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max()))
        ok = err <= 1e-4 and (b == e or st["uncertain_pairs"] == ost["uncertain_pairs"])
        info = dict(P=P, b=b, e=e)
    elif kind == "chunks":
        tgt = int(rng.choice([1, 3, 17, 64, 500]))
        ctx.as_set_chunk_target(tgt)
        try:
            lo, hi, st = ctx.as_render_bounds(tile, batch)
        finally:
            ctx.as_set_chunk_target(0)
        olo, ohi, ost = oracle.render_bounds(w, tile=tile)
        err = float(max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max()))
        ok = err <= 1e-4 and st["uncertain_pairs"] == ost["uncertain_pairs"]
        info = dict(target=tgt, items=st["n_items"])
    else:
        world = int(rng.integers(2, 9))
        nt = ctx.n_tiles(tile)
        cap = -(-nt // world) + int(rng.integers(1, 4))
        flo, fhi, _ = ctx.as_render_bounds(tile, batch)
        tl, th, owned, nown = [], [], [], []
        for r in range(world):
            a, b2, o, k, _ = ctx.as_render_shard(tile, batch, r, world, cap)
            tl.append(a)
            th.append(b2)
            owned.append(o)
            nown.append(k)
        lo, hi = ctx.as_untile(tile, world, cap, np.stack(owned), np.array(nown, np.int32),
                               torch.stack(tl), torch.stack(th))
        # a rank cuts its tiles into chunks for its own share of the pairs, so chunk boundaries
        # (and the fp32 order of the front-to-back composition) can differ from the full render:
        # equal within rounding, not necessarily bit for bit
        err = float(max((lo - flo).abs().max().item(), (hi - fhi).abs().max().item()))
        ok = err <= 1e-6 and sum(nown) == nt
        info = dict(world=world, cap=cap, bitwise=bool(torch.equal(lo, flo) and torch.equal(hi, fhi)))
    rows.append(dict(seed=seed, cfg=w.name, kind=kind, tile=tile, err=err, ok=ok, **info))
    print(json.dumps(rows[-1]), flush=True)
    if not ok:
        fails.append(seed)
ctx.close()
print("\n| cases | failed | subbox ranges | chunk targets | shard worlds | max abs err | wall s |")
print("|---|---|---|---|---|---|---|")
print(f"| {len(rows)} | {len(fails)} {fails[:10]} | {sum(r['kind'] == 'subboxes' for r in rows)} | "
      f"{sum(r['kind'] == 'chunks' for r in rows)} | {sum(r['kind'] == 'shard' for r in rows)} | "
      f"{max(r['err'] for r in rows):.2e} | {time.time() - t0:.0f} |")
