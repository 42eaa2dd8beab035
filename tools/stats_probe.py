"""Integer statistics of one random-sweep case, GPU against the oracle, at the case's tile
size and the others: python tools/stats_probe.py <seed>"""
import sys

sys.path.insert(0, '.')
from oracle import pyoracle as oracle  # noqa: E402
from paper_2503_00308_b200 import Context  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402

seed = int(sys.argv[1])
w, tile, batch = _case(seed)
ctx = Context(0)
ctx.load_workload(w)
keys = ("pairs", "active_pairs", "uncertain_pairs", "fails", "dropped", "straddles")
for ts, bs in ((tile, batch), (tile, 24), (8, 32), (32, 24)):
    _, _, st = ctx.as_render_bounds(ts, bs)
    _, _, ost = oracle.render_bounds(w, tile=ts)
    print(ts, bs, {k: (st[k], ost[k]) for k in keys if st[k] != ost[k]} or "equal", flush=True)
ctx.close()
