"""Per-warp cycle split of k_tile2 (libabsplat_prof.so, -DKT2_PROF): batch barrier wait, bulk
copy wait, staging (phases A+B), walk.  ABSPLAT_LIB=.../libabsplat_prof.so python tools/kt2_prof.py C4"""
import sys

sys.path.insert(0, '.')
from paper_2503_00308_b200 import Context  # noqa: E402
from workloads import make_config  # noqa: E402

w = make_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
ctx = Context(0)
ctx.load_workload(w)
ctx.as_render_bounds(tile=w.tile, batch=w.batch)
ctx.as_debug_counters(1)
ctx.as_render_bounds(tile=w.tile, batch=w.batch)
c = list(ctx.as_debug_counters().values())
tot = sum(c[:4])
print({k: round(v / tot, 3) for k, v in zip(("barrier", "bulk_wait", "staging", "walk"), c[:4])})
