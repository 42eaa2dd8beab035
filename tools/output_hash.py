"""Hash of the bound images of a fixed set of workloads (reduced C1-C5, full C2 / C4, random
sweep cases): run with two library builds (ABSPLAT_LIB) to check a refactor is bit-identical.
usage: python tools/output_hash.py"""
import hashlib
import sys

sys.path.insert(0, '.')
from paper_2503_00308_b200 import Context  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402
from workloads import make_config  # noqa: E402

SMALL = {"C1": dict(), "C2": dict(N=4000, res=72), "C3": dict(N=5000, res=56),
         "C4": dict(N=6000, res=72), "C5": dict(N=4000, res=72)}
ctx = Context(0)
cases = [(n, make_config(n, **kw), None, None) for n, kw in SMALL.items()]
cases += [("C2full", make_config("C2"), None, None), ("C4full", make_config("C4"), None, None)]
cases += [(f"seed{s}",) + _case(s) for s in (5906, 2049, 170189, 1234, 4321)]
for name, w, tile, batch in cases:
    ctx.load_workload(w)
    for ts in ((tile,) if tile else (8, 16, 32)):
        lo, hi, st = ctx.as_render_bounds(ts or w.tile, batch or w.batch)
        h = hashlib.sha1(lo.cpu().numpy().tobytes() + hi.cpu().numpy().tobytes()).hexdigest()[:16]
        print(name, ts, h, st["active_pairs"], st["uncertain_pairs"], flush=True)
ctx.close()
