"""One random-sweep case against the oracle at several tile sizes / batches: max error, its
pixel, and the values.  usage: python tools/case_probe.py <seed>"""
import sys

import numpy as np

sys.path.insert(0, '.')
from oracle import pyoracle as oracle  # noqa: E402
from paper_2503_00308_b200 import Context  # noqa: E402
from tests.test_gpu_random import _case  # noqa: E402

seed = int(sys.argv[1])
w, tile, batch = _case(seed)
ctx = Context(0)
ctx.load_workload(w)
for ts, bs in ((tile, batch), (32, 24), (16, 1), (16, 24), (8, 32)):
    lo, hi, st = ctx.as_render_bounds(ts, bs)
    olo, ohi, ost = oracle.render_bounds(w, tile=ts)
    lo, hi = lo.cpu().numpy(), hi.cpu().numpy()
    el, eh = np.abs(lo - olo), np.abs(hi - ohi)
    k = np.unravel_index(np.argmax(np.maximum(el, eh)), el.shape)
    print(ts, bs, 'max err lo %.2e hi %.2e' % (el.max(), eh.max()), 'at', k,
          'gpu', lo[k], hi[k], 'oracle', olo[k], ohi[k], 'unc', st['uncertain_pairs'], flush=True)
ctx.close()
