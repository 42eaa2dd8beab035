"""C5 exception-path census: rare-path counters and per-phase times at TS 8 / 16."""
import json
import sys

import torch

from paper_2503_00308_b200 import Context
from workloads import make_config

w = make_config("C5")
ctx = Context(0)
ctx.load_workload(w)
for tile, batch in ((8, 32), (16, 24)):
    ctx.as_debug_counters(1)
    lo, hi, st = ctx.as_render_bounds(tile=tile, batch=batch)
    c = ctx.as_debug_counters()
    ctx.as_debug_counters(0)
    for _ in range(3):
        lo, hi, st = ctx.as_render_bounds(tile=tile, batch=batch)
    torch.cuda.synchronize()
    print(json.dumps(dict(tile=tile, batch=batch, counters=c,
                          stats={k: st[k] for k in ("pairs", "uncertain_pairs", "n_items", "ring_len",
                                                    "max_window", "ms_tile", "ms_pairs", "ms_bin")})))
    sys.stdout.flush()
ctx.close()
