"""Per-rank phase times of an emulated N-rank tile-sharded C4 render (as_render_shard on one
GPU), for a few chunk targets: python tools/shard_probe.py [N]."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2503_00308_b200 import Context  # noqa: E402
from workloads import make_config  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = make_config("C4")
ctx = Context(0)
ctx.load_workload(w)
nt = ctx.n_tiles(16)
per = -(-nt // N)
cap = per + max(1, per // 4)
lo = torch.empty((cap, 256, 3), device='cuda')
hi = torch.empty_like(lo)
for ct in (0, 400, 600, 900, 1400):
    ctx.as_set_chunk_target(ct)
    for it in range(3):
        st = ctx.as_render_shard(16, 24, 3, N, cap, lo, hi, stats=True)[-1]
    print(ct, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()
               if k.startswith('ms_') or k in ('pairs', 'n_items', 'host_syncs')})
