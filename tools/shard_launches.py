"""One emulated rank (3 of 8) of a tile-sharded C4 render, rendered 4 times (run under ncu for
the per-kernel launch list of a shard): python tools/shard_launches.py"""
import sys, torch
sys.path.insert(0, '.')
from paper_2503_00308_b200 import Context
from workloads import make_config
N = 8
w = make_config("C4")
ctx = Context(0)
ctx.load_workload(w)
nt = ctx.n_tiles(16); per = -(-nt // N); cap = per + max(1, per // 4)
lo = torch.empty((cap, 256, 3), device='cuda'); hi = torch.empty_like(lo)
for it in range(4):
    st = ctx.as_render_shard(16, 24, 3, N, cap, lo, hi, stats=True)[-1]
torch.cuda.synchronize()
print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items() if k.startswith('ms_') or k in ('pairs','n_items','host_syncs','graph_replay')})
