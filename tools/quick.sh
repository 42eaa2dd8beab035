#!/bin/bash
# quick GPU iteration: parity + edge tests, then the C4 bench (no baselines)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/quick_tests.log
for c in ${CONFIGS:-C4}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
r=d['roofline']; s=d['stats']
print('$c', 'ms/step %.2f'%d['ms_per_step'], 'tile %.2f'%r['tile_kernel_ms_per_step'], 'frac %.3f'%r['frac'], 'setup %.2f bin %.2f pairs %.2f'%(s['ms_setup'],s['ms_bin'],s['ms_pairs']))
" 2>&1 | tail -1
done
