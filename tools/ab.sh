#!/bin/bash
# A/B: default library vs ABSPLAT_LIB alternatives (in-tree builds), tile-kernel time
mkdir -p gpurun_out
for lib in default ${ALTS}; do
  if [ "$lib" = default ]; then unset ABSPLAT_LIB; else export ABSPLAT_LIB=$PWD/paper_2503_00308_b200/$lib; fi
  for c in ${CONFIGS:-C4}; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e ${BARGS} > gpurun_out/ab_${lib}_$c.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab_${lib}_$c.json').read().strip().splitlines()[-1])
print('$lib $c', 'ms %.2f'%d['ms_per_step'], 'tile %.2f'%d['roofline']['tile_kernel_ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'grid', d['stats']['grid'])"
  done
done
