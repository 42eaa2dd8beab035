mkdir -p gpurun_out
for kv in 2; do for bs in 16 24 32 40; do
ABSPLAT_KTILE=$kv timeout 300 python bench.py --config C4 --batch $bs --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw_${kv}_$bs.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/sw_${kv}_$bs.json').read().strip().splitlines()[-1])
print('kver $kv bs $bs', 'tile %.2f'%d['roofline']['tile_kernel_ms_per_step'], 'grid', d['stats']['grid'])"
done; done
for bs in 4 8 12 16; do
ABSPLAT_KTILE=3 timeout 300 python bench.py --config C4 --batch $bs --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw_3_$bs.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/sw_3_$bs.json').read().strip().splitlines()[-1])
print('kver 3 bs $bs', 'tile %.2f'%d['roofline']['tile_kernel_ms_per_step'], 'grid', d['stats']['grid'])"
done
