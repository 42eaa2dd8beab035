mkdir -p gpurun_out/ab
for b in 12 16 24 32 48; do timeout 600 python bench.py --config C5 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab/c5_$b.json 2>/dev/null; done
for b in 16 32; do timeout 600 python bench.py --config C2 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab/c2_$b.json 2>/dev/null; done
