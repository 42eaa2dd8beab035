#!/bin/bash
# round-2 probe: pipe microbenchmark + C4 bench + full ncu of k_tile with source
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipebench tools/pipebench.cu && timeout 120 /tmp/pipebench > gpurun_out/pipebench.txt 2>&1; echo "pipebench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --config ${CFG:-C4}"
timeout 600 $CMD > gpurun_out/plain_${CFG:-C4}.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_tile$ -s 1 -c 1 \
    -o gpurun_out/prof_${CFG:-C4}_${TAG:-r2} $CMD > gpurun_out/ncu_full_${CFG:-C4}.log 2>&1; echo "ncu rc=$?"
