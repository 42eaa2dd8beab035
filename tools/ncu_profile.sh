#!/bin/bash
# Launch list + one full ncu capture of the hot kernel, per B200_PROFILING.md.
# usage: tools/ncu_profile.sh <tag> <bench args...>   (run under gpurun; writes gpurun_out/)
TAG=$1; shift
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^k_tile2?$ -s 1 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu_profile rc=$?"
