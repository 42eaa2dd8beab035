#!/bin/bash
# quick GPU iteration: parity tests, bench on all configs, optional ncu for one config
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
echo "tests_rc=$?"; tail -3 gpurun_out/gpu_tests.log
for c in ${CONFIGS:-C4 C2 C3 C5}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
if [ -n "$PROF" ]; then bash tools/ncu_profile.sh $PROF --config $PROF; fi
