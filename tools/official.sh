#!/bin/bash
# full round-end style run: gpu tests, smoke, default bench (C4, all keys), launch list + full
# ncu capture of k_tile on the bench command, clocks.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_full.log 2>&1; echo "gpu_tests rc=$?"
tail -3 gpurun_out/gpu_tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
bash tools/ncu_profile.sh C4 --config C4
