#!/bin/bash
# Round-end style run (round 2): GPU tests, smoke, default bench (C4, all keys), reference arm,
# the other configs, the emulated multi-GPU ranks, then the ncu launch list and one full ncu
# capture each of k_tile2 (C4) and k_setup (C4).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests_full.log 2>&1; echo "gpu_tests rc=$?"
tail -3 gpurun_out/gpu_tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
for c in C1 C2 C3 C5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
for c in C4 C3; do for n in 2 4 8; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --emulate-world $n > gpurun_out/emu_${c}_$n.json 2>/dev/null; echo "emu $c $n rc=$?"
done; done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --config C4"
$CMD > gpurun_out/plain_C4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $CMD > gpurun_out/ncu_launch_C4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile2 -s 1 -c 1 -o gpurun_out/prof_C4_k_tile2 $CMD > gpurun_out/ncu_full_C4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_setup -s 1 -c 1 -o gpurun_out/prof_C4_k_setup $CMD > gpurun_out/ncu_setup_C4.log 2>&1
echo "ncu rc=$?"
