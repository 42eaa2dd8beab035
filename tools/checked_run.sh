#!/bin/bash
# Device-side bounds checks in lieu of compute-sanitizer (closed on this pool): the GPU parity,
# edge and multi-GPU suites against libabsplat_checked.so (-DABSPLAT_CHECKS: every gathered /
# ring / list / output index of the tile kernels checked, trap on the first violation).
mkdir -p gpurun_out
export ABSPLAT_LIB=$PWD/paper_2503_00308_b200/libabsplat_checked.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_comm.py \
  tests/test_gpu_random.py tests/test_private_means.py tests/test_linear_blend.py \
  tests/test_gpu_syncfree.py -q -m gpu \
  --timeout 300 -p no:cacheprovider > gpurun_out/checked_tests.log 2>&1
echo "checked tests rc=$?"; tail -3 gpurun_out/checked_tests.log
grep -c "DCHECK failed" gpurun_out/checked_tests.log
