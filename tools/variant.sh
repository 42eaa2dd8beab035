#!/bin/bash
# Build an A/B variant of the library: k_tile.cu recompiled with extra flags, linked with the
# default build's other objects.  usage: tools/variant.sh <name> "<nvcc flags>"
set -e
cd "$(dirname "$0")/../paper_2503_00308_b200"
python -c "import build; build.build()" >/dev/null
mkdir -p /tmp/variant_$1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include \
  --expt-relaxed-constexpr $2 -c csrc/k_tile.cu -o /tmp/variant_$1/k_tile.o
objs=$(ls csrc/build/*.o | grep -v k_tile.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o libabsplat_$1.so $objs /tmp/variant_$1/k_tile.o -ldl
echo built libabsplat_$1.so
