#!/bin/bash
# Build K2 ablation variants of libmace_b200.so into /tmp (profiling only) and, with --run,
# time each with tools/profile_k2.py.  Usage: tools/ablate_k2.sh [--build|--run]
set -e
cd "$(dirname "$0")/.."
VARIANTS="0 1 2 4 8 16 32 63"
if [ "$1" != "--run" ]; then
  mkdir -p ablate
  for v in $VARIANTS; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
      -Iinclude -DMACE_ABLATE=$v -shared -o ablate/libmace_ablate_$v.so \
      paper_1911_09278_b200/csrc/mace.cu paper_1911_09278_b200/csrc/cnn.cu paper_1911_09278_b200/csrc/layout.cpp \
      paper_1911_09278_b200/csrc/sysmat.cpp -lcudart &
  done
  wait
fi
if [ "$1" == "--run" ]; then
  for v in $VARIANTS; do
    echo "ablate=$v: $(MACE_LIB=$PWD/ablate/libmace_ablate_$v.so python tools/profile_k2.py --iters 6 2>&1 | tail -1)"
  done
fi
