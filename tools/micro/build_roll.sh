#!/bin/bash
# builds the K5 rolling-accumulator trace tool (cnn.cu with -DK5_TRACE); extra flags are passed on
set -e
cd "$(dirname "$0")"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xptxas -v -DK5_TRACE "$@" -o k5roll k5_trace_roll.cu ../../paper_1911_09278_b200/csrc/cnn.cu -lcuda 2>&1 | grep -A2 "k_conv64_roll" | grep -i "stack\|Used" || true
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a "$@" -o k5roll_prod k5_trace_roll.cu ../../paper_1911_09278_b200/csrc/cnn.cu -lcuda
ls -la k5roll k5roll_prod
