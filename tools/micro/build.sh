#!/bin/bash
# Builds the micro-benchmarks (sm_100a) against the SHARED CUDA runtime, so no executable
# embeds the static runtime's symbol table.  Run on the GPU box before run_*.sh.
set -e
cd "$(dirname "$0")"
INC=../../paper_2509_12494_b200/csrc
for s in ${@:-int_rate bfly_rate mulmod_rate pipe_mix pipe_mix2 shoup_rate}; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cudart shared \
    -I "$INC" -o "$s" "$s.cu"
done
