#!/bin/bash
# Runs the integer-pipe microbenchmarks on a B200 (under gpurun) with clocks sampled.
set -u
OUT=${GRAFT_REPO_ROOT:-.}/gpurun_out/micro
mkdir -p $OUT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $OUT/clocks.csv &
SMI=$!
nvidia-smi -q > $OUT/smi_q.txt 2>&1
./tools/micro/int_rate > $OUT/int_rate.jsonl 2>&1
./tools/micro/mulmod_rate > $OUT/mulmod_rate.jsonl 2>&1
kill $SMI
lscpu > $OUT/lscpu.txt 2>&1
nproc >> $OUT/lscpu.txt
cat $OUT/int_rate.jsonl $OUT/mulmod_rate.jsonl
