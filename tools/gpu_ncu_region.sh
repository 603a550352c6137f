#!/bin/bash
mkdir -p gpurun_out
K=${1:-k_st_insert}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o gpurun_out/prof_$K python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$K.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_$K.log | tail -4
