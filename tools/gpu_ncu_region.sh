#!/bin/bash
# ncu capture of one launch: K=kernel regex, S=launches to skip, MODE=kernel|application
mkdir -p gpurun_out
K=${1:-k_st_probe}; S=${2:-0}; NAME=${3:-prof_probe}
timeout 900 ncu --set full --replay-mode ${MODE:-kernel} --clock-control none --import-source on -k regex:"$K" -s $S -c 1 \
    -o gpurun_out/$NAME python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu ${LOC:+--locality $LOC} > gpurun_out/ncu_$NAME.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_$NAME.log | tail -6
