#!/bin/bash
# ncu (application replay) of the staged kernels on tools/prof_staged.py
mkdir -p gpurun_out
K=${1:-k_st_probe}; C=${2:-2}; NAME=${3:-prof_app}; N=${4:-16777216}
timeout 1200 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:"$K" -s 0 -c $C \
    -o gpurun_out/$NAME python tools/prof_staged.py $N > gpurun_out/ncu_$NAME.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_$NAME.log | tail -4
