#!/bin/bash
# ncu --set full of one kernel of tools/prof_staged.py at 2^28 (second iteration):
# tools/gpu_ncu_kernel.sh REGEX SKIP NAME
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-1} -c 1 \
    -o gpurun_out/$3 python tools/prof_staged.py $((1<<28)) > gpurun_out/ncu_$3.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_$3.log | tail -3
