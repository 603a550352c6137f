#!/bin/bash
# ncu --set full of the deferred-key COPS kernels of one staged insert + lookup (second iteration)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_insert|k_lookup" -s 2 -c 2 \
    -o gpurun_out/prof_deferred python tools/prof_staged.py $((1<<28)) > gpurun_out/ncu_prof_deferred.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_prof_deferred.log | tail -3
