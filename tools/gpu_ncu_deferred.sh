#!/bin/bash
# ncu --set full of the deferred-key COPS kernels and the result gathers of one bench step.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lookup|k_insert|k_st_gather" -s 0 -c 6 \
    -o gpurun_out/prof_deferred python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_deferred.log 2>&1
tail -3 gpurun_out/ncu_deferred.log
