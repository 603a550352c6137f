#!/bin/bash
# ncu --set full of the staged region kernels (insert + lookup) of the second iteration of
# tools/prof_staged.py at 2^28 keys, load 0.95.
mkdir -p gpurun_out
NAME=${1:-prof_regions}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_st_insert_sg|k_st_lookup_q" -s 2 -c 2 \
    -o gpurun_out/$NAME python tools/prof_staged.py $((1<<28)) > gpurun_out/ncu_$NAME.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_$NAME.log | tail -3
