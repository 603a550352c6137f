#!/bin/bash
# ncu --set full of the partition / gather passes of one staged insert + retrieve at 2^28
# (second iteration of tools/prof_staged.py), plus the deferred-key lookup kernel.
mkdir -p gpurun_out
NAME=${1:-prof_reorder}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_st_split|k_st_gather|k_lookup" \
    -s ${SKIP:-13} -c ${COUNT:-13} -o gpurun_out/$NAME python tools/prof_staged.py $((1<<28)) > gpurun_out/ncu_$NAME.log 2>&1
grep -v "^==PROF== Profiling" gpurun_out/ncu_$NAME.log | tail -4
