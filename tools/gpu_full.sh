#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"${1:-k_insert|k_lookup}" -s ${2:-6} -c ${3:-2} \
    -o gpurun_out/${4:-prof} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
