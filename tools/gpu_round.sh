#!/bin/bash
# One GPU session: bench line, sweep, reference arm, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 2 --no-e2e --no-cpu --sweep gpurun_out/sweep.json > /dev/null 2> gpurun_out/sweep.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|tile|split" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_insert|k_lookup" -s 6 -c 2 \
    -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
