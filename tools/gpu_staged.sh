#!/bin/bash
# staged-path iteration: single-table GPU tests, bench line, launch list
mkdir -p gpurun_out
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests/test_gpu_single.py -q -m gpu -p no:cacheprovider -x --timeout 300 2>&1 | tail -25 > gpurun_out/pytest_single.txt
cat gpurun_out/pytest_single.txt
timeout 300 python bench.py --no-cpu ${LOC:+--locality $LOC} > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_|tile" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu ${LOC:+--locality $LOC} > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv 60 | grep -v "k_tile\|k_zero\|k_reset\|k_st_plan" | tail -30
