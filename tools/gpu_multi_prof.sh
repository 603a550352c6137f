#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
  -k regex:"k_" --csv --log-file gpurun_out/launches_multi.csv python tools/bench_configs.py --which multi --reps 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_multi.csv 30
