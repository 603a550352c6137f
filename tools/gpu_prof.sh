#!/bin/bash
# launch list with DRAM bytes + one full capture of the probe kernels
mkdir -p gpurun_out
python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_|tile" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_insert|k_lookup|k_loc_scatter|k_unpermute" -s 8 -c 5 \
    -o gpurun_out/prof_loc python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
