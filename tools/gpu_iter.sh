#!/bin/bash
# iteration: full GPU tests, bench line, launch list with DRAM bytes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --maxfail=10 --timeout 300 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_|tile" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
