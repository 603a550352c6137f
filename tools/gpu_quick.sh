#!/bin/bash
# quick iteration: targeted tests + bench line + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_single.py -q -m gpu -p no:cacheprovider -x --timeout 300 2>&1 | tail -5 > gpurun_out/pytest_single.txt
python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|tile" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
