#!/bin/bash
# Round-2 final measurements: GPU test suite, bench line (default), reference arm, ncu launch
# list of one bench step, ncu --set full of both region kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
bash tools/gpu_ncu_region_pair.sh prof_regions_final > /dev/null 2>&1
cat gpurun_out/bench.json
timeout 600 python tools/bench_configs.py --reps 3 > gpurun_out/configs_final.jsonl 2> gpurun_out/configs_final.err
timeout 300 python tools/kprof.py 27 insert > gpurun_out/kprof_multi_insert.txt 2>&1
timeout 300 python tools/kprof.py 27 retrieve > gpurun_out/kprof_multi_retrieve.txt 2>&1
