#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 2 --no-e2e --no-cpu --sweep gpurun_out/sweep_on.json --locality on > gpurun_out/b_on.json 2>/dev/null
python bench.py --steps 2 --no-e2e --no-cpu --sweep gpurun_out/sweep_off.json --locality off > gpurun_out/b_off.json 2>/dev/null
bash tools/gpu_full.sh "k_insert|k_lookup" 6 2 prof_v3
