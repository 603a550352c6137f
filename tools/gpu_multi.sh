#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x --timeout 300 2>&1 | tail -5
timeout 900 python tools/bench_configs.py --which multi --reps 2 2>&1 | tail -3
