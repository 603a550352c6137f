#!/bin/bash
# functor + multi-value tests, then the multi-value CLI sweep at 2^24 and configs[2] at 2^27
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_functors.py tests/test_gpu_multi.py tests/test_bench_cli.py -m gpu -x -q > gpurun_out/pytest_sel.txt 2>&1
tail -15 gpurun_out/pytest_sel.txt
timeout 600 python -m paper_2009_07914_b200.bench multi-sweep --n 16777216 --multiplicities 1,16,256,4096 \
   --layout packed --group-width 8 --repeats 3 --out gpurun_out/q_multi.csv 2>&1 | tail -8
timeout 600 python tools/bench_configs.py --which multi --reps 3 2>&1 | tail -2
