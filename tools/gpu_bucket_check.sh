#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_kmer.py tests/test_gpu_scale.py -m gpu -x -q -k "bucket or kmer or configs3" > gpurun_out/pytest_sel.txt 2>&1; tail -3 gpurun_out/pytest_sel.txt
python tools/bench_configs.py --which bucket --reps 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bucket_elem.csv python tools/bucket_element_insert.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/bucket_elem.csv 14
