#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_single.py -m gpu -x -q -k "host" > gpurun_out/pytest_sel.txt 2>&1; tail -3 gpurun_out/pytest_sel.txt
timeout 900 python bench.py --steps 5 --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['e2e'], d['verified'])"
