#!/bin/bash
# headline bench (no e2e / cpu) + misses / erase at 2^28 + ncu launch list of one step
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --no-e2e --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('value', d['value'], 'ins', d['insert_gops'], 'ret', d['retrieve_gops'], d['phase_ms'], d['verified'])"
timeout 600 python tools/ops_2p28.py --reps 2 > gpurun_out/ops_q.jsonl 2> gpurun_out/ops_q.err; cat gpurun_out/ops_q.jsonl
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_q.csv | tail -40
fi
