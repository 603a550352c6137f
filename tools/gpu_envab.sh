#!/bin/bash
# A/B of env switches on one build: tools/gpu_envab.sh "VAR=1 VAR2=0" [reps] [tests]
# runs the single-value GPU tests (default env), then bench lines with and without the switches,
# and a launch list of the default.
mkdir -p gpurun_out
if [ -n "$3" ]; then
  timeout 900 python -m pytest $3 -q -m gpu -p no:cacheprovider -x 2>&1 | tail -4 > gpurun_out/pytest_ab.txt
  cat gpurun_out/pytest_ab.txt
fi
for v in A B; do
  for r in $(seq ${2:-2}); do
    if [ $v = B ]; then pre="env $1"; else pre=""; fi
    timeout 300 $pre python bench.py --no-cpu --no-e2e ${BENCH_ARGS} | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value'],3), d['verified'], {k: round(x,3) for k,x in d['phase_ms'].items()})"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches_A.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_A.csv 40 | grep -v "k_tile\|k_reset\|k_st_plan\|k_clear\|ms=   0.00"
