#!/bin/bash
# Bench line + ncu launch list per environment setting:
#   tools/gpu_envsweep.sh "A=1 B=0" "A=0" ...   ("-" = no extra variables)
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  i=$((i+1))
  [ "$cfg" = "-" ] && cfg=""
  r=$(timeout 300 env $cfg python bench.py --no-cpu --no-e2e ${BENCH_ARGS} | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value'],3), d['verified'], {k: round(x,3) for k,x in d['phase_ms'].items()})")
  echo "[$cfg] $r"
  timeout 600 env $cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv \
      --log-file gpurun_out/launches_$i.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_$i.csv 40 | grep -v "k_tile\|k_reset\|k_st_plan\|k_clear\|ms=   0.00"
done
