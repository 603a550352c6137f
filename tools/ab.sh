#!/bin/bash
# A/B of two builds: B is built here with EXTRA="$1" into build_ab/ (travels with gpurun);
# on the GPU box: tools/ab.sh run [reps] -> bench values + launch lists for A (default) and B.
if [ "$1" != run ]; then
  make -C paper_2009_07914_b200/csrc -j8 BUILD=../../build_ab/obj OUT=../../build_ab/libcoophash_b200.so EXTRA="$1" | tail -1
  exit
fi
mkdir -p gpurun_out
for v in A B; do
  [ $v = B ] && export CH_LIB_PATH=$PWD/build_ab/libcoophash_b200.so
  for r in $(seq ${2:-2}); do
    timeout 300 python bench.py --no-cpu --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value'],3), {k: round(x,3) for k,x in d['phase_ms'].items()})"
  done
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  python tools/launches.py gpurun_out/launches_$v.csv 60 | grep -v "k_tile\|k_zero\|k_reset\|k_st_plan\|k_clear" | tail -18
done
