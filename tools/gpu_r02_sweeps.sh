#!/bin/bash
# Round-2 sweeps on the shipped schedule: g x load at 2^28 (bench.py --sweep), the reference
# CLI sweeps through the B200 bench CLI, configs[2]/[3] at 2^27 incl. Zipf s = 0.75, and the
# other single-value operations at 2^28 (misses, erase).
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/sweep_clocks_before.txt
timeout 900 python bench.py --steps 2 --no-e2e --no-cpu --sweep gpurun_out/r02_sweep_g_load.json > gpurun_out/r02_sweep_bench.json 2> gpurun_out/r02_sweep.err
timeout 600 python tools/ops_2p28.py > gpurun_out/r02_ops_2p28.jsonl 2> gpurun_out/r02_ops.err
for L in packed soa; do
  timeout 600 python -m paper_2009_07914_b200.bench single-sweep --n 1048576 --densities 0.8,0.9,0.95 \
     --layout $L --group-width 8 --repeats 10 --out gpurun_out/r02_cli_single_${L}_2p20.csv > gpurun_out/r02_cli_single_${L}.log 2>&1
done
timeout 900 python -m paper_2009_07914_b200.bench single-sweep --n 16777216 --densities 0.8,0.9,0.95 \
   --layout packed --group-width 8 --repeats 3 --out gpurun_out/r02_cli_single_packed_2p24.csv > gpurun_out/r02_cli_single_2p24.log 2>&1
timeout 900 python -m paper_2009_07914_b200.bench multi-sweep --n 16777216 --multiplicities 1,16,256,4096 \
   --layout packed --group-width 8 --repeats 3 --out gpurun_out/r02_cli_multi_2p24.csv > gpurun_out/r02_cli_multi.log 2>&1
timeout 900 python -m paper_2009_07914_b200.bench bucket-sweep --n 16777216 --r 16 --repeats 3 \
   --out gpurun_out/r02_cli_bucket_2p24.csv > gpurun_out/r02_cli_bucket.log 2>&1
timeout 600 python -m paper_2009_07914_b200.bench distributed-sweep --n 4194304 --r 4 --shards 1,2,4,8 --repeats 3 \
   --layout packed --group-width 8 --out gpurun_out/r02_cli_dist_2p22.csv > gpurun_out/r02_cli_dist.log 2>&1
timeout 1200 python tools/bench_configs.py --which multi,bucket --reps 2 > gpurun_out/r02_configs_2p27.jsonl 2> gpurun_out/r02_configs.err
timeout 1200 python tools/bench_configs.py --which multi --zipf 0.75 --reps 1 >> gpurun_out/r02_configs_2p27.jsonl 2>> gpurun_out/r02_configs.err
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/sweep_clocks_after.txt
ls gpurun_out | grep r02_
