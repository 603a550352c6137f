#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=k_ --print-limit 20 \
      python tools/sanitize_multi.py > gpurun_out/san_multi_$tool.txt 2>&1
  echo "== $tool"; tail -6 gpurun_out/san_multi_$tool.txt
done
