#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name kns=k_st --print-limit 20 python tools/sanitize_staged.py > gpurun_out/san_$tool.txt 2>&1
  echo "== $tool"; tail -8 gpurun_out/san_$tool.txt
done
