#!/bin/bash
# GPU tests (optionally a -k filter / file list) with the output kept in gpurun_out/.
mkdir -p gpurun_out
timeout ${T:-1500} python -m pytest ${@:-tests} -m gpu -x -q > gpurun_out/pytest_sel.txt 2>&1
tail -30 gpurun_out/pytest_sel.txt
