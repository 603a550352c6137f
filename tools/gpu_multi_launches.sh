#!/bin/bash
mkdir -p gpurun_out
python tools/multi_r1_probe.py 1
python tools/multi_r1_probe.py 16
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/multi_r1_launches.csv python tools/multi_r1_probe.py 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/multi_r1_launches.csv")))
h = rows[0] if rows else []
for r in rows:
    if len(r) > 10 and r[-3] in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
        pass
import collections
agg = collections.OrderedDict()
for r in rows[1:]:
    try:
        name, metric, val = r[4], r[-3], r[-1]
    except IndexError:
        continue
    if metric == "gpu__time_duration.sum":
        print(f"{name[:60]:60s} {val}")
PY
