"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes): the LAST occurrence
of every kernel sequence of one bench step, in launch order."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
recs = {}
order = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    if key not in recs:
        recs[key] = {"name": d["Kernel Name"]}
        order.append(key)
    recs[key][d["Metric Name"]] = d["Metric Value"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
tot = 0.0
for key in order[-n:]:
    x = recs[key]
    ms = float(x.get("gpu__time_duration.sum", 0)) / 1e6 if "gpu__time_duration.sum" in x else 0
    rd = float(x.get("dram__bytes_read.sum", "0").replace(",", ""))
    wr = float(x.get("dram__bytes_write.sum", "0").replace(",", ""))
    tot += ms
    print(f"{x['name'][:48]:48s} ms={ms:8.3f} rd={rd/1e9:6.2f}GB wr={wr/1e9:6.2f}GB")
print(f"total {tot:.3f} ms")
