"""profiles/ncu_traffic.json from an ncu --set full capture of the staged region kernels
(tools/gpu_ncu_region_pair.sh): DRAM bytes per launch, read by bench.py's roofline `traffic`.
usage: python tools/ncu_traffic.py REPORT.ncu-rep [source note]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]
note = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
col = {name: h.index(name) for name in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                         "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
names = {"k_st_insert_sg": "k_st_insert_sg (staged insert)", "k_st_lookup_q": "k_st_lookup_q (staged retrieve)"}
traffic = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    key = next((v for k, v in names.items() if k in name), None)
    if key is None or key in traffic:
        continue
    val = lambda m: float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    traffic[key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                    "duration_ms": val("gpu__time_duration.sum"),
                    "l2_hit_pct": float(r[col["lts__t_sector_hit_rate.pct"]]), "kernel": name[:90],
                    "source": note}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1, sort_keys=True)
print(json.dumps(traffic, indent=1))
