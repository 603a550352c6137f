"""Round artifacts from tools/gpu_profile_round.sh outputs (gpurun_out/):
profiles/ncu_traffic.json (dram bytes per launch of the staged probe kernels, read by
bench.py's roofline), profiles/r01_ncu_staged_probe.txt (ncu_sass summary), bench lines
and the launch list summary."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "gpurun_out")
prof = os.path.join(ROOT, "profiles")
rep = os.path.join(out, "prof_probe_full.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
col = {name: h.index(name) for name in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                         "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct")}
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
traffic = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    key = "k_st_probe<0> (staged insert)" if "k_st_probe<0" in name else \
        "k_st_probe<1> (staged retrieve)" if "k_st_probe<1" in name else None
    if key is None or key in traffic:
        continue
    val = lambda m: float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    traffic[key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                    "duration_ms": val("gpu__time_duration.sum"),
                    "l2_hit_pct": float(r[col["lts__t_sector_hit_rate.pct"]]), "kernel": name[:90],
                    "source": "profiles/r01_ncu_staged_probe.txt (ncu --set full, kernel replay, 2^28 keys, "
                              "staged schedule)"}
json.dump(traffic, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1, sort_keys=True)
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass.py"), rep, "0.012"],
                      capture_output=True, text=True).stdout
open(os.path.join(prof, "r01_ncu_staged_probe.txt"), "w").write(summ)
for src, dst in (("bench.json", "r01_bench_latest.json"), ("bench_ref.json", "r01_bench_reference.json"),
                 ("launches.csv", "r01_launches_staged.csv")):
    if os.path.exists(os.path.join(out, src)):
        shutil.copy(os.path.join(out, src), os.path.join(prof, dst))
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), os.path.join(out, "launches.csv"),
                       "60"], capture_output=True, text=True).stdout
open(os.path.join(prof, "r01_launches_staged_summary.txt"), "w").write(summ)
print(json.dumps(traffic, indent=1))
