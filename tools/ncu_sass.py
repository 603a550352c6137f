"""Summarise an ncu report: key metrics + SASS hot spots (warp stall samples, instructions, active lanes).

usage: python tools/ncu_sass.py REPORT.ncu-rep [min_frac]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(det))
h = next(r)
want = {"Duration", "DRAM Throughput", "Achieved Occupancy", "Executed Ipc Active", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "No Eligible", "Executed Instructions", "Block Limit Shared Mem",
        "Block Limit Registers", "Registers Per Thread", "Memory Throughput"}
for row in r:
    if row[h.index("Metric Name")] in want:
        print(row[h.index("Kernel Name")][:28], "|", row[h.index("Metric Name")], row[h.index("Metric Value")],
              row[h.index("Metric Unit")])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.split("\n")
blocks, cur = [], None
for ln in src:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    rows = list(csv.reader(b[1:]))
    h = rows[0]
    data = [x for x in rows[1:] if len(x) == len(h)]
    si, ii, at = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index(
        "Avg. Threads Executed")
    tot = sum(int(x[si]) for x in data)
    toti = sum(int(x[ii]) for x in data)
    lanes = sum(int(x[ii]) * float(x[at]) for x in data) / max(1, toti)
    print(b[0][:90])
    print(f"  samples {tot}  warp-instr {toti}  avg active lanes {lanes:.1f}")
    sc = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(int(x[h.index(c)]) for x in data) for c in sc}
    print("  stalls:", ", ".join(f"{k[6:]}={v * 100 // max(1, tot)}%" for k, v in sorted(agg.items(), key=lambda y: -y[1])[:7]))
    for idx, x in enumerate(data):
        if int(x[si]) > tot * thr or int(x[ii]) > toti * thr * 1.5:
            st = sorted(((int(x[h.index(c)]), c[6:]) for c in sc), reverse=True)[:2]
            print(f"  {idx:5d} {int(x[si]):7d} {int(x[ii]):10d} {float(x[at]):5.1f} {x[1][:56]:56s} {st}")
