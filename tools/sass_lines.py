"""Attribute an ncu report's per-SASS-instruction metrics to CUDA source lines.

usage: python tools/sass_lines.py REPORT.ncu-rep KERNEL_SUBSTR CUBIN [top]
The cubin is the kernel's own (cuobjdump -xelf all lib.so); nvdisasm -g maps each
SASS instruction to its file:line (inlined code is attributed to the innermost line).
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, ksub, cubin = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.split("\n")
blocks, cur, name = {}, None, None
for ln in src:
    if ln.startswith('"Kernel Name"'):
        name = next(csv.reader([ln]))[1]
        cur = blocks.setdefault(name, []) if ksub in name and name not in blocks else None
    elif cur is not None:
        cur.append(ln)
(kname, rows), = [(k, v) for k, v in blocks.items()][:1]
r = list(csv.reader(io.StringIO("\n".join(rows))))
h = r[0]
ia, ii, isamp = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ith = h.index("Thread Instructions Executed")
data = [(int(x[ia], 16), int(x[ii] or 0), int(x[isamp] or 0), int(x[ith] or 0)) for x in r[1:] if len(x) > ith]
base = min(d[0] for d in data)
# nvdisasm line table for the kernel
m = re.search(r"chb::(\w+)(?:<([^>]*)>)?\(", kname)
frag = "".join(f"L{'b' if ty == 'bool' else 'i'}{val}E" for ty, val in re.findall(r"\((\w+)\)(\d+)(?=[,>]|$)", m.group(2) or ""))
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
sec, line, lines = None, None, {}
for ln in dis:
    if ln.startswith("//--------------------- .text."):
        sec = ln.split(".text.")[1].split(" ")[0]
        continue
    if sec is None or m.group(1) not in sec or (frag and f"{frag}E" not in sec):
        continue
    mm = re.match(r"\s*//## File \"([^\"]+)\", line (\d+)", ln)
    if mm:
        line = f"{mm.group(1).split('/')[-1]}:{mm.group(2)}"
        continue
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if mo:
        lines[int(mo.group(1), 16)] = line
agg = collections.defaultdict(lambda: [0, 0, 0])
for a, ins, s, th in data:
    key = lines.get(a - base, "?")
    agg[key][0] += ins
    agg[key][1] += s
    agg[key][2] += th
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(kname[:90], f"warp-instr {tot_i:.3e}  samples {tot_s}")
for k, (ins, s, th) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:28s} instr {ins / tot_i * 100:5.1f}%  stall {s / tot_s * 100:5.1f}%  lanes {th / max(ins, 1):4.1f}")
