"""Summarise an ncu launch-list CSV (last N launches)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
d = OrderedDict()
for r in rows[hdr_i + 1:]:
    d.setdefault((r[0], r[ki][:44]), {})[r[mi]] = r[vi]
for (i, k), m in list(d.items())[-last:]:
    f = lambda key: float(m.get(key, "nan").replace(",", "") or "nan")
    print(f"{i:>4} {k:44s} ms={f('gpu__time_duration.sum') / 1e6:8.3f} rd={f('dram__bytes_read.sum') / 1e9:7.2f}GB "
          f"wr={f('dram__bytes_write.sum') / 1e9:6.2f}GB hit={m.get('lts__t_sector_hit_rate.pct', '')}")
