"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
gi = hdr.index("Grid Size")
agg = collections.defaultdict(lambda: [0, 0.0])
tot, n = 0.0, 0
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki]
    v = float(r[vi].replace(",", ""))
    ns = v * {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1)
    key = name.split("(")[0].replace("void ", "").replace("chimera::", "").replace("<unnamed>::", "")
    agg[key][0] += 1
    agg[key][1] += ns
    tot += ns
    n += 1
print(f"launches {n}  total {tot/1e6:.2f} ms (serialised, cold-cache ncu replay)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e6:9.2f} ms {100*t/tot:5.1f}%  n={c:5d}  avg {t/c/1e3:8.1f} us  {k}")
