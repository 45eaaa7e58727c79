"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[ki].split("(")[0]
    if "<" in r[ki]:
        name = r[ki].split("(")[0]
    agg[name[:70]][0] += 1
    agg[name[:70]][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
print(f"{len(rows) - 1} launches, {tot / 1e3:.1f} ms total (serialised, cold-cache under ncu)")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{100 * t / tot:6.2f}%  {t / 1e3:10.2f} ms  n={c:5d}  {k}")
