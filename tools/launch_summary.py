"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].split("<")[0].split("::")[-1]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale[r[ui]]
for name, (cnt, us) in agg.items():
    print(f"{name:32s} {cnt:5d} launches {us / 1000:10.3f} ms total {us / cnt:10.1f} us each")
