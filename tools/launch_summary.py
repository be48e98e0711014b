"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, ni, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
tscale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
bscale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].split("<")[0].split("::")[-1]
    a = agg.setdefault(name, {"ids": set(), "us": 0.0, "gb": 0.0})
    a["ids"].add(r[ii])
    v = float(r[vi].replace(",", ""))
    if r[ni].startswith("gpu__time_duration"):
        a["us"] += v * tscale[r[ui]]
    elif r[ni].startswith("dram__bytes"):
        a["gb"] += v * bscale[r[ui]]
for name, a in agg.items():
    n = len(a["ids"])
    bw = a["gb"] / (a["us"] * 1e-6) if a["us"] else 0.0
    print(f"{name:26s} {n:4d} launches {a['us'] / 1000:9.3f} ms {a['us'] / n:9.1f} us each"
          f"  DRAM {a['gb'] / n:8.3f} GB each  {bw:7.0f} GB/s")
