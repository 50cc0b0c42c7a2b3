"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total ms, share, average us.

  python scripts/launch_summary.py LAUNCHES.csv[.gz]"""
import collections
import csv
import gzip
import re
import sys

path = sys.argv[1]
fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = [r for r in csv.reader(fh) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("<unnamed>::", "")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r[ui]]
    a = agg[name]
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale
tot = sum(a[1] for a in agg.values())
n = sum(a[0] for a in agg.values())
print(f"{'kernel':44s} {'launches':>9s} {'total_ms':>10s} {'share':>6s} {'avg_us':>9s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {c:9d} {t:10.3f} {100 * t / tot:5.1f}% {1e3 * t / c:9.2f}")
print(f"total {n} launches, {tot:.3f} ms (serialised, cold-cache ncu times)")
