"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    n = r[ki].split("(")[0][:70]
    agg[n][0] += 1
    agg[n][1] += float(r[vi].replace(",", ""))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"{'launches':>8} {'total_us':>11} {'avg_us':>9}  kernel")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{c:8d} {t / 1e3:11.1f} {t / c / 1e3:9.2f}  {n}")
