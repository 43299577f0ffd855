"""Per-launch table (time, DRAM bytes) from an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[hdr + 1:]:
    try:
        d.setdefault(r[ii], {"k": r[ki][:34]})[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for k, v in d.items():
    if pat in v["k"]:
        print(k, f"{v['k']:34s} {v.get('gpu__time_duration.sum', 0) / 1e6:7.3f} ms  "
                 f"R {v.get('dram__bytes_read.sum', 0) / 1e9:6.2f} GB  W {v.get('dram__bytes_write.sum', 0) / 1e9:6.2f} GB")
