O=gpurun_out/c2prof
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/prof_c2.py > $O/ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/c2prof/launches_c2.csv")) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    a = agg[r[ki][:100]]
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print("total ms", tot / 1e6)
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{v/1e6:9.3f} ms {n:6d}x  {k}")
PY
