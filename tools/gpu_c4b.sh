set -x
O=gpurun_out/c4b
mkdir -p $O
timeout 900 python bench.py --workload c4 --steps 1 --warmup 1 > $O/c4_n1.json 2> $O/c4_n1.err
cat $O/c4_n1.json; tail -5 $O/c4_n1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 --model-ms 5 --prop-warmup-ms 0 > $O/ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/c4b/launches_c4.csv")) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    a = agg[r[ki][:90]]
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print("total ns", tot)
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{v/1e6:9.3f} ms {n:6d}x  {k}")
PY
