"""Top CUDA source lines by executed instructions / stall samples from
`ncu -i X --page source --csv --print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out, hdr, cur, fn = [], None, None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if want and (fn is None or want not in fn):
        continue
    if hdr and len(r) > 8 and r[0] and r[2] == "-":
        ie = hdr.index("Instructions Executed")
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            out.append((float(r[ie]), float(r[ws]), cur, r[0], r[1][:96]))
        except ValueError:
            pass
tot = sum(x[0] for x in out) or 1
ts = sum(x[1] for x in out) or 1
print(f"total warp-instr {tot / 1e6:.1f}M  samples {ts:.0f}")
for x in sorted(out, reverse=True)[:top]:
    print(f"{100 * x[0] / tot:5.1f}% inst {100 * x[1] / ts:5.1f}% stall  {x[2]}:{x[3]}  {x[4]}")
