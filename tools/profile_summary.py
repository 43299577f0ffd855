"""Summaries committed under profiles/<round>/ from the raw ncu outputs in gpurun_out/<round>/.

  python tools/profile_summary.py gpurun_out/r1f profiles/r1f

writes launches_bench_summary.csv (per-kernel share of the bench launch list),
construct_dram_summary.csv (per-kernel time and DRAM bytes of one C3
construction), traffic.json (DRAM bytes of the generation + sort kernels per
synapse; bench.py reports it as roofline.traffic) and, when an .ncu-rep of a
--set full capture is present, ncu_full_summary.csv.
"""
import collections
import csv
import json
import os
import subprocess
import sys

SYNAPSES = 100_000 * 11_250
GEN_SORT = ("draw_", "tile_hist", "chunk_sum", "chunk_scan", "tile_offsets", "downsweep", "scan_",
            "fused_gen", "fb_")


def launch_rows(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = {}
    for r in rows[hdr + 1:]:
        try:
            d.setdefault(r[ii], {"k": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    return list(d.values())


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    lb = os.path.join(src, "launches_bench.csv")
    if os.path.exists(lb):
        agg = collections.defaultdict(lambda: [0, 0.0])
        for v in launch_rows(lb):
            a = agg[v["k"]]
            a[0] += 1
            a[1] += v.get("gpu__time_duration.sum", 0.0)
        tot = sum(a[1] for a in agg.values())
        with open(os.path.join(dst, "launches_bench_summary.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "launches", "total_us", "avg_us", "share"])
            for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
                w.writerow([k, c, round(t / 1e3, 1), round(t / c / 1e3, 2), round(t / tot, 4)])
    cd = os.path.join(src, "construct_dram.csv")
    if os.path.exists(cd):
        agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
        for v in launch_rows(cd):
            a = agg[v["k"]]
            a[0] += v.get("gpu__time_duration.sum", 0.0)
            a[1] += v.get("dram__bytes_read.sum", 0.0)
            a[2] += v.get("dram__bytes_write.sum", 0.0)
        gs_bytes, gs_ms = 0.0, 0.0
        with open(os.path.join(dst, "construct_dram_summary.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "time_ms", "dram_read_GB", "dram_write_GB"])
            for k, (t, r, wr) in sorted(agg.items(), key=lambda x: -x[1][0]):
                w.writerow([k, round(t / 1e6, 3), round(r / 1e9, 3), round(wr / 1e9, 3)])
                name = k.split("::")[-1]
                if any(name.startswith(p) or p in k for p in GEN_SORT):
                    gs_bytes += r + wr
                    gs_ms += t / 1e6
        fused = any("fused_gen" in k for k in agg)
        json.dump({"what": "DRAM bytes (read+write) of the generation + sort kernels of one C3 construction "
                           "(1.125e9 synapses), ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                           "--clock-control none, tools/prof_construct.py",
                   "store_path": "fused" if fused else "general",
                   "bytes_per_construction": gs_bytes, "bytes_per_synapse": gs_bytes / SYNAPSES,
                   "kernel_time_ms_serialised": gs_ms, "algorithmic_bytes_per_synapse": 20.0,
                   "path_minimum_bytes_per_synapse": 12.0 if fused else 20.0},
                  open(os.path.join(dst, "traffic.json"), "w"), indent=1)
    reps = [x for x in os.listdir(src) if x.endswith(".ncu-rep")]
    if reps:
        metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                   "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                   "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                   "sm__inst_issued.avg.pct_of_peak_sustained_active",
                   "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                   "launch__grid_size", "launch__shared_mem_per_block_dynamic"]
        with open(os.path.join(dst, "ncu_full_summary.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel"] + metrics)
            for rep in reps:
                out = subprocess.run(["ncu", "-i", os.path.join(src, rep), "--page", "raw", "--csv",
                                      "--metrics", ",".join(metrics)], capture_output=True, text=True).stdout
                rows = list(csv.reader(out.splitlines()))
                if len(rows) < 3:
                    continue
                h = rows[0]
                for r in rows[2:]:
                    w.writerow([r[h.index("Kernel Name")][:80]] + [r[h.index(m)] if m in h else "" for m in metrics])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
