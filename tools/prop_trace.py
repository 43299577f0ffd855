"""GPU timeline of C3 propagation (torch profiler, CUDA activities): per
kernel name total time and count over one 20 ms simulate, plus the GPU busy
fraction per stream."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
models.build_balanced_network(c, models.BalancedParams(neurons_per_rank=100_000, k_exc=9000, k_inh=2250))
c.prepare()
c.simulate(0.0, 30.0, record=False)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    rep = c.simulate(0.0, 20.0, record=False)
    torch.cuda.synchronize()
print("rtf", rep.rtf)
prof.export_chrome_trace("/tmp/prop.json")
ev = json.load(open("/tmp/prop.json"))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in gpu)
t1 = max(e["ts"] + e["dur"] for e in gpu)
print(f"span {1e-3 * (t1 - t0):.3f} ms")
agg = collections.defaultdict(lambda: [0, 0.0])
per_stream = collections.defaultdict(float)
for e in gpu:
    a = agg[e["name"][:70]]
    a[0] += 1
    a[1] += e["dur"]
    per_stream[e.get("tid")] += e["dur"]
for k, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"{1e-3 * d:8.3f} ms {n:6d}x {1e-3 * d / n * 1e3:8.2f} us  {k}")
for s, d in per_stream.items():
    print(f"stream {s}: busy {1e-3 * d:.3f} ms")
# gaps on the main stream
main = sorted((e for e in gpu if e.get("tid") == 7), key=lambda e: e["ts"])
gaps = [main[i + 1]["ts"] - (main[i]["ts"] + main[i]["dur"]) for i in range(len(main) - 1)]
if gaps:
    print(f"main-stream gaps: total {1e-3 * sum(g for g in gaps if g > 0):.3f} ms, n={len(gaps)}, "
          f"max {max(gaps):.1f} us")
