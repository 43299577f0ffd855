"""torch.profiler trace of one construction on rank 0 under torchrun: prints
GPU-busy vs wall time and the largest idle gaps with the CPU op active then."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
P = models.BalancedParams(neurons_per_rank=100_000, k_exc=9000, k_inh=2250)
cfg = api.SimConfig(n_ranks=world, comm_mode="collective" if world > 1 else "p2p", seed=12345)


C4 = bool(os.environ.get("C4"))
if C4:  # multi-area model, 4 areas of 129,063 neurons per rank (bench.py --workload c4)
    areas = [models.AreaSpec(f"A{i:02d}", 129_063, 1) for i in range(4 * world)]
    assignment, _ = models.pack_areas(areas, world)
    MA = models.MultiAreaParams(k_intra_exc=3600, k_intra_inh=900, k_inter=44, delay_steps=15)
    cfg = api.SimConfig(n_ranks=world, comm_mode="p2p", seed=12345)


def build():
    torch.zeros(1, device="cuda")  # marks the start of the construction on the GPU timeline
    c = engine.Cluster(cfg)
    if C4:
        models.build_multi_area(c, areas, assignment, MA)
    else:
        models.build_balanced_network(c, P)
    c.prepare()
    torch.cuda.synchronize()
    return c


for _ in range(2):
    c = build()
    del c
dist.barrier()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=bool(os.environ.get("STACK"))) as prof:
    c = build()
dist.barrier()
if rank == 0:
    path = "/tmp/trace.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = sorted((e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
                 if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
    cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("python_function", "user_annotation", "cpu_op")]
    t0, t1 = gpu[0][0], gpu[-1][1]
    busy, last, gaps = 0.0, t0, []
    for a, b, n in gpu:
        if a > last:
            gaps.append((a - last, last, n))
        busy += max(0.0, b - max(a, last))
        last = max(last, b)
    print(f"rank0: GPU span {1e-3 * (t1 - t0):.2f} ms, busy {1e-3 * busy:.2f} ms, idle {1e-3 * (t1 - t0 - busy):.2f} ms")
    for g, at, n in sorted(gaps, reverse=True)[:25]:
        ops = [e["name"] for e in cpu if e["ts"] <= at + g / 2 <= e["ts"] + e["dur"]]
        print(f"  gap {1e-3 * g:6.3f} ms at {1e-3 * (at - t0):7.2f} ms before {n[:40]:40s} cpu: {ops[-3:]}")
    if os.environ.get("TIMELINE"):  # every GPU op >= 20 us: start, duration, stream, host launch time, name
        launch = {e["args"]["correlation"]: e["ts"] for e in ev
                  if e.get("cat") == "cuda_runtime" and "correlation" in e.get("args", {})}
        for e2 in sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
                         key=lambda e: e["ts"]):
            if e2["dur"] >= 20:
                lt = launch.get(e2.get("args", {}).get("correlation"))
                ls = f"{1e-3 * (lt - t0):7.2f}" if lt is not None else "      ?"
                print(f"  gpu {1e-3 * (e2['ts'] - t0):7.2f} +{1e-3 * e2['dur']:7.3f} ms s{e2.get('tid')} launched {ls}  "
                      f"{e2['name'][:60]}")

        fg = min((e for e in ev if e.get("ph") == "X" and e.get("cat") == "kernel" and "fused_gen" in e["name"]),
                 key=lambda e: e["ts"], default=None)
        if fg is not None and not C4:  # everything the GPU and the runtime did while the first pass A ran
            w0, w1 = fg["ts"], fg["ts"] + fg["dur"] + 300
            for e2 in sorted((e for e in ev if e.get("ph") == "X" and w0 <= e["ts"] <= w1 and
                              e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime", "cuda_driver")),
                             key=lambda e: e["ts"]):
                lt = launch.get(e2.get("args", {}).get("correlation"))
                ls = f"{1e-3 * (lt - t0):7.2f}" if lt is not None and e2.get("cat") != "cuda_runtime" else "      -"
                print(f"  win {e2.get('cat')[:7]:7s} {1e-3 * (e2['ts'] - t0):7.2f} +{1e-3 * e2['dur']:7.3f} ms "
                      f"s{e2.get('tid')} launched {ls}  {e2['name'][:60]}")
        for e2 in sorted(cpu, key=lambda e: e["ts"]):
            if e2.get("cat") == "python_function" and e2["dur"] >= 300 and "engine.py" in e2["name"]:
                print(f"  cpu {1e-3 * (e2['ts'] - t0):7.2f} +{1e-3 * e2['dur']:7.3f} ms  {e2['name'][:80]}")
    if os.environ.get("STACK"):  # host functions (>= 30 us) before the first generation launch
        first = min((a for a, b, n in gpu if "draw_" in n or "fused_gen" in n), default=t1)
        for e in sorted(cpu, key=lambda e: e["ts"]):
            if e["ts"] < first and e["dur"] >= 30 and e.get("cat") == "python_function":
                print(f"  host {1e-3 * (e['ts'] - t0):7.2f} +{1e-3 * e['dur']:6.3f} ms  {e['name'][:90]}")
dist.destroy_process_group()
