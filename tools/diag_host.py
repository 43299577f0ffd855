"""Host time per façade call / prepare step of one C3 construction (no
profiler): wall clock around each method, and the CUDA-event span of the
whole construction.  Shows whether the host or the device is the critical
path."""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

T = defaultdict(float)
N = defaultdict(int)
EV = []          # (start, duration, name) of the current iteration (TIMELINE=1)
T0 = [0.0]


def wrap(cls, name):
    f = getattr(cls, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            T[name] += time.perf_counter() - t0
            N[name] += 1
            EV.append((t0 - T0[0], time.perf_counter() - t0, name))
    setattr(cls, name, g)


_call = engine.call


def timed_call(name, *a):
    t0 = time.perf_counter()
    try:
        return _call(name, *a)
    finally:
        T["call:" + name] += time.perf_counter() - t0
        EV.append((t0 - T0[0], time.perf_counter() - t0, "call:" + name))
        N["call:" + name] += 1


engine.call = timed_call
for m in ("_up_index", "_up"):
    f0 = getattr(engine, m)

    def mk(f0, m):
        def g(*a, **k):
            t0 = time.perf_counter()
            try:
                return f0(*a, **k)
            finally:
                T[m] += time.perf_counter() - t0
                N[m] += 1
        return g
    setattr(engine, m, mk(f0, m))
for m in ("create_neurons", "add_poisson_source", "connect_fixed_indegree_distributed", "prepare", "_prepare_rank",
          "_prepare_tables", "_fused_sort", "_fused_eager", "_fused_ready", "_fused_check", "_sort_pending",
          "_alloc_propagation", "_dist_target", "_routes", "_compact", "_delay_stats", "_dist", "_present_ranks",
          "_final_pieces", "_assign", "_syn_class", "_dist_accounting", "_defer", "_tables", "_replay_start",
          "_replay_finish", "_dist_replay", "_dist_tables", "connect", "_emit_records", "_write_syn",
          "_write_syn_random", "_make_wide", "_fused_off", "_gen_deferred", "_prepare_tables", "connect_remote",
          "_remote", "_remote_deferred", "_connect_local", "_validate_conn",
          "_replay_positions"):
    wrap(engine.Cluster, m)
neur = int(os.environ.get("NEURONS", "100000"))
P = models.BalancedParams(neurons_per_rank=neur, k_exc=9000, k_inh=2250)
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
if world > 1:   # under torchrun: one rank per GPU, rank 0 prints
    import torch.distributed as dist
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
cfg = api.SimConfig(n_ranks=world, comm_mode="collective" if world > 1 and not os.environ.get("C4") else "p2p",
                    seed=12345)
for it in range(4):
    T.clear()
    N.clear()
    EV.clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    T0[0] = t0
    e0.record()
    if world > 1:
        dist.barrier()
    c = engine.Cluster(cfg)
    if os.environ.get("C2"):   # PD microcircuit, full scale
        models.build_microcircuit(c, models.MicrocircuitParams(scale=1.0))
    elif os.environ.get("C4"):   # multi-area, 4 areas per rank, p2p
        areas = [models.AreaSpec(f"A{i:02d}", 129_063, 1) for i in range(4 * world)]
        asg, _ = models.pack_areas(areas, world)
        models.build_multi_area(c, areas, asg, models.MultiAreaParams(k_intra_exc=3600, k_intra_inh=900,
                                                                      k_inter=44, delay_steps=15))
    else:
        models.build_balanced_network(c, P)
    c.prepare()
    e1.record()
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    if rank == 0:
        print(f"iter {it}: host {1e3 * host:.2f} ms, gpu span {e0.elapsed_time(e1):.2f} ms, "
              f"store {c.ranks[rank].store_path}", flush=True)
    del c
if rank == 0 and os.environ.get("TIMELINE"):   # host timeline of the last iteration
    for a, d, name in sorted(EV):
        print(f"  t={1e3 * a:8.3f} ms  {1e3 * d:7.3f} ms  {name}")
if rank == 0:
    for k in sorted(T, key=lambda k: -T[k]):
        print(f"  {k:40s} {1e3 * T[k]:8.3f} ms  x{N[k]}")
if world > 1:
    dist.destroy_process_group()
