"""Per-rank construction phase timers under torchrun (one process per GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
P = models.BalancedParams(neurons_per_rank=100_000, k_exc=9000, k_inh=2250)
cfg = api.SimConfig(n_ranks=world, comm_mode="collective", seed=12345)
SAMP = None
if os.environ.get("SAMPLE") and rank == 0:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from stall_sampler import Sampler
    SAMP = Sampler(period=float(os.environ.get("PERIOD", "0.0005"))).start()
for rep in range(int(os.environ.get("REPS", "3"))):
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = engine.Cluster(cfg, profile=True)
    models.build_balanced_network(c, P)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    c.prepare()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = c.ranks[rank]
    if SAMP is not None and rep == int(os.environ.get("REPS", "3")) - 1:
        print("-- build"); SAMP.summarise(t0, t1, top=int(os.environ.get("TOP", "25")))
        print("-- prepare"); SAMP.summarise(t1, t2, top=int(os.environ.get("TOP", "25")))
    print(f"rank {rank} rep {rep}: build {1e3 * (t1 - t0):.1f} prepare {1e3 * (t2 - t1):.1f} "
          f"gen {c.kernel_ms('gen'):.1f} sort {c.kernel_ms('sort'):.1f} records {st.n_records} nodes {st.n_nodes} "
          f"timers { {k: round(v * 1e3, 1) for k, v in c.timers.as_dict().items()} }", flush=True)
    from paper_2512_09502_b200 import _lib
    if _lib.TIMELINE is not None:
        tl = _lib.TIMELINE
        if rank == 0 and rep == int(os.environ.get("REPS", "3")) - 1:
            ref = tl[0]
            for i, (name, h0, h1, e) in enumerate(tl):
                gpu = ref[3].elapsed_time(e)
                print(f"    {name:24s} host {1e3 * (h0 - ref[1]):8.1f}->{1e3 * (h1 - ref[1]):8.1f} ms   gpu done {gpu:8.1f} ms")
        tl.clear()
    del c
dist.destroy_process_group()
