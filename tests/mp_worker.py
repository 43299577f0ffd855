"""Multi-process parity worker: one process per rank (torchrun, NCCL).

Builds a scenario through the GPU Cluster with only the local rank
materialised, checks that rank's tables against the golden fixtures, runs
the simulation with NCCL spike exchange, gathers the per-rank rasters and
checks the merged raster SHA on rank 0.  Exit code 0 = parity.
"""
import json
import faulthandler
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import scenarios  # noqa: E402
import tables  # noqa: E402
from namespaces import gpu_ns  # noqa: E402


if os.environ.get("MP_DUMP"):  # debugging aid: stacks of a hung worker
    faulthandler.dump_traceback_later(int(os.environ["MP_DUMP"]), exit=True)


def main(names):
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    gold_r = json.load(open(os.path.join(HERE, "golden", "rasters.json")))
    bad_all = []
    for name in names:
        c, sim = scenarios.SCENARIOS[name](gpu_ns())
        if c.n_ranks != world:
            continue
        c.prepare()
        gold = dict(np.load(os.path.join(HERE, "golden", f"tables_{name}.npz")))
        mine = tables.canon_gpu(c)
        want = {k: v for k, v in gold.items() if k.startswith(f"r{rank}/")}
        bad = tables.compare(mine, want)
        c.simulate(sim[0], sim[1], record=True)
        ev = c.rank_events(rank)
        parts = [None] * world
        dist.all_gather_object(parts, ev)
        if rank == 0:
            from paper_2512_09502_b200.api import Raster
            r = Raster.from_events(np.concatenate(parts), c.cfg.resolution_ms)
            if name not in scenarios.NON_DYADIC and r.sha256() != gold_r[name]["sha256"]:
                bad.append(f"raster {r.n_events} events vs {gold_r[name]['n_events']}")
        c.close()
        if bad:
            bad_all.append((name, rank, bad[:5]))
        print(f"[rank {rank}] {name}: {'OK' if not bad else bad[:3]}", flush=True)
    flags = [None] * world
    dist.all_gather_object(flags, bad_all)
    dist.destroy_process_group()
    if any(flags):
        sys.exit(1)


if __name__ == "__main__":
    main(sys.argv[1:])
