"""One C3-style construction (+ optional propagation steps) for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--neurons", type=int, default=100_000)
ap.add_argument("--k-exc", type=int, default=9000)
ap.add_argument("--k-inh", type=int, default=2250)
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
for _ in range(a.repeat):
    c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
    models.build_balanced_network(c, models.BalancedParams(neurons_per_rank=a.neurons, k_exc=a.k_exc, k_inh=a.k_inh))
    c.prepare()
    for _ in range(a.steps):
        c.step()
    torch.cuda.synchronize()
    del c
print("done")
