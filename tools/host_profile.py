"""cProfile of the host side of one warm C3 construction (1 GPU): where the
Python time before the first generation launch goes."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

P = models.BalancedParams(neurons_per_rank=100_000, k_exc=9000, k_inh=2250)


def build():
    c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
    models.build_balanced_network(c, P)
    c.prepare()
    torch.cuda.synchronize()
    c.close()


for _ in range(3):
    build()
pr = cProfile.Profile()
pr.enable()
build()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(int(os.environ.get("TOP", "30")))
st.sort_stats("cumulative").print_stats("engine.py", int(os.environ.get("TOP", "30")))
