"""Propagation RTF on the C3 network (one construction, repeated runs)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--neurons", type=int, default=100_000)
ap.add_argument("--k-exc", type=int, default=9000)
ap.add_argument("--k-inh", type=int, default=2250)
ap.add_argument("--ms", type=float, default=100.0)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
c.use_graphs = not a.no_graph
models.build_balanced_network(c, models.BalancedParams(neurons_per_rank=a.neurons, k_exc=a.k_exc, k_inh=a.k_inh))
c.prepare()
for r in range(a.runs):
    rep = c.simulate(0.0, a.ms, record=True)
    print(f"run {r}: rtf={rep.rtf:.4f} us/step={rep.rtf * 100:.2f} spikes={rep.n_spike_events} "
          f"rate_hz={rep.n_spike_events / (a.neurons * a.ms * 1e-3):.2f} graph={c.use_graphs}", flush=True)
