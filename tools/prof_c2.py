"""One full-scale C2 (PD microcircuit) construction, for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09502_b200 import api, engine, models  # noqa: E402

c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
models.build_microcircuit(c, models.MicrocircuitParams(scale=1.0))
c.prepare()
torch.cuda.synchronize()
print("done")
