"""Look-back statistics of pass A (variant built with -DSMX_FG_LBSTAT)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09502_b200 import _lib, api, engine, models  # noqa: E402

L = _lib.lib()
out = (ctypes.c_ulonglong * 4)()
for it in range(3):
    c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
    models.build_balanced_network(c, models.BalancedParams(neurons_per_rank=100_000, k_exc=9000, k_inh=2250))
    c.prepare()
    torch.cuda.synchronize()
    L.smx_fg_lbstat(out, 1)
    t, s, u, w = list(out)
    print(f"tiles {t}: steps/tile {s / max(t, 1):.2f}, descriptors/tile {u / max(t, 1):.2f}, waits/tile {w / max(t, 1):.2f}")
    del c
