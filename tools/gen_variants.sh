for v in 0 1 2 3; do
  echo "variant $v"
  SMX_GEN_VARIANT=$v timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2512_09502_b200 import api, engine, models
for r in range(3):
    c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345), profile=True)
    models.build_balanced_network(c, models.BalancedParams(neurons_per_rank=100000, k_exc=9000, k_inh=2250))
    torch.cuda.synchronize()
    print('gen ms', round(c.kernel_ms('gen'), 2))
    del c
" 2>&1 | tail -1
done
