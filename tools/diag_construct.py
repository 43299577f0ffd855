import sys, time, gc
sys.path.insert(0, '/root/repo')
import os
if os.environ.get('SPIN'):
    from paper_2512_09502_b200 import _lib as _l0
    print('spin rc', _l0.lib().smx_set_sync_policy(int(os.environ['SPIN'])))
import torch
from paper_2512_09502_b200 import api, engine, models
from paper_2512_09502_b200 import _lib
P = models.BalancedParams(neurons_per_rank=100000, k_exc=9000, k_inh=2250)
import os
sys.path.insert(0, '/root/repo/tools')
from stall_sampler import Sampler
SAMP = Sampler(period=float(os.environ.get('PERIOD', '0.005'))).start()
x = torch.randn(8192, 8192, device='cuda')
for rep in range(int(os.environ.get('REPS', '4'))):
    if os.environ.get('PREWARM'):
        for _ in range(20): y = x @ x
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
    models.build_balanced_network(c, P)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    c.prepare()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    s = torch.cuda.memory_stats()
    if (t2 - t0) > 0.2 or os.environ.get('SAMPLE_ALL'):
        SAMP.summarise(t0, t2, top=int(os.environ.get('TOP', '8')))
    print(f"rep {rep}: build {1e3*(t1-t0):.1f} ms  prepare {1e3*(t2-t1):.1f} ms  timers={ {k: round(v*1e3,1) for k,v in c.timers.as_dict().items()} } "
          f"segments={s['segment.all.current']} alloc_retries={s['num_alloc_retries']} reserved={s['reserved_bytes.all.current']/1e9:.1f}GB cudaMalloc={s.get('num_device_alloc', '?')}", flush=True)
    if _lib.TIMELINE is not None:
        tl = _lib.TIMELINE
        ref = tl[0]
        for i, (name, h0, h1, e) in enumerate(tl):
            gpu = ref[3].elapsed_time(e)
            if os.environ.get('ALL') or h1 - h0 > 3e-3 or i == len(tl) - 1 or (i and gpu - ref[3].elapsed_time(tl[i-1][3]) > 3):
                print(f"    {name:24s} host {1e3*(h0-ref[1]):8.1f}->{1e3*(h1-ref[1]):8.1f} ms   gpu done {gpu:8.1f} ms")
        _lib.TIMELINE.clear()
    del c; gc.collect()
from paper_2512_09502_b200 import _lib
if _lib.TRACE is not None:
    for k, (n, t) in sorted(_lib.TRACE.items(), key=lambda x: -x[1][1]):
        print(f"  {k:28s} n={n:4d} total={1e3*t:9.1f} ms")
