"""Micro-benchmark of smx_sort_records on random keys (tuning knobs via env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_09502_b200 import _lib  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_125_000_000
M = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000
dev = torch.device("cuda")
torch.zeros(1, device=dev)
_lib.call("smx_pool_setup", 0)
g = torch.Generator(device=dev).manual_seed(1)
keys = torch.randint(0, M, (n,), device=dev, dtype=torch.int32, generator=g)
vals = torch.arange(n, device=dev, dtype=torch.int32)
scratch = torch.empty(2 * n, device=dev, dtype=torch.int32)
kb, vb = scratch[:n], scratch[n:]
counts = torch.empty(M, dtype=torch.int32, device=dev)
which = np.zeros(1, dtype=np.int32)
bits = max(1, int(M - 1).bit_length())
st = torch.cuda.current_stream().cuda_stream
ka, va = keys.clone(), vals.clone()
times = []
for it in range(int(os.environ.get('ITERS', '4'))):
    keys.copy_(ka)
    vals.copy_(va)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("smx_sort_records", keys.data_ptr(), vals.data_ptr(), kb.data_ptr(), vb.data_ptr(), n, bits, 0, 0,
              counts.data_ptr(), M, which.ctypes.data, st)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
out = vb if which[0] else vals
# check: stable sort of (key, original index)
if n <= 50_000_000 or os.environ.get("CHECK"):
    order = torch.argsort(ka.long() * n + va.long())
    ok = torch.equal(out[:n], va[order])
else:
    s = ka[out[:n].long()]
    ok = bool((s[1:] >= s[:-1]).all())
ref_counts = torch.bincount(ka.long(), minlength=M)[:M].to(torch.int32)
ok = ok and torch.equal(counts, ref_counts)
print(f"n={n:.3g} M={M} bits={bits} env={ {k: v for k, v in os.environ.items() if k.startswith('SMX_')} } "
      f"ms={min(times):.2f} GB/s(20B)={20 * n / min(times) / 1e6:.0f} ok={ok} all={[round(t, 1) for t in times]}")
