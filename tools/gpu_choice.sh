set -x
O=gpurun_out/choice
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rng.py -k choice_rows -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -15 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -k "no_multapse" tests/test_gpu_multiprocess.py -q -p no:cacheprovider > $O/pytest2.log 2>&1; tail -5 $O/pytest2.log
timeout 600 python - <<'PY' > $O/timing.log 2>&1
import sys, time, torch
sys.path.insert(0, "tests")
import device_rng as dr
from paper_2512_09502_b200.api import stream_key
for n, k, rows in [(100_000, 1000, 10_000), (100_000, 11_250, 1000), (80_000, 900, 100_000)]:
    key = stream_key(1, ("t", n, k))
    dr.choice_rows(key, 0, n, k, 100)
    torch.cuda.synchronize(); t = time.perf_counter()
    out, cur = dr.choice_rows(key, 0, n, k, rows)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"n={n} k={k} rows={rows}: {dt*1e3:.1f} ms, {rows*k/dt:.3e} values/s, cursor {cur}")
PY
cat $O/timing.log
