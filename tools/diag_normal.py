"""Where the device ziggurat differs from the oracle (glibc) on a long stream."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle.rng import OracleStream
import device_rng as dr
from paper_2512_09502_b200.api import stream_key
for seed in (1, 2):
    k = stream_key(seed, ("normal-scale", seed))
    o = OracleStream(0, key=k)
    want = o.normal(0.0, 1.0, size=10_000_000)
    got, used = dr.normal(k, 0.0, 1.0, 10_000_000)
    got = got.cpu().numpy()
    bad = np.flatnonzero(got.view(np.int64) != want.view(np.int64))
    print(f"seed {seed}: {len(bad)} mismatches, words dev {used} oracle {o.words_used}")
    for i in bad[:10]:
        print(f"  i={i} got={got[i]!r} want={want[i]!r} ulps={int(got[i:i+1].view(np.int64)[0]) - int(want[i:i+1].view(np.int64)[0])}")
    big = np.abs(want) > 3.6541528853610087963519472518
    print(f"  tail samples (|z| > R): {int(big.sum())}, mismatches among them: {int(big[bad].sum()) if len(bad) else 0}")
