"""Reference-layout drop-in kernels (kernels_b200) against the reference's
kernel semantics restated in numpy (sm/kernels/_numpy_impl.py:16-58)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lif_numpy(v, ref, real, inputs, decay, vr, vreset, vth, refsteps, out):
    realb = real.astype(bool)
    refr = realb & (ref > 0)
    act = realb & ~refr
    integ = vr + (v - vr) * decay + inputs
    spk = act & (integ >= vth)
    v[act] = integ[act]
    v[spk] = vreset[spk]
    v[refr] = vreset[refr]
    ref[refr] -= 1
    ref[spk] = refsteps[spk]
    out[:] = 0
    out[spk] = 1


def test_lif_step_bit_exact():
    from paper_2512_09502_b200 import kernels_b200 as kb
    rng = np.random.default_rng(3)
    n = 100_003
    v = rng.normal(-55, 6, n)
    ref = rng.integers(0, 3, n).astype(np.int64)
    real = (rng.random(n) < 0.9).astype(np.uint8)
    inputs = rng.integers(-64, 65, n) / 64.0
    decay = np.full(n, np.exp(-0.1 / 10.0))
    vr, vreset, vth = np.full(n, -65.0), np.full(n, -65.0), np.full(n, -50.0)
    refsteps = np.full(n, 20, dtype=np.int64)
    want = [a.copy() for a in (v, ref)] + [np.zeros(n, np.uint8)]
    _lif_numpy(want[0], want[1], real, inputs, decay, vr, vreset, vth, refsteps, want[2])
    out = np.zeros(n, np.uint8)
    kb.lif_step(v, ref, real, inputs, decay, vr, vreset, vth, refsteps, out)
    assert np.array_equal(v.view(np.int64), want[0].view(np.int64))
    assert np.array_equal(ref, want[1]) and np.array_equal(out, want[2])


def test_deliver_spikes_exact_dyadic():
    from paper_2512_09502_b200 import kernels_b200 as kb
    rng = np.random.default_rng(4)
    M, P, L, S = 500, 2, 11, 20_000
    src = np.sort(rng.integers(0, M, S))
    fi = np.zeros(M + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=M), out=fi[1:])
    tgt = rng.integers(0, M, S).astype(np.int64)
    port = rng.integers(0, P, S).astype(np.int64)
    delay = rng.integers(1, L, S).astype(np.int64)
    w = rng.integers(-64, 65, S) / 256.0
    nodes = rng.choice(M, 60, replace=False).astype(np.int64)
    mults = rng.integers(1, 3, 60).astype(np.int64)
    buf = np.zeros((M, P, L))
    want = buf.copy()
    for node, m in zip(nodes, mults):
        lo, hi = fi[node], fi[node + 1]
        np.add.at(want, (tgt[lo:hi], port[lo:hi], (7 + delay[lo:hi]) % L), w[lo:hi] * m)
    kb.deliver_spikes(nodes, mults, fi, tgt, port, delay, w, buf, 7)
    assert np.array_equal(buf, want)
