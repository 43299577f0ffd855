"""Device RNG kernels against the golden vectors (numpy 2.3.5 via the
reference) and against the CPU oracle at larger sizes."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng.npz")
pytestmark = pytest.mark.gpu


def _keys(z):
    i = 0
    while f"s{i}/key" in z:
        yield i, tuple(int(x) for x in z[f"s{i}/key"])
        i += 1


def test_words_golden():
    import device_rng as dr
    z = np.load(GOLDEN)
    for i, k in _keys(z):
        got = dr.words(k, 0, 64).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, z[f"s{i}/words"])
        # random access at an odd offset
        assert np.array_equal(dr.words(k, 37, 20).cpu().numpy().view(np.uint64), z[f"s{i}/words"][37:57])


def test_integers_golden_with_cursor():
    import device_rng as dr
    z = np.load(GOLDEN)
    for i, k in _keys(z):
        cur = 0
        j = 0
        while f"s{i}/int{j}" in z:
            lo, hi, n = (int(x) for x in z[f"s{i}/int{j}/spec"])
            v, cur = dr.integers(k, cur, lo, hi, n)
            assert np.array_equal(v.cpu().numpy(), z[f"s{i}/int{j}"]), (i, j)
            j += 1


@pytest.mark.parametrize("lo,hi,n", [(0, 8000, 8_000_000), (0, 640_000, 3_000_000), (7, 3_000_000_007, 200_000),
                                     (0, 2, 100_001), (0, 2**32, 5000)])
def test_integers_vs_oracle_large(lo, hi, n):
    from oracle.rng import OracleStream
    import device_rng as dr
    from paper_2512_09502_b200.api import stream_key
    k = stream_key(99, ("big", lo, n))
    o = OracleStream(0, key=k)
    a = o.integers(lo, hi, size=n)
    used_a = o.u32_used
    b = o.integers(lo, hi, size=3)
    v, cur = dr.integers(k, 0, lo, hi, n)
    assert np.array_equal(v.cpu().numpy(), a)
    assert cur == used_a  # the device cursor is the u32 position after the n-th accept
    v2, _ = dr.integers(k, cur, lo, hi, 3)
    assert np.array_equal(v2.cpu().numpy(), b)


def test_init_v_golden():
    import device_rng as dr
    z = np.load(GOLDEN)
    gids = z["initv/gids"]
    for seed in (11, 12345):
        got = dr.init_v(seed, gids, -58.0, 5.0).cpu().numpy()
        assert np.array_equal(got.view(np.int64), z[f"initv/seed{seed}"].view(np.int64)), seed


def test_init_v_vs_oracle_many():
    from oracle.rng import OracleStream
    import device_rng as dr
    gids = np.arange(0, 20000, 7, dtype=np.int64)
    want = np.array([OracleStream(5, ("init-v", int(g))).normal(-58.0, 5.0) for g in gids])
    got = dr.init_v(5, gids, -58.0, 5.0).cpu().numpy()
    assert np.array_equal(got, want)


def test_poisson_golden_steps():
    import device_rng as dr
    z = np.load(GOLDEN)
    for i, k in _keys(z):
        ps = dr.PoissonStream(k, 1.1)
        assert np.array_equal(ps.draw(20000).cpu().numpy(), z[f"s{i}/poisson"])
        ps = dr.PoissonStream(k, 1.1)
        steps = np.stack([ps.draw(333).cpu().numpy() for _ in range(20)])
        assert np.array_equal(steps, z[f"s{i}/poisson_steps"])


@pytest.mark.parametrize("lam,n,batches", [(1.1, 1_000_000, 3), (0.3, 200_000, 4), (6.5, 300_000, 2),
                                           (10.0, 300_000, 2), (27.5, 300_000, 2), (150.0, 200_000, 2)])
def test_poisson_vs_oracle_large(lam, n, batches):
    from oracle.rng import OracleStream
    import device_rng as dr
    from paper_2512_09502_b200.api import stream_key
    k = stream_key(3, ("poisson", 0, int(lam * 10)))
    o = OracleStream(0, key=k)
    ps = dr.PoissonStream(k, lam)
    for _ in range(batches):
        assert np.array_equal(ps.draw(n).cpu().numpy().astype(np.int64), o.poisson(lam, size=n))
    assert ps.word_cursor == o.words_used


_VARIANT_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from oracle.rng import OracleStream
import device_rng as dr
from paper_2512_09502_b200.api import stream_key
for lo, hi, n in [(0, 8000, 1_000_000), (7, 3_000_000_007, 200_000), (0, 2, 100_001), (0, 100_000, 2047),
                  (0, 100_000, 2048), (0, 100_000, 2049), (0, 2**32, 5000), (5, 9, 1)]:
    for u0 in (0, 3, 4093):
        k = stream_key(7, ("variant", lo, n, u0))
        o = OracleStream(0, key=k)
        if u0:
            o.integers(0, 2**32, size=u0)  # consume u0 raw u32 draws (a full-range draw never rejects)
        a = o.integers(lo, hi, size=n)
        b = o.integers(lo, hi, size=3)
        v, cur = dr.integers(k, u0, lo, hi, n)
        assert np.array_equal(v.cpu().numpy(), a), (lo, hi, n, u0)
        v2, _ = dr.integers(k, cur, lo, hi, 3)
        assert np.array_equal(v2.cpu().numpy(), b), (lo, hi, n, u0, "cursor")
print("ok")
"""


@pytest.mark.parametrize("env", [{"SMX_DRAW_TILE_RT": "256"}, {"SMX_DRAW_TILE_RT": "4096"},
                                 {"SMX_DRAW_SHORT_WINDOW": "1"}, {"SMX_DRAW_ONEPASS": "0"},
                                 {"SMX_DRAW_ONEPASS": "0", "SMX_DRAW_SHORT_WINDOW": "1"}])
def test_integers_draw_variants(env):
    """The one-pass draw at extreme tile sizes (deep look-back chains with 256),
    the widen-and-retry path (a window of exactly n raw positions), and the
    two-pass A/B path, all against the oracle stream incl. the cursor.  The
    switches are read once per process, hence a subprocess per variant."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("seed", [1, 2])
def test_normal_slow_paths_at_scale(seed):
    """1e7 ziggurat normals from one stream (~1.5e5 wedge/tail samples, the
    branches that call exp / log1p) bit-exact against the oracle (glibc)."""
    from oracle.rng import OracleStream
    import device_rng as dr
    from paper_2512_09502_b200.api import stream_key
    k = stream_key(seed, ("normal-scale", seed))
    o = OracleStream(0, key=k)
    want = o.normal(-58.0, 5.0, size=10_000_000)
    got, used = dr.normal(k, -58.0, 5.0, 10_000_000)
    got = got.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    assert used == o.words_used


@pytest.mark.parametrize("lam", [12.5, 150.0])
def test_ptrs_at_scale(lam):
    """numpy's PTRS sampler (lam >= 10, CUDA log in the squeeze test):
    1e7 samples bit-exact against the oracle."""
    from oracle.rng import OracleStream
    import device_rng as dr
    from paper_2512_09502_b200.api import stream_key
    k = stream_key(8, ("ptrs-scale", int(lam)))
    o = OracleStream(0, key=k)
    ps = dr.PoissonStream(k, lam)
    assert np.array_equal(ps.draw(10_000_000).cpu().numpy().astype(np.int64), o.poisson(lam, size=10_000_000))
    assert ps.word_cursor == o.words_used


def test_init_v_many_gids():
    """Per-gid init-v streams (blake2b on the device) for 2e5 gids spread over
    0 .. 4.1e6 (the C4 neuron count) against the oracle."""
    from oracle.rng import OracleStream
    import device_rng as dr
    gids = np.unique(np.random.default_rng(5).integers(0, 4_130_000, 200_000)).astype(np.int64)
    want = np.array([OracleStream(12345, ("init-v", int(g))).normal(-58.0, 5.0) for g in gids])
    got = dr.init_v(12345, gids, -58.0, 5.0).cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("n,k,rows", [(1000, 40, 3000), (5, 5, 50), (20_000, 900, 40), (50_000, 600, 200),
                                      (3, 1, 100), (100_000, 1, 20_000),
                                      (2_200_000_000, 20, 2000)])
def test_choice_rows_parallel_chain(n, k, rows):
    """smx_choice_rows draws rows concurrently (one warp per row) after
    resolving the chain of row starts; the rows and the final cursor equal
    numpy's back-to-back choice(n, k, replace=False) calls on one stream
    (Floyd + shuffle, the tail branch for n > 10000 and k > n // 50, n == k,
    a long chain, and ranges just above 2^31 where about half the draws are
    Lemire rejections, so nearly every row shifts the ones after it)."""
    import device_rng as dr
    from oracle.rng import OracleStream
    from paper_2512_09502_b200.api import stream_key
    key = stream_key(5, ("choice-rows", n, k, rows))
    got, cur = dr.choice_rows(key, 0, n, k, rows)
    o = OracleStream(0, key=key)
    want = np.stack([o.choice_no_replace(n, k) for _ in range(rows)])
    assert np.array_equal(got.cpu().numpy().view(np.uint32).astype(np.int64), want.astype(np.int64))
    assert cur == o.u32_used


def test_draw_chain_does_not_leak_past_a_failed_call():
    """A chain set for a draw call that then fails before drawing (bad key
    mode) is dropped with it: the next, unrelated draw starts at its own
    cursor (csrc/common.cuh DrawChainScope)."""
    import ctypes
    import torch
    import device_rng as dr
    from oracle.rng import OracleStream
    from paper_2512_09502_b200 import _lib
    from paper_2512_09502_b200.api import stream_key
    L = _lib.lib()
    cur = torch.tensor([12345], dtype=torch.int64, device="cuda")
    assert L.smx_draw_chain(ctypes.c_void_p(cur.data_ptr()), None) == 0
    rc = L.smx_gen_draw(1, 2, 0, 100, 10, 99, 0, None, None, 1, None, None, None, None, 0, 0, 0, 0, None,
                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == -1
    key = stream_key(3, ("chain-scope",))
    got, c = dr.integers(key, 0, 0, 1000, 5000)
    o = OracleStream(0, key=key)
    assert np.array_equal(got.cpu().numpy(), o.integers(0, 1000, size=5000))
