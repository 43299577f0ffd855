"""The CPU oracle's RNG restatement (oracle/rng.c) against numpy 2.3.5
itself and against the golden vectors generated from the reference."""
import os

import numpy as np
import pytest

from oracle.rng import OracleStream, stream_key, words

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng.npz")


def test_golden_key_vector():
    # (seed=7, ("dist-indegree", 1, 0))
    assert stream_key(7, ("dist-indegree", 1, 0)) == (0x3761F6E86C6D088B, 0xFD6F20DCBAC23712)


def _numpy_stream(seed, sid):
    k0, k1 = stream_key(seed, sid)
    return np.random.Generator(np.random.Philox(key=k0 | (k1 << 64)))


@pytest.mark.parametrize("sid", [("a", 1), ("init-v", 5), ("remote-src", 0, 1, 3)])
def test_against_numpy(sid):
    if np.__version__ != "2.3.5":
        pytest.skip("numpy 2.3.5 pins the stream semantics")
    g, o = _numpy_stream(3, sid), OracleStream(3, sid)
    for lo, hi, n in [(0, 36, 1000), (0, 640000, 10000), (5, 3_000_000_000, 5000), (0, 1, 10),
                      (0, 2**32, 100), (1, 21, 333), (0, 7, 3)]:
        assert np.array_equal(g.integers(lo, hi, size=n), o.integers(lo, hi, size=n))
    assert np.array_equal(g.normal(-58, 5, size=5000), o.normal(-58, 5, size=5000))
    assert np.array_equal(g.poisson(1.1, size=5000), o.poisson(1.1, size=5000))
    assert np.array_equal(g.uniform(0, 1, size=100), o.uniform(0, 1, size=100))


def test_against_golden():
    z = np.load(GOLDEN)
    i = 0
    while f"s{i}/key" in z:
        k0, k1 = (int(x) for x in z[f"s{i}/key"])
        assert np.array_equal(words(k0, k1, 0, 64), z[f"s{i}/words"])
        o = OracleStream(0, key=(k0, k1))
        j = 0
        while f"s{i}/int{j}" in z:
            lo, hi, n = (int(x) for x in z[f"s{i}/int{j}/spec"])
            assert np.array_equal(o.integers(lo, hi, size=n), z[f"s{i}/int{j}"]), (i, j)
            j += 1
        assert np.array_equal(OracleStream(0, key=(k0, k1)).normal(-58.0, 5.0, size=4000), z[f"s{i}/normal"])
        assert np.array_equal(OracleStream(0, key=(k0, k1)).poisson(1.1, size=20000), z[f"s{i}/poisson"])
        p = OracleStream(0, key=(k0, k1))
        steps = np.stack([p.poisson(1.1, size=333) for _ in range(20)])
        assert np.array_equal(steps, z[f"s{i}/poisson_steps"])
        i += 1
    assert i == 3
    gids = z["initv/gids"]
    for seed in (11, 12345):
        got = np.array([OracleStream(seed, ("init-v", int(g))).normal(-58.0, 5.0) for g in gids])
        assert np.array_equal(got, z[f"initv/seed{seed}"])


@pytest.mark.parametrize("n,k", [(10, 3), (100, 50), (1000, 1000), (20000, 400), (20000, 401), (10001, 201),
                                 (10000, 5000), (50000, 3000), (7, 0), (300, 299)])
def test_choice_no_replace_matches_numpy(n, k):
    """Generator.choice(n, k, replace=False) restated (sm/core.py:140-141):
    Floyd + shuffle / tail shuffle, three consecutive calls per stream (the
    reference draws one row per target from one stream)."""
    from numpy.random import Generator, Philox
    from oracle.rng import OracleStream
    g = Generator(Philox(key=(7 << 64) | 11))
    o = OracleStream(0, key=(11, 7))
    for _ in range(3):
        assert np.array_equal(o.choice_no_replace(n, k), g.choice(n, size=k, replace=False))
    assert o.next64() == int(g.bit_generator.random_raw())


@pytest.mark.parametrize("lam", [10.0, 11.5, 30.0, 100.0, 1234.5])
def test_poisson_ptrs_matches_numpy(lam):
    """numpy random_poisson_ptrs (lam >= 10) restated: counts and cursor."""
    from numpy.random import Generator, Philox
    g = Generator(Philox(key=(5 << 64) | 9))
    o = OracleStream(0, key=(9, 5))
    assert np.array_equal(o.poisson(lam, size=50_000), g.poisson(lam, size=50_000))
    assert o.next64() == int(g.bit_generator.random_raw())
