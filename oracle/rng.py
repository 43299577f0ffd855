"""CPU ORACLE -- test infrastructure only (tests/, smoke(), bench cpu_baseline).

ctypes front end of `oracle/rng.c`: a keyed stream with the call surface of
the reference's `RngStream` (sm/core.py:110-148).  Keys follow
sm/core.py:99-107 (canonical bytes) and :119-126 (blake2b-128 digest,
little-endian, split into the two Philox key words).  The arithmetic is the
C restatement of numpy 2.3.5's Philox / Lemire / ziggurat / Poisson
(see the header of rng.c).
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_rng.so")
_lib = None


def build() -> str:
    """Compile the oracle restatement (make -C oracle)."""
    subprocess.check_call(["make", "-s", "-C", _HERE], stdout=subprocess.DEVNULL)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        u64, i64, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
        L.orc_init.argtypes = [p, u64, u64]
        L.orc_next64.argtypes = [p]
        L.orc_next64.restype = u64
        L.orc_next32.argtypes = [p]
        L.orc_next32.restype = ctypes.c_uint32
        L.orc_next_double.argtypes = [p]
        L.orc_next_double.restype = ctypes.c_double
        L.orc_words_used.argtypes = [p]
        L.orc_words_used.restype = u64
        L.orc_u32_used.argtypes = [p]
        L.orc_u32_used.restype = u64
        L.orc_integers.argtypes = [p, i64, u64, i64, p]
        L.orc_integers.restype = ctypes.c_int
        L.orc_choice.argtypes = [p, i64, i64, p]
        L.orc_choice.restype = ctypes.c_int
        L.orc_normal.argtypes = [p, ctypes.c_double, ctypes.c_double, i64, p]
        L.orc_uniform.argtypes = [p, ctypes.c_double, ctypes.c_double, i64, p]
        L.orc_poisson.argtypes = [p, ctypes.c_double, ctypes.c_double, i64, p]
        L.orc_poisson.restype = ctypes.c_int
        L.orc_words.argtypes = [u64, u64, u64, i64, p]
        L.orc_philox_block.argtypes = [u64, u64, u64, p]
        L.orc_sizeof_stream.restype = ctypes.c_int
        _lib = L
    return _lib


def canonical_bytes(obj) -> bytes:
    """sm/core.py:99-107: tuples -> '(a,b)', str -> 's:..', int -> 'i:..'."""
    if isinstance(obj, (tuple, list)):
        return b"(" + b",".join(canonical_bytes(x) for x in obj) + b")"
    if isinstance(obj, str):
        return b"s:" + obj.encode("utf-8")
    if isinstance(obj, (int, np.integer)):
        return b"i:" + str(int(obj)).encode("ascii")
    raise TypeError(f"stream ids may contain only ints, strings and tuples, got {type(obj)!r}")


def stream_key(seed: int, stream_id) -> tuple[int, int]:
    """(k0, k1) Philox key words of RngStream(seed, stream_id) (sm/core.py:119-126)."""
    digest = hashlib.blake2b(canonical_bytes((int(seed), stream_id)), digest_size=16).digest()
    key = int.from_bytes(digest, "little")
    return key & 0xFFFFFFFFFFFFFFFF, key >> 64


class OracleStream:
    """Restated numpy Generator(Philox(key)) with the RngStream draw surface."""

    def __init__(self, seed: int, stream_id=None, key: tuple[int, int] | None = None):
        self.k0, self.k1 = key if key is not None else stream_key(seed, stream_id)
        L = lib()
        self._buf = ctypes.create_string_buffer(L.orc_sizeof_stream())
        self._p = ctypes.cast(self._buf, ctypes.c_void_p)
        L.orc_init(self._p, self.k0, self.k1)

    # raw ---------------------------------------------------------------
    def next64(self) -> int:
        return lib().orc_next64(self._p)

    def next32(self) -> int:
        return lib().orc_next32(self._p)

    @property
    def words_used(self) -> int:
        return lib().orc_words_used(self._p)

    @property
    def u32_used(self) -> int:
        return lib().orc_u32_used(self._p)

    # distributions -------------------------------------------------------
    def integers(self, low, high, size=None):
        n = 1 if size is None else int(size)
        ex = int(high) - int(low)
        if ex < 1:
            raise ValueError("high <= low")
        if ex > (1 << 32):
            raise ValueError("oracle supports integer ranges up to 2^32")
        out = np.empty(n, dtype=np.int64)
        if n:
            rc = lib().orc_integers(self._p, int(low), ex, n, out.ctypes.data)
            if rc:
                raise ValueError("bad integer range")
        return int(out[0]) if size is None else out

    def choice_no_replace(self, n: int, k: int) -> np.ndarray:
        """numpy Generator.choice(n, size=k, replace=False) (sm/core.py:140-141)."""
        out = np.empty(max(int(k), 0), dtype=np.int64)
        rc = lib().orc_choice(self._p, int(n), int(k), out.ctypes.data)
        if rc:
            raise ValueError("Cannot take a larger sample than population when replace is False"
                             if rc == -1 else "oracle choice: allocation failed")
        return out

    def normal(self, loc, scale, size=None):
        n = 1 if size is None else int(size)
        out = np.empty(n, dtype=np.float64)
        if n:
            lib().orc_normal(self._p, float(loc), float(scale), n, out.ctypes.data)
        return float(out[0]) if size is None else out

    def uniform(self, low, high, size=None):
        n = 1 if size is None else int(size)
        out = np.empty(n, dtype=np.float64)
        if n:
            lib().orc_uniform(self._p, float(low), float(high), n, out.ctypes.data)
        return float(out[0]) if size is None else out

    def poisson(self, lam, size=None):
        n = 1 if size is None else int(size)
        out = np.empty(n, dtype=np.int64)
        if n:
            rc = lib().orc_poisson(self._p, float(lam), math.exp(-float(lam)), n, out.ctypes.data)
            if rc:
                raise ValueError("lam < 0")
        return int(out[0]) if size is None else out


def words(k0: int, k1: int, w0: int, n: int) -> np.ndarray:
    """Random access to raw 64-bit words [w0, w0+n) of a keyed stream."""
    out = np.empty(n, dtype=np.uint64)
    if n:
        lib().orc_words(k0, k1, w0, n, out.ctypes.data)
    return out
