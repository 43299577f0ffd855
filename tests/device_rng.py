"""Test helper: the library's keyed-stream draw entry points (raw Philox
words, Generator.integers, per-gid init-v normals, the Poisson drive's
counts) called one by one through the C ABI, so the parity tests can compare
each against numpy / the oracle.  Not part of the product package."""
from __future__ import annotations

import math

import numpy as np
import torch

from paper_2512_09502_b200 import _lib
from paper_2512_09502_b200._lib import call
from paper_2512_09502_b200.api import canonical_bytes


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


def words(key, w0: int, n: int, device="cuda") -> torch.Tensor:
    out = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    call("smx_philox_words", key[0], key[1], w0, n, out.data_ptr(), _stream(out.device))
    return out[:n]


def integers(key, u32_cursor: int, lo: int, hi: int, n: int, device="cuda"):
    """numpy Generator.integers(lo, hi, size=n) from a u32 cursor; returns
    (values int64 tensor, cursor after the draws)."""
    out = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    cur = np.zeros(1, dtype=np.uint64)
    call("smx_integers", key[0], key[1], u32_cursor, lo, hi - lo, n, out.data_ptr(), cur.ctypes.data,
         _stream(out.device))
    return out[:n], int(cur[0])


def choice_rows(key, u32_cursor: int, n: int, k: int, rows: int, device="cuda"):
    """rows back-to-back Generator.choice(n, k, replace=False) draws from a
    u32 cursor; returns (rows x k int32 tensor, cursor after the last row)."""
    out = torch.empty(max(rows * k, 1), dtype=torch.int32, device=device)
    cur = np.zeros(1, dtype=np.uint64)
    call("smx_choice_rows", key[0], key[1], u32_cursor, n, k, rows, out.data_ptr(), cur.ctypes.data,
         _stream(out.device))
    return out[: rows * k].view(rows, k) if rows * k else out[:0], int(cur[0])


def init_v(seed: int, gids, mu: float, sd: float, device="cuda") -> torch.Tensor:
    g = torch.as_tensor(np.asarray(gids, dtype=np.int64)).to(device)
    v = torch.empty(max(g.numel(), 1), dtype=torch.float64, device=device)
    pre = canonical_bytes((int(seed), ("init-v", 0)))
    prefix = pre[: pre.rindex(b"i:0))") + 2]
    call("smx_init_v", prefix, len(prefix), b"))", 2, g.data_ptr(), g.numel(), float(mu), float(sd),
         v.data_ptr(), _stream(v.device))
    return v[: g.numel()]


class PoissonStream:
    """numpy Generator.poisson(lam, size=n) calls on one stream, on the device."""

    def __init__(self, key, lam: float, device="cuda"):
        self.key, self.lam, self.enlam = key, float(lam), math.exp(-float(lam))
        self.dev = torch.device(device)
        self.cursor = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.ping = 0
        self.err = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def draw(self, n: int) -> torch.Tensor:
        L = _lib.lib()
        chunks = L.smx_poisson_chunks_for(n, self.lam)
        ws = torch.empty(int(L.smx_poisson_workspace(chunks)), dtype=torch.uint8, device=self.dev)
        out = torch.empty(max(n, 1), dtype=torch.uint8, device=self.dev)
        cin = self.cursor[self.ping:]
        cout = self.cursor[1 - self.ping:]
        fn, par = ("smx_poisson_counts_ptrs", self.lam) if self.lam >= 10.0 else ("smx_poisson_counts", self.enlam)
        call(fn, self.key[0], self.key[1], cin.data_ptr(), par, n, chunks,
             ws.data_ptr(), out.data_ptr(), cout.data_ptr(), self.err.data_ptr(), _stream(self.dev))
        self.ping = 1 - self.ping
        if int(self.err.item()):
            raise RuntimeError(f"poisson chain error {int(self.err.item())}")
        return out[:n]

    @property
    def word_cursor(self) -> int:
        return int(self.cursor[self.ping].item())


def normal(key, loc: float, scale: float, n: int, device="cuda"):
    """numpy Generator.normal(loc, scale, size=n) from the start of a stream
    (ziggurat, variable words per sample); returns (values, words used)."""
    L = _lib.lib()
    dev = torch.device(device)
    chunks = L.smx_normal_chunks_for(n)
    ws = torch.empty(int(L.smx_poisson_workspace(chunks)), dtype=torch.uint8, device=dev)
    cur = torch.zeros(2, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    call("smx_normal_fill", key[0], key[1], cur.data_ptr(), float(loc), float(scale), n, chunks, ws.data_ptr(),
         out.data_ptr(), cur[1:].data_ptr(), err.data_ptr(), _stream(dev))
    if int(err.item()):
        raise RuntimeError(f"normal chain error {int(err.item())}")
    return out[:n], int(cur[1].item())
