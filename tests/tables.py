"""Canonical per-rank table dumps of the three implementations (reference,
CPU oracle, GPU Cluster) and their comparison.

Canonical keys per rank r:
  r{r}/{src,tgt,weight,delay,port,first_index}      sorted store (sm/core.py:299-324)
  r{r}/map/{g}/{s}/{R,L}                            remote-source maps
  r{r}/mirror/{t}                                   p2p mirrors S
  r{r}/roster/{g}/{s}, r{r}/lookup/{g}/{s}          H and I
  r{r}/tp, r{r}/gq                                  routes flattened to (node, dest, pos) rows
"""
from __future__ import annotations

import numpy as np


def _routes(d):
    rows = []
    for s in sorted(d):
        a, b = d[s]
        for x, y in zip(np.asarray(a).tolist(), np.asarray(b).tolist()):
            rows.append((int(s), int(x), int(y)))
    return np.array(rows, dtype=np.int64).reshape(-1, 3)


def canon_reference(c) -> dict:
    out = {}
    for st in c.ranks:
        p = f"r{st.rank}/"
        s = st.store
        out[p + "src"], out[p + "tgt"] = s.src, s.tgt
        out[p + "weight"], out[p + "delay"], out[p + "port"] = s.weight, s.delay, s.port
        out[p + "first_index"] = s.first_index
        for (g, sr), m in st.remote_maps.items():
            if m.n:
                out[p + f"map/{g}/{sr}/R"], out[p + f"map/{g}/{sr}/L"] = m.remote, m.image
        for t, v in st.mirrors.items():
            out[p + f"mirror/{t}"] = v
        for (g, sr), v in st.rosters.items():
            out[p + f"roster/{g}/{sr}"] = v
        for (g, sr), v in st.image_lookups.items():
            out[p + f"lookup/{g}/{sr}"] = v
        out[p + "tp"] = _routes(st.point_routes)
        out[p + "gq"] = _routes(st.group_routes)
    return out


def canon_oracle(c) -> dict:
    out = {}
    for st in c.ranks:
        p = f"r{st.rank}/"
        out[p + "src"], out[p + "tgt"] = st.src, st.tgt
        out[p + "weight"], out[p + "delay"], out[p + "port"] = st.weight, st.delay, st.port
        out[p + "first_index"] = st.first_index
        for (g, sr), (R, L) in st.maps.items():
            if len(R):
                out[p + f"map/{g}/{sr}/R"], out[p + f"map/{g}/{sr}/L"] = R, L
        for t, v in st.mirrors.items():
            out[p + f"mirror/{t}"] = v
        for (g, sr), v in st.rosters.items():
            out[p + f"roster/{g}/{sr}"] = v
        for (g, sr), v in st.lookups.items():
            out[p + f"lookup/{g}/{sr}"] = v
        out[p + "tp"] = _routes(st.point_routes)
        out[p + "gq"] = _routes(st.group_routes)
    return out


def canon_gpu(c) -> dict:
    out = {}
    for r in sorted(c.ranks):
        e = c.export(r)
        p = f"r{r}/"
        for k in ("src", "tgt", "weight", "delay", "port", "first_index"):
            out[p + k] = e[k]
        for (g, sr), (R, L) in e["maps"].items():
            if len(R):
                out[p + f"map/{g}/{sr}/R"], out[p + f"map/{g}/{sr}/L"] = R, L
        for t, v in e["mirrors"].items():
            out[p + f"mirror/{t}"] = v
        for (g, sr), v in e["rosters"].items():
            out[p + f"roster/{g}/{sr}"] = v
        for (g, sr), v in e["lookups"].items():
            out[p + f"lookup/{g}/{sr}"] = v
        out[p + "tp"] = _routes(e["point_routes"])
        out[p + "gq"] = _routes(e["group_routes"])
    return out


def compare(a: dict, b: dict) -> list[str]:
    """Bit-exact comparison; returns human-readable mismatches."""
    bad = []
    for k in sorted(set(a) | set(b)):
        if k not in a or k not in b:
            # empty route tables / empty arrays may be absent on one side
            v = a.get(k, b.get(k))
            if np.asarray(v).size:
                bad.append(f"{k}: only in {'first' if k in a else 'second'}")
            continue
        x, y = np.asarray(a[k]), np.asarray(b[k])
        if x.shape != y.shape:
            bad.append(f"{k}: shape {x.shape} vs {y.shape}")
        elif x.dtype.kind == "f" or y.dtype.kind == "f":
            if not np.array_equal(x.astype(np.float64).view(np.int64), y.astype(np.float64).view(np.int64)):
                bad.append(f"{k}: float bits differ at {int(np.flatnonzero(x != y)[:1][0]) if (x != y).any() else -1}")
        elif not np.array_equal(x.astype(np.int64), y.astype(np.int64)):
            i = int(np.flatnonzero(x.astype(np.int64) != y.astype(np.int64))[0])
            bad.append(f"{k}: differs at {i} ({x.reshape(-1)[i]} vs {y.reshape(-1)[i]})")
    return bad


def digests(t: dict) -> dict:
    """SHA-256 of every non-empty canonical array (integers as int64, floats
    as float64 bits, C order) -- full-size tables compared by digest."""
    import hashlib
    out = {}
    for k in sorted(t):
        x = np.asarray(t[k])
        if not x.size:
            continue
        x = np.ascontiguousarray(x.astype(np.float64) if x.dtype.kind == "f" else x.astype(np.int64))
        out[k] = dict(sha256=hashlib.sha256(x.tobytes()).hexdigest(), shape=list(x.shape))
    return out
