"""Public value types of the façade, mirroring the reference package surface
(sm/__init__.py:10-41): SimConfig, ConnSpec, SynSpec, LifParams, RngStream,
Raster, SpikePacket, POINT_TO_POINT and the error classes.  Host-side only;
nothing here touches the device.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

POINT_TO_POINT = -1  # sm/core.py:17


class DelayRangeError(ValueError):
    """A connection or buffer delay falls outside the representable range."""


class ArenaUnderflowError(RuntimeError):
    """More bytes freed from an arena than were ever allocated."""


class ProtocolError(RuntimeError):
    """A transport round was violated (missing rank, bad destination...)."""


class ConsistencyError(RuntimeError):
    """Internal bookkeeping disagrees with itself."""


COMM_MODES = ("p2p", "collective")


@dataclass
class SimConfig:
    """Static per-run configuration (sm/core.py:58-92), same fields and checks."""

    n_ranks: int = 1
    resolution_ms: float = 0.1
    comm_mode: str = "p2p"
    opt_level: int = 2
    block_size: int = 1024
    flag_threshold: float = 1.0
    seed: int = 0

    def __post_init__(self):
        problems = []
        if self.n_ranks < 1:
            problems.append(f"n_ranks must be >= 1, got {self.n_ranks}")
        if not self.resolution_ms > 0.0:
            problems.append(f"resolution_ms must be > 0, got {self.resolution_ms}")
        if self.comm_mode not in COMM_MODES:
            problems.append(f"comm_mode must be one of {COMM_MODES}, got {self.comm_mode!r}")
        if self.opt_level not in (0, 1, 2, 3):
            problems.append(f"opt_level must be in 0..3, got {self.opt_level}")
        if self.block_size < 1:
            problems.append(f"block_size must be >= 1, got {self.block_size}")
        if not self.flag_threshold > 0.0:
            problems.append(f"flag_threshold must be > 0, got {self.flag_threshold}")
        if self.seed < 0:
            problems.append(f"seed must be >= 0, got {self.seed}")
        if problems:
            raise ValueError("; ".join(problems))

    def steps_for(self, span_ms: float) -> int:
        if span_ms < 0.0:
            raise ValueError(f"time span must be >= 0 ms, got {span_ms}")
        return int(round(span_ms / self.resolution_ms))


@dataclass
class LifParams:
    """LIF parameters (sm/dynamics.py:26-55)."""

    v_rest: float = -65.0
    v_reset: float = -65.0
    v_th: float = -50.0
    tau_m: float = 10.0
    c_m: float = 250.0
    t_ref: float = 2.0
    i_e: float = 0.0

    def __post_init__(self):
        if self.tau_m <= 0.0:
            raise ValueError(f"tau_m must be > 0, got {self.tau_m}")
        if self.t_ref < 0.0:
            raise ValueError(f"t_ref must be >= 0, got {self.t_ref}")
        if self.v_reset > self.v_th:
            raise ValueError("v_reset above threshold would spike forever")

    def decay_factor(self, dt_ms: float) -> float:
        return math.exp(-dt_ms / self.tau_m)

    def ref_steps(self, dt_ms: float) -> int:
        return int(round(self.t_ref / dt_ms))


CONNECTION_RULES = ("one_to_one", "all_to_all", "fixed_indegree", "fixed_outdegree",
                    "fixed_total", "assigned")


@dataclass
class ConnSpec:
    """Connection rule (sm/construction.py:92-121)."""

    rule: str
    k_in: int | None = None
    k_out: int | None = None
    n_total: int | None = None
    allow_autapses: bool = True
    allow_multapses: bool = True

    def validate(self, n_src: int, n_tgt: int) -> None:
        if self.rule not in CONNECTION_RULES:
            raise ValueError(f"unknown connection rule {self.rule!r}")
        if self.rule in ("one_to_one", "assigned") and n_src != n_tgt:
            raise ValueError(f"{self.rule} needs equally long source/target lists, "
                             f"got {n_src} and {n_tgt}")
        if self.rule == "fixed_indegree":
            if self.k_in is None or self.k_in < 0:
                raise ValueError(f"fixed_indegree needs k_in >= 0, got {self.k_in}")
            if not self.allow_multapses and self.k_in > n_src:
                raise ValueError(f"k_in {self.k_in} > {n_src} sources with multapses disabled")
        if self.rule == "fixed_outdegree" and (self.k_out is None or self.k_out < 0):
            raise ValueError(f"fixed_outdegree needs k_out >= 0, got {self.k_out}")
        if self.rule == "fixed_total" and (self.n_total is None or self.n_total < 0):
            raise ValueError(f"fixed_total needs n_total >= 0, got {self.n_total}")


@dataclass
class SynSpec:
    """Weight/delay realization (sm/construction.py:124-154): scalars,
    ("normal", mean, std) / ("uniform_int", lo, hi), or per-record arrays."""

    weight: object = 1.0
    delay_steps: object = 1

    def validate(self) -> None:
        w, d = self.weight, self.delay_steps
        if isinstance(w, tuple):
            if len(w) != 3 or w[0] != "normal" or w[2] < 0:
                raise ValueError(f"bad weight spec {w!r}")
        elif isinstance(w, (list, np.ndarray)):
            np.asarray(w, dtype=np.float64)
        else:
            float(w)
        if isinstance(d, tuple):
            if len(d) != 3 or d[0] != "uniform_int" or d[1] < 1 or d[2] < d[1]:
                raise ValueError(f"bad delay spec {d!r}")
        elif isinstance(d, (list, np.ndarray)):
            arr = np.asarray(d, dtype=np.int64)
            if arr.size and arr.min() < 1:
                raise ValueError("per-record delays must all be >= 1 step")
        elif int(d) < 1:
            raise ValueError(f"delays must be >= 1 step, got {d}")

    @property
    def is_constant(self) -> bool:
        return not isinstance(self.weight, (tuple, list, np.ndarray)) and \
            not isinstance(self.delay_steps, (tuple, list, np.ndarray))


def canonical_bytes(obj) -> bytes:
    """Stream-id encoding (sm/core.py:99-107)."""
    if isinstance(obj, (tuple, list)):
        return b"(" + b",".join(canonical_bytes(x) for x in obj) + b")"
    if isinstance(obj, str):
        return b"s:" + obj.encode("utf-8")
    if isinstance(obj, (int, np.integer)):
        return b"i:" + str(int(obj)).encode("ascii")
    raise TypeError(f"stream ids may contain only ints, strings and tuples, got {type(obj)!r}")


def stream_key(seed: int, stream_id) -> tuple[int, int]:
    """Philox key words (k0, k1) of a keyed stream (sm/core.py:119-126)."""
    digest = hashlib.blake2b(canonical_bytes((int(seed), stream_id)), digest_size=16).digest()
    key = int.from_bytes(digest, "little")
    return key & 0xFFFFFFFFFFFFFFFF, key >> 64


class RngStream:
    """Host-side keyed stream with the reference's surface (sm/core.py:110-148).

    The construction and propagation draws never go through this class: the
    device kernels consume the same keyed Philox streams directly.  It exists
    for model scripts (e.g. ExplicitNetwork.generate) and API parity.
    """

    def __init__(self, seed: int, stream_id):
        self.seed = int(seed)
        self.stream_id = stream_id
        self.key = stream_key(self.seed, stream_id)
        self._key = self.key[0] | (self.key[1] << 64)
        self.gen = np.random.Generator(np.random.Philox(key=self._key))

    def integers(self, low, high, size=None):
        return self.gen.integers(low, high, size=size)

    def normal(self, loc, scale, size=None):
        return self.gen.normal(loc, scale, size=size)

    def uniform(self, low, high, size=None):
        return self.gen.uniform(low, high, size=size)

    def poisson(self, lam, size=None):
        return self.gen.poisson(lam, size=size)

    def choice_no_replace(self, n: int, k: int):
        return self.gen.choice(n, size=k, replace=False)

    @property
    def state(self):
        return self.gen.bit_generator.state

    def __repr__(self):
        return f"RngStream(seed={self.seed}, stream_id={self.stream_id!r})"


@dataclass
class SpikePacket:
    """Spikes one rank sends (sm/transport.py:29-52)."""

    src_rank: int
    positions: np.ndarray
    multiplicities: np.ndarray

    def __post_init__(self):
        self.positions = np.asarray(self.positions, dtype=np.int64)
        self.multiplicities = np.asarray(self.multiplicities, dtype=np.int64)
        if len(self.positions) != len(self.multiplicities):
            raise ValueError("positions and multiplicities must align")

    @property
    def n_pairs(self) -> int:
        return len(self.positions)


@dataclass
class Raster:
    """Merged spike raster (sm/dynamics.py:290-346): (step, gid) sorted by
    time then gid; text form gid<TAB>time_ms; SHA-256 of the text."""

    events: np.ndarray
    resolution_ms: float

    @classmethod
    def from_events(cls, events, resolution_ms: float) -> "Raster":
        events = np.asarray(events, dtype=np.int64).reshape(-1, 2)
        order = np.lexsort((events[:, 1], events[:, 0]))
        return cls(events[order], float(resolution_ms))

    @property
    def n_events(self) -> int:
        return int(self.events.shape[0])

    def spikes_of(self, gid: int) -> np.ndarray:
        return self.events[self.events[:, 1] == gid, 0]

    def to_text(self) -> str:
        lines = [f"{g}\t{s * self.resolution_ms:.3f}" for s, g in self.events.tolist()]
        return "\n".join(lines) + ("\n" if lines else "")

    def sha256(self) -> str:
        return hashlib.sha256(self.to_text().encode("ascii")).hexdigest()
