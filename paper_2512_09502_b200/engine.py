"""The GPU `Cluster`: the reference façade (sm/engine.py:197-399) over
sm_100a kernels.

Every heavy step is a call through the C ABI (`_lib`) on device buffers owned
by torch tensors (plumbing only).  Host work is bookkeeping per façade call:
stream keys (blake2b of the stream id), call counters, argument validation
and buffer sizing.  There is no CPU fallback: without a CUDA device or the
built library every method raises.

Rank placement.  The reference keeps every rank in one process.  Here a
process owns a set of *local* ranks:
  * single process (default): all ranks are local, placed on `devices`
    (default cuda:0) -- the layout used by the parity tests;
  * one process per GPU (torch.distributed initialised with
    world_size == n_ranks): only rank == dist.get_rank() is local.  Every
    process runs the whole construction script; calls that touch no local
    rank only advance counters, exactly like the paper's per-process scripts.
Construction and preparation never communicate (check_construction_silent).
"""
from __future__ import annotations

import ctypes
import math
import os
import time
from contextlib import contextmanager
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _lib
from .memory import RankMemory
from ._lib import call, check
from .exchange import fixed_allgather, fixed_p2p
from .api import (POINT_TO_POINT, ConnSpec, ConsistencyError, DelayRangeError, LifParams,
                  ProtocolError, Raster, SimConfig, SynSpec, canonical_bytes, stream_key)

TMP_KEY = 0x80000000
ROW_MASK = 0xFFFFFF
MAX_CLASSES = 256
MAX_LIF_BLOCK = 16   # steps per lif_block_kernel launch (csrc/propagate.cu MAX_BLOCK)
PHASES = ("construction", "preparation", "propagation")


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


H2D_BYTES = [0]


def _up(arr, dev) -> torch.Tensor:
    """Host -> device upload (counted for the end-to-end byte accounting),
    staged through pinned memory so the host does not wait for the work
    already queued on the stream."""
    a = np.ascontiguousarray(arr)
    H2D_BYTES[0] += a.nbytes
    return torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)


def _run_info(a: np.ndarray):
    """(consecutive, min, max) of an int64 node array in one pass when it is
    a run (the common population case).  Not cached: a caller may reuse and
    refill an array between calls."""
    n = len(a)
    if n == 0:
        return False, 0, -1
    f, l = int(a[0]), int(a[-1])
    cons = n > 1 and l - f == n - 1 and bool((np.diff(a) == 1).all())
    return (cons, f, l) if cons else (cons, int(a.min()), int(a.max()))


def _consecutive(a: np.ndarray) -> bool:
    """a is one run first, first + 1, ... (the common population case)."""
    return _run_info(a)[0]


def _up_index(arr, dev) -> torch.Tensor:
    """int64 node-index upload; a consecutive run (the common population
    case) is materialised on the device from its first index instead of
    being copied from pageable host memory."""
    a = np.ascontiguousarray(arr, dtype=np.int64)
    n = len(a)
    if n > 1024 and _consecutive(a):
        H2D_BYTES[0] += 16
        return torch.arange(int(a[0]), int(a[0]) + n, dtype=torch.int64, device=dev)
    return _up(a, dev)


_PREP_STREAMS: dict = {}
_GEN_STREAMS: dict = {}
_CAPTURE_STREAMS: dict = {}


def _capture_stream(dev) -> "torch.cuda.Stream":
    """Block-graph capture stream of a device (torch's default capture stream
    is one process-wide stream on whichever device was current first)."""
    key = torch.device(dev).index
    if key not in _CAPTURE_STREAMS:
        _CAPTURE_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _CAPTURE_STREAMS[key]


def _gen_stream(dev) -> "torch.cuda.Stream":
    """Stream of the fused path's pass A (one per device): the draws of a
    call overlap the host work and small kernels of the calls that follow."""
    key = torch.device(dev).index
    if key not in _GEN_STREAMS:
        _GEN_STREAMS[key] = _nonblocking_stream(dev)
    return _GEN_STREAMS[key]


def _nonblocking_stream(dev):
    """A CUDA stream created with cudaStreamNonBlocking (csrc/capi.cu): it does
    not serialise with the legacy default stream that torch's default stream
    is, so its kernels run beside the default stream's small kernels."""
    p = ctypes.c_void_p()
    with torch.cuda.device(dev):
        call("smx_stream_create", 0, ctypes.byref(p))
    return torch.cuda.ExternalStream(p.value, device=dev)


def _prep_stream(dev) -> "torch.cuda.Stream":
    """One preparation side stream per device for the whole process (its
    caching-allocator pool is then reused by every Cluster)."""
    key = torch.device(dev).index
    if key not in _PREP_STREAMS:
        _PREP_STREAMS[key] = _nonblocking_stream(dev)
    return _PREP_STREAMS[key]


def _record_stream(obj, stream, depth: int = 0) -> None:
    """Tell the caching allocator that the tensors reachable from obj are used
    on `stream` (they were allocated on a preparation side stream)."""
    if isinstance(obj, torch.Tensor):
        obj.record_stream(stream)
    elif depth < 3 and isinstance(obj, dict):
        for v in obj.values():
            _record_stream(v, stream, depth + 1)
    elif depth < 3 and isinstance(obj, (list, tuple)):
        for v in obj:
            _record_stream(v, stream, depth + 1)


def _popcount_dev(b):
    """Set bits of an int32-word bitmap as a 0-dim device tensor (no sync)."""
    excl = torch.zeros(b.numel() + 1, dtype=torch.int64, device=b.device)
    if b.numel():
        call("smx_bits_prefix", _ptr(b), b.numel(), _ptr(excl), torch.cuda.current_stream(b.device).cuda_stream)
    return excl[-1]


def _popcounts(bitmaps) -> list:
    """Set bits of each bitmap (int32 words), one host synchronisation."""
    outs = []
    for b in bitmaps:
        excl = torch.empty(b.numel() + 1, dtype=torch.int64, device=b.device)
        if b.numel():
            call("smx_bits_prefix", _ptr(b), b.numel(), _ptr(excl), torch.cuda.current_stream(b.device).cuda_stream)
        else:
            excl.zero_()
        outs.append(excl[-1:])
    if not outs:
        return []
    return [int(x) for x in torch.cat([o.to(outs[0].device) for o in outs]).cpu().numpy()]


def _all_distinct(a: np.ndarray) -> bool:
    """True when a has no repeated value (O(n) for the usual ascending ids)."""
    if len(a) < 2 or bool((a[1:] > a[:-1]).all()):
        return True
    return len(np.unique(a)) == len(a)


def _syn_is_constant(syn) -> bool:
    """Scalar weight and delay.  Reads only the two fields the reference's
    SynSpec has (sm/construction.py:125-154), so reference objects work."""
    return not isinstance(syn.weight, (tuple, list, np.ndarray)) and \
        not isinstance(syn.delay_steps, (tuple, list, np.ndarray))


def _words(nbits: int) -> int:
    return (int(nbits) + 31) // 32


@dataclass
class PhaseTimers:
    """sm/engine.py:40-52 (seconds per phase).  A façade call is not
    synchronised at its end -- the host prepares the next call while the
    device works -- so each call records CUDA events on its streams; when the
    timers are read, a call counts max(host time, device span of its work)."""

    initialization: float = 0.0
    node_creation: float = 0.0
    local_connection: float = 0.0
    remote_connection: float = 0.0
    preparation: float = 0.0
    propagation: float = 0.0
    _pending: list = field(default_factory=list, repr=False)

    def resolve(self) -> None:
        pending, self._pending = self._pending, []
        for bucket, host_s, pairs in pending:
            gpu_s = 0.0
            for a, b in pairs:
                b.synchronize()
                gpu_s = max(gpu_s, a.elapsed_time(b) * 1e-3)
            setattr(self, bucket, getattr(self, bucket) + max(host_s, gpu_s))

    def as_dict(self) -> dict:
        self.resolve()
        return {k: v for k, v in asdict(self).items() if not k.startswith("_")}


@dataclass
class RunReport:
    """sm/engine.py:55-82; host/device peaks are the modeled-byte arenas of
    memory.py (the reference's cost table and placement plans)."""

    n_ranks: int
    comm_mode: str
    opt_level: int
    seed: int
    kernel_backend: str
    n_neurons: int
    n_synapses: int
    timers: dict
    warmup_s: float
    model_time_s: float
    rtf: float
    host_peak_bytes: list
    device_peak_bytes: list
    transport_messages: dict
    transport_bytes: dict
    n_spike_events: int
    raster_sha256: str | None


class _Buf:
    """Growable 1-D device buffer."""

    def __init__(self, dtype, device, cap=0, fill=None):
        self.dtype, self.device, self.fill = dtype, device, fill
        self.t = self._alloc(max(cap, 16))
        self.n = 0

    def _alloc(self, cap):
        if self.fill is None:
            return torch.empty(cap, dtype=self.dtype, device=self.device)
        return torch.full((cap,), self.fill, dtype=self.dtype, device=self.device)

    def reserve(self, n, headroom: float = 0.0):
        """Capacity for n entries; a reallocation copies the used part only.
        headroom: extra fraction of n allocated on growth (record buffers use
        it so a later, smaller connect call does not move the earlier ones)."""
        if n > self.t.numel():
            cap = max(n + int(n * headroom), int(self.t.numel() * 1.5) + 16)
            nt = self._alloc(cap)
            if self.n:
                nt[: self.n].copy_(self.t[: self.n])
            self.t = nt

    def view(self, a=0, b=None):
        return self.t[a: self.n if b is None else b]


class _Map:
    """Dense remote-source map (group, source rank) on a target rank:
    img_of[value] (-1 = no image) plus a presence bitmap.  (R, L) of the
    reference is the compaction of the bitmap (sm/construction.py:183-242)."""

    def __init__(self, device):
        self.img_of = _Buf(torch.int32, device, fill=-1)
        self.present = _Buf(torch.int32, device, fill=0)
        # node-value intervals that may hold images (host-side knowledge, for _dist_speculate)
        self.imaged: list = []
        self.runs: dict = {}   # (lo, hi) source run imaged whole and consecutively -> its first image id

    def ensure(self, n_values: int):
        nw = _words(n_values)
        self.present.reserve(nw)
        self.present.n = max(self.present.n, nw)
        self.img_of.reserve(nw * 32)
        self.img_of.n = max(self.img_of.n, nw * 32)


class _Bits:
    """Growable bitmap over node values."""

    def __init__(self, device):
        self.b = _Buf(torch.int32, device, fill=0)

    def ensure(self, n_values):
        nw = _words(n_values)
        self.b.reserve(nw)
        self.b.n = max(self.b.n, nw)
        return self

    @property
    def t(self):
        return self.b.view()


class _Rank:
    """Everything one local rank owns on its device."""

    def __init__(self, rank: int, device: torch.device):
        self.rank = rank
        self.device = device
        self.n_nodes = 0
        self.n_real = 0
        self.node2row = _Buf(torch.int32, device, fill=-1)     # device node -> row
        self.row2node: list[np.ndarray] = []
        self.row_gid: list[np.ndarray] = []
        self.row_param: list[np.ndarray] = []
        self.v0: list[torch.Tensor] = []
        self.keys = _Buf(torch.int32, device)
        self.vals = _Buf(torch.int32, device)
        self.wide = False
        self.w_rows = self.w_w = self.w_meta = None
        self.lut = _Buf(torch.int32, device)
        self.maps: dict[tuple, _Map] = {}
        self.mirrors: dict[int, _Bits] = {}
        self.rosters: dict[tuple, _Bits] = {}
        self.devices: list[dict] = []
        self.used_classes: set[int] = set()
        self.mem: RankMemory | None = None   # modeled-byte arenas (memory.py)
        self.prepared = False
        # fixed-in-degree draws whose generation is deferred to prepare, where
        # it runs fused with the first sort pass (csrc/fused.cu); any other
        # record-producing call first generates them into the pending
        # buffers, in call order (fused_ok then stays False)
        self.deferred: list[dict] = []
        self.pending_errs: list = []   # device error flags of asynchronous syn-stream chains
        self.fused_ok = True
        self.fz = None     # fused-path session: record format and every call's digit regions

    @property
    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def map_for(self, group, src_rank) -> _Map:
        key = (int(group), int(src_rank))
        if key not in self.maps:
            self.maps[key] = _Map(self.device)
        return self.maps[key]

    RECORD_HEADROOM = 0.5

    def reserve_records(self, n_new):
        need = self.keys.n + n_new
        h = self.RECORD_HEADROOM
        self.keys.reserve(need, h)
        self.vals.reserve(need, h)
        if self.wide:
            self.w_rows.reserve(need, h)
            self.w_w.reserve(need, h)
            self.w_meta.reserve(need, h)
        return self.keys.n

    def commit_records(self, n_new):
        self.keys.n += n_new
        self.vals.n += n_new
        if self.wide:
            self.w_rows.n += n_new
            self.w_w.n += n_new
            self.w_meta.n += n_new


class Cluster:
    """GPU cluster with the reference façade (sm/engine.py:197-399)."""

    def __init__(self, cfg: SimConfig, devices=None, local_ranks=None, profile: bool = False):
        t0 = time.perf_counter()
        self.prof = {"gen": [], "sort": []} if profile else None
        if not torch.cuda.is_available():
            raise RuntimeError("spikemesh-b200 needs a CUDA device (no CPU fallback)")
        _lib.lib()
        self.cfg = cfg
        self.timers = PhaseTimers()
        self.now = 0
        self.prepared = False
        self.n_ranks = cfg.n_ranks
        dist = torch.distributed
        self.distributed = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        if local_ranks is None:
            if self.distributed:
                if dist.get_world_size() != cfg.n_ranks:
                    raise ValueError("one process per rank: world_size must equal n_ranks")
                local_ranks = [dist.get_rank()]
            else:
                local_ranks = list(range(cfg.n_ranks))
        self.local = sorted(int(r) for r in local_ranks)
        if devices is None:
            if self.distributed:
                devices = [torch.device("cuda", torch.cuda.current_device())]
            else:
                devices = [torch.device("cuda", 0)]
        devices = [torch.device(d) for d in devices]
        if len({(d.type, d.index) for d in devices}) > 1:
            # native calls run on the current device's stream and per-device
            # kernel attributes are configured once per process: several
            # devices need one process each (torchrun), not one Cluster
            raise ValueError("one Cluster drives one device; use one process per GPU (torchrun) for several")
        # native calls launch on the current device (kernel attributes and the
        # error word are per device): every façade call makes this one current
        self.device = devices[0]
        self._on_device()
        self.ranks: dict[int, _Rank] = {
            r: _Rank(r, devices[i % len(devices)]) for i, r in enumerate(self.local)}
        for st in self.ranks.values():
            st.mem = RankMemory(cfg.opt_level, cfg.block_size)
        for d in {st.device for st in self.ranks.values()}:
            with torch.cuda.device(d):
                torch.cuda.current_stream(d)  # make sure the context exists
                call("smx_pool_setup", d.index if d.index is not None else 0)
        # host-side counters and node counts for every rank (scripts run everywhere)
        self.n_nodes = [0] * cfg.n_ranks
        self.images_made = [False] * cfg.n_ranks
        self.local_ctr = [0] * cfg.n_ranks
        self.pair_ctr: dict[tuple, int] = {}
        self.dist_ctr = 0
        self.groups: dict[int, tuple] = {}
        self.params: list[LifParams] = []
        self._ref_min = None
        self.param_index: dict = {}
        self.classes: list[tuple] = []      # (weight, delay, port)
        self.class_index: dict = {}
        self.any_p2p = False
        self.min_remote_delay = None
        self.use_graphs = True
        self.fused_enabled = self.FUSED_ENABLED   # fused generation + sort (tests switch it off for A/B)
        # distributed calls whose pass A started on predicted keys (_dist_speculate)
        self.spec_stats = {"confirmed": 0, "redone": 0, "dropped": 0}
        self._graph = None
        self._xgraph_ok = None   # exchange captured in the block graph (None: not tried yet)
        self._pg = None
        self.messages = {p: 0 for p in PHASES}
        self.bytes = {p: 0 for p in PHASES}
        self.phase = "construction"
        self.timers.initialization += time.perf_counter() - t0

    # ------------------------------------------------------------------ utils
    def is_local(self, r) -> bool:
        return int(r) in self.ranks

    def _key(self, sid):
        return stream_key(self.cfg.seed, sid)

    @contextmanager
    def _timed(self, bucket):
        """Phase timer of one façade call (sm/engine.py:212-219), with an NVTX
        range of the same name for nsys / ncu timelines."""
        self._on_device()
        starts = [(st, self._event(st)) for st in self.ranks.values()]
        t0 = time.perf_counter()
        torch.cuda.nvtx.range_push(bucket)
        try:
            yield
        finally:
            torch.cuda.nvtx.range_pop()
            host_s = time.perf_counter() - t0
            self.timers._pending.append((bucket, host_s, [(a, self._event(st)) for st, a in starts]))

    def _on_device(self):
        if self.device.index is not None and torch.cuda.current_device() != self.device.index:
            torch.cuda.set_device(self.device)

    @staticmethod
    def _event(st):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(st.device))
        return e

    def kernel_ms(self, what: str) -> float:
        """Summed CUDA-event time of the profiled C-ABI calls ('gen', 'sort')."""
        torch.cuda.synchronize()
        return float(sum(a.elapsed_time(b) for a, b in self.prof[what]))

    def _require_unprepared(self):
        if self.prepared:
            raise ConsistencyError("construction after preparation")

    def _param_id(self, p: LifParams) -> int:
        key = tuple(asdict(p).values())
        if key not in self.param_index:
            self.param_index[key] = len(self.params)
            self.params.append(p)
        return self.param_index[key]

    def _class_id(self, weight: float, delay: int, port: int):
        key = (float(weight), int(delay), int(port))
        if key not in self.class_index:
            self.class_index[key] = len(self.classes)
            self.classes.append(key)
        return self.class_index[key]

    # ------------------------------------------------------------ node creation
    def declare_group(self, group_id: int, members) -> None:
        with self._timed("initialization"):
            members = tuple(int(m) for m in members)
            if group_id < 0:
                raise ValueError(f"group ids must be >= 0, got {group_id}")
            if len(set(members)) != len(members) or not members:
                raise ValueError(f"group members must be a non-empty unique list, got {members}")
            for m in members:
                if not 0 <= m < self.n_ranks:
                    raise ValueError(f"group member rank {m} out of range")
            if group_id in self.groups:
                raise ValueError(f"group {group_id} already declared")
            self.groups[group_id] = members

    def create_neurons(self, rank: int, n: int, params: LifParams | None = None, v_init=None,
                       gids=None) -> range:
        """sm/construction.py:335-370; initial V per gid drawn on the device."""
        with self._timed("node_creation"):
            self._require_unprepared()
            if n <= 0:
                raise ValueError(f"need n >= 1 neurons, got {n}")
            params = params if params is not None else LifParams()
            start = self.n_nodes[rank]
            if not self.is_local(rank) and self.images_made[rank]:
                raise NotImplementedError(
                    "node ranges of a remote rank are unknown after it created images")
            gids_run = gids is None   # the default gids are a run: no host scan to upload them
            if gids_run:
                gids = np.arange(start, start + n, dtype=np.int64)
            else:
                gids = np.asarray(gids, dtype=np.int64)
                if len(gids) != n:
                    raise ValueError("gids must have one entry per neuron")
            self.n_nodes[rank] = start + n
            # smallest refractory period of the whole network (every process
            # runs the script): bounds the spikes per neuron in an exchange block
            ref = int(round(params.t_ref / self.cfg.resolution_ms))
            self._ref_min = ref if self._ref_min is None else min(self._ref_min, ref)
            if not self.is_local(rank):
                return range(start, start + n)
            st = self.ranks[rank]
            st.mem.later("neurons", n)
            dev = st.device
            if v_init is None:
                v = torch.full((n,), float(params.v_rest), dtype=torch.float64, device=dev)
            elif isinstance(v_init, tuple):
                if len(v_init) != 3 or v_init[0] != "normal":
                    raise ValueError(f"bad v_init spec {v_init!r}")
                v = torch.empty(n, dtype=torch.float64, device=dev)
                if gids_run:
                    H2D_BYTES[0] += 16   # as _up_index counts a run
                    g = torch.arange(start, start + n, dtype=torch.int64, device=dev)
                else:
                    g = _up_index(gids, dev)
                pre = canonical_bytes((int(self.cfg.seed), ("init-v", 0)))
                prefix = pre[: pre.rindex(b"i:0))") + 2]
                suffix = b"))"
                call("smx_init_v", prefix, len(prefix), suffix, len(suffix), _ptr(g), n,
                     float(v_init[1]), float(v_init[2]), _ptr(v), st.stream)
            elif np.ndim(v_init) == 0:
                v = torch.full((n,), float(v_init), dtype=torch.float64, device=dev)
            else:
                v = _up(np.asarray(v_init, dtype=np.float64), dev)
                if v.numel() != n:
                    raise ValueError("v_init must have one entry per neuron")
            row0 = st.n_real
            st.node2row.reserve(start + n)
            st.node2row.t[start: start + n] = torch.arange(row0, row0 + n, dtype=torch.int32, device=dev)
            st.node2row.n = start + n
            st.row2node.append(np.arange(start, start + n, dtype=np.int64))
            st.row_gid.append(gids)
            st.row_param.append(np.full(n, self._param_id(params), dtype=np.int32))
            st.v0.append(v)
            st.n_real += n
            st.n_nodes = start + n
            if st.n_real > ROW_MASK:
                raise ValueError("more than 2^24 real neurons on one rank")
            return range(start, start + n)

    def add_poisson_source(self, rank: int, rate_hz: float, weight: float, delay_steps: int, targets,
                           port: int = 0):
        """sm/construction.py:373-384 (stream ("poisson", rank, device index))."""
        with self._timed("node_creation"):
            self._require_unprepared()
            if rate_hz < 0.0:
                raise ValueError(f"rate must be >= 0, got {rate_hz}")
            if delay_steps < 1:
                raise ValueError(f"delay must be >= 1 step, got {delay_steps}")
            targets = np.asarray(targets, dtype=np.int64)
            if len(targets) and (targets.min() < 0 or targets.max() >= self.n_nodes[rank]):
                raise ValueError("poisson targets outside the rank's node range")
            lam = float(rate_hz) * self.cfg.resolution_ms * 1e-3
            if not self.is_local(rank):
                return None
            st = self.ranks[rank]
            d = dict(index=len(st.devices), key=self._key(("poisson", rank, len(st.devices))), lam=lam,
                     enlam=math.exp(-lam), weight=float(weight), delay=int(delay_steps),
                     port=int(port), targets=targets)
            st.devices.append(d)
            return d

    # -------------------------------------------------------------- connections
    @staticmethod
    def _check_real_targets(st: _Rank, targets):
        """Connection targets must be real neurons of the target rank (rows of
        the store), not image nodes: checked against the rank's node ranges."""
        if st.n_nodes == st.n_real or not len(targets):
            return   # no images on the rank: every node index in range is real
        starts = np.array([int(r[0]) for r in st.row2node], dtype=np.int64)
        ends = np.array([int(r[0]) + len(r) for r in st.row2node], dtype=np.int64)
        t = np.asarray(targets, dtype=np.int64)
        if _consecutive(t):   # a population run: its two ends decide
            t = t[[0, -1]]
        i = np.searchsorted(starts, t, side="right") - 1
        if (i < 0).any() or (t >= ends[np.maximum(i, 0)]).any():
            raise ValueError("connection targets must be real neurons of the target rank")

    def _tables(self, st: _Rank, sources, targets, cls, tmp_base=None):
        self._check_real_targets(st, targets)
        dev = st.device
        src = _up_index(sources, dev)
        tgt = _up_index(targets, dev)
        key_tab = torch.empty(len(sources), dtype=torch.int32, device=dev)
        pay_tab = torch.empty(len(targets), dtype=torch.int32, device=dev)
        call("smx_key_table", _ptr(src), len(sources), 0 if tmp_base is None else tmp_base,
             0 if tmp_base is None else 1, _ptr(key_tab), st.stream)
        call("smx_pay_table", _ptr(tgt), len(targets), _ptr(st.node2row.t), st.node2row.n,
             cls & 0xFF, _ptr(pay_tab), st.stream)
        return src, tgt, key_tab, pay_tab

    def _syn_class(self, st: _Rank, syn: SynSpec, port: int):
        """Class id for a constant SynSpec in packed mode, or None (wide)."""
        if _syn_is_constant(syn) and not st.wide:
            cid = self._class_id(float(syn.weight), int(syn.delay_steps), port)
            if cid < MAX_CLASSES:
                st.used_classes.add(cid)
                return cid
        return None

    def _make_wide(self, st: _Rank):
        if st.wide:
            return
        dev = st.device
        n = st.keys.n
        st.w_rows = _Buf(torch.int32, dev, cap=st.keys.t.numel())
        st.w_w = _Buf(torch.float64, dev, cap=st.keys.t.numel())
        st.w_meta = _Buf(torch.int32, dev, cap=st.keys.t.numel())
        if n:
            cw, cm = self._class_tables(dev)
            call("smx_promote_wide", _ptr(st.vals.t), n, _ptr(cw), _ptr(cm), _ptr(st.w_rows.t),
                 _ptr(st.w_w.t), _ptr(st.w_meta.t), st.stream)
        st.w_rows.n = st.w_w.n = st.w_meta.n = n
        st.wide = True

    def _class_tables(self, dev):
        cw = torch.zeros(MAX_CLASSES, dtype=torch.float64)
        cm = torch.zeros(MAX_CLASSES, dtype=torch.int64)
        for i, (w, d, p) in enumerate(self.classes[:MAX_CLASSES]):
            cw[i] = w
            cm[i] = (d & 0xFFFFFF) | (p << 24)
        return _up(cw.numpy(), dev), _up(cm.to(torch.int32).numpy(), dev)

    def _write_syn(self, st: _Rank, syn: SynSpec, port: int, base: int, n: int, syn_key):
        """Per-record weights/delays for wide ranks (sm/construction.py:157-176)."""
        dev = st.device
        w, d = syn.weight, syn.delay_steps
        if isinstance(w, tuple) or isinstance(d, tuple):
            return self._write_syn_random(st, syn, port, base, n, syn_key)
        wv = np.asarray(w, dtype=np.float64)
        dv = np.asarray(d, dtype=np.int64)
        if wv.ndim and len(wv) != n:
            raise ValueError(f"{len(wv)} weights for {n} records")
        if dv.ndim and len(dv) != n:
            raise ValueError(f"{len(dv)} delays for {n} records")
        if dv.ndim and len(dv) and dv.min() < 1:
            raise DelayRangeError(f"connection delays must be >= 1 step, got {dv.min()}")
        if (dv.max() if dv.size else 0) > ROW_MASK or port > 255:
            raise DelayRangeError("delay >= 2^24 steps or port > 255 not representable")
        seg_w = st.w_w.t[base: base + n]
        seg_m = st.w_meta.t[base: base + n]
        if wv.ndim == 0 and dv.ndim == 0:
            call("smx_fill_wide_const", _ptr(seg_w), _ptr(seg_m), n, float(wv),
                 (int(dv) & ROW_MASK) | (port << 24), st.stream)
        else:
            seg_w.copy_(_up(np.broadcast_to(wv, (n,)).copy(), seg_w.device))
            meta = (np.broadcast_to(dv, (n,)).astype(np.int64) & ROW_MASK) | (port << 24)
            seg_m.copy_(_up(meta.astype(np.uint32).view(np.int32), seg_m.device))

    def _write_syn_random(self, st: _Rank, syn: SynSpec, port: int, base: int, n: int, syn_key, out=None):
        """Random syn specs drawn on the device from the call's syn stream:
        normal weights (next64 words) then uniform_int delays continuing at
        the next u32 (sm/construction.py:157-176).  out: (weights, meta)
        tensors to fill instead of the record range [base, base + n)."""
        dev = st.device
        w, d = syn.weight, syn.delay_steps
        seg_w, seg_m = out if out is not None else (st.w_w.t[base: base + n], st.w_meta.t[base: base + n])
        if port > 255:
            raise DelayRangeError("port > 255 not representable")
        u32 = 0
        if isinstance(w, tuple):
            L = _lib.lib()
            chunks = L.smx_normal_chunks_for(n)
            ws = torch.empty(int(L.smx_poisson_workspace(chunks)), dtype=torch.uint8, device=dev)
            cur = torch.zeros(2, dtype=torch.int64, device=dev)
            err = torch.zeros(1, dtype=torch.int32, device=dev)
            call("smx_normal_fill", syn_key[0], syn_key[1], _ptr(cur), float(w[1]), float(w[2]), n, chunks,
                 _ptr(ws), _ptr(seg_w), _ptr(cur[1:]), _ptr(err), st.stream)
            st.pending_errs.append(err)   # checked at prepare (no synchronisation per call)
            # next32 after next64 words starts at the next word: u32 cursor = 2 x words,
            # handed to the delay draw on the device
            u32 = cur[1:2] * 2
        else:
            wv = np.asarray(w, dtype=np.float64)
            if wv.ndim:
                if len(wv) != n:
                    raise ValueError(f"{len(wv)} weights for {n} records")
                seg_w.copy_(_up(wv, dev))
            else:
                seg_w.fill_(float(wv))
        if isinstance(d, tuple):
            lo, hi = int(d[1]), int(d[2])
            if hi > ROW_MASK:
                raise DelayRangeError("delay >= 2^24 steps not representable")
            if isinstance(u32, torch.Tensor):   # continues after the normal weights (device cursor)
                call("smx_draw_chain", _ptr(u32), 0)
                call("smx_delay_fill", syn_key[0], syn_key[1], 0, lo, hi - lo + 1, n, port, _ptr(seg_m), 0,
                     st.stream)
            else:
                call("smx_delay_fill", syn_key[0], syn_key[1], u32, lo, hi - lo + 1, n, port, _ptr(seg_m), 0,
                     st.stream)
        else:
            dv = np.asarray(d, dtype=np.int64)
            if dv.ndim:
                if len(dv) != n:
                    raise ValueError(f"{len(dv)} delays for {n} records")
                meta = (dv & ROW_MASK) | (port << 24)
                seg_m.copy_(_up(meta.astype(np.uint32).view(np.int32), dev))
            else:
                seg_m.fill_(int((int(dv) & ROW_MASK) | (port << 24)) - (1 << 32 if port >= 128 else 0))

    def _emit_records(self, st: _Rank, conn: ConnSpec, sources, targets, syn: SynSpec, port: int,
                      aligned_key, local_key, syn_key, tmp_base=None, pos_bits=None, autapse_fix=False):
        """Realize one call's records into the pending buffers (target side).
        Returns the record count.  sm/construction.py:410-432 + 530-534."""
        n_src, n_tgt = len(sources), len(targets)
        cls = self._syn_class(st, syn, port)
        rule = conn.rule
        if (rule == "fixed_indegree" and conn.allow_multapses and tmp_base is None and pos_bits is None
                and not autapse_fix and self._defer_ok(st, cls, n_src, int(conn.k_in) * n_tgt)):
            # local fixed in-degree draws: generated at prepare, fused with the sort
            src, tgt, key_tab, pay_tab = self._tables(st, sources, targets, cls, None)
            self._defer(st, aligned_key, n_src, int(conn.k_in) * n_tgt, 1, key_tab, pay_tab, int(conn.k_in),
                        n_tgt, cls, src_host=np.asarray(sources, dtype=np.int64))
            return int(conn.k_in) * n_tgt, src
        if (rule == "fixed_total" and local_key == aligned_key and tmp_base is None and pos_bits is None
                and not autapse_fix and self._defer_ok(st, cls, n_src, int(conn.n_total))
                and (st.deferred or int(conn.n_total) >= self.FUSED_TOTAL_MIN)):
            # local fixed total: the target draws continue the stream where the
            # position draws end -- that cursor from a count-only pass, the
            # targets' payloads drawn per record, the positions deferred to
            # pass A with those payloads (kdiv 1)
            n = int(conn.n_total)
            src, tgt, key_tab, pay_tab = self._tables(st, sources, targets, cls, None)
            cdev = torch.zeros(1, dtype=torch.int64, device=st.device)   # stream cursor, chained on the device
            piece = 1 << 31   # one draw call takes < 2^32 records
            for j0 in range(0, n, piece):   # count-only: where the position draws end
                call("smx_draw_chain", _ptr(cdev) if j0 else 0, _ptr(cdev))
                call("smx_gen_draw", aligned_key[0], aligned_key[1], 0, n_src, min(piece, n - j0), 0, 0, 0, 0, 1,
                     0, 0, 0, 0, 0, 0, 0, 0, 0, st.stream)
            rec_pay = torch.empty(max(n, 1), dtype=torch.int32, device=st.device)
            for j0 in range(0, n, piece):   # the targets' payloads, continuing that stream
                call("smx_draw_chain", _ptr(cdev), _ptr(cdev))
                call("smx_gen_draw", local_key[0], local_key[1], 0, n_tgt, min(piece, n - j0), 0, 1, 0,
                     _ptr(pay_tab), 1, 0, _ptr(rec_pay[j0:]), 0, 0, 0, 0, 0, 0, 0, st.stream)
            d = self._defer(st, aligned_key, n_src, n, 1, key_tab, rec_pay, 1, n, cls,
                            src_host=np.asarray(sources, dtype=np.int64))
            return n, src
        self._fused_off(st)
        if cls is None:
            self._make_wide(st)
        src, tgt, key_tab, pay_tab = self._tables(st, sources, targets, 0 if cls is None else cls, tmp_base)
        if rule in ("one_to_one", "assigned"):
            n = n_src
        elif rule == "all_to_all":
            n = n_src * n_tgt
        elif rule == "fixed_indegree":
            n = int(conn.k_in) * n_tgt
        elif rule == "fixed_outdegree":
            n = int(conn.k_out) * n_src
        else:
            n = int(conn.n_total)
        base = st.reserve_records(n)
        keys = st.keys.t[base:]
        vals = (st.w_rows.t if st.wide else st.vals.t)[base:]
        cur = np.zeros(1, dtype=np.uint64)
        # the stream cursor comes back to the host (a synchronisation) only
        # when a later draw continues the same stream
        cur_out = cur.ctypes.data if (autapse_fix or rule == "fixed_total") else 0
        sk = st.stream
        ev0 = self._event(st) if self.prof is not None else None
        if n:
            if rule in ("one_to_one", "assigned"):
                call("smx_gen_pairs", 0, n, n_src, _ptr(key_tab), _ptr(pay_tab), _ptr(keys), _ptr(vals), sk)
            elif rule == "all_to_all":
                call("smx_gen_pairs", 1, n, n_src, _ptr(key_tab), _ptr(pay_tab), _ptr(keys), _ptr(vals), sk)
            elif rule == "fixed_indegree" and not conn.allow_multapses:
                # one choice(n_src, k, replace=False) row per target (sm/construction.py:403-404)
                pos = torch.empty(n, dtype=torch.int32, device=st.device)
                call("smx_choice_rows", aligned_key[0], aligned_key[1], 0, n_src, int(conn.k_in), n_tgt, _ptr(pos),
                     cur.ctypes.data, sk)
                call("smx_records_from_values", _ptr(pos), n, _ptr(key_tab), _ptr(pay_tab), int(conn.k_in),
                     _ptr(keys), _ptr(vals), _ptr(pos_bits), 0, sk)
            elif rule == "fixed_indegree":
                call("smx_gen_draw", aligned_key[0], aligned_key[1], 0, n_src, n, 1, 2, _ptr(key_tab),
                     _ptr(pay_tab), int(conn.k_in), _ptr(keys), _ptr(vals), _ptr(pos_bits), 0,
                     _words(n_src), 0, 0, 0, cur_out, sk)
            elif rule == "fixed_outdegree":
                call("smx_gen_draw", local_key[0], local_key[1], 0, n_tgt, n, 2, 1, _ptr(key_tab),
                     _ptr(pay_tab), int(conn.k_out), _ptr(keys), _ptr(vals), 0, 0, 0, 0, 0, 0, cur_out, sk)
            else:  # fixed_total: positions (aligned) then targets (local; same stream locally)
                same = local_key == aligned_key
                if same and not autapse_fix:
                    # the target draw starts where the position draw ended: cursor chained on the device
                    cdev = torch.empty(1, dtype=torch.int64, device=st.device)
                    call("smx_draw_chain", 0, _ptr(cdev))
                    call("smx_gen_draw", aligned_key[0], aligned_key[1], 0, n_src, n, 1, 0, _ptr(key_tab),
                         0, 1, _ptr(keys), 0, _ptr(pos_bits), 0, _words(n_src), 0, 0, 0, 0, sk)
                    call("smx_draw_chain", _ptr(cdev), 0)
                    call("smx_gen_draw", local_key[0], local_key[1], 0, n_tgt, n, 0, 1, 0,
                         _ptr(pay_tab), 1, 0, _ptr(vals), 0, 0, 0, 0, 0, 0, 0, sk)
                else:
                    call("smx_gen_draw", aligned_key[0], aligned_key[1], 0, n_src, n, 1, 0, _ptr(key_tab),
                         0, 1, _ptr(keys), 0, _ptr(pos_bits), 0, _words(n_src), 0, 0, 0, cur_out, sk)
                    u0 = int(cur[0]) if same else 0
                    call("smx_gen_draw", local_key[0], local_key[1], u0, n_tgt, n, 0, 1, 0,
                         _ptr(pay_tab), 1, 0, _ptr(vals), 0, 0, 0, 0, 0, 0, cur_out, sk)
        if self.prof is not None:
            self.prof["gen"].append((ev0, self._event(st)))
        if autapse_fix and n:
            # redraw self-connections from the same stream, continuing after
            # the pair draws (sm/construction.py:524-529)
            u0 = int(cur[0])
            call("smx_autapse_fix", local_key[0], local_key[1], u0, n_src, _ptr(key_tab), _ptr(keys), _ptr(vals),
                 n, _ptr(st.node2row.t), st.node2row.n, cur.ctypes.data, sk)
        if st.wide:
            self._write_syn(st, syn, port, base, n, syn_key)
        st.commit_records(n)
        return n, src

    def _defer(self, st: _Rank, key, ex, n, kmode, ktab, pay_tab, kdiv, n_tgt, cls, src_host=None, acct=None):
        """Register a fixed in-degree draw for the fused path and launch its
        pass A; when the record format cannot take it, every deferred call
        (this one included) goes through the general path instead."""
        lm_thr = 0 if ex == (1 << 32) else ((1 << 32) - ex) % ex
        d = dict(key=key, ex=int(ex), n=int(n), kmode=kmode, ktab=ktab, pay_tab=pay_tab, cls=int(cls),
                 kdiv=int(kdiv), n_tgt=int(n_tgt), src_host=src_host, acct=acct, prej=lm_thr / 4294967296.0,
                 src_run=src_host is not None and _consecutive(np.asarray(src_host)))
        st.deferred.append(d)
        if not self._fused_eager(st, d):
            self._fused_off(st)
        return d

    def _validate_conn(self, rank, sources, targets, conn, syn, what="connect", ranges=True):
        """Argument checks of a connect call.  ranges=False (a call that no
        local rank takes part in, one process per GPU) skips the O(n) node
        range scans: the processes that do take part raise on bad ranges."""
        sources = np.asarray(sources, dtype=np.int64)
        targets = np.asarray(targets, dtype=np.int64)
        if len(sources) == 0 or len(targets) == 0:
            raise ValueError("connect needs non-empty source and target sets")
        for name, arr, r in (("source", sources, rank[0]), ("target", targets, rank[1])) if ranges else ():
            _, lo, hi = _run_info(arr)
            if lo < 0 or hi >= self.n_nodes[r]:
                raise ValueError(f"{name} index outside the rank's node range")
        conn.validate(len(sources), len(targets))
        syn.validate()
        return sources, targets

    def connect(self, rank: int, sources, targets, conn: ConnSpec, syn: SynSpec, port: int = 0) -> int:
        """sm/construction.py:507-534."""
        with self._timed("local_connection"):
            return self._connect_local(rank, sources, targets, conn, syn, port)

    def _connect_local(self, rank, sources, targets, conn, syn, port, validated=False):
        self._require_unprepared()
        if not validated:
            sources, targets = self._validate_conn((rank, rank), sources, targets, conn, syn,
                                                   ranges=self.is_local(rank))
        if port < 0:
            raise ValueError("ports must be >= 0")
        self.local_ctr[rank] += 1
        if not self.is_local(rank):
            return 0
        st = self.ranks[rank]
        ctr = self.local_ctr[rank]
        k = self._key(("conn-local", rank, ctr))
        n, _ = self._emit_records(st, conn, sources, targets, syn, port, k, k,
                                  self._key(("syn-local", rank, ctr)),
                                  autapse_fix=not conn.allow_autapses and conn.rule in ("fixed_indegree",
                                                                                       "fixed_total"))
        st.mem.later("store_append", n)
        return n

    def connect_remote(self, src_rank: int, sources, tgt_rank: int, targets, conn: ConnSpec,
                       syn: SynSpec, port: int = 0, group: int = POINT_TO_POINT) -> int:
        """sm/construction.py:550-637."""
        with self._timed("remote_connection"):
            return self._remote(src_rank, sources, tgt_rank, targets, conn, syn, port, group)

    def _flagging(self, conn, n_src, n_tgt) -> bool:
        """sm/construction.py:439-451."""
        if conn.rule == "fixed_indegree":
            return int(conn.k_in) * n_tgt / n_src < self.cfg.flag_threshold
        if conn.rule == "fixed_total":
            return int(conn.n_total) / n_src < self.cfg.flag_threshold
        return False

    def _note_remote_delay(self, syn: SynSpec):
        d = syn.delay_steps
        if isinstance(d, tuple):
            m = int(d[1])
        elif isinstance(d, (list, np.ndarray)):
            m = int(np.min(d)) if len(d) else None
        else:
            m = int(d)
        if m is not None:
            self.min_remote_delay = m if self.min_remote_delay is None else min(self.min_remote_delay, m)

    def _bump_pair(self, sr, tr) -> int:
        idx = self.pair_ctr.get((sr, tr), 0) + 1
        self.pair_ctr[(sr, tr)] = idx
        return idx

    def _remote(self, sr, sources, tr, targets, conn, syn, port, group):
        for r in (sr, tr):
            if not 0 <= r < self.n_ranks:
                raise ValueError(f"rank {r} out of range 0..{self.n_ranks - 1}")
        if sr == tr:
            return self._connect_local(sr, sources, targets, conn, syn, port)
        self._require_unprepared()
        members = None
        if group != POINT_TO_POINT:
            members = self.groups.get(group)
            if members is None:
                raise ValueError(f"group {group} is not declared")
            if sr not in members or tr not in members:
                raise ValueError(f"ranks {sr} and {tr} must both belong to group {group}")
        involved = self.is_local(sr) or self.is_local(tr) or (
            members is not None and any(self.is_local(m) for m in members))
        sources, targets = self._validate_conn((sr, tr), sources, targets, conn, syn, ranges=involved)
        n_src, n_tgt = len(sources), len(targets)
        if group == POINT_TO_POINT:
            self.any_p2p = True
        if not self.is_local(tr):
            self.images_made[tr] = True  # the target may have grown images
        self._note_remote_delay(syn)
        idx = self._bump_pair(sr, tr)
        flag = self._flagging(conn, n_src, n_tgt)
        k_src = self._key(("remote-src", sr, tr, idx))
        k_tgt = self._key(("remote-tgt", sr, tr, idx))
        k_syn = self._key(("remote-syn", sr, tr, idx))
        n_rec = 0
        used_pos = None
        if not involved:   # nothing local: the counters above are all this process needs
            return n_rec
        span = _run_info(sources)[2] + 1
        if self.is_local(tr) and self._remote_defer_ok(self.ranks[tr], conn, syn, port, n_src, n_tgt):
            n_rec, used_pos = self._remote_deferred(self.ranks[tr], sr, sources, targets, conn, syn, port, group,
                                                    k_src, flag, span)
        elif self.is_local(tr):
            st = self.ranks[tr]
            dev = st.device
            pos_bits = torch.zeros(_words(n_src), dtype=torch.int32, device=dev) if flag else None
            lut_base = st.lut.n
            n_rec, src_dev = self._emit_records(st, conn, sources, targets, syn, port, k_src, k_tgt, k_syn,
                                                tmp_base=lut_base, pos_bits=pos_bits)
            vbits = torch.zeros(_words(span), dtype=torch.int32, device=dev)
            call("smx_mark_values", _ptr(pos_bits), _ptr(src_dev), n_src, _ptr(vbits), st.stream)
            if flag:
                used_pos = pos_bits
            m = st.map_for(group, sr)
            m.ensure(span)
            self._assign(st, vbits, [(0, _words(span), m)], [[(int(sources.min()), span)]])
            st.lut.reserve(lut_base + n_src)
            call("smx_gather_lut", _ptr(src_dev), n_src, _ptr(m.img_of.t), _ptr(st.lut.t[lut_base:]), st.stream)
            st.lut.n = lut_base + n_src
            st.mem.later("remote_batch", n_src, (int(group), sr), _popcount_dev(m.present.view()), n_rec)
        # source side
        if group == POINT_TO_POINT:
            if self.is_local(sr):
                ss = self.ranks[sr]
                dev = ss.device
                src_dev = _up(sources, dev)
                pb = None
                if flag:
                    if used_pos is not None and used_pos.device == dev:
                        pb = used_pos
                    else:
                        pb = self._replay_positions(ss, conn, n_src, n_tgt, k_src)
                mir = ss.mirrors.setdefault(tr, _Bits(dev)).ensure(span)
                call("smx_mark_values", _ptr(pb), _ptr(src_dev), n_src, _ptr(mir.t), ss.stream)
                ss.mem.later("mirror_size", tr, _popcount_dev(mir.t))
        else:
            for mbr in members:
                if self.is_local(mbr):
                    ms = self.ranks[mbr]
                    src_dev = _up(sources, ms.device)
                    ros = ms.rosters.setdefault((group, sr), _Bits(ms.device)).ensure(span)
                    call("smx_mark_values", 0, _ptr(src_dev), n_src, _ptr(ros.t), ms.stream)
        return n_rec

    def _remote_defer_ok(self, st: _Rank, conn, syn, port, n_src, n_tgt) -> bool:
        return (conn.rule == "fixed_indegree" and conn.allow_multapses and
                self._defer_ok(st, self._syn_class(st, syn, port), n_src, int(conn.k_in) * n_tgt))

    def _remote_deferred(self, st: _Rank, sr, sources, targets, conn, syn, port, group, k_src, flag, span):
        """Target side of a remote fixed in-degree call on the fused path
        (sm/construction.py:550-612): the images come first -- every source
        (unflagged call) or the used ones, from a marking-only replay of the
        position draws (flagged call) -- so the call's keys are final image
        ids and its draws go to pass A like a local call's."""
        dev = st.device
        n_src, n_tgt = len(sources), len(targets)
        k_in = int(conn.k_in)
        cls = self._syn_class(st, syn, port)
        src_dev = _up_index(sources, dev)
        pos_bits = self._replay_positions(st, conn, n_src, n_tgt, k_src) if flag else None
        vbits = torch.zeros(_words(span), dtype=torch.int32, device=dev)
        call("smx_mark_values", _ptr(pos_bits), _ptr(src_dev), n_src, _ptr(vbits), st.stream)
        m = st.map_for(group, sr)
        m.ensure(span)
        # image ids on the host without a readback: a consecutive source run
        # whose values had no images gets n_nodes, n_nodes + 1, ... (every
        # source imaged when unflagged); a run imaged that way before keeps them
        cons, lo, hi = _run_info(sources)
        known = m.runs.get((lo, hi + 1)) if cons else None
        fresh = (cons and not flag and known is None and
                 not any(a < hi + 1 and lo < b for a, b in m.imaged))
        n0 = st.n_nodes
        n_new = self._assign(st, vbits, [(0, _words(span), m)], [[(lo, span)]])
        if fresh and n_new == n_src:
            known = m.runs[(lo, hi + 1)] = n0
        key_tab = torch.empty(n_src, dtype=torch.int32, device=dev)
        call("smx_gather_lut", _ptr(src_dev), n_src, _ptr(m.img_of.t), _ptr(key_tab), st.stream)
        self._check_real_targets(st, targets)
        tgt = _up_index(targets, dev)
        pay_tab = torch.empty(n_tgt, dtype=torch.int32, device=dev)
        call("smx_pay_table", _ptr(tgt), n_tgt, _ptr(st.node2row.t), st.node2row.n, cls & 0xFF, _ptr(pay_tab),
             st.stream)
        n = k_in * n_tgt
        src_host = np.arange(known, known + n_src, dtype=np.int64) if known is not None else key_tab.cpu().numpy()
        self._defer(st, k_src, n_src, n, 1, key_tab, pay_tab, k_in, n_tgt, cls, src_host=src_host)
        st.mem.later("remote_batch", n_src, (int(group), sr), _popcount_dev(m.present.view()), n)
        return n, pos_bits

    def _replay_positions(self, ss: _Rank, conn, n_src, n_tgt, k_src):
        """Source-side replay of the aligned position draws (sm/construction.py:620-627)."""
        pb = torch.zeros(_words(n_src), dtype=torch.int32, device=ss.device)
        n = int(conn.k_in) * n_tgt if conn.rule == "fixed_indegree" else int(conn.n_total)
        cur = np.zeros(1, dtype=np.uint64)
        if n and conn.rule == "fixed_indegree" and not conn.allow_multapses:
            pos = torch.empty(n, dtype=torch.int32, device=ss.device)
            call("smx_choice_rows", k_src[0], k_src[1], 0, n_src, int(conn.k_in), n_tgt, _ptr(pos),
                 cur.ctypes.data, ss.stream)
            call("smx_records_from_values", _ptr(pos), n, 0, 0, 1, 0, 0, _ptr(pb), 0, ss.stream)
        elif n:
            call("smx_gen_draw", k_src[0], k_src[1], 0, n_src, n, 1, 0, 0, 0, 1, 0, 0, _ptr(pb), 0,
                 _words(n_src), 0, 0, 0, cur.ctypes.data, ss.stream)
        return pb

    @staticmethod
    def _rank_intervals(runs, r, total) -> list:
        """Node intervals [a, b) of source rank r in a call's runs."""
        starts, rks, nds = runs
        ends = np.append(starts[1:], total)
        return [(int(nds[i]), int(nds[i]) + int(ends[i] - starts[i])) for i in range(len(starts)) if int(rks[i]) == r]

    def _assign(self, st: _Rank, vbits, segs, hulls=None):
        """New images for set bits of vbits, segments in ascending source-rank
        order: ids n_nodes, n_nodes+1, ... (sm/construction.py:473-486)."""
        arr = (ctypes_segment * len(segs))()
        for i, (w0, nw, m) in enumerate(segs):
            if m is not None:   # the values that may get images here
                h = hulls[i] if hulls is not None else None
                m.imaged.extend(h if h is not None else [(0, 1 << 62)])
            arr[i].word0 = w0
            arr[i].nwords = nw
            arr[i].present = _ptr(m.present.t) if m is not None else 0
            arr[i].img_of = _ptr(m.img_of.t) if m is not None else 0
        n_new = np.zeros(1, dtype=np.int64)
        call("smx_assign_images", _ptr(vbits), vbits.numel(), ctypes_addr(arr), len(segs),
             st.n_nodes, n_new.ctypes.data, st.stream)
        n_new = int(n_new[0])
        if n_new:
            st.node2row.reserve(st.n_nodes + n_new)
            st.node2row.t[st.n_nodes: st.n_nodes + n_new] = -1
            st.n_nodes += n_new
            st.node2row.n = st.n_nodes
            self.n_nodes[st.rank] = st.n_nodes
            self.images_made[st.rank] = True
        return n_new

    def connect_fixed_indegree_distributed(self, source_pops, target_pops, k_in: int, syn: SynSpec,
                                           port: int = 0, group: int = POINT_TO_POINT,
                                           allow_multapses: bool = True) -> int:
        """sm/construction.py:640-703, one fused pass per target rank."""
        with self._timed("remote_connection"):
            return self._dist(source_pops, target_pops, k_in, syn, port, group, allow_multapses)

    def _dist(self, source_pops, target_pops, k_in, syn, port, group, allow_multapses):
        self._require_unprepared()
        if k_in < 0:
            raise ValueError(f"k_in must be >= 0, got {k_in}")
        src_ranks = [int(r) for r, _ in source_pops]
        src_nodes = [np.asarray(nodes, dtype=np.int64) for _, nodes in source_pops]
        if not src_nodes or any(len(a) == 0 for a in src_nodes):
            raise ValueError("source populations must be non-empty")
        syn.validate()
        if not _syn_is_constant(syn) and (not isinstance(syn.weight, (tuple, float, int)) or
                                    not isinstance(syn.delay_steps, (tuple, int, np.integer))):
            # per-record arrays cannot match every source-rank batch (the
            # reference's _realize_syn raises on the first length mismatch)
            raise ValueError("per-record weight/delay arrays are not valid in the distributed rule")
        all_rank = np.concatenate([np.full(len(a), r, dtype=np.int32) for r, a in zip(src_ranks, src_nodes)])
        all_node = np.concatenate(src_nodes)
        total = len(all_node)
        if not allow_multapses and k_in > total:
            raise ValueError(f"k_in {k_in} > population size {total} without multapses")
        self._dist_multi, self._dist_kin = bool(allow_multapses), int(k_in)
        self._runs_total = total
        self._runs_cache = (self.dist_ctr + 1, self._pops_runs(src_ranks, src_nodes))
        for r, a in zip(src_ranks, src_nodes):
            if a.min() < 0 or a.max() >= self.n_nodes[r]:
                raise ValueError("source index outside the source rank's node range")
        self.dist_ctr += 1
        call_idx = self.dist_ctr
        if group == POINT_TO_POINT and (len(set(src_ranks)) > 1 or
                                        any(int(t) not in src_ranks for t, _ in target_pops)):
            self.any_p2p = True
        # value segments per source rank, ascending rank, word aligned
        ranks_sorted = sorted(set(src_ranks))
        span = {r: int(max(a.max() for rr, a in zip(src_ranks, src_nodes) if rr == r)) + 1 for r in ranks_sorted}
        vbase = np.zeros(self.n_ranks, dtype=np.int64)
        seg_words = {}
        acc = 0
        for r in ranks_sorted:
            vbase[r] = acc * 32
            seg_words[r] = (acc, _words(span[r]))
            acc += _words(span[r])
        total_words = acc
        self._dist_arrays = (all_rank, all_node)
        self._seg_nwords = {r: nw for r, (w0, nw) in seg_words.items()}
        n_created = 0
        members = self.groups.get(group) if group != POINT_TO_POINT else None
        if group != POINT_TO_POINT and members is None:
            raise ValueError(f"group {group} is not declared")
        tgt_bits: dict[int, torch.Tensor] = {}   # per target rank: used-value bitmap (when computed)
        work = []
        for tr, tg in target_pops:
            tr = int(tr)
            tg = np.asarray(tg, dtype=np.int64)
            if len(tg) == 0:
                raise ValueError("target populations must be non-empty")
            if not self.is_local(tr) and any(r != tr for r in src_ranks):
                self.images_made[tr] = True
            if any(r != tr for r in src_ranks):
                self._note_remote_delay(syn)
            key = self._key(("dist-indegree", call_idx, tr))
            n = k_in * len(tg)
            need_bits = self.is_local(tr) or any(
                self.is_local(r) for r in (members or ranks_sorted))
            if need_bits and n:
                work.append((tr, tg, key, n))
        # 0. local targets whose keys can be predicted start their pass A first
        #    (it then runs beside every replay below)
        specs = {}
        if self._dist_multi:
            runs0 = self._runs(all_rank, all_node)
            for tr, tg, key, n in work:
                if self.is_local(tr) and runs0 is not None and bool((runs0[1] != tr).any()):
                    st = self.ranks[tr]
                    if tg.min() < 0 or tg.max() >= self.n_nodes[tr]:
                        raise ValueError("target index outside the rank's node range")
                    specs[tr] = self._dist_speculate(st, key, tr, tg, k_in, total, runs0, group, syn, port)
        # 1. source-side replays of the remote targets, launched before the local
        #    draws; their completion checks and presence flags come back in one
        #    asynchronous read, so the host does not wait for the local draw
        remote = []                               # (target rank, replay state or None, bitmap)
        for tr, tg, key, n in work:
            if self.is_local(tr):
                continue
            dev = next(iter(self.ranks.values())).device
            if self._dist_multi:
                R = self._replay_start(dev, key, tr, total, all_rank, all_node, vbase, total_words, n)
                remote.append((tr, R, R["vbits"]))
            else:
                remote.append((tr, None, self._dist_replay(dev, key, tr, total, all_rank, all_node, vbase,
                                                           total_words, n)))
        chk_host, chk_ev = None, None
        if remote:
            big = torch.full((1,), 1 << 62, dtype=torch.int64, device=remote[0][2].device)
            rows = []
            for tr, R, vb in remote:
                ex = R["excl"][-1:] if R is not None and R["first"] < R["n"] else big
                fl = torch.stack([vb[w0: w0 + nw].ne(0).any() for w0, nw in (seg_words[r] for r in ranks_sorted)])
                rows.append(torch.cat([ex, fl.to(torch.int64)]))
            chk = torch.stack(rows)
            chk_host = torch.empty(chk.shape, dtype=torch.int64, pin_memory=True)
            chk_host.copy_(chk, non_blocking=True)
            chk_ev = torch.cuda.Event()
            chk_ev.record()
        # 2. the local targets: replay, images, draw
        for tr, tg, key, n in work:
            if not self.is_local(tr):
                continue
            st = self.ranks[tr]
            if tg.min() < 0 or tg.max() >= self.n_nodes[tr]:
                raise ValueError("target index outside the rank's node range")
            tgt_bits[tr] = self._dist_target(st, key, tr, tg, k_in, total, all_rank, all_node, vbase,
                                             seg_words, total_words, syn, port, group, ranks_sorted,
                                             spec=specs.get(tr, "none"))
        # 3. remote bitmaps and their source ranks (the rare incomplete first
        #    piece continues synchronously)
        if remote:
            chk_ev.synchronize()
            got = chk_host.numpy()
            for (tr, R, vb), row in zip(remote, got):
                if R is not None and int(row[0]) < R["n_distinct"]:
                    vb = self._replay_finish([R])[0]
                    row = [0] + [int(vb[w0: w0 + nw].ne(0).any()) for w0, nw in (seg_words[r] for r in ranks_sorted)]
                tgt_bits[tr] = (vb, [r for r, a in zip(ranks_sorted, row[1:]) if a])
        # counters, in the reference's (target, source-rank) call order
        ros_segs: dict = {}
        for tr, tg in target_pops:
            tr = int(tr)
            if tr not in tgt_bits:
                continue
            vb, present = tgt_bits[tr]
            for sr in present:
                if sr == tr:
                    self.local_ctr[tr] += 1
                else:
                    self._bump_pair(sr, tr)
            if self.is_local(tr):
                n_created += k_in * len(tg)
            # source side: mirrors (p2p) / rosters (collective)
            for sr in present:
                if sr == tr:
                    continue
                w0, nw = seg_words[sr]
                if group == POINT_TO_POINT:
                    if self.is_local(sr):
                        ss = self.ranks[sr]
                        mir = ss.mirrors.setdefault(tr, _Bits(ss.device)).ensure(span[sr])
                        seg = vb[w0: w0 + nw].to(ss.device)
                        call("smx_bits_or", _ptr(mir.t), _ptr(seg), nw, ss.stream)
                        ss.mem.later("mirror_size", tr, _popcount_dev(mir.t))
                else:
                    for mbr in members:
                        if self.is_local(mbr):
                            ros_segs.setdefault((mbr, sr), []).append(vb[w0: w0 + nw].to(self.ranks[mbr].device))
        # rosters: the segments of every target merged in one launch per (member, source rank)
        for (mbr, sr), segs in ros_segs.items():
            ms = self.ranks[mbr]
            ros = ms.rosters.setdefault((group, sr), _Bits(ms.device)).ensure(span[sr])
            ptrs = (ctypes.c_void_p * len(segs))(*[s.data_ptr() for s in segs])
            call("smx_bits_or_many", _ptr(ros.t), ctypes.addressof(ptrs), len(segs), seg_words[sr][1], ms.stream)
        return n_created

    def _present_ranks(self, vb, ranks_sorted, seg_words):
        counts = []
        for r in ranks_sorted:
            w0, nw = seg_words[r]
            counts.append(vb[w0: w0 + nw])
        any_set = torch.stack([c.ne(0).any() for c in counts]).cpu().numpy()
        return [r for r, a in zip(ranks_sorted, any_set) if a]

    def _dist_tables(self, dev, stream, tr, total, all_rank, all_node, vbase, lut_base):
        rk = _up(all_rank, dev)
        nd = _up(all_node, dev)
        vb = _up(vbase.astype(np.uint32).view(np.int32), dev)
        key_tab = torch.empty(total, dtype=torch.int32, device=dev)
        gv_tab = torch.empty(total, dtype=torch.int32, device=dev)
        call("smx_dist_tables", _ptr(rk), _ptr(nd), total, _ptr(vb), tr, lut_base, _ptr(key_tab),
             _ptr(gv_tab), stream)
        return key_tab, gv_tab, rk, nd

    @staticmethod
    def _pops_runs(src_ranks, src_nodes, max_pieces=8):
        """_pieces_of computed from the populations (no concatenated arrays)."""
        starts, rks, nds = [], [], []
        at = 0
        for r, a in zip(src_ranks, src_nodes):
            if len(a) == 0:
                continue
            brk = np.flatnonzero(np.diff(a) != 1) + 1
            for b0 in np.concatenate([[0], brk]):
                b0 = int(b0)
                if starts and rks[-1] == r and nds[-1] + (at + b0 - starts[-1]) == int(a[b0]):
                    pass  # continues the previous run (same rank, next node)
                else:
                    starts.append(at + b0)
                    rks.append(int(r))
                    nds.append(int(a[b0]))
                if len(starts) > max_pieces:
                    return None
            at += len(a)
        if not starts:
            return None
        return np.array(starts, np.int64), np.array(rks, np.int64), np.array(nds, np.int64)

    @staticmethod
    def _pieces_of(all_rank, all_node, max_pieces=8):
        """Runs of consecutive nodes on one source rank: (starts, ranks, first
        nodes), or None beyond max_pieces runs."""
        r = np.asarray(all_rank, dtype=np.int64)
        nd = np.asarray(all_node, dtype=np.int64)
        if len(r) == 0:
            return None
        brk = np.flatnonzero((r[1:] != r[:-1]) | (nd[1:] != nd[:-1] + 1)) + 1
        starts = np.concatenate([[0], brk]).astype(np.int64)
        if len(starts) > max_pieces:
            return None
        return starts, r[starts], nd[starts]

    @staticmethod
    def _pack_pieces(starts, keys0):
        delta = (np.asarray(keys0, dtype=np.int64) - starts) & 0xFFFFFFFF
        return np.concatenate([[len(starts)], starts, delta]).astype(np.uint32)

    def _dist_speculate(self, st, key, tr, tg, k_in, total, runs, group, syn, port):
        """Deferred call with predicted keys, or None.  With every remote map
        of the call fresh and every source value drawn (a fixed in-degree
        draw of K x N_tgt from N_src values covers them all unless K N_tgt is
        small against N_src ln N_src), the images are assigned in (rank, node)
        order from st.n_nodes: the key pieces are known before the replay and
        pass A can run beside it.  _dist_target checks the prediction."""
        starts, rks, nds = runs
        n = k_in * len(tg)
        remote = [r for r in sorted(set(int(x) for x in rks)) if r != tr]
        mode = os.environ.get("SMX_SPECULATE", "1")   # "0": never, "force": whatever the coverage odds
        if mode == "0" or not self._dist_multi or not n or total < 2:
            return None
        if mode != "force" and n < 2.0 * total * (math.log(total) + 6.0):
            return None   # full coverage unlikely
        for r in remote:   # none of the call's remote sources may have an image yet
            m = st.maps.get((int(group), r))
            if m is not None and any(a < y and x < b for a, b in self._rank_intervals(runs, r, total)
                                     for x, y in m.imaged):
                return None
        cls = self._syn_class(st, syn, port)
        if not self._defer_ok(st, cls, total, n):
            return None
        ends = np.append(starts[1:], total)
        keys0 = np.zeros(len(starts), dtype=np.int64)
        nxt = st.n_nodes
        for r in remote:   # images in ascending (rank, node) order
            idx = [i for i in range(len(starts)) if int(rks[i]) == r]
            idx.sort(key=lambda i: int(nds[i]))
            last = -1
            for i in idx:
                nd0, ln = int(nds[i]), int(ends[i] - starts[i])
                if nd0 <= last:
                    return None   # overlapping runs of one rank
                keys0[i] = nxt
                nxt += ln
                last = nd0 + ln - 1
        for i in range(len(starts)):
            if int(rks[i]) == tr:
                keys0[i] = int(nds[i])
        pieces = self._pack_pieces(starts, keys0)
        self._check_real_targets(st, tg)
        dev = st.device
        tgt = _up_index(tg, dev)
        pay_tab = torch.empty(len(tg), dtype=torch.int32, device=dev)
        call("smx_pay_table", _ptr(tgt), len(tg), _ptr(st.node2row.t), st.node2row.n, cls, _ptr(pay_tab), st.stream)
        d = self._defer(st, key, total, n, 3, pieces, pay_tab, k_in, len(tg), cls)
        return d if st.fused_ok else None

    def _final_pieces(self, st, tr, group, runs, total, present):
        """Key pieces with final source rows (local node or image id) when
        every remote run's images are consecutive; None otherwise."""
        starts, rks, nds = runs
        ends = np.append(starts[1:], total)
        keys0 = np.zeros(len(starts), dtype=np.int64)
        checks = []
        for i, (s0, r, nd0) in enumerate(zip(starts, rks, nds)):
            r, nd0, ln = int(r), int(nd0), int(ends[i] - s0)
            if r == tr:
                keys0[i] = nd0
                continue
            if r not in present:
                continue  # no draw falls in this run
            img = st.maps[(int(group), r)].img_of.t[nd0: nd0 + ln]
            ar = torch.arange(ln, dtype=img.dtype, device=img.device)
            checks.append((i, img[0:1], ((img - img[0]) != ar).any().reshape(1)))
        if checks:
            first = torch.cat([c[1] for c in checks]).cpu().numpy()
            bad = torch.cat([c[2] for c in checks]).cpu().numpy()
            if bad.any() or (first < 0).any():
                return None
            for (i, _, _), f in zip(checks, first):
                keys0[i] = int(f)
        return self._pack_pieces(starts, keys0)

    def _dist_target(self, st, key, tr, tg, k_in, total, all_rank, all_node, vbase, seg_words,
                     total_words, syn, port, group, ranks_sorted, spec="none"):
        dev, sk = st.device, st.stream
        lut_base = st.lut.n
        n = k_in * len(tg)
        multi = self._dist_multi
        runs = self._runs(all_rank, all_node) if multi else None
        remote = bool((runs[1] != tr).any()) if runs is not None else bool((np.asarray(all_rank) != tr).any())
        speculated = spec != "none"   # _dist already tried (spec: its deferred call or None)
        spec = spec if speculated else None
        if runs is None:
            # general table: keys gathered from key_tab, used values marked by the draw
            key_tab, gv_tab = self._dist_tables(dev, sk, tr, total, all_rank, all_node, vbase, lut_base)[:2]
            vbits = torch.zeros(max(total_words, 1), dtype=torch.int32, device=dev)
        elif remote:
            # pass A starts before the replay when the keys can be predicted:
            # fresh maps and every source value drawn (checked below)
            if not speculated:
                spec = self._dist_speculate(st, key, tr, tg, k_in, total, runs, group, syn, port)
            # used source values from the early-exit replay of the same stream (what
            # every source rank runs anyway), so images exist before the draw
            vbits = self._dist_replay(dev, key, tr, total, all_rank, all_node, vbase, total_words, n)
        else:
            vbits = torch.zeros(max(total_words, 1), dtype=torch.int32, device=dev)
            if n and total:
                b = int(vbase[tr])
                vbits[b >> 5: (b >> 5) + 1] |= int(np.uint32(1 << (b & 31)).view(np.int32))

        def assign(present):
            segs, hulls = [], []
            for r in ranks_sorted:
                sw0, snw = seg_words[r]
                m = None
                if r != tr and r in present:
                    m = st.map_for(group, r)
                    m.ensure(snw * 32)
                segs.append((sw0, snw, m))
                hulls.append(self._rank_intervals(runs, r, total) if runs is not None else None)
            self._assign(st, vbits, segs, hulls)

        pieces, tmp_keys, present = None, True, None
        if runs is not None:
            if remote:
                present = self._present_ranks(vbits, ranks_sorted, seg_words)
                assign(present)
            else:  # all sources local: nothing to assign, present iff anything was drawn
                present = [tr] if n and total else []
            pieces = self._final_pieces(st, tr, group, runs, total, present)
            if remote and spec is not None:
                d = spec
                if not st.fused_ok or d not in st.deferred:
                    raise ConsistencyError("speculative fused call left the fused path early")
                if pieces is not None:
                    d["acct"] = self._dist_accounting(st, tr, group, n, 0, present, runs, pieces, False, lut_base,
                                                      vbase, seg_words, deferred=True)
                    same = np.array_equal(pieces, d["ktab"])
                    self.spec_stats["confirmed" if same else "redone"] += 1
                    if not same:
                        # some value never drawn: pass A again with the real keys, same place in the order
                        d["ktab"] = pieces
                        if not self._fused_eager(st, d, slot=d["zi"]):
                            self._fused_off(st)   # generates it (real keys, counted) with the others
                    return vbits, present
                # temporary keys needed: drop the speculative call, general path below
                self.spec_stats["dropped"] += 1
                st.deferred.remove(d)
                self._fused_off(st)
            tmp_keys = pieces is None
            if pieces is None:  # images not consecutive: temporary keys resolved through the LUT
                starts, rks, nds = runs
                keys0 = np.where(rks == tr, nds, TMP_KEY | (lut_base + np.asarray(vbase, np.int64)[rks] + nds))
                pieces = self._pack_pieces(starts, keys0)
        cls = self._syn_class(st, syn, port)
        defer = multi and pieces is not None and not tmp_keys and self._defer_ok(st, cls, total, n)
        if not defer:
            self._fused_off(st)
        if cls is None:
            self._make_wide(st)
        self._check_real_targets(st, tg)
        tgt = _up_index(tg, dev)
        pay_tab = torch.empty(len(tg), dtype=torch.int32, device=dev)
        call("smx_pay_table", _ptr(tgt), len(tg), _ptr(st.node2row.t), st.node2row.n,
             0 if cls is None else cls, _ptr(pay_tab), sk)
        if defer:
            # pass A now (fused with the draw), pass B at prepare
            acct = self._dist_accounting(st, tr, group, n, 0, present, runs, pieces, False, lut_base, vbase,
                                         seg_words, deferred=True)
            self._defer(st, key, total, n, 3, pieces, pay_tab, k_in, len(tg), cls, acct=acct)
            return vbits, present
        base = st.reserve_records(n)
        vals = (st.w_rows.t if st.wide else st.vals.t)[base:]
        cur = np.zeros(1, dtype=np.uint64)
        ev0 = self._event(st) if self.prof is not None else None
        mark = runs is None
        if not multi:  # one choice(total, k_in, replace=False) row per target (sm/construction.py:680-683)
            pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            call("smx_choice_rows", key[0], key[1], 0, total, k_in, len(tg), _ptr(pos), cur.ctypes.data, sk)
            call("smx_records_from_values", _ptr(pos), n, _ptr(key_tab), _ptr(pay_tab), k_in,
                 _ptr(st.keys.t[base:]), _ptr(vals), _ptr(vbits), _ptr(gv_tab), sk)
        else:
            kmode, ktab = (1, _ptr(key_tab)) if pieces is None else (3, pieces.ctypes.data)
            # nothing follows on this stream: no cursor, no host synchronisation
            call("smx_gen_draw", key[0], key[1], 0, total, n, kmode, 2, ktab, _ptr(pay_tab), k_in,
                 _ptr(st.keys.t[base:]), _ptr(vals), _ptr(vbits) if mark else 0, 0, vbits.numel(), 1, lut_base,
                 int(vbase[tr]), 0, sk)
        if self.prof is not None:
            self.prof["gen"].append((ev0, self._event(st)))
        if st.wide and not _syn_is_constant(syn):
            self._dist_syn(st, syn, port, key, tr, total, n, base, runs, vbase, total_words, ranks_sorted,
                           pos if not multi else None, None if multi else gv_tab)
        elif st.wide:
            self._write_syn(st, syn, port, base, n, None)
        st.commit_records(n)
        if present is None:
            present = self._present_ranks(vbits, ranks_sorted, seg_words)
            assign(present)
        if tmp_keys:
            # LUT over the concatenated value space: lut[base + gv] = img_of[rank][value]
            st.lut.reserve(lut_base + total_words * 32)
            for r in present:
                if r == tr:
                    continue
                sw0, snw = seg_words[r]
                m = st.maps[(int(group), r)]
                st.lut.t[lut_base + sw0 * 32: lut_base + (sw0 + snw) * 32].copy_(m.img_of.t[: snw * 32])
            st.lut.n = lut_base + total_words * 32
        self._dist_accounting(st, tr, group, n, base, present, runs, pieces, tmp_keys, lut_base, vbase,
                              seg_words)
        return vbits, present

    def _dist_syn(self, st, syn, port, key, tr, total, n, base, runs, vbase, total_words, ranks_sorted,
                  pos, gv_tab):
        """Random weights / delays of a distributed call (sm/construction.py:
        689-703): the reference appends one batch per source rank, its records
        in (source rank, source) order (stable lexsort of the draws), and draws
        each batch's syn values from that batch's stream -- ("syn-local", r, c)
        for its own rank, ("remote-syn", s, r, idx) for the others.  Here the
        call's draws are regenerated as global source values gv (ascending in
        (rank, source)), stably sorted, the batches drawn in sorted order and
        scattered back to the records."""
        dev, sk = st.device, st.stream
        gvk = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        if pos is not None:  # choice rows: the drawn positions are already here
            gvk[:n] = gv_tab[pos[:n].long()]
        elif runs is not None:
            starts, rks, nds = runs
            gvp = self._pack_pieces(starts, np.asarray(vbase, np.int64)[rks] + nds)
            call("smx_gen_draw", key[0], key[1], 0, total, n, 3, 0, gvp.ctypes.data, 0, 1, _ptr(gvk), 0, 0, 0, 0, 0,
                 0, 0, 0, sk)
        else:
            gv_all = self._dist_tables(dev, sk, tr, total, *self._dist_arrays, vbase, 0)[1]
            call("smx_gen_draw", key[0], key[1], 0, total, n, 1, 0, _ptr(gv_all), 0, 1, _ptr(gvk), 0, 0, 0, 0, 0,
                 0, 0, 0, sk)
        nv = max(total_words * 32, 1)
        scratch = torch.empty(2 * max(n, 1), dtype=torch.int32, device=dev)
        idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        counts = torch.empty(nv, dtype=torch.int32, device=dev)
        which = np.zeros(1, dtype=np.int32)
        call("smx_sort_records", _ptr(gvk), _ptr(idx), _ptr(scratch), _ptr(scratch[max(n, 1):]), n,
             max(1, int(nv - 1).bit_length()), 1, 0, _ptr(counts), nv, which.ctypes.data, sk)
        order = (scratch[max(n, 1):] if which[0] else idx)[:n].long()
        per_rank = {}
        csum = torch.cumsum(counts.long(), 0)
        for r in ranks_sorted:
            lo = int(vbase[r])
            per_rank[r] = (lo, lo + 32 * int(self._seg_nwords[r]))
        zero = torch.zeros((), dtype=csum.dtype, device=dev)
        bounds = torch.stack([torch.stack([csum[lo - 1] if lo else zero, csum[hi - 1]])
                              for lo, hi in per_rank.values()]).cpu().numpy()
        tmp_w = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        tmp_m = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        for r, (b0, b1) in zip(per_rank, bounds):
            b0, b1 = int(b0), int(b1)
            if b1 <= b0:
                continue
            if r == tr:
                skey = self._key(("syn-local", tr, self.local_ctr[tr] + 1))
            else:
                skey = self._key(("remote-syn", r, tr, self.pair_ctr.get((r, tr), 0) + 1))
            self._write_syn_random(st, syn, port, 0, b1 - b0, skey, out=(tmp_w[b0:b1], tmp_m[b0:b1]))
        st.w_w.t[base: base + n][order] = tmp_w[:n]
        st.w_meta.t[base: base + n][order] = tmp_m[:n]

    def _dist_accounting(self, st, tr, group, n, base, present, runs, pieces, tmp_keys, lut_base, vbase,
                         seg_words, deferred=None):
        """Modeled bytes of one distributed call on its target rank: the
        reference appends one batch per source rank present, ascending, the
        remote ones through remote_connect (sm/construction.py:689-703)."""
        remote = [r for r in present if r != tr]
        if not remote:
            st.mem.later("store_append", n)
            return None
        # records per source rank: disjoint key ranges of the call's records,
        # counted on the preparation side stream (memory-bound, it overlaps the
        # next call's compute-bound draws)
        los, his, owner = [], [], []
        if runs is not None:
            starts, rks, _ = runs
            m = int(pieces[0])
            lens = np.diff(np.append(starts, self._runs_total))
            for i in range(m):
                k0 = (int(pieces[1 + i]) + int(pieces[1 + m + i])) & 0xFFFFFFFF
                los.append(k0)
                his.append(k0 + int(lens[i]))
                owner.append(int(rks[i]))
        else:
            los.append(0)
            his.append(TMP_KEY)
            owner.append(tr)
            for r in remote:
                sw0, snw = seg_words[r]
                los.append(TMP_KEY | (lut_base + sw0 * 32))
                his.append(TMP_KEY | (lut_base + (sw0 + snw) * 32))
                owner.append(r)
        rng = np.array([len(los)] + los + his, dtype=np.uint64).astype(np.uint32)
        if deferred:  # counted once the records are sorted (prepare): returns (ranges, counts)
            cnt = torch.zeros(len(los), dtype=torch.int64, device=st.device)
            sizes = torch.stack([_popcount_dev(st.maps[(int(group), r)].present.view()) for r in remote])
            st.mem.later("dist_batches", tr, int(group), list(present), owner, cnt, sizes)
            return rng, cnt
        main = torch.cuda.current_stream(st.device)
        side = _prep_stream(st.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            cnt = torch.zeros(len(los), dtype=torch.int64, device=st.device)
            call("smx_count_ranges", _ptr(st.keys.t[base:]), n, rng.ctypes.data, _ptr(cnt), side.cuda_stream)
        # (resolved in prepare on this same side stream; the keys stay untouched
        # until the sort, which only reads them)
        sizes = torch.stack([_popcount_dev(st.maps[(int(group), r)].present.view()) for r in remote])
        st.mem.later("dist_batches", tr, int(group), list(present), owner, cnt, sizes)

    def _dist_replay(self, dev, key, tr, total, all_rank, all_node, vbase, total_words, n):
        """Source-side replay of a remote target's draws: used-value bitmap only
        (compute only, no communication).  Coupon-collector early exit: the
        draws are replayed in growing pieces and the replay stops once every
        distinct source value is marked -- no later draw can add a bit, so the
        bitmap equals the full replay's (SURVEY §7 hard part 6).  The first
        piece is sized for coupon collection (V (ln V + 6) draws for V distinct
        values), so a full-coverage call needs one check."""
        stream = torch.cuda.current_stream(dev).cuda_stream
        if not self._dist_multi:  # the rows form one chain: replay all of them
            _, gv_all, _, _ = self._dist_tables(dev, stream, tr, total, all_rank, all_node, vbase, 0)
            vbits = torch.zeros(max(total_words, 1), dtype=torch.int32, device=dev)
            k = self._dist_kin
            pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            cur = np.zeros(1, dtype=np.uint64)
            call("smx_choice_rows", key[0], key[1], 0, total, k, n // k if k else 0, _ptr(pos), cur.ctypes.data,
                 stream)
            call("smx_records_from_values", _ptr(pos), n, 0, 0, 1, 0, 0, _ptr(vbits), _ptr(gv_all), stream)
            return vbits
        return self._replay_finish([self._replay_start(dev, key, tr, total, all_rank, all_node, vbase,
                                                       total_words, n)])[0]

    def _replay_start(self, dev, key, tr, total, all_rank, all_node, vbase, total_words, n):
        """First piece of an early-exit replay, launched without any host
        synchronisation (the cursor is not read back)."""
        stream = torch.cuda.current_stream(dev).cuda_stream
        R = dict(dev=dev, key=key, total=total, n=n, stream=stream)
        runs = self._runs(all_rank, all_node)
        if runs is None:
            R["gv_all"] = self._dist_tables(dev, stream, tr, total, all_rank, all_node, vbase, 0)[1]
        else:  # mark through keys TMP | gv (piecewise affine): no table
            starts, rks, nds = runs
            R["gvp"] = self._pack_pieces(starts, TMP_KEY | (np.asarray(vbase, np.int64)[rks] + nds))
        R["vbits"] = torch.zeros(max(total_words, 1), dtype=torch.int32, device=dev)
        R["n_distinct"] = self._n_distinct_gv(all_rank, all_node, vbase, total_words)
        R["excl"] = torch.empty(R["vbits"].numel() + 1, dtype=torch.int64, device=dev)
        R["piece"] = max(int(R["n_distinct"] * (math.log(max(R["n_distinct"], 2)) + self.REPLAY_C)), 1 << 20)
        k = min(R["piece"], n)
        if k:
            self._replay_piece(R, 0, k, None)
            if k < n:
                call("smx_bits_prefix", _ptr(R["vbits"]), R["vbits"].numel(), _ptr(R["excl"]), stream)
        R["first"] = k
        return R

    def _replay_piece(self, R, u0, k, cur):
        vb = R["vbits"]
        cptr = cur.ctypes.data if cur is not None else 0
        if "gv_all" in R:
            call("smx_gen_draw", R["key"][0], R["key"][1], u0, R["total"], k, 1, 0, 0, 0, 1, 0, 0, _ptr(vb),
                 _ptr(R["gv_all"]), vb.numel(), 0, 0, 0, cptr, R["stream"])
        else:
            call("smx_gen_draw", R["key"][0], R["key"][1], u0, R["total"], k, 3, 0, R["gvp"].ctypes.data, 0, 1, 0, 0,
                 _ptr(vb), 0, vb.numel(), 1, 0, 0xFFFFFFFF, cptr, R["stream"])

    def _replay_finish(self, states) -> list:
        """Completes the replays: one batched check of the first pieces; the
        rare incomplete ones continue in doubling pieces."""
        need = [R for R in states if R["first"] < R["n"]]
        if need:
            got = torch.stack([R["excl"][-1] for R in need]).cpu().numpy()
            for R, g in zip(need, got):
                if int(g) >= R["n_distinct"]:
                    continue
                # redo the first piece with its cursor, then keep drawing
                cur = np.zeros(1, dtype=np.uint64)
                self._replay_piece(R, 0, R["first"], cur)
                u0, done, piece = int(cur[0]), R["first"], R["piece"] * 2
                while done < R["n"]:
                    k = min(piece, R["n"] - done)
                    self._replay_piece(R, u0, k, cur)
                    u0 = int(cur[0])
                    done += k
                    if done < R["n"]:
                        call("smx_bits_prefix", _ptr(R["vbits"]), R["vbits"].numel(), _ptr(R["excl"]), R["stream"])
                        if int(R["excl"][-1].item()) >= R["n_distinct"]:
                            break
                        piece *= 2
        return [R["vbits"] for R in states]

    def _runs(self, all_rank, all_node):
        """_pieces_of for the current distributed call (computed once per call)."""
        self._runs_total = len(all_node)
        cache = getattr(self, "_runs_cache", None)
        if cache is not None and cache[0] == self.dist_ctr:
            return cache[1]
        runs = self._pieces_of(all_rank, all_node)
        self._runs_cache = (self.dist_ctr, runs)
        return runs

    def _n_distinct_gv(self, all_rank, all_node, vbase, total_words):
        """Distinct (rank, node) source values of a distributed call (cached per call)."""
        cache = getattr(self, "_gv_cache", None)
        if cache is not None and cache[0] == self.dist_ctr:
            return cache[1]
        runs = self._runs(all_rank, all_node)
        if runs is not None:  # union of the runs' node intervals per rank
            starts, rks, nds = runs
            lens = np.diff(np.append(starts, len(all_node)))
            nd = 0
            for r in np.unique(rks):
                iv = sorted((int(a), int(a) + int(b)) for a, b in zip(nds[rks == r], lens[rks == r]))
                hi = -1
                for a, b in iv:
                    nd += max(0, b - max(a, hi))
                    hi = max(hi, b)
            self._gv_cache = (self.dist_ctr, nd)
            return nd
        mask = np.zeros(max(total_words, 1) * 32, dtype=bool)
        mask[vbase[all_rank].astype(np.int64) + all_node] = True
        nd = int(mask.sum())
        self._gv_cache = (self.dist_ctr, nd)
        return nd

    # -------------------------------------------------------------- preparation
    def prepare(self) -> None:
        if self.prepared:
            raise ConsistencyError("cluster already prepared")
        self.phase = "preparation"
        with self._timed("preparation"):
            if not self.distributed:
                gids = np.concatenate([g for st in self.ranks.values() for g in st.row_gid] or
                                      [np.empty(0, np.int64)])
                if not _all_distinct(gids):
                    raise ConsistencyError("neuron gids must be globally unique")
            for st in self.ranks.values():
                self._delay_stats(st)
            self.block = self._block_size()
            self.group_slots = {g: i for i, g in enumerate(sorted(self.groups))}
            for st in self.ranks.values():
                self._prepare_rank(st)
        self.has_p2p = self._compute_has_p2p()
        self.group_ids = sorted(self.groups)
        self.prepared = True

    def _compute_has_p2p(self):
        """sm/engine.py:268-271.  With one process per rank a process cannot
        see the other ranks' maps without communicating, so the round runs
        whenever the (identical) script issued any cross-rank p2p call."""
        if self.distributed:
            return self.any_p2p
        return any(bool(st.mirrors) or any(k[0] == POINT_TO_POINT for k in st.maps)
                   for st in self.ranks.values())

    def _delay_stats(self, st: _Rank):
        """Delays and ports in use (sm/construction.py:759-768) plus the
        smallest record delay (it bounds the multi-step LIF block)."""
        max_delay, max_port, min_delay = 1, 0, None
        if st.wide and st.w_meta.n:
            mm = torch.zeros(3, dtype=torch.int32, device=st.device)
            call("smx_max_meta", _ptr(st.w_meta.t), st.w_meta.n, _ptr(mm), st.stream)
            mm = mm.cpu().numpy().view(np.uint32)
            max_delay, max_port, min_delay = max(max_delay, int(mm[0])), max(max_port, int(mm[1])), int(mm[2])
        elif not st.wide:
            for c in st.used_classes:
                _, d, p = self.classes[int(c)]
                max_delay, max_port = max(max_delay, d), max(max_port, p)
                min_delay = d if min_delay is None else min(min_delay, d)
        for d in st.devices:
            max_delay, max_port = max(max_delay, d["delay"]), max(max_port, d["port"])
        st.max_delay, st.max_port, st.min_delay = max_delay, max_port, min_delay

    def _prepare_rank(self, st: _Rank):
        dev, sk = st.device, st.stream
        n_nodes = st.n_nodes
        st.L = max(2, st.max_delay + 1)
        st.P = 1 + st.max_port
        if n_nodes >= (1 << 31):
            raise ValueError("more than 2^31 nodes on one rank")
        main = torch.cuda.current_stream(dev)
        pre_sort = torch.cuda.Event()
        pre_sort.record(main)  # maps / mirrors / rosters written so far
        # sort the store first (sm/core.py:299-324): it is the long kernel
        # sequence, and everything below up to the first_index check is host
        # work or independent small kernels that overlap it on a side stream
        fused = self._fused_ready(st)
        if st.deferred and st.fused_ok and not fused:
            self._fused_off(st)   # the regions cannot be sorted in one pass B: general path
        if fused:
            self._fused_sort(st)
            sorted_state = None
        else:
            sorted_state = self._sort_pending(st)
        side = _prep_stream(dev)
        side.wait_event(pre_sort)  # not on the sort itself: the side work overlaps it
        with torch.cuda.stream(side):
            self._prepare_tables(st)
        main.wait_stream(side)
        _record_stream(st.__dict__, main)  # side-stream allocations are used on main
        check(_lib.lib().smx_check_device_errors(sk), "construction")  # asynchronous draws
        # every small device result the checks below read, in one transfer
        # (the stream is idle here; each separate .item() would be a round trip)
        probe = self._prepare_probe(st, fused)
        if probe["err"]:
            raise RuntimeError(f"normal weight chain error {probe['err']}")
        if fused and not self._fused_check(st, probe):
            # a digit region overflowed or a raw window was short (both ~never):
            # regenerate every deferred call into the pending buffers and sort
            self._fused_off(st)
            sorted_state = self._sort_pending(st)
            probe = self._prepare_probe(st, False)
            if probe["err"]:
                raise RuntimeError(f"normal weight chain error {probe['err']}")
        n = st.n_records
        if n and probe["fi_last"] != n:
            raise ConsistencyError(f"record source beyond node count {n_nodes}")
        if not probe["rows_ok"]:
            raise ValueError("poisson targets must be real neurons")
        # modeled bytes of construction + prepare (sm/construction.py:763-807);
        # record counts of deferred calls exist only now
        st.mem.resolve()
        st.mem.prepare(st.N, st.P, st.L, st.n_nodes, {k: int(v.numel()) for k, v in st.H.items()}, st.rank,
                       {k: int(v.numel()) for k, v in st.S.items()})
        # record lists are dropped only after the sort has consumed them
        del sorted_state
        st.keys = st.vals = None
        st.w_rows = st.w_w = st.w_meta = None
        st.lut = None
        st.fz = None
        st.deferred = []
        max_len = probe["max_len"]
        max_chunks = max(1, -(-max_len // 1024))
        st.owner_cap = st.N * self.block * max_chunks + 16
        st.owner = torch.zeros(st.owner_cap, dtype=torch.int32, device=dev)
        self._place(st)
        st.prepared = True

    @staticmethod
    def _place(st: _Rank):
        """The optimisation level's placement plan made real
        (sm/construction.py:43-71): structures the plan puts on the host move
        to pinned host memory, which the kernels read in place over the host
        link (zero-copy; same pointer under unified addressing); counts the
        plan drops (level 2) are freed.  Results never depend on the
        placement, only speed and HBM use do."""
        from .memory import HOST
        plan = st.mem.plan

        def host(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)   # ordered on the rank's stream before every later kernel
            return h
        if plan.first_index == HOST:
            st.first_index = host(st.first_index)
        if plan.counts is None:
            st.counts = None
        elif plan.counts == HOST and st.counts is not None:
            st.counts = host(st.counts)
        if plan.remote_source_maps == HOST:
            st.RL = {k: tuple(host(x) for x in v) for k, v in st.RL.items()}
        if plan.image_maps == HOST:
            st.I = {k: host(v) for k, v in st.I.items()}

    def _sort_pending(self, st: _Rank):
        """General path: stable LSD sort of the pending (key, value) records by
        source (sm/core.py:299-324), per-source counts and first_index.
        Returns the scratch that must outlive the asynchronous sort."""
        dev, sk = st.device, st.stream
        n_nodes = st.n_nodes
        n = st.keys.n
        st.n_records = n
        st.store_path = "general"
        key_bits = max(1, int(n_nodes - 1).bit_length())
        st.counts = torch.empty(max(n_nodes, 1), dtype=torch.int32, device=dev)
        # scratch pair in one allocation: the sort's intermediate passes use it
        # as n (key, value) records
        scratch = torch.empty(2 * max(n, 1), dtype=torch.int32, device=dev)
        kb, vb = scratch[: max(n, 1)], scratch[max(n, 1):]
        which = np.zeros(1, dtype=np.int32)
        ev0 = self._event(st) if self.prof is not None else None
        call("smx_sort_records", _ptr(st.keys.t), _ptr(st.vals.t), _ptr(kb), _ptr(vb), n, key_bits,
             1 if st.wide else 0, _ptr(st.lut.t), _ptr(st.counts), n_nodes, which.ctypes.data, sk)
        sorted_vals = (vb if which[0] else st.vals.t)[:n]
        if self.prof is not None:
            self.prof["sort"].append((ev0, self._event(st)))
        st.first_index = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
        call("smx_counts_to_offsets", _ptr(st.counts), n_nodes, _ptr(st.first_index), sk)
        if st.wide:
            st.payload = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            st.ww = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
            st.wm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            call("smx_gather_wide", _ptr(sorted_vals), n, _ptr(st.w_rows.t), _ptr(st.w_w.t), _ptr(st.w_meta.t),
                 _ptr(st.payload), _ptr(st.ww), _ptr(st.wm), sk)
        else:
            st.payload = sorted_vals if n else torch.empty(1, dtype=torch.int32, device=dev)
            st.ww = st.wm = None
        return (scratch, st.keys, st.vals, st.lut)

    # ------------------------------------------------- fused generation + sort
    FUSED_ENABLED = os.environ.get("SMX_FUSED", "1") != "0"
    # Poisson drive batch: at least this many steps per batch (the batch's
    # sequential composition kernels are a fixed cost; longer batches
    # amortise them, at the price of generating up to one batch ahead)
    POIS_MIN_STEPS = int(os.environ.get("SMX_POIS_MIN_STEPS", "64"))
    # fixed_total calls take the fused path when the rank is on it already, or
    # from this size on (below it the general path's two draws + sort are
    # faster; above it they do not fit: 32-bit record index, 20 B/synapse)
    FUSED_TOTAL_MIN = int(os.environ.get("SMX_FUSED_TOTAL_MIN", str(1 << 31)))
    # first replay piece V (ln V + c) draws: covers every value with
    # probability exp(-e^-c) (c = 6: 0.9975); a miss continues in pieces
    REPLAY_C = float(os.environ.get("SMX_REPLAY_C", "6"))
    # SMs pass A leaves to the replays of later calls in multi-rank runs; the
    # replays grow with the rank count (one per remote target rank), so by
    # default 2 per rank up to 16 (measured at 4 GPUs: 8 -> 25.2 ms, 4 -> 31.7)
    PASS_A_FREE_SMS = int(os.environ["SMX_PASS_A_FREE_SMS"]) if "SMX_PASS_A_FREE_SMS" in os.environ else None

    def _defer_ok(self, st: _Rank, cls, ex: int, n: int) -> bool:
        return (self.fused_enabled and st.fused_ok and cls is not None and not st.wide and ex >= 2 and n > 0
                and ex <= (1 << 32))

    def _fused_off(self, st: _Rank):
        """Leave the fused path for good: the deferred calls are generated into
        the pending buffers (same draws, call order) by the general path."""
        if not st.fused_ok:
            return
        st.fused_ok = False
        st.fz = None   # regions of pass A (if any) are dropped
        for d in st.deferred:
            self._gen_deferred(st, d)
        st.deferred = []

    def _gen_deferred(self, st: _Rank, d: dict):
        n = d["n"]

        base = st.reserve_records(n)
        keys, vals = st.keys.t[base:], st.vals.t[base:]
        sk = st.stream
        ev0 = self._event(st) if self.prof is not None else None
        ktab = d["ktab"].ctypes.data if d["kmode"] == 3 else _ptr(d["ktab"])
        call("smx_gen_draw", d["key"][0], d["key"][1], 0, d["ex"], n, d["kmode"], 2, ktab, _ptr(d["pay_tab"]),
             d["kdiv"], _ptr(keys), _ptr(vals), 0, 0, 0, 0, 0, 0, 0, sk)
        if self.prof is not None:
            self.prof["gen"].append((ev0, self._event(st)))
        st.commit_records(n)
        if d["acct"] is not None:  # records per source rank (modeled bytes), as _dist_accounting does
            rng, cnt = d["acct"]
            main = torch.cuda.current_stream(st.device)
            side = _prep_stream(st.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                call("smx_count_ranges", _ptr(keys), n, rng.ctypes.data, _ptr(cnt), side.cuda_stream)

    @staticmethod
    def _call_key_ranges(d: dict) -> list:
        """Key intervals [a, b) a deferred call's draws can produce."""
        if d["kmode"] == 1:
            s = d["src_host"]
            if d.get("src_run"):   # keys a, a + 1, ..., b - 1
                return [(int(s[0]), int(s[-1]) + 1)]
            return [(int(s.min()), int(s.max()) + 1)]
        pc = d["ktab"]
        m = int(pc[0])
        starts = [int(x) for x in pc[1: 1 + m]] + [d["ex"]]
        return [((starts[i] + int(pc[1 + m + i])) & 0xFFFFFFFF,
                 ((starts[i] + int(pc[1 + m + i])) & 0xFFFFFFFF) + starts[i + 1] - starts[i]) for i in range(m)
                if starts[i + 1] > starts[i]]

    @staticmethod
    def _digit_probs(d: dict, B: int) -> np.ndarray:
        """Probability of each low key digit (key mod B) for one draw of a
        deferred call: uniform positions mapped to keys (exact)."""
        cnt = np.zeros(B, dtype=np.float64)
        if d["kmode"] == 1 and not d.get("src_run"):
            cnt += np.bincount(np.asarray(d["src_host"], dtype=np.int64) & (B - 1), minlength=B)
        else:
            for a, b in Cluster._call_key_ranges(d):
                ln = b - a
                cnt += ln // B
                rem = ln % B
                if rem:
                    np.add.at(cnt, (a + np.arange(rem)) & (B - 1), 1.0)
        return cnt / float(d["ex"])

    def _fused_eager(self, st: _Rank, d: dict, slot=None) -> bool:
        """Pass A of one deferred call, launched at call time (it overlaps the
        host work of the calls that follow): the call's draws ranked by the
        low key digit into its own digit regions (csrc/fused.cu).  The record
        format (digit split, row / class bits) is fixed by the rank's first
        call; False when this call does not fit it."""
        z = st.fz
        dev, sk = st.device, st.stream
        if z is None:
            # the call's own keys may lie past the current nodes (predicted images)
            top = max([st.n_nodes] + [b for _, b in self._call_key_ranges(d)])
            key_bits = max(1, int(top - 1).bit_length())
            env_lo = os.environ.get("SMX_FUSED_LO")
            lo = int(env_lo) if env_lo is not None else (
                0 if key_bits <= 11 else max(key_bits - 11, min(9, key_bits - 8)))
            if lo > 9:
                return False
            # payload of 20 bits (with the <= 11-bit high digit: 31-bit records)
            z = st.fz = dict(lo=lo, pbits=20, cidx={}, calls=[], flag=torch.zeros(2, dtype=torch.int64, device=dev))
        # the call's payload split: its target rows (real neurons so far) in
        # the low bits, the class index above (pass B decodes per call)
        row_bits = max(1, int(st.n_real - 1).bit_length())
        if row_bits > z["pbits"] or (slot is None and len(z["calls"]) >= 512):
            return False
        if d["cls"] not in z["cidx"]:
            z["cidx"][d["cls"]] = len(z["cidx"])
        if z["cidx"][d["cls"]] >= (1 << min(8, z["pbits"] - row_bits)):
            return False
        B = 1 << z["lo"]
        p = self._digit_probs(d, B)
        n = float(d["n"])
        # the raw window's slack (accepted draws past the last record) lands
        # in the regions too
        slack = 1.25 * n * d["prej"] + 12.0 * math.sqrt(n * d["prej"] + 1.0) + 64.0
        if (n + slack) * float(p.max()) * 1.05 + 1e4 >= (1 << 30):
            return False   # look-back descriptors hold 30-bit counts
        cap = np.ceil((n + slack) * p + 8.0 * np.sqrt(n * p * (1.0 - p)) + 64.0).astype(np.int64)
        cap = (cap + 31) // 32 * 32
        rstart = np.zeros(B, dtype=np.int64)
        rstart[1:] = np.cumsum(cap)[:-1]
        slots = int(rstart[-1] + cap[-1])
        region = torch.empty(slots, dtype=torch.int32, device=dev)
        meta = _up(np.concatenate([rstart, cap]), dev)
        fills = torch.zeros((2, B), dtype=torch.int64, device=dev)
        total = torch.zeros(1, dtype=torch.int64, device=dev)
        cls_field = z["cidx"][d["cls"]] << row_bits   # pass A packs row | class index << row bits
        # pass A runs on the generation stream: the main stream keeps only the
        # small map / image kernels that the preparation side stream waits on
        gen = _gen_stream(dev)
        gen.wait_stream(torch.cuda.current_stream(dev))
        ev0 = torch.cuda.Event(enable_timing=True) if self.prof is not None else None
        if ev0 is not None:
            ev0.record(gen)
        ktab = d["ktab"].ctypes.data if d["kmode"] == 3 else _ptr(d["ktab"])
        # SMs left free for the replays / small kernels of later calls: only
        # a multi-rank construction has any
        free = self.PASS_A_FREE_SMS if self.PASS_A_FREE_SMS is not None else min(16, 2 * self.n_ranks)
        call("smx_set_pass_a_free_sms", 0 if self.n_ranks == 1 else free)
        call("smx_fused_gen", d["key"][0], d["key"][1], d["ex"], d["n"], d["kmode"], ktab, d["kdiv"],
             _ptr(d["pay_tab"]), cls_field,
             z["lo"], z["pbits"], _ptr(region), slots, _ptr(meta[:B]), _ptr(meta[B:]), _ptr(fills[0]),
             _ptr(fills[1]), _ptr(total), _ptr(z["flag"]), gen.cuda_stream)
        if ev0 is not None:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(gen)
            self.prof["gen"].append((ev0, ev1))
        for tnsr in (region, meta, fills, total, z["flag"], d["pay_tab"]):
            tnsr.record_stream(gen)
        if d["kmode"] == 1:
            d["ktab"].record_stream(gen)
        zc = dict(region=region, rstart=rstart, cap=cap.astype(np.uint64), meta=meta, fill=fills[1],
                  fills=fills, total=total, n=int(d["n"]), row_bits=row_bits)
        if slot is None:   # in call order (pass B keeps it within every key)
            d["zi"] = len(z["calls"])
            z["calls"].append(zc)
        else:              # the same call again (keys corrected): its place in the order stays
            z["calls"][slot] = zc
        return True

    def _fused_ready(self, st: _Rank) -> bool:
        """At prepare: can pass B take the rank's regions (the high digit fits
        12 bits with the final node count; accounted calls own their keys)?"""
        z = st.fz
        if z is None or not st.fused_ok or not st.deferred:
            return False
        key_bits = max(1, int(st.n_nodes - 1).bit_length())
        z["hi"] = max(8, key_bits - z["lo"])
        if z["hi"] > 12 or z["hi"] + z["pbits"] > 32:
            return False
        if z["hi"] + z["pbits"] == 32:
            # 32-bit records: the all-ones word is the sentinel, so no call may
            # be able to produce an all-ones payload (row 2^row_bits - 1 with
            # the largest class index of its split)
            n_cls = len(z["cidx"])
            for zc in z["calls"]:
                rb = zc["row_bits"]
                if (st.n_real >= (1 << rb) and n_cls >= (1 << min(8, z["pbits"] - rb))):
                    return False
        # records per source rank of distributed calls (modeled bytes) come
        # from the per-key counts: every accounted call's keys must be its own
        calls = st.deferred
        acct = [i for i, d in enumerate(calls) if d["acct"] is not None]
        if acct:
            rngs = [self._call_key_ranges(d) for d in calls]
            for i in acct:
                for j, rj in enumerate(rngs):
                    if j != i and any(a < y and x < b for a, b in rngs[i] for x, y in rj):
                        return False
        return True

    def _fused_sort(self, st: _Rank):
        """Pass B over every call's regions, in (low digit, call) order: the
        store's payloads, per-key counts and first_index (csrc/fused.cu)."""
        dev, sk = st.device, st.stream
        z = st.fz
        calls = z["calls"]
        C, B = len(calls), 1 << z["lo"]
        rptr = np.empty((B, C), dtype=np.int64)
        rcap = np.empty((B, C), dtype=np.uint64)
        for c, zc in enumerate(calls):
            rptr[:, c] = zc["region"].data_ptr() + 4 * zc["rstart"]
            rcap[:, c] = zc["cap"]
        rptr_t = _up(rptr.reshape(-1), dev)
        rcap = np.ascontiguousarray(rcap.reshape(-1))
        torch.cuda.current_stream(dev).wait_stream(_gen_stream(dev))   # every call's pass A
        fill = torch.stack([zc["fill"] for zc in calls], dim=1).reshape(-1).contiguous()
        n = sum(zc["n"] for zc in calls)
        st.n_records = n
        cls_map = np.zeros(256, dtype=np.uint32)
        for cls, i in z["cidx"].items():
            cls_map[i] = np.uint32(cls) << np.uint32(24)
        cls_map_t = _up(cls_map.view(np.int32), dev)
        st.counts = torch.empty(max(st.n_nodes, 1), dtype=torch.int32, device=dev)
        st.payload = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        ev0 = self._event(st) if self.prof is not None else None
        rbits = np.array([zc["row_bits"] for zc in calls], dtype=np.uint8)
        call("smx_fused_sort", _ptr(rptr_t), _ptr(fill), rcap.ctypes.data, C, z["lo"], z["hi"], z["pbits"],
             rbits.ctypes.data, _ptr(cls_map_t), _ptr(st.counts), st.n_nodes, n, _ptr(st.payload), _ptr(z["flag"][1:]), sk)
        st.first_index = torch.empty(st.n_nodes + 1, dtype=torch.int64, device=dev)
        call("smx_counts_to_offsets", _ptr(st.counts), st.n_nodes, _ptr(st.first_index), sk)
        if self.prof is not None:
            self.prof["sort"].append((ev0, self._event(st)))
        st.ww = st.wm = None
        st.store_path = "fused"
        # records per source rank of accounted distributed calls: sums of the
        # per-key counts over the call's key ranges (keys are the call's own)
        cs = None
        for d in st.deferred:
            if d["acct"] is None:
                continue
            if cs is None:
                cs = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(st.counts.long(), 0)])
            rng, cnt = d["acct"]
            m = int(rng[0])
            los = _up(rng[1: 1 + m].astype(np.int64), dev).clamp(max=st.n_nodes)
            his = _up(rng[1 + m: 1 + 2 * m].astype(np.int64), dev).clamp(max=st.n_nodes)
            cnt.copy_(cs[his] - cs[los])
        z["keep"] = (rptr_t, fill, cls_map_t)

    @staticmethod
    def _prepare_probe(st: _Rank, fused: bool) -> dict:
        """The device scalars prepare checks after the sort, fetched with one
        device->host copy: the normal-chain error word, the fused flags and
        per-call totals, first_index's last entry and the longest key run."""
        parts, names = [], []

        def add(name, t):
            t = t.reshape(-1).to(torch.int64)
            names.append((name, t.numel()))
            parts.append(t)

        if st.pending_errs:
            add("err", torch.stack(st.pending_errs).max())
            st.pending_errs = []
        if fused:
            add("flag", st.fz["flag"])
            add("totals", torch.cat([zc["total"] for zc in st.fz["calls"]]))
        fi = st.first_index
        if st.n_records:
            add("fi_last", fi[-1])
        if st.n_nodes:
            add("max_len", (fi[1:] - fi[:-1]).max())
        oks = [d["rows_ok"] for d in st.devices if d.get("rows_ok") is not None]
        if oks:
            add("rows_ok", torch.stack(oks).all())
        flat = torch.cat(parts).cpu().numpy() if parts else np.empty(0, np.int64)
        out = {"err": 0, "fi_last": 0, "max_len": 0, "rows_ok": 1}
        at = 0
        for name, k in names:
            out[name] = flat[at: at + k] if name in ("flag", "totals") else int(flat[at])
            at += k
        return out

    def _fused_check(self, st: _Rank, probe: dict) -> bool:
        z = st.fz
        f = probe["flag"]
        if int(f[0]):
            return False   # a region overflowed: its records are incomplete (pass B saw a clamped fill)
        if int(f[1]):
            raise ConsistencyError(f"fused sort: device error {int(f[1])}")
        want = np.array([zc["n"] for zc in z["calls"]], dtype=np.int64)
        return bool((probe["totals"] >= want).all())

    def _prepare_tables(self, st: _Rank):
        """Everything of prepare that does not read the sorted store: neuron
        state, class tables, (R, L), S, H, I, T/P, G/Q, propagation buffers."""
        dev = st.device
        dt = self.cfg.resolution_ms
        # neuron state, real rows only (sm/dynamics.py:153-189)
        N = st.n_real
        st.N = N
        # per-row parameters gathered on the device from the (small) table of
        # distinct LifParams; decay = exp(-dt / tau) from the host (glibc)
        tab = np.array([[math.exp(-dt / p.tau_m), p.v_rest, p.v_reset, p.v_th, p.i_e] for p in self.params] or
                       [[0.0] * 5], dtype=np.float64)
        rs = np.array([int(round(p.t_ref / dt)) for p in self.params] or [0], dtype=np.int32)
        pid = [(int(p[0]), len(p)) for p in st.row_param]
        prm = (torch.cat([torch.full((k,), i, dtype=torch.int64, device=dev) for i, k in pid]) if pid
               else torch.zeros(0, dtype=torch.int64, device=dev))
        tab_t = _up(np.ascontiguousarray(tab.T), dev)
        st.decay, st.v_rest, st.v_reset, st.v_th, st.i_e = (tab_t[j][prm].contiguous() for j in range(5))
        st.ref_steps = _up(rs, dev)[prm].contiguous()
        st.v = torch.cat(st.v0) if st.v0 else torch.empty(0, dtype=torch.float64, device=dev)
        st.ref = torch.zeros(N, dtype=torch.int32, device=dev)
        st.row2node_np = np.concatenate(st.row2node) if st.row2node else np.empty(0, np.int64)
        st.row2node_t = (torch.cat([torch.arange(int(r[0]), int(r[0]) + len(r), dtype=torch.int32, device=dev)
                                    for r in st.row2node]) if st.row2node
                         else torch.zeros(0, dtype=torch.int32, device=dev))
        st.gid_np = np.concatenate(st.row_gid) if st.row_gid else np.empty(0, np.int64)
        st.gid_t = (torch.cat([_up_index(g, dev) for g in st.row_gid]) if st.row_gid
                    else torch.zeros(0, dtype=torch.int64, device=dev))
        st.ring = torch.zeros(st.L * st.P * max(N, 1), dtype=torch.float64, device=dev)
        st.cls_w, cm = self._class_tables(dev)
        cmn = cm.cpu().numpy().view(np.uint32)
        st.cls_delay = _up((cmn & ROW_MASK).astype(np.int32), dev)
        st.cls_port = _up((cmn >> 24).astype(np.int32), dev)
        # maps -> sorted (R, L) (sm/construction.py:183-242)
        st.RL = {}
        for key, m in st.maps.items():
            st.RL[key] = self._compact(st, m.present.view(), m.img_of.view())
        # mirrors -> S (source side of each p2p pair)
        st.S = {tr: self._compact(st, b.t, None)[0] for tr, b in st.mirrors.items()}
        # rosters -> H; image lookups I (sm/construction.py:780-803)
        st.H, st.I = {}, {}
        for key in sorted(st.rosters):
            st.H[key] = self._compact(st, st.rosters[key].t, None)[0]
        for key in sorted(st.H):
            g, sr = key
            if sr == st.rank:
                continue
            m = st.maps.get(key)
            if m is not None:
                rw = st.rosters[key].t
                pw = m.present.view()
                nw = min(rw.numel(), pw.numel())
                extra = (pw[:nw] & ~rw[:nw]).ne(0).any() or pw[nw:].ne(0).any()
                if bool(extra):
                    raise ConsistencyError(f"rank {st.rank}: map keys for {key} missing from roster")
                m.ensure(rw.numel() * 32)
                st.I[key] = self._compact(st, rw, m.img_of.view())[1]
            else:
                st.I[key] = torch.full((st.H[key].numel(),), -1, dtype=torch.int64, device=dev)
        # routing tables: T/P from mirrors (dest = target rank, ascending),
        # G/Q from own rosters (dest = group slot, groups ascending)
        st.TP = self._routes(st, [(tr, st.mirrors[tr].t) for tr in sorted(st.mirrors)])
        own = [(self.group_slots[g], st.rosters[(g, sr)].t) for (g, sr) in sorted(st.rosters) if sr == st.rank]
        st.GQ = self._routes(st, own)
        # propagation buffers
        self._alloc_propagation(st)

    def _compact(self, st, bits, img_of):
        nw = bits.numel()
        excl = torch.empty(nw + 1, dtype=torch.int64, device=st.device)
        call("smx_bits_prefix", _ptr(bits), nw, _ptr(excl), st.stream)
        cnt = int(excl[-1].item())
        vals = torch.empty(max(cnt, 1), dtype=torch.int64, device=st.device)
        imgs = torch.empty(max(cnt, 1), dtype=torch.int64, device=st.device)
        call("smx_bits_compact", _ptr(bits), nw, _ptr(excl), _ptr(vals), _ptr(img_of), _ptr(imgs), st.stream)
        return vals[:cnt], imgs[:cnt]

    def _routes(self, st, tables):
        dev = st.device
        n_nodes = st.n_nodes
        if not tables:  # no mirror / roster: empty routing table, no kernel and no readback
            empty = torch.zeros(1, dtype=torch.int32, device=dev)
            return dict(first=torch.zeros(n_nodes + 1, dtype=torch.int64, device=dev), dest=empty[:0], pos=empty[:0],
                        n=0)
        arr = (ctypes_route * max(len(tables), 1))()
        keep = []
        for i, (dest, bits) in enumerate(tables):
            excl = torch.empty(bits.numel() + 1, dtype=torch.int64, device=dev)
            call("smx_bits_prefix", _ptr(bits), bits.numel(), _ptr(excl), st.stream)
            keep.append(excl)
            arr[i].bits = _ptr(bits)
            arr[i].excl = _ptr(excl)
            arr[i].nwords = bits.numel()
            arr[i].dest = int(dest)
        first = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
        cnt = torch.empty(max(n_nodes, 1), dtype=torch.int32, device=dev)
        ne_h = np.zeros(1, dtype=np.int64)
        call("smx_build_routes", ctypes_addr(arr), len(tables), n_nodes, _ptr(cnt), _ptr(first), 0, 0,
             ne_h.ctypes.data, st.stream)
        ne = int(ne_h[0])
        dest = torch.empty(max(ne, 1), dtype=torch.int32, device=dev)
        pos = torch.empty(max(ne, 1), dtype=torch.int32, device=dev)
        call("smx_build_routes", ctypes_addr(arr), len(tables), n_nodes, _ptr(cnt), _ptr(first), _ptr(dest),
             _ptr(pos), ne_h.ctypes.data, st.stream)
        return dict(first=first, dest=dest[:ne], pos=pos[:ne], n=ne)

    def _alloc_propagation(self, st):
        dev = st.device
        N = st.N
        B = self.block
        st.spike_bits = torch.zeros(max(_words(N), 1), dtype=torch.int32, device=dev)
        st.now_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        st.record_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        # packets of one exchange block (B steps): p2p per destination rank,
        # collective per group slot; entries are (position, emission step)
        st.pk_cap = max(N, 1) * B
        st.p2p_packets = torch.zeros(self.n_ranks * st.pk_cap * 2, dtype=torch.int32, device=dev)
        st.p2p_counts = torch.zeros(self.n_ranks, dtype=torch.int32, device=dev)
        ng = max(len(self.groups), 1)
        st.g_packets = torch.zeros(ng * st.pk_cap * 2, dtype=torch.int32, device=dev)
        st.g_counts = torch.zeros(ng, dtype=torch.int32, device=dev)
        st.src_cap = N + self.n_ranks * st.pk_cap + 16
        st.src_nodes = torch.zeros(st.src_cap, dtype=torch.int32, device=dev)
        st.src_steps = torch.zeros(st.src_cap, dtype=torch.int32, device=dev)
        st.n_src = torch.zeros(1, dtype=torch.int32, device=dev)
        st.wprefix = torch.zeros(st.src_cap, dtype=torch.int32, device=dev)
        st.n_work = torch.zeros(1, dtype=torch.int32, device=dev)
        st.err = torch.zeros(1, dtype=torch.int32, device=dev)
        # device raster: (step, gid) pairs, spilled to the host every
        # rec_spill_steps steps of a recording run (a bound that cannot fill
        # half the buffer: one spike per refractory period per neuron)
        st.rec_cap = int(min(1 << 23, max(1 << 16, 64 * max(N, 1))))
        per_step = -(-max(N, 1) // (max(self._ref_min or 0, 0) + 1))
        st.rec_spill_steps = max(B, (st.rec_cap // 2) // per_step // B * B)
        st.rec = torch.zeros(2 * st.rec_cap, dtype=torch.int64, device=dev)
        st.n_rec = torch.zeros(1, dtype=torch.int64, device=dev)
        st.spike_total = torch.zeros(1, dtype=torch.int32, device=dev)
        st.sent = torch.zeros(1, dtype=torch.int64, device=dev)   # exchanged pairs (byte counter)
        st.rec_spill = []
        st.p2p_desc = ctypes_routes_desc(st.TP, st.p2p_packets, st.p2p_counts, self.n_ranks, st.pk_cap)
        st.g_desc = ctypes_routes_desc(st.GQ, st.g_packets, st.g_counts, len(self.groups), st.pk_cap)
        st.graph = None
        st.xplan = None
        st.pois_stream = torch.cuda.Stream(device=dev)
        st.pois_ready = None
        st.pois_next = -1
        st.pois_have = -1
        # Poisson devices: numpy-exact counts generated for S steps at a time
        # (S a multiple of the exchange block, so a block never straddles two
        # batches and can be replayed from a CUDA graph).  The fused kernels
        # add a count at its arrival step now = t + d, reading back up to d
        # steps: S >= max Poisson delay keeps that inside the previous batch.
        max_pd = max([int(d["delay"]) for d in st.devices] + [self.POIS_MIN_STEPS])
        st.pois_steps = B * max(1, -(-max_pd // B))
        for d in st.devices:
            nt = len(d["targets"])
            # node -> row on the device (no host copy of the node map)
            tg = _up_index(d["targets"], dev)
            rows = st.node2row.t[tg] if len(d["targets"]) else torch.empty(0, dtype=torch.int32, device=dev)
            d["rows"] = rows.to(torch.int32)
            d["rows_ok"] = (rows >= 0).all() if len(d["targets"]) else None
            d["nt"] = nt
            d["active"] = nt > 0 and d["lam"] != 0.0
            if not d["active"]:
                continue
            S = st.pois_steps
            # ring of 3 batches: the one being consumed, the previous one (read
            # back by delay) and the next one (generated on the side stream)
            d["counts"] = torch.zeros(3 * S * nt, dtype=torch.uint8, device=dev)
            d["cursor"] = torch.zeros(2, dtype=torch.int64, device=dev)
            d["ping"] = 0
            d["chunks"] = _lib.lib().smx_poisson_chunks_for(S * nt, d["lam"])
            d["ws"] = torch.empty(int(_lib.lib().smx_poisson_workspace(d["chunks"])), dtype=torch.uint8,
                                  device=dev)
            d["batch0"] = -1
        # fused step path: every active device hits each row at most once
        act = [d for d in st.devices if d["active"]]
        # rows are distinct iff the targets are (node -> row is injective on real neurons)
        st.fused = len(act) <= 8 and all(_all_distinct(np.asarray(d["targets"])) for d in act)
        st.ctr = torch.zeros(2, dtype=torch.int64, device=dev)
        # multi-step LIF blocks: every record delay >= block length (Poisson
        # devices are applied by their target row's own thread)
        st.block_ok = st.min_delay is None or st.min_delay >= B
        st.fdev = (ctypes_fdev * max(len(act), 1))()
        for k, d in enumerate(act):
            inv = torch.full((max(N, 1),), -1, dtype=torch.int32, device=dev)
            inv[d["rows"].long()] = torch.arange(d["nt"], dtype=torch.int32, device=dev)
            d["inv"] = inv
            st.fdev[k].counts = _ptr(d["counts"])
            st.fdev[k].inv = _ptr(d["inv"])
            st.fdev[k].n_t = d["nt"]
            st.fdev[k].w = d["weight"]
            st.fdev[k].delay = d["delay"]
            st.fdev[k].port = d["port"]
        st.n_fdev = len(act)

    # -------------------------------------------------------------- propagation
    def _block_size(self) -> int:
        """Steps per exchange round.  A spike emitted at step t over a remote
        connection of delay d >= D is consumed at t + d, so exchanging every D
        = min remote delay steps delivers every spike before its slot is read
        (the script-level minimum is identical on every rank)."""
        if self.n_ranks == 1 or self.min_remote_delay is None:
            # no exchange: the block only sets the CUDA-graph / LIF-block length
            mins = [st.min_delay for st in self.ranks.values() if st.min_delay is not None]
            m = min(mins) if mins else 32
            return int(min(m, 32)) if m >= 4 else 16
        return int(max(1, min(self.min_remote_delay, 32)))

    def _poisson_gen(self, st, b0, stream):
        """Counts for steps [b0, b0 + S) of every active device into ring third
        (b0 / S) % 3, on `stream` (numpy-exact, cursor carried on the device)."""
        S = st.pois_steps
        half = (b0 // S) % 3
        for d in st.devices:
            if not d["active"]:
                continue
            cin = d["cursor"][d["ping"]:]
            cout = d["cursor"][1 - d["ping"]:]
            fn, par = ("smx_poisson_counts_ptrs", d["lam"]) if d["lam"] >= 10.0 else ("smx_poisson_counts", d["enlam"])
            call(fn, d["key"][0], d["key"][1], _ptr(cin), par, S * d["nt"],
                 d["chunks"], _ptr(d["ws"]), _ptr(d["counts"][half * S * d["nt"]:]), _ptr(cout), _ptr(st.err),
                 stream.cuda_stream)
            d["ping"] = 1 - d["ping"]

    def _poisson_batch(self, st, b0):
        """Make batch b0 ready for the main stream and start generating batch
        b0 + S on a side stream, overlapped with the propagation of batch b0
        (the Poisson chain only depends on the previous batch's cursor)."""
        if not any(d["active"] for d in st.devices):
            return
        S = st.pois_steps
        main = torch.cuda.current_stream(st.device)
        if st.pois_next != b0:  # first batch, or steps were skipped: generate in line
            self._poisson_gen(st, b0, main)
        else:
            main.wait_event(st.pois_ready)
        # batch b0 + S reuses the third of batch b0 - 2S, last read by batch
        # b0 - S's steps: everything queued on the main stream so far must
        # finish first
        freed = torch.cuda.Event()
        freed.record(main)
        st.pois_stream.wait_event(freed)
        self._poisson_gen(st, b0 + S, st.pois_stream)
        st.pois_ready = torch.cuda.Event()
        st.pois_ready.record(st.pois_stream)
        st.pois_next = b0 + S

    def _step_kernels(self, st, offset: int = 0):
        """One step of one rank, every argument device-resident (graph-safe):
        consume + LIF, Poisson emission, spike list / raster / packets, local
        delivery (sm/engine.py:285-296)."""
        sk = st.stream
        if st.fused:
            call("smx_step", _ptr(st.v), _ptr(st.ref), _ptr(st.decay), _ptr(st.v_rest), _ptr(st.v_reset),
                 _ptr(st.v_th), _ptr(st.ref_steps), _ptr(st.i_e), st.N, _ptr(st.ring), st.P, st.L, _ptr(st.now_dev),
                 offset, _ptr(st.record_dev), 3 * st.pois_steps, ctypes_addr(st.fdev), st.n_fdev, _ptr(st.row2node_t),
                 _ptr(st.gid_t), _ptr(st.first_index), _ptr(st.src_nodes), _ptr(st.src_steps), _ptr(st.wprefix),
                 _ptr(st.owner), st.owner_cap, _ptr(st.ctr), st.src_cap, _ptr(st.rec), _ptr(st.n_rec), st.rec_cap,
                 _ptr(st.err), ctypes_addr(st.p2p_desc), ctypes_addr(st.g_desc), _ptr(st.payload), _ptr(st.cls_w),
                 _ptr(st.cls_delay), _ptr(st.cls_port), _ptr(st.ww), _ptr(st.wm), sk)
            return
        call("smx_lif_update", _ptr(st.v), _ptr(st.ref), _ptr(st.decay), _ptr(st.v_rest), _ptr(st.v_reset),
             _ptr(st.v_th), _ptr(st.ref_steps), _ptr(st.i_e), st.N, _ptr(st.ring), st.P, st.L, _ptr(st.now_dev),
             _ptr(st.spike_bits), sk)
        for d in st.devices:
            if d["active"]:
                call("smx_poisson_emit", _ptr(d["counts"]), 3 * st.pois_steps, d["nt"], _ptr(d["rows"]), d["weight"],
                     _ptr(st.ring), st.N, st.P, st.L, d["delay"], d["port"], _ptr(st.now_dev), sk)
        call("smx_spikes", _ptr(st.spike_bits), st.N, _ptr(st.row2node_t), _ptr(st.gid_t), _ptr(st.now_dev),
             _ptr(st.src_nodes), _ptr(st.src_steps), _ptr(st.n_src), st.src_cap, _ptr(st.record_dev),
             _ptr(st.rec), _ptr(st.n_rec), st.rec_cap, _ptr(st.spike_total), _ptr(st.err),
             ctypes_addr(st.p2p_desc), ctypes_addr(st.g_desc), sk)
        self._deliver(st)

    def _block_kernels(self, st, n_steps: int, offset: int = 0):
        """n_steps (<= MAX_LIF_BLOCK) steps of one rank from block step
        `offset`, in two launches (smx_block)."""
        call("smx_block", _ptr(st.v), _ptr(st.ref), _ptr(st.decay), _ptr(st.v_rest), _ptr(st.v_reset),
             _ptr(st.v_th), _ptr(st.ref_steps), _ptr(st.i_e), st.N, _ptr(st.ring), st.P, st.L, _ptr(st.now_dev),
             offset, n_steps, _ptr(st.record_dev), 3 * st.pois_steps, ctypes_addr(st.fdev), st.n_fdev, _ptr(st.row2node_t),
             _ptr(st.gid_t), _ptr(st.first_index), _ptr(st.src_nodes), _ptr(st.src_steps), _ptr(st.wprefix),
             _ptr(st.owner), st.owner_cap, _ptr(st.ctr), st.src_cap, _ptr(st.rec), _ptr(st.n_rec), st.rec_cap,
             _ptr(st.err), ctypes_addr(st.p2p_desc), ctypes_addr(st.g_desc), _ptr(st.payload), _ptr(st.cls_w),
             _ptr(st.cls_delay), _ptr(st.cls_port), _ptr(st.ww), _ptr(st.wm), st.stream)

    def _deliver(self, st):
        call("smx_deliver", _ptr(st.src_nodes), _ptr(st.src_steps), _ptr(st.n_src), _ptr(st.wprefix),
             _ptr(st.n_work), _ptr(st.first_index), _ptr(st.payload), _ptr(st.cls_w), _ptr(st.cls_delay),
             _ptr(st.cls_port), _ptr(st.ww), _ptr(st.wm), _ptr(st.ring), st.N, st.P, st.L, 0, st.stream)

    def _block_body(self, n_steps: int):
        for st in self.ranks.values():
            if st.fused and st.block_ok and n_steps > 1:
                # the LIF block kernel stages at most MAX_LIF_BLOCK steps of
                # inputs; longer exchange blocks run as consecutive sub-blocks
                for s0 in range(0, n_steps, MAX_LIF_BLOCK):
                    self._block_kernels(st, min(MAX_LIF_BLOCK, n_steps - s0), s0)
            else:
                for j in range(n_steps):
                    self._step_kernels(st, j)
        if self.n_ranks > 1 and not self.distributed:
            self._exchange_local()

    def _run_block(self, n_steps: int, use_graph: bool):
        """n_steps steps of every local rank, then one exchange round."""
        now = self.now
        for st in self.ranks.values():
            b0 = now - now % st.pois_steps
            if st.pois_have != b0:
                self._poisson_batch(st, b0)
                st.pois_have = b0
        for st in self.ranks.values():
            st.now_dev.fill_(now)  # block start; fused steps add their offset
        nccl = self.n_ranks > 1 and self.distributed
        if use_graph:
            if self._graph is None:
                if nccl and self._xgraph_ok is None:
                    # one eager round first: communicators and exchange buffers exist
                    # before the capture of the whole block (NCCL rounds included)
                    self._block_body(n_steps)
                    self._exchange_nccl()
                    self._zero_counts()
                    self._xgraph_ok = True
                    self._count_rounds(n_steps)
                    self.now += n_steps
                    return
                for st in self.ranks.values():
                    torch.cuda.synchronize(st.device)
                g = torch.cuda.CUDAGraph()
                ok = True
                try:
                    with torch.cuda.graph(g, stream=_capture_stream(self._dev0())):
                        self._block_body(n_steps)
                        if nccl and self._xgraph_ok:
                            self._exchange_nccl()
                            self._zero_counts()
                except RuntimeError as e:
                    if not nccl:
                        raise
                    ok = False
                    import sys
                    print(f"[spikemesh-b200] ranks {list(self.ranks)}: exchange not captured ({e})", file=sys.stderr)
                if nccl and self._xgraph_ok:
                    # every rank must replay the same collectives: agree on the outcome
                    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=self._dev0())
                    torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
                    if not int(flag.item()):
                        # collectives not capturable here: graph the block, exchange eagerly
                        self._xgraph_ok = False
                        for st in self.ranks.values():
                            torch.cuda.synchronize(st.device)
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=_capture_stream(self._dev0())):
                            self._block_body(n_steps)
                self._graph = g
            self._graph.replay()
            if nccl and not self._xgraph_ok:
                self._exchange_nccl()
                self._zero_counts()
            elif not nccl:
                self._zero_counts()
        else:
            self._block_body(n_steps)
            if nccl:
                self._exchange_nccl()
            self._zero_counts()
        self._count_rounds(n_steps)
        self.now += n_steps

    def close(self) -> None:
        """Release the block graph (it may hold captured NCCL rounds: drop it
        before torch.distributed.destroy_process_group)."""
        self._sync()
        self._graph = None
        self._xgraph_ok = None
        self._sync()

    def _dev0(self):
        return next(iter(self.ranks.values())).device

    def _zero_counts(self):
        for st in self.ranks.values():
            X = getattr(st, "xplan", None)
            if X is not None and X.get("peer") is not None:
                continue   # the peer round clears them (csrc/peer.cu)
            st.p2p_counts.zero_()
            st.g_counts.zero_()

    def _count_rounds(self, n_steps):
        """Message counters as the reference's lockstep transport would count
        them: one p2p round (n(n-1) messages) and one allgather per group per
        step (sm/transport.py:128,165)."""
        per = (self.n_ranks * (self.n_ranks - 1) if self.has_p2p else 0)
        per += sum(len(self.groups[g]) for g in self.group_ids)
        self.messages["propagation"] += per * n_steps

    def step(self) -> dict:
        """One step of every rank including its exchange round; returns the
        spiking nodes of each local rank, ascending (sm/engine.py:277-310).
        The spikes are read back through the device raster buffer (one
        readback per step); simulate() keeps everything on the device."""
        if not self.prepared:
            raise ConsistencyError("prepare() the cluster before stepping")
        self._on_device()
        keep = self._recording
        marks = {r: int(st.n_rec.item()) for r, st in self.ranks.items()}
        self._set_record(True)
        self._run_block(1, use_graph=False)
        self._set_record(keep)
        out = {}
        for r, st in self.ranks.items():
            n1 = int(st.n_rec.item())
            if n1 > st.rec_cap:
                raise ProtocolError(f"rank {r}: raster buffer overflow")
            gids = st.rec[2 * marks[r]: 2 * n1].view(-1, 2)[:, 1].cpu().numpy()
            out[r] = np.sort(self._gid_to_node(st, gids))
            if not keep:
                st.n_rec.fill_(marks[r])
        return out

    @staticmethod
    def _gid_to_node(st, gids: np.ndarray) -> np.ndarray:
        if getattr(st, "gid_order", None) is None:
            st.gid_order = np.argsort(st.gid_np, kind="stable")
        pos = np.searchsorted(st.gid_np, gids, sorter=st.gid_order)
        return st.row2node_np[st.gid_order[pos]]

    def _set_record(self, on: bool):
        for st in self.ranks.values():
            st.record_dev.fill_(1 if on else 0)

    def _advance(self, n_steps: int):
        """Advance n_steps in exchange blocks; whole blocks aligned on the block
        size replay one captured CUDA graph."""
        B = self.block
        done = 0
        spill = min(st.rec_spill_steps for st in self.ranks.values())
        since = 0
        while done < n_steps:
            if self._recording and since >= spill:
                self._spill_rec()
                since = 0
            since += min(B, n_steps - done)
            if self.now % B == 0 and n_steps - done >= B:
                self._run_block(B, use_graph=self.use_graphs)
                done += B
            else:
                k = min(n_steps - done, B - self.now % B)
                self._run_block(k, use_graph=False)
                done += k

    def _exchange_local(self):
        """One p2p round (if any p2p routing exists) then one allgather round
        per group (sm/engine.py:297-308), as device-resident packet reads
        between ranks of this process."""
        for st in self.ranks.values():
            st.n_src.zero_()
            # pairs put on the wire this round (sm/transport.py:128-129,165-166)
            if self.has_p2p:
                st.sent += st.p2p_counts.sum()
            if self.group_ids:
                st.sent += st.g_counts.sum()
        if self.has_p2p:
            for st in self.ranks.values():
                for sr in range(self.n_ranks):
                    if sr == st.rank:
                        continue
                    src = self.ranks[sr]
                    rl = st.RL.get((POINT_TO_POINT, sr))
                    if rl is None:
                        continue
                    pk = src.p2p_packets[st.rank * src.pk_cap * 2:]
                    cnt = src.p2p_counts[st.rank:]
                    call("smx_unpack", _ptr(pk), _ptr(cnt), src.pk_cap, _ptr(rl[1]), rl[1].numel(), _ptr(st.src_nodes),
                         _ptr(st.src_steps), _ptr(st.n_src), st.src_cap, _ptr(st.err), st.stream)
        for g in self.group_ids:
            slot = self.group_slots[g]
            members = self.groups[g]
            for m in members:
                st = self.ranks[m]
                for sr in sorted(members):
                    if sr == m:
                        continue
                    lk = st.I.get((g, sr))
                    if lk is None:
                        continue
                    src = self.ranks[sr]
                    pk = src.g_packets[slot * src.pk_cap * 2:]
                    cnt = src.g_counts[slot:]
                    call("smx_unpack", _ptr(pk), _ptr(cnt), src.pk_cap, _ptr(lk), lk.numel(), _ptr(st.src_nodes),
                         _ptr(st.src_steps), _ptr(st.n_src), st.src_cap, _ptr(st.err), st.stream)
        for st in self.ranks.values():
            self._deliver(st)

    def _xplan(self, st):
        """Fixed-capacity exchange buffers.  A neuron spikes at
        most ceil(B / (ref_steps + 1)) times in a block of B steps, so a
        group round carries at most (largest roster) x that many packets and a
        p2p pair (mirror size) x that many: every size is known to sender and
        receiver without a count round, and no host synchronisation is needed
        per block.  Rosters are replicated on every member; a target's p2p map
        has exactly the source's mirror entries."""
        dev = st.device
        me = st.rank
        ref_min = max(self._ref_min or 0, 0)   # network-wide: both sides of a round agree
        m = -(-self.block // (ref_min + 1))
        plan = dict(groups={}, m=m)
        for g in self.group_ids:
            members = sorted(self.groups[g])
            if me not in members:
                continue
            # identical on every member (no local clamp: sizes must agree)
            cap = max(max([int(st.H[(g, sr)].numel()) for sr in members if (g, sr) in st.H] + [0]) * m, 1)
            plan["groups"][g] = dict(members=members, cap=cap,
                                     send=torch.zeros(2 + 2 * cap, dtype=torch.int32, device=dev),
                                     recv=torch.zeros(len(members) * (2 + 2 * cap), dtype=torch.int32, device=dev))
        if self.has_p2p:
            # a sender's mirror and the receiver's map hold the same sources, so
            # both sides derive the same size (no local clamp)
            out_c = [int(st.S[d].numel()) * m if d in st.S and d != me else 0 for d in range(self.n_ranks)]
            in_c = [int(st.RL[(POINT_TO_POINT, s)][0].numel()) * m
                    if (POINT_TO_POINT, s) in st.RL and s != me else 0 for s in range(self.n_ranks)]
            out_sz = [2 + 2 * c if c else 0 for c in out_c]
            in_sz = [2 + 2 * c if c else 0 for c in in_c]
            plan["p2p"] = dict(out_c=out_c, in_c=in_c, out_sz=out_sz, in_sz=in_sz,
                               send=torch.zeros(max(sum(out_sz), 1), dtype=torch.int32, device=dev),
                               recv=torch.zeros(max(sum(in_sz), 1), dtype=torch.int32, device=dev))
        plan["sent"] = torch.zeros(1, dtype=torch.int64, device=dev)    # packets sent (byte counter)
        plan["over"] = torch.zeros(1, dtype=torch.int32, device=dev)    # capacity check
        plan["peer"] = self._peer_setup(st, plan)
        return plan

    PEER_EXCHANGE = os.environ.get("SMX_PEER_EXCHANGE", "1") != "0"

    def _exchange_nccl(self):
        """One process per rank: the exchange round of a block (sm/transport.py:
        92-168) with fixed-capacity receive blocks, each led by its count.
        Default: every sender writes its occupied packets straight into the
        receivers' HBM over NVLink (CUDA IPC peer memory, csrc/peer.cu); with
        SMX_PEER_EXCHANGE=0 (or without peer access) NCCL moves the
        fixed-capacity buffers: one all_gather per group, one all_to_all for
        p2p pairs.  Nothing is read back to the host either way."""
        dist = torch.distributed
        (st,) = self.ranks.values()
        me = st.rank
        if self._pg is None:
            self._pg = {g: dist.new_group(sorted(self.groups[g])) for g in sorted(self.groups)}
        if st.xplan is None:
            st.xplan = self._xplan(st)
        X = st.xplan
        peer = X.get("peer")
        if peer is not None:
            # sends (+ capacity check, byte counter, list reset), then wait +
            # unpack in place: two kernels, then the delivery of the round
            for g in peer["solo"]:   # a group with this rank alone: no message, its pairs still count
                X["sent"] += st.g_counts[self.group_slots[g]]
            call("smx_peer_exchange", ctypes_addr(peer["sends"]), peer["n_send"], ctypes_addr(peer["slots"]),
                 peer["n_slot"], _ptr(peer["seq"]), _ptr(X["sent"]), _ptr(X["over"]), _ptr(st.src_nodes),
                 _ptr(st.src_steps), _ptr(st.n_src), st.src_cap, _ptr(st.err), _ptr(peer["done"]),
                 _ptr(st.p2p_counts), st.p2p_counts.numel(), _ptr(st.g_counts), st.g_counts.numel(), st.stream)
            self._deliver(st)
            return
        st.n_src.zero_()
        if self.has_p2p:
            P = X["p2p"]
            for d, c in enumerate(P["out_c"]):
                if c:
                    X["over"].bitwise_or_((st.p2p_counts[d: d + 1] > c).to(torch.int32))
            X["sent"] += st.p2p_counts.sum()
        for g, G in X["groups"].items():
            slot = self.group_slots[g]
            X["over"].bitwise_or_((st.g_counts[slot: slot + 1] > G["cap"]).to(torch.int32))
            X["sent"] += st.g_counts[slot]
        if self.has_p2p:
            P = X["p2p"]
            rv, offs = fixed_p2p(st.p2p_counts, st.p2p_packets, st.pk_cap, P["out_c"], P["in_c"], P["send"],
                                 P["recv"])
            for sr in range(self.n_ranks):
                if not P["in_c"][sr]:
                    continue
                rl = st.RL.get((POINT_TO_POINT, sr))
                if rl is None:
                    raise ProtocolError(f"rank {me}: spikes from rank {sr} but no map for that pair")
                off = offs[sr]
                call("smx_unpack", _ptr(rv[off + 2:]), _ptr(rv[off:]), P["in_c"][sr], _ptr(rl[1]), rl[1].numel(),
                     _ptr(st.src_nodes), _ptr(st.src_steps), _ptr(st.n_src), st.src_cap, _ptr(st.err), st.stream)
        for g, G in X["groups"].items():
            slot, cap, members = self.group_slots[g], G["cap"], G["members"]
            recv = fixed_allgather(st.g_counts[slot: slot + 1],
                                   st.g_packets[slot * st.pk_cap * 2: (slot + 1) * st.pk_cap * 2], cap,
                                   G["send"], G["recv"], self._pg[g])
            for i, sr in enumerate(members):
                if sr == me:
                    continue
                lk = st.I.get((g, sr))
                if lk is None:
                    continue
                base = i * (2 + 2 * cap)
                call("smx_unpack", _ptr(recv[base + 2:]), _ptr(recv[base:]), cap, _ptr(lk), lk.numel(),
                     _ptr(st.src_nodes), _ptr(st.src_steps), _ptr(st.n_src), st.src_cap, _ptr(st.err), st.stream)
        self._deliver(st)

    def _peer_setup(self, st, X):
        """Receive area of this rank (CUDA IPC, one per process) and the
        mapped slots of every peer it sends to.  Every receiver publishes its
        slot layout with its IPC handle (one host all_gather at setup); the
        per-block rounds are kernels only.  None when peer access is not
        available (different nodes, no NVLink P2P): NCCL is used instead."""
        dist = torch.distributed
        me = st.rank
        if not self.PEER_EXCHANGE or dist.get_backend() != "nccl":
            return None
        # slot keys received by this rank: ("g", group, source) and ("p", source)
        slots = []
        for g, G in X["groups"].items():
            for sr in G["members"]:
                if sr != me:
                    slots.append((("g", g, sr), G["cap"]))
        if self.has_p2p:
            for sr, c in enumerate(X["p2p"]["in_c"]):
                if c and sr != me:
                    slots.append((("p", sr), c))
        layout, words = {}, 0
        for key, cap in slots:
            sz = (4 + 2 * cap + 3) // 4 * 4   # 16-byte aligned slots
            layout[key] = (words, words + sz, cap)
            words += 2 * sz
        words = (words + 3) // 4 * 4
        fl0 = words // 2   # flags (u64) after the slots: two per slot
        for i, (key, cap) in enumerate(slots):
            w0, w1, c = layout[key]
            layout[key] = (w0, w1, fl0 + 2 * i, fl0 + 2 * i + 1, c)
        nbytes = 4 * words + 16 * max(len(slots), 1)
        ptr = ctypes.c_void_p()
        call("smx_peer_alloc", nbytes, ctypes.byref(ptr))
        handle = ctypes.create_string_buffer(64)
        call("smx_peer_handle", ptr, handle)
        infos = [None] * self.n_ranks
        dist.all_gather_object(infos, (bytes(handle.raw), layout))
        mapped = {}
        # sends: group members (all_gather semantics) and p2p destinations
        sends, solo = [], []
        for g, G in X["groups"].items():
            slot = self.group_slots[g]
            first = True
            for m in G["members"]:
                if m != me:   # the group's pairs count once per round (sm/transport.py:165-166)
                    sends.append((m, ("g", g, me), st.g_counts[slot: slot + 1], st.g_packets[slot * st.pk_cap * 2:],
                                  first))
                    first = False
            if first:
                solo.append(g)
        if self.has_p2p:
            for d, c in enumerate(X["p2p"]["out_c"]):
                if c and d != me:
                    sends.append((d, ("p", me), st.p2p_counts[d: d + 1], st.p2p_packets[d * st.pk_cap * 2:], True))
        S = (ctypes_peer_send * max(len(sends), 1))()
        for i, (dst, key, cnt, pk, account) in enumerate(sends):
            if dst not in mapped:
                rp = ctypes.c_void_p()
                call("smx_peer_open", ctypes.create_string_buffer(infos[dst][0], 64), ctypes.byref(rp))
                mapped[dst] = rp.value
            w0, w1, f0, f1, cap = infos[dst][1][key]
            base = mapped[dst]
            S[i].count, S[i].packets = _ptr(cnt), _ptr(pk)
            S[i].slot0, S[i].slot1 = base + 4 * w0, base + 4 * w1
            S[i].flag0, S[i].flag1 = base + 8 * f0, base + 8 * f1
            S[i].cap = cap
            S[i].account = 1 if account else 0
        W = (ctypes_peer_slot * max(len(slots), 1))()
        for i, (key, cap) in enumerate(slots):
            w0, w1, f0, f1, _ = layout[key]
            W[i].slot0, W[i].slot1 = ptr.value + 4 * w0, ptr.value + 4 * w1
            W[i].flag0, W[i].flag1 = ptr.value + 8 * f0, ptr.value + 8 * f1
            # lookup of the source's positions: roster lookups I (groups) or
            # map images L (p2p); none -> the round is waited for, not delivered
            tab = st.I.get((key[1], key[2])) if key[0] == "g" else st.RL[(POINT_TO_POINT, key[1])][1]
            W[i].table = _ptr(tab)
            W[i].table_len = 0 if tab is None else tab.numel()
            W[i].cap = cap
        seq = torch.zeros(1, dtype=torch.int64, device=st.device)
        done = torch.zeros(1, dtype=torch.int32, device=st.device)
        return dict(area=ptr.value, mapped=mapped, sends=S, n_send=len(sends), slots=W, n_slot=len(slots), seq=seq,
                    done=done, solo=solo)

    def _settle_exchange(self):
        """Byte counter and capacity check of the fixed-capacity rounds (read
        once per simulate, not per block)."""
        for st in self.ranks.values():
            if getattr(st, "sent", None) is not None:
                self.bytes["propagation"] += 8 * int(st.sent.item())
                st.sent.zero_()
            X = getattr(st, "xplan", None)
            if X is None:
                continue
            over = X["over"].clone()
            if self.distributed:  # every rank raises together (no rank left waiting in a collective)
                torch.distributed.all_reduce(over, op=torch.distributed.ReduceOp.MAX)
            if int(over.item()):
                raise ProtocolError(f"rank {st.rank}: exchange capacity exceeded")
            self.bytes["propagation"] += 8 * int(X["sent"].item())
            X["sent"].zero_()

    _recording = False

    def _per_rank(self, fn) -> list:
        """fn(rank state) for every rank, in rank order; with one process per
        rank the values are summed over processes (each fills its own)."""
        vals = [0] * self.n_ranks
        for r, st in self.ranks.items():
            vals[r] = int(fn(st))
        if self.distributed:
            import torch.distributed as dist
            dev = next(iter(self.ranks.values())).device
            t = torch.tensor(vals, dtype=torch.int64,
                             device=dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(t)
            vals = [int(x) for x in t.cpu().numpy()]
        return vals

    def simulate(self, warmup_ms: float = 0.0, model_ms: float = 0.0, record: bool = True) -> RunReport:
        """sm/engine.py:312-359.  RTF = propagation wall time / model time, the
        wall time bracketed by device synchronisations."""
        if not self.prepared:
            self.prepare()
        self._on_device()
        warm = self.cfg.steps_for(warmup_ms)
        steps = self.cfg.steps_for(model_ms)
        self.phase = "propagation"
        self._recording = False
        self._set_record(False)
        self._sync()
        t0 = time.perf_counter()
        self._advance(warm)
        self._sync()
        warm_s = time.perf_counter() - t0
        self._recording = record
        self._set_record(record)
        torch.cuda.nvtx.range_push("propagation")
        t1 = time.perf_counter()
        self._advance(steps)
        self._sync()
        prop = time.perf_counter() - t1
        torch.cuda.nvtx.range_pop()
        self._recording = False
        self._set_record(False)
        self.timers.propagation += prop
        self._settle_exchange()
        self._check_errors()
        model_s = steps * self.cfg.resolution_ms * 1e-3
        raster = self.merged_raster() if record else None
        n_neurons = sum(self._per_rank(lambda st: st.n_real))
        n_synapses = sum(self._per_rank(lambda st: st.n_records))
        return RunReport(
            n_ranks=self.n_ranks, comm_mode=self.cfg.comm_mode, opt_level=self.cfg.opt_level,
            seed=self.cfg.seed, kernel_backend="cuda-sm_100a",
            n_neurons=n_neurons, n_synapses=n_synapses,
            timers=self.timers.as_dict(), warmup_s=warm_s, model_time_s=model_s,
            rtf=prop / model_s if model_s > 0 else 0.0,
            host_peak_bytes=self._per_rank(lambda st: st.mem.host.peak_bytes),
            device_peak_bytes=self._per_rank(lambda st: st.mem.device.peak_bytes),
            transport_messages=dict(self.messages), transport_bytes=dict(self.bytes),
            n_spike_events=raster.n_events if raster is not None else 0,
            raster_sha256=raster.sha256() if raster is not None else None)

    def _sync(self):
        for st in self.ranks.values():
            torch.cuda.synchronize(st.device)

    def _check_errors(self):
        for st in self.ranks.values():
            e = int(st.err.item())
            if e:
                raise ProtocolError(f"rank {st.rank}: device error code {e} during propagation")

    # -------------------------------------------------------------- inspection
    def _spill_rec(self):
        """Move the recorded events of every rank to the host and reset the
        device buffers (they keep their addresses: the block graph stays valid)."""
        for st in self.ranks.values():
            n = int(st.n_rec.item())
            if n > st.rec_cap:
                raise ProtocolError(f"rank {st.rank}: raster buffer overflow ({n} > {st.rec_cap} events)")
            if n:
                st.rec_spill.append(st.rec[: 2 * n].view(-1, 2).cpu().numpy())
                st.n_rec.zero_()

    def rank_events(self, rank) -> np.ndarray:
        st = self.ranks[rank]
        n = int(st.n_rec.item())
        if n > st.rec_cap:
            raise ProtocolError(f"rank {rank}: raster buffer overflow ({n} > {st.rec_cap} events)")
        cur = st.rec[: 2 * n].view(-1, 2).cpu().numpy()
        return np.concatenate(st.rec_spill + [cur]) if st.rec_spill else cur

    def merged_raster(self) -> Raster:
        parts = [self.rank_events(r) for r in self.ranks]
        ev = np.concatenate(parts) if parts else np.empty((0, 2), np.int64)
        return Raster.from_events(ev, self.cfg.resolution_ms)

    def check_construction_silent(self) -> None:
        for phase in ("construction", "preparation"):
            if self.messages[phase] or self.bytes[phase]:
                raise ConsistencyError(f"transport was used during {phase}")

    def check_alignment(self) -> None:
        """sm/engine.py:378-399: mirrors S equal map keys R for every p2p pair."""
        if not self.prepared:
            raise ConsistencyError("prepare() first")
        for tr, st in self.ranks.items():
            for (g, sr), rl in st.RL.items():
                if g != POINT_TO_POINT or sr not in self.ranks:
                    continue
                s = self.ranks[sr].S.get(tr)
                if s is None or not torch.equal(s.cpu(), rl[0].cpu()):
                    raise ConsistencyError(f"mirror of rank {sr} for rank {tr} does not match the map keys")
        for sr, ss in self.ranks.items():
            for tr, s in ss.S.items():
                if tr not in self.ranks:
                    continue
                rl = self.ranks[tr].RL.get((POINT_TO_POINT, sr))
                if rl is None or not torch.equal(s.cpu(), rl[0].cpu()):
                    raise ConsistencyError(f"map of rank {tr} for source rank {sr} does not match the mirror")

    def export(self, rank) -> dict:
        """Every table of one rank as numpy arrays, in the reference's terms:
        store columns sorted by source, first_index, (R, L) per map, mirrors
        S, rosters H, lookups I, routes T/P and G/Q, neuron state."""
        st = self.ranks[rank]
        fi = st.first_index.cpu().numpy()
        n = st.n_records
        src = np.repeat(np.arange(st.n_nodes, dtype=np.int64), np.diff(fi))
        pay = st.payload[:n].cpu().numpy().view(np.uint32).astype(np.int64)
        if st.ww is not None:
            rows = pay
            w = st.ww[:n].cpu().numpy()
            meta = st.wm[:n].cpu().numpy().view(np.uint32).astype(np.int64)
            delay, port = meta & ROW_MASK, meta >> 24
        else:
            rows = pay & ROW_MASK
            cls = pay >> 24
            ctab = np.array(self.classes or [(0.0, 0, 0)], dtype=object)
            w = np.array([self.classes[c][0] for c in range(len(self.classes))] or [0.0])[cls]
            delay = np.array([c[1] for c in self.classes] or [0], dtype=np.int64)[cls]
            port = np.array([c[2] for c in self.classes] or [0], dtype=np.int64)[cls]
            del ctab
        tgt = st.row2node_np[rows] if n else np.empty(0, np.int64)
        out = dict(src=src, tgt=tgt, weight=np.asarray(w, dtype=np.float64), delay=delay, port=port,
                   first_index=fi, n_nodes=st.n_nodes)
        out["maps"] = {k: (v[0].cpu().numpy(), v[1].cpu().numpy()) for k, v in st.RL.items()}
        out["mirrors"] = {k: v.cpu().numpy() for k, v in st.S.items()}
        out["rosters"] = {k: v.cpu().numpy() for k, v in st.H.items()}
        out["lookups"] = {k: v.cpu().numpy() for k, v in st.I.items()}
        inv_slot = {v: k for k, v in self.group_slots.items()}
        for name, tab, mapper in (("point_routes", st.TP, lambda d: d), ("group_routes", st.GQ, lambda d: inv_slot[d])):
            f = tab["first"].cpu().numpy()
            dst = tab["dest"].cpu().numpy()
            pos = tab["pos"].cpu().numpy().view(np.uint32).astype(np.int64)
            routes = {}
            for s in np.flatnonzero(np.diff(f)):
                a, b = f[s], f[s + 1]
                routes[int(s)] = (np.array([mapper(int(x)) for x in dst[a:b]], dtype=np.int64), pos[a:b])
            out[name] = routes
        out["v"] = st.v.cpu().numpy()
        out["ref"] = st.ref.cpu().numpy()
        out["gid"] = st.gid_np
        out["row2node"] = st.row2node_np
        return out


# ---------------------------------------------------------------- ctypes structs


class ctypes_segment(ctypes.Structure):
    _fields_ = [("word0", ctypes.c_uint64), ("nwords", ctypes.c_uint64),
                ("present", ctypes.c_void_p), ("img_of", ctypes.c_void_p)]


class ctypes_route(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_void_p), ("excl", ctypes.c_void_p), ("nwords", ctypes.c_uint64),
                ("dest", ctypes.c_int32)]


class ctypes_fdev(ctypes.Structure):
    _fields_ = [("counts", ctypes.c_void_p), ("inv", ctypes.c_void_p), ("n_t", ctypes.c_uint32),
                ("w", ctypes.c_double), ("delay", ctypes.c_int), ("port", ctypes.c_int)]


class ctypes_peer_send(ctypes.Structure):   # csrc/peer.cu PeerSend
    _fields_ = [("count", ctypes.c_void_p), ("packets", ctypes.c_void_p), ("slot0", ctypes.c_void_p),
                ("slot1", ctypes.c_void_p), ("flag0", ctypes.c_void_p), ("flag1", ctypes.c_void_p),
                ("cap", ctypes.c_uint32), ("account", ctypes.c_int)]


class ctypes_peer_slot(ctypes.Structure):   # csrc/peer.cu PeerSlot
    _fields_ = [("slot0", ctypes.c_void_p), ("slot1", ctypes.c_void_p), ("flag0", ctypes.c_void_p),
                ("flag1", ctypes.c_void_p), ("table", ctypes.c_void_p), ("table_len", ctypes.c_uint64),
                ("cap", ctypes.c_uint32)]


class ctypes_routes(ctypes.Structure):
    _fields_ = [("first", ctypes.c_void_p), ("dest", ctypes.c_void_p), ("pos", ctypes.c_void_p),
                ("n_dest", ctypes.c_int), ("packets", ctypes.c_void_p), ("counts", ctypes.c_void_p),
                ("cap", ctypes.c_uint32)]


def ctypes_routes_desc(tab, packets, counts, n_dest, cap):
    d = ctypes_routes()
    d.first = _ptr(tab["first"])
    d.dest = _ptr(tab["dest"])
    d.pos = _ptr(tab["pos"])
    d.n_dest = int(n_dest) if tab["n"] else 0
    d.packets = _ptr(packets)
    d.counts = _ptr(counts)
    d.cap = int(cap)
    return d


def ctypes_addr(obj) -> int:
    return ctypes.addressof(obj)
