"""CPU ORACLE -- test infrastructure only.

Only tests/, `__graft_entry__.smoke()` and bench.py's CPU-baseline leg may
import this module, and only as the checker / the timed CPU port.  The
product (paper_2512_09502_b200) never imports it.

A numpy restatement of the reference's construction path and the
propagation loop that consumes it (`spikemesh` 0.1.0 under
/root/reference/pkg/src/spikemesh, cited below as sm/<file>:<line>).  Every
random draw goes through `oracle.rng.OracleStream`, the C restatement of
numpy 2.3.5's Philox/Lemire/ziggurat/Poisson (pinned against numpy by
tests/test_oracle_rng.py).  The restatement is pinned against the reference
itself by tests/golden/ (fixtures written by tests/golden/make_golden.py,
which imports the reference in the build container).

Scope is the hot path of SURVEY.md §8(a): keyed streams, node creation with
per-gid initial V, the connection rules, the remote-connection machinery
(flag / extract / image maps / mirrors / rosters), distributed fixed
in-degree, preparation (stable sort by source, first-index, H/I, T/P, G/Q)
and the lockstep step loop.  Memory arenas (modeled bytes) are out of scope.
"""
from __future__ import annotations

import hashlib
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .rng import OracleStream

P2P = -1  # sm/core.py:17  POINT_TO_POINT


class ConsistencyError(RuntimeError):
    pass


class ProtocolError(RuntimeError):
    pass


class DelayRangeError(ValueError):
    pass


# ---------------------------------------------------------------------------
# Specs (sm/core.py:58-92, sm/construction.py:92-176, sm/dynamics.py:26-55)
# ---------------------------------------------------------------------------

@dataclass
class Config:
    n_ranks: int = 1
    resolution_ms: float = 0.1
    comm_mode: str = "p2p"
    opt_level: int = 2
    block_size: int = 1024
    flag_threshold: float = 1.0
    seed: int = 0

    def steps_for(self, span_ms: float) -> int:
        return int(round(span_ms / self.resolution_ms))


@dataclass
class Lif:
    v_rest: float = -65.0
    v_reset: float = -65.0
    v_th: float = -50.0
    tau_m: float = 10.0
    c_m: float = 250.0
    t_ref: float = 2.0
    i_e: float = 0.0


@dataclass
class Conn:
    rule: str
    k_in: int | None = None
    k_out: int | None = None
    n_total: int | None = None
    allow_autapses: bool = True
    allow_multapses: bool = True


@dataclass
class Syn:
    weight: object = 1.0
    delay_steps: object = 1


def _syn_draws(syn, n, stream):
    """sm/construction.py:157-176 -- weights first, then delays, one stream."""
    w = syn.weight
    if isinstance(w, tuple):
        weights = stream.normal(w[1], w[2], size=n)
    elif isinstance(w, (list, np.ndarray)):
        weights = np.array(w, dtype=np.float64)
        if len(weights) != n:
            raise ValueError(f"{len(weights)} weights for {n} records")
    else:
        weights = np.full(n, float(w))
    d = syn.delay_steps
    if isinstance(d, tuple):
        delays = stream.integers(d[1], d[2] + 1, size=n)
    elif isinstance(d, (list, np.ndarray)):
        delays = np.array(d, dtype=np.int64)
        if len(delays) != n:
            raise ValueError(f"{len(delays)} delays for {n} records")
    else:
        delays = np.full(n, int(d), dtype=np.int64)
    return weights, delays


def _positions(conn, n_src, n_tgt, aligned):
    """sm/construction.py:391-407 -- the only consumer of the aligned stream."""
    if conn.rule == "fixed_indegree":
        k = int(conn.k_in)
        if not conn.allow_multapses:  # one row per target (sm/construction.py:403-404)
            rows = [aligned.choice_no_replace(n_src, k) for _ in range(n_tgt)]
            return np.concatenate(rows).astype(np.int64) if rows else np.empty(0, np.int64)
        return aligned.integers(0, n_src, size=k * n_tgt)
    if conn.rule == "fixed_total":
        return aligned.integers(0, n_src, size=int(conn.n_total))
    return None


def _pairs(conn, n_src, targets, aligned, local):
    """sm/construction.py:410-432 -- (source positions, target indices)."""
    n_tgt = len(targets)
    r = conn.rule
    if r in ("one_to_one", "assigned"):
        return np.arange(n_src, dtype=np.int64), targets.copy()
    if r == "all_to_all":
        return np.tile(np.arange(n_src, dtype=np.int64), n_tgt), np.repeat(targets, n_src)
    if r == "fixed_indegree":
        return _positions(conn, n_src, n_tgt, aligned), np.repeat(targets, int(conn.k_in))
    if r == "fixed_outdegree":
        k = int(conn.k_out)
        return (np.repeat(np.arange(n_src, dtype=np.int64), k),
                targets[local.integers(0, n_tgt, size=k * n_src)])
    if r == "fixed_total":
        pos = _positions(conn, n_src, n_tgt, aligned)
        return pos, targets[local.integers(0, n_tgt, size=int(conn.n_total))]
    raise ValueError(f"unknown connection rule {r!r}")


def _flagging(conn, n_src, n_tgt, xi):
    """sm/construction.py:439-451."""
    if conn.rule == "fixed_indegree":
        return int(conn.k_in) * n_tgt / n_src < xi
    if conn.rule == "fixed_total":
        return int(conn.n_total) / n_src < xi
    return False


def _used_sorted(values, flags):
    """sm/construction.py:461-470 -- used (positions, values) by value, stable."""
    positions = np.flatnonzero(flags)
    vals = values[positions]
    order = np.argsort(vals, kind="stable")
    return positions[order], vals[order]


# ---------------------------------------------------------------------------
# Per-rank state (sm/construction.py:183-312, sm/dynamics.py:96-208)
# ---------------------------------------------------------------------------

class Rank:
    def __init__(self, rank: int):
        self.rank = rank
        # node rows: real flag, params, v_init, gid  (sm/dynamics.py:109)
        self.real: list[bool] = []
        self.params: list = []
        self.v0: list[float] = []
        self.gids: list[int] = []
        self.batches: list[tuple] = []          # (src, tgt, w, d, port)
        self.maps: dict[tuple, list] = {}       # (group, σ) -> [R, L]
        self.mirrors: dict[int, np.ndarray] = {}
        self.roster_sets: dict[tuple, set] = {}
        self.rosters: dict[tuple, np.ndarray] = {}
        self.lookups: dict[tuple, np.ndarray] = {}
        self.point_routes: dict[int, tuple] = {}
        self.group_routes: dict[int, tuple] = {}
        self.groups: dict[int, tuple] = {}
        self.pair_ctr: dict[tuple, int] = {}
        self.dist_ctr = 0
        self.local_ctr = 0
        self.devices: list[dict] = []
        self.prepared = False
        self.rec_steps: list[np.ndarray] = []
        self.rec_gids: list[np.ndarray] = []

    @property
    def n_nodes(self) -> int:
        return len(self.real)

    # sorted store (sm/core.py:299-324)
    def finalize(self):
        n = self.n_nodes
        if self.batches:
            cols = [np.concatenate([b[i] for b in self.batches]) for i in range(5)]
        else:
            cols = [np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0),
                    np.empty(0, np.int64), np.empty(0, np.int64)]
        order = np.argsort(cols[0], kind="stable")
        self.src, self.tgt, self.weight, self.delay, self.port = (c[order] for c in cols)
        if len(self.src) and self.src[-1] >= n:
            raise ConsistencyError("record source beyond node count")
        self.first_index = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.src, minlength=n), out=self.first_index[1:])
        self.batches = []

    def freeze(self, dt, max_delay, n_ports):
        """sm/dynamics.py:153-189 (buffers span all M rows like the reference)."""
        m = self.n_nodes
        self.v = np.zeros(m)
        self.ref = np.zeros(m, dtype=np.int64)
        self.mask = np.array(self.real, dtype=bool)
        self.decay = np.zeros(m)
        self.vrest = np.zeros(m)
        self.vreset = np.zeros(m)
        self.vth = np.full(m, np.inf)
        self.refsteps = np.zeros(m, dtype=np.int64)
        self.ie = np.zeros(m)
        self.gid = np.full(m, -1, dtype=np.int64)
        for i in np.flatnonzero(self.mask):
            p = self.params[i]
            self.v[i] = self.v0[i]
            self.decay[i] = math.exp(-dt / p.tau_m)
            self.vrest[i], self.vreset[i], self.vth[i] = p.v_rest, p.v_reset, p.v_th
            self.refsteps[i] = int(round(p.t_ref / dt))
            self.ie[i] = p.i_e
            self.gid[i] = self.gids[i]
        self.n_ports = max(1, int(n_ports))
        self.L = max(2, int(max_delay) + 1)
        self.buf = np.zeros((m, self.n_ports, self.L))


# ---------------------------------------------------------------------------
# Cluster façade (sm/engine.py:197-359)
# ---------------------------------------------------------------------------

class OracleCluster:
    def __init__(self, cfg: Config):
        self.cfg = cfg
        self.ranks = [Rank(r) for r in range(cfg.n_ranks)]
        self.now = 0
        self.prepared = False
        self.timers = {k: 0.0 for k in ("node_creation", "local_connection",
                                         "remote_connection", "preparation", "propagation")}

    def _stream(self, sid):
        return OracleStream(self.cfg.seed, sid)

    # -- node creation (sm/construction.py:335-384) --------------------------
    def declare_group(self, gid, members):
        members = tuple(int(m) for m in members)
        for st in self.ranks:
            if gid in st.groups:
                raise ValueError(f"group {gid} already declared")
            st.groups[gid] = members

    def create_neurons(self, rank, n, params=None, v_init=None, gids=None):
        t0 = time.perf_counter()
        st = self.ranks[rank]
        p = params if params is not None else Lif()
        start = st.n_nodes
        g = np.arange(start, start + n, dtype=np.int64) if gids is None else np.asarray(gids, np.int64)
        if v_init is None:
            v = np.full(n, p.v_rest)
        elif isinstance(v_init, tuple):
            v = np.array([self._stream(("init-v", int(x))).normal(v_init[1], v_init[2]) for x in g])
        elif np.ndim(v_init) == 0:
            v = np.full(n, float(v_init))
        else:
            v = np.asarray(v_init, dtype=np.float64)
        st.real += [True] * n
        st.params += [p] * n
        st.v0 += v.tolist()
        st.gids += g.tolist()
        self.timers["node_creation"] += time.perf_counter() - t0
        return range(start, start + n)

    def add_poisson_source(self, rank, rate_hz, weight, delay_steps, targets, port=0):
        st = self.ranks[rank]
        dev = dict(stream=self._stream(("poisson", rank, len(st.devices))),
                   lam=float(rate_hz) * self.cfg.resolution_ms * 1e-3, weight=float(weight),
                   delay=int(delay_steps), targets=np.asarray(targets, np.int64), port=int(port))
        st.devices.append(dev)
        return dev

    def _add_image(self, st) -> int:
        idx = st.n_nodes
        st.real.append(False)
        st.params.append(None)
        st.v0.append(0.0)
        st.gids.append(-1)
        return idx

    # -- connect (sm/construction.py:507-534) --------------------------------
    def connect(self, rank, sources, targets, conn, syn, port=0):
        t0 = time.perf_counter()
        n = self._connect_local(self.ranks[rank], np.asarray(sources, np.int64),
                                np.asarray(targets, np.int64), conn, syn, port)
        self.timers["local_connection"] += time.perf_counter() - t0
        return n

    def _connect_local(self, st, sources, targets, conn, syn, port):
        st.local_ctr += 1
        stream = self._stream(("conn-local", st.rank, st.local_ctr))
        pos, tgt = _pairs(conn, len(sources), targets, stream, stream)
        src = sources[pos]
        if not conn.allow_autapses and conn.rule in ("fixed_indegree", "fixed_total"):
            bad = np.flatnonzero(src == tgt)
            while len(bad):
                src[bad] = sources[stream.integers(0, len(sources), size=len(bad))]
                bad = bad[src[bad] == tgt[bad]]
        w, d = _syn_draws(syn, len(src), self._stream(("syn-local", st.rank, st.local_ctr)))
        return self._append(st, src, tgt, w, d, port)

    def _append(self, st, src, tgt, w, d, port):
        n = len(src)
        if n == 0:
            return 0
        if d.min() < 1:
            raise DelayRangeError("connection delays must be >= 1 step")
        st.batches.append((np.asarray(src, np.int64), np.asarray(tgt, np.int64),
                           np.asarray(w, np.float64), np.asarray(d, np.int64),
                           np.full(n, int(port), dtype=np.int64)))
        return n

    # -- remote connect (sm/construction.py:550-637) -------------------------
    def connect_remote(self, src_rank, sources, tgt_rank, targets, conn, syn, port=0, group=P2P):
        t0 = time.perf_counter()
        n = self._remote(src_rank, np.asarray(sources, np.int64), tgt_rank,
                         np.asarray(targets, np.int64), conn, syn, port, group)
        self.timers["remote_connection"] += time.perf_counter() - t0
        return n

    def _remote(self, sr, sources, tr, targets, conn, syn, port, group):
        if sr == tr:
            return self._connect_local(self.ranks[sr], sources, targets, conn, syn, port)
        S, T = self.ranks[sr], self.ranks[tr]
        members = T.groups.get(group) if group != P2P else None
        key = (sr, tr)
        a, b = S.pair_ctr.get(key, 0) + 1, T.pair_ctr.get(key, 0) + 1
        if a != b:
            raise ConsistencyError("pair counters diverged")
        S.pair_ctr[key] = T.pair_ctr[key] = a
        n_src, n_tgt = len(sources), len(targets)
        flag = _flagging(conn, n_src, n_tgt, self.cfg.flag_threshold)
        pos, tgt = _pairs(conn, n_src, targets, self._stream(("remote-src", sr, tr, a)),
                          self._stream(("remote-tgt", sr, tr, a)))
        w, d = _syn_draws(syn, len(pos), self._stream(("remote-syn", sr, tr, a)))
        used = np.zeros(n_src, bool)
        if flag:
            used[pos] = True
        else:
            used[:] = True
        upos, uvals = _used_sorted(sources, used)
        uniq = np.unique(uvals)
        pos_img = np.full(n_src, -1, dtype=np.int64)
        if len(uniq):
            m = T.maps.setdefault((group, sr), [np.empty(0, np.int64), np.empty(0, np.int64)])
            R, L = m
            at = np.searchsorted(R, uniq)
            hit = np.zeros(len(uniq), bool)
            ok = at < len(R)
            hit[ok] = R[at[ok]] == uniq[ok]
            imgs = np.full(len(uniq), -1, dtype=np.int64)
            imgs[hit] = L[at[hit]]
            missing = uniq[~hit]
            if len(missing):
                new = np.array([self._add_image(T) for _ in missing], dtype=np.int64)
                ins = np.searchsorted(R, missing)
                m[0] = np.insert(R, ins, missing)
                m[1] = np.insert(L, ins, new)
                imgs[~hit] = new
            pos_img[upos] = imgs[np.searchsorted(uniq, uvals)]
        rec_src = pos_img[pos]
        if len(rec_src) and rec_src.min() < 0:
            raise ConsistencyError("connection references a source with no image")
        n = self._append(T, rec_src, tgt, w, d, port)
        # source side
        if group == P2P:
            if flag:
                p2 = _positions(conn, n_src, n_tgt, self._stream(("remote-src", sr, tr, a)))
                f2 = np.zeros(n_src, bool)
                f2[p2] = True
            else:
                f2 = np.ones(n_src, bool)
            _, v2 = _used_sorted(sources, f2)
            if len(v2):
                old = S.mirrors.get(tr)
                S.mirrors[tr] = np.union1d(old, v2) if old is not None else np.unique(v2)
        else:
            for mbr in members:
                self.ranks[mbr].roster_sets.setdefault((group, sr), set()).update(sources.tolist())
        return n

    # -- distributed fixed in-degree (sm/construction.py:640-703) ------------
    def connect_fixed_indegree_distributed(self, source_pops, target_pops, k_in, syn,
                                           port=0, group=P2P, allow_multapses=True):
        t0 = time.perf_counter()
        s_rank = np.concatenate([np.full(len(n), int(r), np.int64) for r, n in source_pops])
        s_node = np.concatenate([np.asarray(n, np.int64) for _, n in source_pops])
        total = len(s_node)
        for st in self.ranks:
            st.dist_ctr += 1
        call = self.ranks[0].dist_ctr
        made = 0
        for tr, tg in target_pops:
            tr = int(tr)
            tg = np.asarray(tg, np.int64)
            stream = self._stream(("dist-indegree", call, tr))
            if allow_multapses:
                flat = stream.integers(0, total, size=k_in * len(tg))
            else:  # sm/construction.py:680-683
                flat = np.concatenate([stream.choice_no_replace(total, k_in) for _ in tg]).astype(np.int64)
            sig, sv, tv = s_rank[flat], s_node[flat], np.repeat(tg, k_in)
            order = np.lexsort((sv, sig))
            sig, sv, tv = sig[order], sv[order], tv[order]
            us, starts = np.unique(sig, return_index=True)
            ends = list(starts[1:]) + [len(sig)]
            for s_r, b, e in zip(us, starts, ends):
                spec = Conn("assigned")
                if int(s_r) == tr:
                    made += self._connect_local(self.ranks[tr], sv[b:e], tv[b:e], spec, syn, port)
                else:
                    made += self._remote(int(s_r), sv[b:e], tr, tv[b:e], spec, syn, port, group)
        self.timers["remote_connection"] += time.perf_counter() - t0
        return made

    # -- preparation (sm/construction.py:742-807) ----------------------------
    def prepare(self):
        t0 = time.perf_counter()
        dt = self.cfg.resolution_ms
        for st in self.ranks:
            md = max([int(b[3].max()) for b in st.batches] + [d["delay"] for d in st.devices] + [1])
            mp = max([int(b[4].max()) for b in st.batches] + [d["port"] for d in st.devices] + [0])
            st.freeze(dt, md, 1 + mp)
            st.finalize()
            for key in sorted(st.roster_sets):
                st.rosters[key] = np.array(sorted(st.roster_sets[key]), dtype=np.int64)
            for key in sorted(st.rosters):
                if key[1] == st.rank:
                    continue
                H = st.rosters[key]
                lk = np.full(len(H), -1, dtype=np.int64)
                m = st.maps.get(key)
                if m is not None and len(m[0]):
                    at = np.searchsorted(H, m[0])
                    if (at >= len(H)).any() or (H[at] != m[0]).any():
                        raise ConsistencyError("map keys missing from roster")
                    lk[at] = m[1]
                st.lookups[key] = lk
            routes: dict[int, list] = {}
            for tr in sorted(st.mirrors):
                for i, s in enumerate(st.mirrors[tr].tolist()):
                    routes.setdefault(s, []).append((tr, i))
            st.point_routes = {s: (np.array([a for a, _ in v], np.int64), np.array([b for _, b in v], np.int64))
                               for s, v in routes.items()}
            groutes: dict[int, list] = {}
            for (g, sr) in sorted(st.rosters):
                if sr != st.rank:
                    continue
                for i, s in enumerate(st.rosters[(g, sr)].tolist()):
                    groutes.setdefault(s, []).append((g, i))
            st.group_routes = {s: (np.array([a for a, _ in v], np.int64), np.array([b for _, b in v], np.int64))
                               for s, v in groutes.items()}
            st.prepared = True
        self.has_p2p = any(st.mirrors or any(k[0] == P2P for k in st.maps) for st in self.ranks)
        self.group_ids = sorted(self.ranks[0].groups)
        self.prepared = True
        self.timers["preparation"] += time.perf_counter() - t0

    # -- propagation (sm/engine.py:89-190, 277-310; kernels/_numpy_impl.py) --
    @staticmethod
    def _deliver(st, nodes, mults, now):
        fi = st.first_index
        for node, mult in zip(nodes.tolist(), mults.tolist()):
            lo, hi = fi[node], fi[node + 1]
            if lo == hi:
                continue
            slot = (now + st.delay[lo:hi]) % st.L
            np.add.at(st.buf, (st.tgt[lo:hi], st.port[lo:hi], slot), st.weight[lo:hi] * mult)

    def step(self):
        now = self.now
        spikes, out_p2p = {}, {}
        gather = {g: {} for g in self.group_ids}
        for st in self.ranks:
            cur = now % st.L
            inputs = st.buf[:, :, cur].sum(axis=1)
            st.buf[:, :, cur] = 0.0
            inputs = inputs + st.ie
            refr = st.mask & (st.ref > 0)
            act = st.mask & ~refr
            integ = st.vrest + (st.v - st.vrest) * st.decay + inputs
            spk = act & (integ >= st.vth)
            st.v[act] = integ[act]
            st.v[spk] = st.vreset[spk]
            st.v[refr] = st.vreset[refr]
            st.ref[refr] -= 1
            st.ref[spk] = st.refsteps[spk]
            spiking = np.flatnonzero(spk)
            spikes[st.rank] = spiking
            if self._recording and len(spiking):
                st.rec_steps.append(np.full(len(spiking), now, np.int64))
                st.rec_gids.append(st.gid[spiking])
            for dev in st.devices:
                if len(dev["targets"]) == 0 or dev["lam"] == 0.0:
                    continue
                c = dev["stream"].poisson(dev["lam"], size=len(dev["targets"]))
                hit = c > 0
                if hit.any():
                    np.add.at(st.buf, (dev["targets"][hit], dev["port"], (now + dev["delay"]) % st.L),
                              dev["weight"] * c[hit].astype(np.float64))
            if len(spiking):
                self._deliver(st, spiking, np.ones(len(spiking), np.int64), now)
            pk: dict[int, list] = {}
            gk: dict[int, list] = {}
            for s in spiking.tolist():
                r = st.point_routes.get(s)
                if r is not None:
                    for d, p in zip(r[0].tolist(), r[1].tolist()):
                        pk.setdefault(d, []).append(p)
                r = st.group_routes.get(s)
                if r is not None:
                    for g, p in zip(r[0].tolist(), r[1].tolist()):
                        gk.setdefault(g, []).append(p)
            out_p2p[st.rank] = {d: np.array(v, np.int64) for d, v in pk.items()}
            for g, v in gk.items():
                gather[g][st.rank] = np.array(v, np.int64)
        if self.has_p2p:
            for st in self.ranks:
                for src in range(len(self.ranks)):
                    if src == st.rank:
                        continue
                    pos = out_p2p[src].get(st.rank)
                    if pos is None or len(pos) == 0:
                        continue
                    m = st.maps.get((P2P, src))
                    if m is None or pos.max() >= len(m[0]):
                        raise ProtocolError("bad point-to-point position")
                    self._deliver(st, m[1][pos], np.ones(len(pos), np.int64), now)
        for g in self.group_ids:
            members = self.ranks[0].groups[g]
            for m_ in members:
                st = self.ranks[m_]
                for src in sorted(members):
                    if src == m_:
                        continue
                    pos = gather[g].get(src)
                    if pos is None or len(pos) == 0:
                        continue
                    lk = st.lookups.get((g, src))
                    if lk is None or pos.max() >= len(lk):
                        raise ProtocolError("bad roster position")
                    img = lk[pos]
                    img = img[img >= 0]
                    if len(img):
                        self._deliver(st, img, np.ones(len(img), np.int64), now)
        self.now += 1
        return spikes

    _recording = False

    def simulate(self, warmup_ms=0.0, model_ms=0.0, record=True):
        if not self.prepared:
            self.prepare()
        self._recording = False
        for _ in range(self.cfg.steps_for(warmup_ms)):
            self.step()
        self._recording = record
        n = self.cfg.steps_for(model_ms)
        t0 = time.perf_counter()
        for _ in range(n):
            self.step()
        wall = time.perf_counter() - t0
        self.timers["propagation"] += wall
        self._recording = False
        model_s = n * self.cfg.resolution_ms * 1e-3
        return dict(rtf=wall / model_s if model_s > 0 else 0.0, propagation_s=wall,
                    model_time_s=model_s, n_steps=n)

    # -- raster (sm/dynamics.py:290-346) ------------------------------------
    def raster(self) -> np.ndarray:
        parts = [np.column_stack((np.concatenate(st.rec_steps), np.concatenate(st.rec_gids)))
                 for st in self.ranks if st.rec_steps]
        ev = np.concatenate(parts) if parts else np.empty((0, 2), np.int64)
        order = np.lexsort((ev[:, 1], ev[:, 0]))
        return ev[order]

    def raster_sha256(self) -> str:
        return raster_sha256(self.raster(), self.cfg.resolution_ms)


def raster_sha256(events: np.ndarray, resolution_ms: float) -> str:
    lines = [f"{g}\t{s * resolution_ms:.3f}" for s, g in np.asarray(events).tolist()]
    text = "\n".join(lines) + ("\n" if lines else "")
    return hashlib.sha256(text.encode("ascii")).hexdigest()
