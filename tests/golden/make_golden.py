"""Generate the golden fixtures from the REFERENCE itself.

Runs in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box); the outputs are committed:
  tests/golden/rng.npz           raw Philox words, integers (with rejections
                                 and continued cursors), normals, poisson
                                 chains, per-gid init-v -- numpy 2.3.5
  tests/golden/tables_<name>.npz per-rank construction tables of each
                                 scenario in tests/scenarios.py
  tests/golden/rasters.json      raster SHA-256 / event counts per scenario
  tests/golden/memory.json       modeled host/device peak bytes per rank after
                                 prepare, per scenario and optimisation level
  tests/golden/c1_digests.json   C1 (10k neurons, K=1000, seed 12345) at full
                                 size: SHA-256 of every table column, raster
                                 SHA over 100 ms, per-neuron spike counts
  tests/golden/transport.json    messages / bytes per phase after simulate()
Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(HERE))
os.environ["SPIKEMESH_PURE_PYTHON"] = "1"

import spikemesh as sm  # noqa: E402
from spikemesh import models as smm  # noqa: E402

import scenarios  # noqa: E402
import tables  # noqa: E402


def ref_namespace():
    # the PD microcircuit script (C2) has no reference counterpart: the
    # reference Cluster runs this repository's script (it only calls façade
    # methods and duck-typed ConnSpec/SynSpec/LifParams)
    sys.path.insert(0, ROOT)
    from paper_2512_09502_b200 import models as mm
    return SimpleNamespace(
        build_microcircuit=mm.build_microcircuit, MicrocircuitParams=mm.MicrocircuitParams,
        SimConfig=sm.SimConfig, make_cluster=sm.Cluster, ConnSpec=sm.ConnSpec, SynSpec=sm.SynSpec,
        LifParams=sm.LifParams, build_balanced_network=smm.build_balanced_network,
        BalancedParams=smm.BalancedParams, ExplicitNetwork=smm.ExplicitNetwork,
        build_multi_area=smm.build_multi_area, AreaSpec=smm.AreaSpec, pack_areas=smm.pack_areas,
        MultiAreaParams=smm.MultiAreaParams)


def gen_rng():
    assert np.__version__ == "2.3.5", np.__version__
    out = {}
    streams = [(7, ("dist-indegree", 1, 0)), (12345, ("conn-local", 0, 3)), (11, ("init-v", 42))]
    for i, (seed, sid) in enumerate(streams):
        st = sm.RngStream(seed, sid)
        k = st._key
        out[f"s{i}/key"] = np.array([k & (2**64 - 1), k >> 64], dtype=np.uint64)
        out[f"s{i}/words"] = sm.RngStream(seed, sid).gen.bit_generator.random_raw(64).astype(np.uint64)
        g = sm.RngStream(seed, sid)
        # integers with continued cursors, odd lengths (buffered high half),
        # ranges with many rejections (ex = 3e9) and ex = 1 (no draws)
        seq = [(0, 36, 101), (0, 640000, 1001), (5, 3_000_000_005, 777), (0, 1, 9), (0, 2**32, 33),
               (1, 21, 500), (0, 8000, 2048)]
        for j, (lo, hi, n) in enumerate(seq):
            out[f"s{i}/int{j}"] = g.integers(lo, hi, size=n)
            out[f"s{i}/int{j}/spec"] = np.array([lo, hi, n], dtype=np.int64)
        out[f"s{i}/normal"] = sm.RngStream(seed, sid).normal(-58.0, 5.0, size=4000)
        out[f"s{i}/poisson"] = sm.RngStream(seed, sid).poisson(1.1, size=20000)
        p = sm.RngStream(seed, sid)
        out[f"s{i}/poisson_steps"] = np.stack([p.poisson(1.1, size=333) for _ in range(20)])
    gids = np.array([0, 1, 2, 7, 99, 1000, 12345, 99999, 4_000_000, 2**40 + 3], dtype=np.int64)
    out["initv/gids"] = gids
    out["initv/seed11"] = np.array([sm.RngStream(11, ("init-v", int(g))).normal(-58.0, 5.0) for g in gids])
    out["initv/seed12345"] = np.array([sm.RngStream(12345, ("init-v", int(g))).normal(-58.0, 5.0) for g in gids])
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def gen_tables():
    ns = ref_namespace()
    rasters = {}
    for name, fn in scenarios.SCENARIOS.items():
        c, sim = fn(ns)
        c.prepare()
        t = tables.canon_reference(c)
        np.savez_compressed(os.path.join(HERE, f"tables_{name}.npz"), **t)
        if sim is not None:
            rep = c.simulate(sim[0], sim[1], record=True)
            rasters[name] = dict(sha256=rep.raster_sha256, n_events=rep.n_spike_events,
                                 warmup_ms=sim[0], model_ms=sim[1])
        print(name, "records", sum(len(st.store.src) for st in c.ranks), rasters.get(name), file=sys.stderr)
    with open(os.path.join(HERE, "rasters.json"), "w") as fh:
        json.dump(rasters, fh, indent=1, sort_keys=True)


def gen_memory():
    """Arena peaks of the reference (sm/core.py:155-182) for every scenario at
    optimisation levels 0..3 (placement plans, sm/construction.py:59-71)."""
    import functools
    out = {}
    for name, fn in scenarios.SCENARIOS.items():
        for level in (0, 1, 2, 3):
            ns = ref_namespace()
            ns.SimConfig = functools.partial(sm.SimConfig, opt_level=level)
            c, _ = fn(ns)
            c.prepare()
            out[f"{name}/L{level}"] = dict(host=[int(st.host.peak_bytes) for st in c.ranks],
                                          device=[int(st.device.peak_bytes) for st in c.ranks])
        print(name, out[f"{name}/L2"], file=sys.stderr)
    with open(os.path.join(HERE, "memory.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


C1 = dict(neurons_per_rank=10_000, k_exc=800, k_inh=200)   # BASELINE configs[0]
C1_SEED, C1_MODEL_MS = 12345, 100.0


def gen_c1():
    """C1 at full size (1e7 synapses, 1 rank, seed 12345): SHA-256 digests of
    every canonical table column and the raster over 100 ms (sm/models.py:
    106-144; reference numpy backend)."""
    ns = ref_namespace()
    c = sm.Cluster(sm.SimConfig(n_ranks=1, comm_mode="p2p", seed=C1_SEED))
    smm.build_balanced_network(c, smm.BalancedParams(**C1))
    c.prepare()
    dig = tables.digests(tables.canon_reference(c))
    rep = c.simulate(0.0, C1_MODEL_MS, record=True)
    counts = np.zeros(C1["neurons_per_rank"], dtype=np.int64)
    ev = c.merged_raster().events
    np.add.at(counts, np.asarray([e[1] for e in ev], dtype=np.int64), 1)
    out = dict(config=dict(C1, seed=C1_SEED, comm_mode="p2p", model_ms=C1_MODEL_MS),
               n_synapses=int(sum(len(st.store.src) for st in c.ranks)), tables=dig,
               raster=dict(sha256=rep.raster_sha256, n_events=rep.n_spike_events),
               spike_counts_sha256=hashlib.sha256(counts.tobytes()).hexdigest())
    with open(os.path.join(HERE, "c1_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("C1", out["n_synapses"], out["raster"], file=sys.stderr)
    del ns


C2_SEED = 12345


def gen_c2():
    """C2 at full size (PD microcircuit, 77,169 neurons, ~3e8 synapses, 1 rank,
    seed 12345): SHA-256 digests of every canonical table column, built by
    the reference Cluster from this repository's microcircuit script (the
    reference has no PD builder; the script only calls façade methods)."""
    import time
    ns = ref_namespace()
    t0 = time.time()
    c = sm.Cluster(sm.SimConfig(n_ranks=1, comm_mode="p2p", seed=C2_SEED))
    ns.build_microcircuit(c, ns.MicrocircuitParams(scale=1.0))
    c.prepare()
    t1 = time.time()
    dig = tables.digests(tables.canon_reference(c))
    out = dict(config=dict(model="PD microcircuit", scale=1.0, seed=C2_SEED, comm_mode="p2p"),
               n_neurons=int(sum(st.n_real for st in c.ranks)) if hasattr(c.ranks[0], "n_real") else None,
               n_synapses=int(sum(len(st.store.src) for st in c.ranks)), tables=dig,
               reference_construction_s=round(t1 - t0, 1))
    with open(os.path.join(HERE, "c2_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("C2", out["n_synapses"], round(t1 - t0, 1), "s", file=sys.stderr)


def gen_transport():
    """Transport counters of each simulated scenario (sm/transport.py:55-67,
    128-129, 165-166): messages and bytes per phase after simulate()."""
    ns = ref_namespace()
    out = {}
    for name, fn in scenarios.SCENARIOS.items():
        c, sim = fn(ns)
        if sim is None:
            continue
        rep = c.simulate(sim[0], sim[1], record=False)
        out[name] = dict(messages=rep.transport_messages, bytes=rep.transport_bytes)
    with open(os.path.join(HERE, "transport.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    if "--transport-only" in sys.argv:
        gen_transport()
        sys.exit(0)
    if "--c1-only" in sys.argv:
        gen_c1()
        sys.exit(0)
    if "--c2-only" in sys.argv:
        gen_c2()
        sys.exit(0)
    if "--memory-only" in sys.argv:
        gen_memory()
        sys.exit(0)
    gen_rng()
    gen_tables()
    gen_memory()
    gen_c1()
    gen_transport()
