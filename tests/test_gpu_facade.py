"""The façade contract (sm/engine.py:197-399) on the GPU Cluster: reference
objects and builders as inputs, step() results, transport counters, the C1
configuration at full size, long-delay / synapse-free networks, and the
single-device rule."""
import dataclasses
import json
import os
import re

import numpy as np
import pytest

import scenarios
import tables
from namespaces import gpu_ns, oracle_ns, ref_gpu_ns, ref_module

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
RASTERS = json.load(open(os.path.join(GOLD, "rasters.json")))
ROOT = os.path.dirname(HERE)


@dataclasses.dataclass
class BareSynSpec:
    """Only the reference SynSpec's fields and method (sm/construction.py:125-154)."""
    weight: object = 1.0
    delay_steps: object = 1

    def validate(self):
        pass


def test_bare_synspec_objects():
    """A SynSpec without any repository-only attribute drives every path
    (local, remote, distributed) and gives the golden tables."""
    from paper_2512_09502_b200 import api
    ns = gpu_ns()
    ns.SynSpec = BareSynSpec
    for name in ("balanced_4r_p2p", "remote_p2p", "rules_local"):
        c, _ = scenarios.SCENARIOS[name](ns)
        c.prepare()
        gold = dict(np.load(os.path.join(GOLD, f"tables_{name}.npz")))
        bad = tables.compare(tables.canon_gpu(c), gold)
        assert not bad, (name, bad[:5])
    assert not hasattr(BareSynSpec(), "is_constant") and hasattr(api.SynSpec(), "is_constant")


REF_SCENARIOS = ["balanced_4r_p2p", "balanced_4r_coll", "explicit_3r_p2p", "explicit_3r_coll", "multi_area_2r",
                 "rules_local", "rules_wide", "remote_p2p", "dist_random_p2p", "no_multapse_coll"]


@pytest.mark.parametrize("name", REF_SCENARIOS)
def test_reference_builders_drive_gpu_cluster(name):
    """The unmodified reference's config/spec classes and model builders
    (baseline/_ref) build on the GPU Cluster: tables equal the goldens and
    the raster equals the reference's."""
    ns = ref_gpu_ns()
    if ns is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    c, sim = scenarios.SCENARIOS[name](ns)
    c.prepare()
    gold = dict(np.load(os.path.join(GOLD, f"tables_{name}.npz")))
    bad = tables.compare(tables.canon_gpu(c), gold)
    assert not bad, bad[:10]
    if sim is not None and name not in scenarios.NON_DYADIC:
        rep = c.simulate(sim[0], sim[1], record=True)
        assert rep.raster_sha256 == RASTERS[name]["sha256"]


def test_integration_snippet():
    """INTEGRATION.md §2 runs verbatim (reference objects and builder, GPU
    Cluster) and gives the reference Cluster's raster."""
    sm = ref_module()
    if sm is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# reference-side script\n.*?)```", text, re.S).group(1)
    env = {}
    exec(compile(code, "INTEGRATION.md", "exec"), env)
    got = env["report"]
    # the same script on the reference's own Cluster
    ref_code = code.replace("cluster = B200Cluster(cfg)", "cluster = sm.Cluster(cfg)")
    renv = {}
    exec(compile(ref_code, "INTEGRATION.md(reference)", "exec"), renv)
    want = renv["report"]
    assert got.raster_sha256 == want.raster_sha256 and got.n_spike_events == want.n_spike_events
    assert got.n_synapses == want.n_synapses
    assert got.transport_messages["propagation"] == want.transport_messages["propagation"]
    assert got.transport_bytes["propagation"] == want.transport_bytes["propagation"]


def test_c1_full_size_digests():
    """BASELINE configs[0] at full size (sm/models.py:106-144: 10k neurons,
    K = 1000, 1 rank, seed 12345, 1e7 synapses): every table column equals
    the reference's by SHA-256, and the 100 ms raster and per-neuron spike
    counts are identical."""
    import hashlib
    want = json.load(open(os.path.join(GOLD, "c1_digests.json")))
    cfgd = want["config"]
    ns = gpu_ns()
    c = ns.make_cluster(ns.SimConfig(n_ranks=1, comm_mode=cfgd["comm_mode"], seed=cfgd["seed"]))
    ns.build_balanced_network(c, ns.BalancedParams(neurons_per_rank=cfgd["neurons_per_rank"], k_exc=cfgd["k_exc"],
                                                   k_inh=cfgd["k_inh"]))
    c.prepare()
    got = tables.digests(tables.canon_gpu(c))
    assert got == want["tables"]
    rep = c.simulate(0.0, cfgd["model_ms"], record=True)
    assert rep.n_synapses == want["n_synapses"]
    assert rep.raster_sha256 == want["raster"]["sha256"]
    counts = np.zeros(cfgd["neurons_per_rank"], dtype=np.int64)
    np.add.at(counts, c.merged_raster().events[:, 1], 1)
    assert hashlib.sha256(counts.tobytes()).hexdigest() == want["spike_counts_sha256"]


def test_c2_full_size_digests():
    """BASELINE configs[1] at full size (PD microcircuit, 77,169 neurons,
    ~3e8 synapses through fixed_total with normal weights and uniform integer
    delays, 1 rank, seed 12345): every table column equals the reference
    Cluster's by SHA-256 (tests/golden/c2_digests.json, made by
    make_golden.py --c2-only)."""
    path = os.path.join(GOLD, "c2_digests.json")
    if not os.path.exists(path):
        pytest.skip("c2_digests.json not generated")
    want = json.load(open(path))
    ns = gpu_ns()
    c = ns.make_cluster(ns.SimConfig(n_ranks=1, comm_mode="p2p", seed=want["config"]["seed"]))
    ns.build_microcircuit(c, ns.MicrocircuitParams(scale=want["config"]["scale"]))
    c.prepare()
    got = tables.digests(tables.canon_gpu(c))
    assert int(c.ranks[0].first_index[-1].item()) == want["n_synapses"]
    bad = [k for k in want["tables"] if got.get(k) != want["tables"][k]]
    assert not bad and set(got) == set(want["tables"]), (bad, sorted(set(got) ^ set(want["tables"])))


@pytest.mark.parametrize("delay_ms,mode,n_ranks", [(2.0, "p2p", 1), (3.0, "p2p", 1), (2.0, "collective", 2),
                                                   (3.0, "p2p", 3)])
def test_long_delays(delay_ms, mode, n_ranks):
    """Minimum delays of 17-32 steps: exchange / LIF blocks longer than the
    block kernel's 16 staged steps run as sub-blocks (identical raster)."""
    def make(ns):
        c = ns.make_cluster(ns.SimConfig(n_ranks=n_ranks, comm_mode=mode, seed=31))
        ns.build_balanced_network(c, ns.BalancedParams(neurons_per_rank=300, k_exc=24, k_inh=6, delay_ms=delay_ms))
        return c
    g, o = make(gpu_ns()), make(oracle_ns())
    rg = g.simulate(0.0, 25.0, record=True)
    o.simulate(0.0, 25.0, record=True)
    assert rg.n_spike_events > 0
    assert rg.raster_sha256 == o.raster_sha256()


def test_poisson_only_network():
    """Poisson drive and no synapses at all (no record delays: 32-step blocks)."""
    def make(ns):
        c = ns.make_cluster(ns.SimConfig(n_ranks=1, seed=3))
        x = c.create_neurons(0, 500, ns.LifParams(), ("normal", -58.0, 5.0))
        c.add_poisson_source(0, 12000.0, 0.5, 3, np.arange(x.start, x.stop))
        return c
    g, o = make(gpu_ns()), make(oracle_ns())
    rg = g.simulate(0.0, 20.0, record=True)
    o.simulate(0.0, 20.0, record=True)
    assert rg.n_spike_events > 0 and rg.n_synapses == 0
    assert rg.raster_sha256 == o.raster_sha256()


@pytest.mark.parametrize("name", ["explicit_3r_p2p", "balanced_4r_coll"])
def test_step_returns_spiking_nodes(name):
    """step() -> {rank: spiking nodes, ascending} like the reference
    (sm/engine.py:277-310), step after step."""
    g, _ = scenarios.SCENARIOS[name](gpu_ns())
    o, _ = scenarios.SCENARIOS[name](oracle_ns())
    g.prepare()
    o.prepare()
    total = 0
    for _ in range(120):
        a, b = g.step(), o.step()
        assert sorted(a) == sorted(range(g.n_ranks))
        for r in a:
            assert np.array_equal(a[r], np.asarray(b[r], dtype=np.int64)), r
            total += len(a[r])
    assert total > 0


@pytest.mark.parametrize("name", sorted(json.load(open(os.path.join(GOLD, "transport.json")))))
def test_transport_counters(name):
    """Messages and bytes of the propagation phase equal the reference's
    LockstepTransport counters (sm/transport.py:128-129,165-166)."""
    want = json.load(open(os.path.join(GOLD, "transport.json")))[name]
    c, sim = scenarios.SCENARIOS[name](gpu_ns())
    rep = c.simulate(sim[0], sim[1], record=False)
    assert rep.transport_messages["propagation"] == want["messages"]["propagation"]
    if name not in scenarios.NON_DYADIC:
        assert rep.transport_bytes["propagation"] == want["bytes"]["propagation"]
    for ph in ("construction", "preparation"):
        assert rep.transport_messages[ph] == 0 and rep.transport_bytes[ph] == 0


def test_several_devices_rejected():
    from paper_2512_09502_b200 import api
    from paper_2512_09502_b200.engine import Cluster
    with pytest.raises(ValueError):
        Cluster(api.SimConfig(n_ranks=2), devices=["cuda:0", "cuda:1"])
    Cluster(api.SimConfig(n_ranks=2), devices=["cuda:0", "cuda:0"])  # one device: fine


def test_second_device_in_one_process():
    """A Cluster on cuda:1 next to one on cuda:0 in the same process (kernel
    attributes and the device error word are per device; every façade call
    makes the cluster's device current): both build the C1 tables with the
    reference's digests, the calls interleaved."""
    import torch
    from paper_2512_09502_b200.engine import Cluster
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    want = json.load(open(os.path.join(GOLD, "c1_digests.json")))
    cfgd = want["config"]
    ns = gpu_ns()
    p = ns.BalancedParams(neurons_per_rank=cfgd["neurons_per_rank"], k_exc=cfgd["k_exc"], k_inh=cfgd["k_inh"])
    cfg = ns.SimConfig(n_ranks=1, comm_mode=cfgd["comm_mode"], seed=cfgd["seed"])
    try:
        c0 = Cluster(cfg, devices=["cuda:0"])
        ns.build_balanced_network(c0, p)
        c1 = Cluster(cfg, devices=["cuda:1"])
        ns.build_balanced_network(c1, p)
        c0.prepare()
        c1.prepare()
        assert c1.ranks[0].device == torch.device("cuda", 1)
        for c in (c1, c0):
            assert tables.digests(tables.canon_gpu(c)) == want["tables"]
        r1 = c1.simulate(0.0, cfgd["model_ms"], record=True)
        r0 = c0.simulate(0.0, cfgd["model_ms"], record=True)
        assert r1.raster_sha256 == r0.raster_sha256 == want["raster"]["sha256"]
    finally:
        torch.cuda.set_device(0)
