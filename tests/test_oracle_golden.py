"""The CPU oracle's construction + propagation restatement against the
fixtures generated from the reference (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

import scenarios
import tables
from namespaces import oracle_ns

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RASTERS = json.load(open(os.path.join(GOLD, "rasters.json")))


@pytest.mark.parametrize("name", sorted(scenarios.SCENARIOS))
def test_tables_and_raster(name):
    c, sim = scenarios.SCENARIOS[name](oracle_ns())
    c.prepare()
    gold = dict(np.load(os.path.join(GOLD, f"tables_{name}.npz")))
    bad = tables.compare(tables.canon_oracle(c), gold)
    assert not bad, bad[:10]
    if sim is not None:
        c.simulate(sim[0], sim[1], record=True)
        assert c.raster().shape[0] == RASTERS[name]["n_events"]
        assert c.raster_sha256() == RASTERS[name]["sha256"]


def test_c1_full_size():
    """C1 at full size (1e7 synapses): every table column by SHA-256 and the
    100 ms raster equal the reference's (tests/golden/c1_digests.json)."""
    want = json.load(open(os.path.join(GOLD, "c1_digests.json")))
    cfg = want["config"]
    ns = oracle_ns()
    c = ns.make_cluster(ns.SimConfig(n_ranks=1, comm_mode=cfg["comm_mode"], seed=cfg["seed"]))
    ns.build_balanced_network(c, ns.BalancedParams(neurons_per_rank=cfg["neurons_per_rank"], k_exc=cfg["k_exc"],
                                                   k_inh=cfg["k_inh"]))
    c.prepare()
    assert tables.digests(tables.canon_oracle(c)) == want["tables"]
    c.simulate(0.0, cfg["model_ms"], record=True)
    assert c.raster_sha256() == want["raster"]["sha256"]

