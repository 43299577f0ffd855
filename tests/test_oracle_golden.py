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
