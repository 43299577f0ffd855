"""GPU construction tables and spike rasters against the golden fixtures
generated from the reference (bit-exact tables, identical raster SHA)."""
import json
import os

import numpy as np
import pytest

import scenarios
import tables

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RASTERS = json.load(open(os.path.join(GOLD, "rasters.json")))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(scenarios.SCENARIOS))
def test_tables(name):
    from namespaces import gpu_ns
    c, _ = scenarios.SCENARIOS[name](gpu_ns())
    c.prepare()
    gold = dict(np.load(os.path.join(GOLD, f"tables_{name}.npz")))
    bad = tables.compare(tables.canon_gpu(c), gold)
    assert not bad, bad[:10]
    c.check_alignment()
    c.check_construction_silent()


@pytest.mark.parametrize("name", sorted(scenarios.SCENARIOS))
def test_raster(name):
    from namespaces import gpu_ns
    c, sim = scenarios.SCENARIOS[name](gpu_ns())
    rep = c.simulate(sim[0], sim[1], record=True)
    want = RASTERS[name]["n_events"]
    if name in scenarios.NON_DYADIC:
        # non-dyadic weights over the full span: last-ulp differences of the
        # input sums can flip a rare threshold tie late in the run; exact
        # per-neuron counts over a short run: test_non_dyadic_short_run
        assert abs(rep.n_spike_events - want) <= max(2, 0.01 * want)
    else:
        assert rep.n_spike_events == want
        assert rep.raster_sha256 == RASTERS[name]["sha256"]


@pytest.mark.parametrize("name", sorted(scenarios.NON_DYADIC))
def test_non_dyadic_short_run(name):
    """Per-synapse normal weights: the fp64 input sums depend on the order of
    the delivery atomics (last-ulp differences).  Over a short run (3 ms)
    every neuron's spike count equals the oracle's (the reference's
    sequential order) exactly, and EVERY neuron's V agrees within
    V_TOL = 1e-9 mV (the north star's fp32 tolerance would be ~4e-6 mV at
    -65 mV)."""
    from namespaces import gpu_ns, oracle_ns
    V_TOL = 1e-9
    g, sim = scenarios.SCENARIOS[name](gpu_ns())
    o, _ = scenarios.SCENARIOS[name](oracle_ns())
    g.simulate(0.0, 3.0, record=True)
    o.simulate(0.0, 3.0, record=True)
    ge, oe = g.merged_raster().events, o.raster()
    gids_g, cnt_g = np.unique(ge[:, 1], return_counts=True)
    gids_o, cnt_o = np.unique(oe[:, 1], return_counts=True)
    assert np.array_equal(gids_g, gids_o) and np.array_equal(cnt_g, cnt_o)
    for r in sorted(g.ranks):
        e = g.export(r)
        st = o.ranks[r]
        ov = st.v[np.flatnonzero(st.mask)]
        assert len(ov) == len(e["v"])
        assert float(np.max(np.abs(e["v"] - ov), initial=0.0)) <= V_TOL


def test_v_after_run_matches_oracle():
    """Membrane potentials bit-exact against the oracle after a short run
    (dyadic weights: fp64 sums are order-independent)."""
    from namespaces import gpu_ns, oracle_ns
    g, sim = scenarios.SCENARIOS["balanced_4r_p2p"](gpu_ns())
    o, _ = scenarios.SCENARIOS["balanced_4r_p2p"](oracle_ns())
    g.simulate(0.0, 15.0, record=False)
    o.simulate(0.0, 15.0, record=False)
    for r in range(4):
        e = g.export(r)
        st = o.ranks[r]
        real = np.flatnonzero(st.mask)
        assert np.array_equal(e["v"], st.v[real])
        assert np.array_equal(e["ref"].astype(np.int64), st.ref[real])
