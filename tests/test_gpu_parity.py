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
        # non-dyadic weights: fp64 input sums depend on atomic order (1 ulp);
        # spike counts agree over short runs up to rare threshold ties
        assert abs(rep.n_spike_events - want) <= max(2, 0.01 * want)
    else:
        assert rep.n_spike_events == want
        assert rep.raster_sha256 == RASTERS[name]["sha256"]


@pytest.mark.parametrize("name", sorted(scenarios.NON_DYADIC))
def test_v_tolerance_non_dyadic(name):
    """V within 1e-9 (relative) of the oracle for >= 99% of neurons after a
    short run with per-synapse normal weights (north star: fp32 tolerance)."""
    from namespaces import gpu_ns, oracle_ns
    g, sim = scenarios.SCENARIOS[name](gpu_ns())
    o, _ = scenarios.SCENARIOS[name](oracle_ns())
    g.simulate(0.0, 3.0, record=False)
    o.simulate(0.0, 3.0, record=False)
    close = total = 0
    for r in sorted(g.ranks):
        e = g.export(r)
        st = o.ranks[r]
        ov = st.v[np.flatnonzero(st.mask)]
        close += int(np.sum(np.abs(e["v"] - ov) <= 1e-9 * np.abs(ov)))
        total += len(ov)
    assert close >= 0.99 * total, (close, total)


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
