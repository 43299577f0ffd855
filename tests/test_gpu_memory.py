"""Modeled-byte arenas: host/device peak bytes per rank after
prepare equal the reference's (tests/golden/memory.json, generated from the
reference by tests/golden/make_golden.py) for every scenario at optimisation
levels 0..3 (placement plans, sm/construction.py:59-71)."""
import functools
import json
import os

import pytest

import scenarios
from namespaces import gpu_ns

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "memory.json")))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(scenarios.SCENARIOS))
def test_arena_peaks(name):
    from paper_2512_09502_b200 import api
    for level in (0, 1, 2, 3):
        ns = gpu_ns()
        ns.SimConfig = functools.partial(api.SimConfig, opt_level=level)
        c, _ = scenarios.SCENARIOS[name](ns)
        c.prepare()
        got = dict(host=c._per_rank(lambda st: st.mem.host.peak_bytes),
                   device=c._per_rank(lambda st: st.mem.device.peak_bytes))
        assert got == GOLD[f"{name}/L{level}"], (name, level, got, GOLD[f"{name}/L{level}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["balanced_2r_p2p", "multi_area_2r_coll", "remote_p2p"])
def test_real_placement(name):
    """Levels 0/1 place first_index, counts, the (R, L) maps (level 0) and the
    image lookups in pinned host memory that the kernels read in place;
    level 2 drops the counts; tables and rasters are identical at every
    level (sm/construction.py:43-71: behaviour never depends on placement)."""
    import tables
    from paper_2512_09502_b200 import api
    out = {}
    for level in (0, 1, 2, 3):
        ns = gpu_ns()
        ns.SimConfig = functools.partial(api.SimConfig, opt_level=level)
        c, sim = scenarios.SCENARIOS[name](ns)
        c.prepare()
        for st in c.ranks.values():
            host = level in (0, 1)
            assert st.first_index.is_cuda != host and (not host or st.first_index.is_pinned())
            assert (st.counts is None) == (level == 2)
            for v in st.I.values():
                assert v.is_cuda != host
            for r, l in st.RL.values():
                assert l.is_cuda == (level != 0)
        t = tables.canon_gpu(c)
        rep = c.simulate(sim[0], sim[1], record=True) if sim is not None else None
        out[level] = (t, rep.raster_sha256 if rep is not None else None)
    for level in (0, 1, 3):
        assert not tables.compare(out[level][0], out[2][0]), level
        assert out[level][1] == out[2][1], level
