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
