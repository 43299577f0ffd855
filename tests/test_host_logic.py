"""CPU checks of host-side helpers of the engine (no device calls)."""
import numpy as np
import pytest

from paper_2512_09502_b200.engine import Cluster


@pytest.mark.parametrize("seed", range(20))
def test_population_runs_match_concatenated(seed):
    """Runs of consecutive nodes per source rank, from the populations and from
    the concatenated arrays (the distributed rule's piecewise key tables)."""
    rng = np.random.default_rng(seed)
    ranks, nodes = [], []
    for _ in range(rng.integers(1, 5)):
        r = int(rng.integers(0, 3))
        start = int(rng.integers(0, 50))
        a = np.arange(start, start + int(rng.integers(1, 30)), dtype=np.int64)
        if rng.random() < 0.3 and len(a) > 3:
            a = np.delete(a, int(rng.integers(1, len(a) - 1)))
        ranks.append(r)
        nodes.append(a)
    all_rank = np.concatenate([np.full(len(a), r) for r, a in zip(ranks, nodes)])
    all_node = np.concatenate(nodes)
    got = Cluster._pops_runs(ranks, nodes, max_pieces=64)
    want = Cluster._pieces_of(all_rank, all_node, max_pieces=64)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_run_info():
    """_run_info: one consecutive run (bounds from the ends) or the general
    min / max; empty arrays; no caching across refills of one array."""
    import numpy as np
    from paper_2512_09502_b200.engine import _consecutive, _run_info
    a = np.arange(7, 107, dtype=np.int64)
    assert _run_info(a) == (True, 7, 106) and _consecutive(a)
    a[50] = 3   # refilled in place: seen afresh
    assert _run_info(a) == (False, 3, 106) and not _consecutive(a)
    assert _run_info(np.array([5], dtype=np.int64)) == (False, 5, 5)
    assert _run_info(np.array([], dtype=np.int64))[0] is False
    assert _run_info(np.array([9, 8, 7], dtype=np.int64)) == (False, 7, 9)
