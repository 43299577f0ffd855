"""Source-side replay (the path every process of a multi-GPU run uses for
the ranks it does not own) against the target-side bitmaps, on one GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["balanced_4r_coll", "balanced_4r_p2p", "remote_p2p", "remote_random_coll"])
def test_single_rank_processes_match(name):
    """Build the scenario once per rank with only that rank local (what one
    process per GPU does) and compare every table with the all-local build."""
    import scenarios
    import tables
    from namespaces import gpu_ns
    full, _ = scenarios.SCENARIOS[name](gpu_ns())
    full.prepare()
    want = tables.canon_gpu(full)
    for r in range(full.n_ranks):
        part, _ = scenarios.SCENARIOS[name](gpu_ns(local_ranks=[r]))
        part.prepare()
        got = tables.canon_gpu(part)
        sub = {k: v for k, v in want.items() if k.startswith(f"r{r}/")}
        bad = tables.compare(got, sub)
        assert not bad, (r, bad[:5])
