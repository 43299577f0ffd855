"""Full-size (C3: 1e5 neurons, K = 9000 + 2250, 1.125e9 synapses) properties
of the GPU construction that do not need the whole oracle run:

* record count and first_index close (every record has a source row),
* exact in-degree: every target receives exactly k_exc + k_inh records,
* stable order: inside each source row the target rows never decrease (the
  records of a row keep the generation order, target-major),
* the draws of the first and of the last target of each distributed call
  equal the oracle's numpy-exact stream (the last one after skipping every
  earlier target's draws, rejections included).
"""
import numpy as np
import pytest

ROW_MASK = 0xFFFFFF


@pytest.mark.gpu
def test_c3_fullsize_properties():
    import torch

    from oracle.rng import OracleStream
    from paper_2512_09502_b200 import api, engine, models

    P = models.BalancedParams(neurons_per_rank=100_000, k_exc=9000, k_inh=2250)
    c = engine.Cluster(api.SimConfig(n_ranks=1, seed=12345))
    models.build_balanced_network(c, P)
    c.prepare()
    st = c.ranks[0]
    n = st.n_records
    assert n == 100_000 * 11_250
    fi = st.first_index
    assert int(fi[-1].item()) == n
    rows = st.payload[:n]
    dev = rows.device
    indeg = torch.zeros(st.N, dtype=torch.int64, device=dev)
    bad_order = 0
    chunk = 1 << 27
    starts = torch.zeros(n + 1, dtype=torch.bool, device=dev)  # row-boundary marks
    starts[fi.clamp(max=n)] = True
    for a in range(0, n, chunk):
        b = min(n, a + chunk + 1)
        r = rows[a:b] & ROW_MASK
        indeg += torch.bincount(r[: min(chunk, n - a)].long(), minlength=st.N)[: st.N]
        dec = (r[1:] < r[:-1]).nonzero().flatten() + a + 1  # positions where the row decreases
        bad_order += int((~starts[dec]).sum().item())        # ... not at a source-row boundary
    assert bad_order == 0
    assert int(indeg.min().item()) == 11_250 and int(indeg.max().item()) == 11_250

    # draws of the first and the last target of each call against the oracle
    fi_h = fi.cpu().numpy()
    row_of = st.node2row.t[: st.n_nodes].cpu().numpy()

    def sources_of(target_node):
        row = int(row_of[target_node])
        pos = ((rows & ROW_MASK) == row).nonzero().flatten().cpu().numpy()
        return np.sort(np.searchsorted(fi_h, pos, side="right") - 1)

    for call, lo, total, k in ((1, 0, 80_000, 9000), (2, 80_000, 20_000, 2250)):
        s = OracleStream(12345, ("dist-indegree", call, 0))
        first = s.integers(0, total, size=k)
        left = 99_998                      # skip targets 1 .. 99998 (rejections included)
        while left:
            m = min(left, 1000)
            s.integers(0, total, size=k * m)
            left -= m
        last = s.integers(0, total, size=k)
        got0, got1 = sources_of(0), sources_of(99_999)
        # target 0 / 99999 records of this call: sources inside the call's population
        m0 = (got0 >= lo) & (got0 < lo + total)
        m1 = (got1 >= lo) & (got1 < lo + total)
        assert np.array_equal(got0[m0], np.sort(first + lo))
        assert np.array_equal(got1[m1], np.sort(last + lo))
