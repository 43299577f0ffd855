"""The fused generation + sort path (csrc/fused.cu) against the general
path (smx_gen_draw + smx_sort_records, itself pinned to the reference's
goldens): identical tables for every digit split, several calls, both key
modes, rejections, and the overflow fallback."""
import numpy as np
import pytest

import scenarios
import tables
from namespaces import gpu_ns

pytestmark = pytest.mark.gpu


def _build(fused, fn, monkeypatch=None, lo=None):
    if lo is not None:
        monkeypatch.setenv("SMX_FUSED_LO", str(lo))
    ns = gpu_ns()
    make = ns.make_cluster

    def mk(cfg):
        c = make(cfg)
        c.fused_enabled = fused
        return c
    ns.make_cluster = mk
    c = fn(ns)
    c.prepare()
    return c


def _balanced(n_ranks, mode, per_rank, k_exc, k_inh, seed=7):
    def fn(ns):
        c, _ = scenarios.balanced(ns, n_ranks, mode, per_rank, k_exc, k_inh, seed)
        return c
    return fn


def _local_mix(ns):
    """Local fixed in-degree calls with key tables (scattered sources), a
    distributed call, overlapping populations and two classes."""
    c = ns.make_cluster(ns.SimConfig(n_ranks=1, seed=19))
    a = c.create_neurons(0, 3000, ns.LifParams(), -60.0)
    b = c.create_neurons(0, 1000, ns.LifParams(), -61.0)
    A, Bn = np.arange(a.start, a.stop), np.arange(b.start, b.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    rng = np.random.default_rng(3)
    c.connect(0, A, Bn, S("fixed_indegree", k_in=40), Sy(0.25, 3))
    c.connect(0, rng.permutation(A)[:777], A, S("fixed_indegree", k_in=9), Sy(-0.5, 4))
    c.connect(0, Bn, A, S("fixed_indegree", k_in=13), Sy(0.25, 3))
    c.connect_fixed_indegree_distributed([(0, Bn), (0, A[:500])], [(0, A)], 11, Sy(0.125, 2))
    return c


def _fixed_total_mix(ns):
    """Local fixed_total calls (targets drawn per record, continuing the
    position stream) between fixed in-degree calls, two classes, a scattered
    source set."""
    c = ns.make_cluster(ns.SimConfig(n_ranks=1, seed=37))
    a = c.create_neurons(0, 2500, ns.LifParams(), -60.0)
    b = c.create_neurons(0, 700, ns.LifParams(), -61.0)
    A, Bn = np.arange(a.start, a.stop), np.arange(b.start, b.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    rng = np.random.default_rng(5)
    c.connect(0, A, Bn, S("fixed_total", n_total=90_000), Sy(0.25, 3))
    c.connect(0, A, A, S("fixed_indegree", k_in=17), Sy(-0.5, 4))
    c.connect(0, rng.permutation(A)[:333], A, S("fixed_total", n_total=41_111), Sy(-0.5, 4))
    c.connect(0, Bn, Bn, S("fixed_total", n_total=5), Sy(0.25, 3))
    return c


CASES = {
    "balanced_1r": _balanced(1, "p2p", 3000, 240, 60),
    "balanced_4r_coll": _balanced(4, "collective", 700, 80, 20),
    "balanced_8r_coll": _balanced(8, "collective", 600, 80, 20),   # 8 source pieces: the generic key mode
    "balanced_3r_p2p": _balanced(3, "p2p", 900, 100, 25),
    "local_mix": _local_mix,
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_fused_equals_general(name):
    g = _build(False, CASES[name])
    f = _build(True, CASES[name])
    assert all(st.store_path == "general" for st in g.ranks.values())
    assert all(st.store_path == "fused" for st in f.ranks.values()), [st.store_path for st in f.ranks.values()]
    bad = tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))
    assert not bad, bad[:10]


def _small(ns):
    c, _ = scenarios.balanced(ns, 2, "collective", 500, 40, 10, 5)   # 11-bit keys: lo = 0 possible
    return c


@pytest.mark.parametrize("lo,case", [(0, "small"), (2, "small"), (0, "local_mix"), (1, "local_mix"), (3, "local_mix"),
                                     (6, "local_mix"), (7, "local_mix"), (8, "local_mix"), (9, "local_mix")])
def test_fused_digit_splits(lo, case, monkeypatch):
    """Every low-digit width of pass A (the high digit takes the rest, 8..12
    bits; local_mix at lo = 0 has 12-bit keys: the 12-bit pass B with
    32-bit records)."""
    fn = _small if case == "small" else CASES["local_mix"]
    g = _build(False, fn)
    f = _build(True, fn, monkeypatch, lo)
    assert all(st.store_path == "fused" for st in f.ranks.values())
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))


def test_fused_with_rejections():
    """A source range whose Lemire threshold rejects draws (ex = 300,000:
    p = 3.9e-5 per draw): the look-back carries the accept counts."""
    def fn(ns):
        c = ns.make_cluster(ns.SimConfig(n_ranks=1, seed=23))
        a = c.create_neurons(0, 300_000, ns.LifParams(), -60.0)
        A = np.arange(a.start, a.stop)
        c.connect(0, A, A[:40_000], ns.ConnSpec("fixed_indegree", k_in=60), ns.SynSpec(0.25, 3))
        return c
    g, f = _build(False, fn), _build(True, fn)
    assert f.ranks[0].store_path == "fused"
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))


def test_fused_overflow_falls_back(monkeypatch):
    """Regions too small for the draws: the overflow flag sends the rank
    through the general path, with identical tables."""
    from paper_2512_09502_b200.engine import Cluster
    real = Cluster._digit_probs

    def tiny(d, B):
        return real(d, B) / 3.0   # regions sized for a third of the draws
    g = _build(False, CASES["balanced_1r"])
    monkeypatch.setattr(Cluster, "_digit_probs", staticmethod(tiny))
    f = _build(True, CASES["balanced_1r"])
    assert f.ranks[0].store_path == "general"
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))


def test_fused_then_general_call_flushes_in_order():
    """A deferred call followed by a call the fused path cannot take (random
    weights): the deferred draws are generated first, in call order."""
    def fn(ns):
        c = ns.make_cluster(ns.SimConfig(n_ranks=1, seed=29))
        a = c.create_neurons(0, 500, ns.LifParams(), -60.0)
        A = np.arange(a.start, a.stop)
        c.connect(0, A, A, ns.ConnSpec("fixed_indegree", k_in=20), ns.SynSpec(0.25, 3))
        c.connect(0, A, A, ns.ConnSpec("fixed_indegree", k_in=5), ns.SynSpec(("normal", 0.5, 0.1), 2))
        return c
    g, f = _build(False, fn), _build(True, fn)
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))


@pytest.mark.parametrize("case,outcome", [("dense", "confirmed"), ("sparse", "dropped")])
def test_speculative_distributed_keys(case, outcome, monkeypatch):
    """Distributed calls with remote sources start pass A on predicted keys
    (fresh maps, every source value drawn) before the replay: a dense call
    confirms the prediction; a sparse one (forced; most values undrawn, so
    the images are not consecutive) drops to the general path.  Tables equal
    the general path's either way."""
    monkeypatch.setenv("SMX_SPECULATE", "force")
    k = (100, 25) if case == "dense" else (3, 1)

    def fn(ns):
        c, _ = scenarios.balanced(ns, 3, "p2p", 900, k[0], k[1], 11)
        return c
    g = _build(False, fn)
    f = _build(True, fn)
    assert f.spec_stats[outcome] > 0, f.spec_stats
    if outcome == "confirmed":
        assert all(st.store_path == "fused" for st in f.ranks.values())
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))


@pytest.mark.parametrize("min_total", [0, 100_000])
def test_fused_fixed_total(min_total, monkeypatch):
    """Local fixed_total on the fused path (cursor from a count-only draw,
    targets per record, positions through pass A), always (0) or only once
    the rank is on the fused path (the first, smaller call then takes the
    general path and so does the rest): identical tables either way."""
    from paper_2512_09502_b200.engine import Cluster
    g = _build(False, _fixed_total_mix)
    monkeypatch.setattr(Cluster, "FUSED_TOTAL_MIN", min_total)
    f = _build(True, _fixed_total_mix)
    assert f.ranks[0].store_path == ("fused" if min_total == 0 else "general")
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))


def test_speculation_redone_when_a_remote_run_is_never_drawn(monkeypatch):
    """A remote source run that no draw hits gets no images, so the real key
    pieces differ from the predicted ones while staying consecutive: pass A
    is redone with the real keys in the call's place (spec_stats 'redone')."""
    monkeypatch.setenv("SMX_SPECULATE", "force")

    def fn(ns):
        c = ns.make_cluster(ns.SimConfig(n_ranks=2, comm_mode="collective", seed=43))
        a = c.create_neurons(0, 10_000, ns.LifParams(), -60.0)
        b = c.create_neurons(1, 1, ns.LifParams(), -60.0, gids=np.array([10_000]))
        A, Bn = np.arange(a.start, a.stop), np.arange(b.start, b.stop)
        c.declare_group(0, [0, 1])
        c.connect_fixed_indegree_distributed([(0, A), (1, Bn)], [(0, A[:100])], 1, ns.SynSpec(0.125, 2), group=0)
        return c
    g = _build(False, fn)
    f = _build(True, fn)
    assert f.spec_stats["redone"] == 1, f.spec_stats
    assert f.ranks[0].store_path == "fused"
    assert not tables.compare(tables.canon_gpu(f), tables.canon_gpu(g))
