"""Construction scenarios shared by the golden-fixture generator (reference),
the oracle tests (CPU) and the parity tests (GPU).

Each scenario takes a namespace `ns` with the façade classes (Cluster,
SimConfig, ConnSpec, SynSpec, LifParams) and the model builders, builds a
network, and returns (cluster, sim) where sim = (warmup_ms, model_ms) or
None (tables only).
"""
from __future__ import annotations

import numpy as np


def balanced(ns, n_ranks, mode, per_rank, k_exc, k_inh, seed, sim=(0.0, 20.0), **kw):
    cfg = ns.SimConfig(n_ranks=n_ranks, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    ns.build_balanced_network(c, ns.BalancedParams(neurons_per_rank=per_rank, k_exc=k_exc, k_inh=k_inh, **kw))
    return c, sim


def explicit(ns, n_ranks, mode, n_neurons=300, n_edges=6000, net_seed=5, seed=11, sim=(0.0, 30.0)):
    net = ns.ExplicitNetwork.generate(n_neurons, n_edges, seed=net_seed)
    cfg = ns.SimConfig(n_ranks=n_ranks, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    rank_of = np.arange(n_neurons) % n_ranks if n_ranks > 1 else np.zeros(n_neurons, dtype=np.int64)
    net.instantiate(c, rank_of)
    return c, sim


def rules_local(ns, seed=3):
    """Every connection rule on one rank with constant syn (packed tables)."""
    cfg = ns.SimConfig(n_ranks=1, seed=seed)
    c = ns.make_cluster(cfg)
    a = c.create_neurons(0, 40, ns.LifParams(), ("normal", -60.0, 3.0), gids=np.arange(40))
    b = c.create_neurons(0, 25, ns.LifParams(i_e=0.5), -62.5, gids=np.arange(40, 65))
    A = np.arange(a.start, a.stop)
    B = np.arange(b.start, b.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect(0, A, B, S("fixed_indegree", k_in=7), Sy(0.25, 3))
    c.connect(0, B, A, S("fixed_total", n_total=333), Sy(-0.5, 2))
    c.connect(0, A[:25], B, S("one_to_one"), Sy(0.125, 1))
    c.connect(0, B[:5], A[:7], S("all_to_all"), Sy(0.0625, 4))
    c.connect(0, A[3:9], B, S("fixed_outdegree", k_out=6), Sy(0.5, 5))
    c.connect(0, A[[1, 1, 5]], B[[2, 3, 2]], S("assigned"), Sy(1.0, 6), port=1)
    c.connect(0, A, A, S("fixed_indegree", k_in=1), Sy(0.25, 3))   # single-source draws
    c.connect(0, A[:1], B, S("fixed_indegree", k_in=2), Sy(0.25, 3))  # ex == 1: no draws
    return c, (0.0, 5.0)


def rules_wide(ns, seed=4):
    """Per-record weight / delay arrays (wide tables)."""
    cfg = ns.SimConfig(n_ranks=1, seed=seed)
    c = ns.make_cluster(cfg)
    a = c.create_neurons(0, 30, ns.LifParams(i_e=0.375), ("normal", -60.0, 3.0), gids=np.arange(30))
    A = np.arange(a.start, a.stop)
    rng = np.random.default_rng(1)
    src = rng.integers(0, 30, 500)
    tgt = rng.integers(0, 30, 500)
    w = rng.integers(-64, 65, 500) / 256.0
    d = rng.integers(1, 9, 500)
    c.connect(0, A[src], A[tgt], ns.ConnSpec("assigned"), ns.SynSpec(w, d))
    c.connect(0, A, A, ns.ConnSpec("fixed_indegree", k_in=3), ns.SynSpec(0.5, 2))
    return c, (0.0, 5.0)


def rules_random(ns, seed=5):
    """Random SynSpec draws: normal weights then uniform_int delays from the
    call's syn stream (sm/construction.py:157-176), every draw-based rule."""
    cfg = ns.SimConfig(n_ranks=1, seed=seed)
    c = ns.make_cluster(cfg)
    a = c.create_neurons(0, 60, ns.LifParams(i_e=0.25), ("normal", -60.0, 3.0), gids=np.arange(60))
    A = np.arange(a.start, a.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect(0, A, A, S("fixed_indegree", k_in=9), Sy(("normal", 0.25, 0.05), ("uniform_int", 1, 8)))
    c.connect(0, A[:30], A[30:], S("fixed_total", n_total=1111), Sy(("normal", -0.5, 0.1), 3))
    c.connect(0, A[:7], A, S("fixed_outdegree", k_out=20), Sy(0.125, ("uniform_int", 2, 2)))
    c.connect(0, A[5:25], A[10:30], S("one_to_one"), Sy(("normal", 0.0, 1.0), ("uniform_int", 1, 30)))
    c.connect(0, A[:4], A[:9], S("all_to_all"), Sy(0.25, ("uniform_int", 3, 9)))
    return c, (0.0, 5.0)


def rules_no_autapse(ns, seed=8):
    """allow_autapses=False: self-connections redrawn from the call's stream
    (sm/construction.py:524-529); tiny populations force several rounds."""
    cfg = ns.SimConfig(n_ranks=1, seed=seed)
    c = ns.make_cluster(cfg)
    a = c.create_neurons(0, 40, ns.LifParams(i_e=0.3), ("normal", -60.0, 3.0), gids=np.arange(40))
    A = np.arange(a.start, a.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect(0, A, A, S("fixed_indegree", k_in=12, allow_autapses=False), Sy(0.25, 2))
    c.connect(0, A[:3], A[:3], S("fixed_indegree", k_in=40, allow_autapses=False), Sy(0.125, 3))
    c.connect(0, A[:6], A[:6], S("fixed_total", n_total=300, allow_autapses=False), Sy(("normal", 0.1, 0.01), 2))
    c.connect(0, A, A, S("fixed_total", n_total=500, allow_autapses=False), Sy(-0.25, ("uniform_int", 1, 4)))
    return c, (0.0, 5.0)


def no_multapse(ns, mode="p2p", seed=21):
    """allow_multapses=False: one numpy choice(n, k, replace=False) row per
    target (sm/construction.py:403-404, 680-683) -- the tail-shuffle variant
    (n > 10000, k > n // 50), Floyd's variant, a flagged remote call (the
    source rank replays the rows) and the distributed rule."""
    cfg = ns.SimConfig(n_ranks=2, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    group = -1
    if mode == "collective":
        group = 0
        c.declare_group(0, [0, 1])
    a = c.create_neurons(0, 12000, ns.LifParams(i_e=0.2), ("normal", -60.0, 2.0), gids=np.arange(12000))
    b = c.create_neurons(1, 500, ns.LifParams(i_e=0.4), ("normal", -58.0, 3.0), gids=np.arange(12000, 12500))
    A, B = np.arange(a.start, a.stop), np.arange(b.start, b.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect(0, A, A[:50], S("fixed_indegree", k_in=300, allow_multapses=False), Sy(0.125, 2))
    c.connect(1, B, B, S("fixed_indegree", k_in=20, allow_multapses=False), Sy(0.25, 3))
    c.connect_remote(0, A[:1000], 1, B[:100], S("fixed_indegree", k_in=5, allow_multapses=False),
                     Sy(0.5, 2), group=group)
    c.connect_fixed_indegree_distributed([(0, A[:2000]), (1, B)], [(0, A[:30]), (1, B[:30])], 40,
                                         Sy(-0.25, 2), group=group, allow_multapses=False)
    return c, (0.0, 5.0)


def poisson_high(ns, seed=41):
    """Poisson drive with lam >= 10 (numpy's PTRS branch, two words per
    trial): lam = 12 and 35 per step next to a lam = 1.1 device."""
    cfg = ns.SimConfig(n_ranks=1, seed=seed)
    c = ns.make_cluster(cfg)
    a = c.create_neurons(0, 200, ns.LifParams(), ("normal", -60.0, 3.0), gids=np.arange(200))
    A = np.arange(a.start, a.stop)
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.add_poisson_source(0, 120_000.0, 0.03125, 2, A[:120])
    c.add_poisson_source(0, 350_000.0, 0.015625, 3, A[60:])
    c.add_poisson_source(0, 11_000.0, 0.125, 4, A[::2])
    c.connect(0, A, A, S("fixed_indegree", k_in=20), Sy(-0.125, 2))
    return c, (0.0, 10.0)


def dist_random(ns, mode="p2p", seed=31):
    """Random SynSpec in the distributed rule: each source-rank batch draws its
    weights / delays from its own stream in (rank, source) order
    (sm/construction.py:689-703); a remote call first leaves pre-existing
    images (non-consecutive image ids), the second call is without multapses."""
    cfg = ns.SimConfig(n_ranks=3, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    group = -1
    if mode == "collective":
        group = 0
        c.declare_group(0, [0, 1, 2])
    pops = []
    for r in range(3):
        x = c.create_neurons(r, 60, ns.LifParams(i_e=0.25), ("normal", -58.0, 4.0), gids=r * 60 + np.arange(60))
        pops.append(np.arange(x.start, x.stop))
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect_remote(1, pops[1][::3], 0, pops[0][:20], S("fixed_indegree", k_in=3), Sy(0.125, 3), group=group)
    c.connect_fixed_indegree_distributed([(r, pops[r]) for r in range(3)], [(r, pops[r]) for r in range(3)], 12,
                                         Sy(("normal", 0.1, 0.02), ("uniform_int", 2, 6)), group=group)
    c.connect_fixed_indegree_distributed([(0, pops[0][:30]), (2, pops[2])], [(1, pops[1]), (2, pops[2][:25])], 7,
                                         Sy(-0.25, ("uniform_int", 3, 5)), group=group, allow_multapses=False)
    return c, (0.0, 5.0)


def poisson_multi(ns, mode="p2p", seed=12):
    """Several Poisson devices per rank with overlapping, permuted targets and
    delays below / above the exchange block (all records delay >= 5, so ranks
    run multi-step LIF blocks of 5)."""
    cfg = ns.SimConfig(n_ranks=2, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    group = -1
    if mode == "collective":
        group = 0
        c.declare_group(0, [0, 1])
    pops = []
    for r in range(2):
        x = c.create_neurons(r, 90, ns.LifParams(), ("normal", -60.0, 3.0), gids=r * 90 + np.arange(90))
        pops.append(np.arange(x.start, x.stop))
    S, Sy = ns.ConnSpec, ns.SynSpec
    for r in range(2):
        c.connect(r, pops[r], pops[r], S("fixed_indegree", k_in=8), Sy(0.25, 5))
        c.add_poisson_source(r, 8000.0, 0.125, 2, pops[r])
        c.add_poisson_source(r, 5000.0, 0.25, 9, pops[r][::-1][:40])
        c.add_poisson_source(r, 3000.0, 0.5, 5, pops[r][10:70:3])
    c.connect_remote(0, pops[0], 1, pops[1], S("fixed_indegree", k_in=6), Sy(0.125, 5), group=group)
    c.connect_remote(1, pops[1], 0, pops[0], S("fixed_indegree", k_in=6), Sy(-0.25, 7), group=group)
    return c, (0.0, 12.0)


def remote_random(ns, mode="p2p", seed=6):
    cfg = ns.SimConfig(n_ranks=2, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    group = -1
    if mode == "collective":
        group = 0
        c.declare_group(0, [0, 1])
    pops = []
    for r in range(2):
        x = c.create_neurons(r, 80, ns.LifParams(i_e=0.2), ("normal", -58.0, 4.0), gids=r * 80 + np.arange(80))
        pops.append(np.arange(x.start, x.stop))
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect_remote(0, pops[0], 1, pops[1], S("fixed_indegree", k_in=6), Sy(("normal", 0.2, 0.02), ("uniform_int", 2, 9)),
                     group=group)
    c.connect_remote(1, pops[1], 0, pops[0][:10], S("fixed_indegree", k_in=2), Sy(("normal", 0.3, 0.01), 4),
                     group=group)  # flagged
    c.connect_remote(1, pops[1][:40], 0, pops[0], S("fixed_total", n_total=500), Sy(0.125, ("uniform_int", 2, 5)),
                     group=group)
    return c, (0.0, 5.0)


def microcircuit(ns, scale=0.02, seed=77):
    cfg = ns.SimConfig(n_ranks=1, seed=seed)
    c = ns.make_cluster(cfg)
    ns.build_microcircuit(c, ns.MicrocircuitParams(scale=scale))
    return c, (0.0, 5.0)


def remote_mix(ns, mode="p2p", seed=9):
    """Remote connections of every rule across 3 ranks, sparse (flagged) and
    dense (unflagged), p2p or collective."""
    cfg = ns.SimConfig(n_ranks=3, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    group = -1
    if mode == "collective":
        group = 0
        c.declare_group(0, [0, 1, 2])
    pops = []
    for r in range(3):
        x = c.create_neurons(r, 50, ns.LifParams(), ("normal", -58.0, 4.0), gids=r * 50 + np.arange(50))
        pops.append(np.arange(x.start, x.stop))
    S, Sy = ns.ConnSpec, ns.SynSpec
    c.connect_remote(0, pops[0], 1, pops[1][:3], S("fixed_indegree", k_in=4), Sy(0.25, 2), group=group)   # flagged
    c.connect_remote(0, pops[0], 1, pops[1], S("fixed_indegree", k_in=5), Sy(0.125, 3), group=group)      # dense
    c.connect_remote(1, pops[1][10:40], 2, pops[2], S("fixed_total", n_total=12), Sy(0.5, 2), group=group)  # flagged
    c.connect_remote(2, pops[2][:20], 0, pops[0][:20], S("one_to_one"), Sy(0.25, 1), group=group)
    c.connect_remote(2, pops[2][5:9], 1, pops[1][:6], S("all_to_all"), Sy(-0.25, 4), group=group)
    c.connect_remote(1, pops[1][:4], 0, pops[0], S("fixed_outdegree", k_out=9), Sy(0.125, 2), group=group)
    c.connect_remote(0, pops[0][[7, 3, 7]], 2, pops[2][[1, 2, 3]], S("assigned"), Sy(0.75, 3), group=group)
    c.connect_remote(0, pops[0], 1, pops[1][5:9], S("fixed_indegree", k_in=2), Sy(0.25, 2), group=group)  # flagged again
    for r in range(3):
        c.connect(r, pops[r], pops[r], S("fixed_indegree", k_in=6), Sy(0.0625, 2))
        c.add_poisson_source(r, 16000.0, 0.25, 2, pops[r])
    return c, (0.0, 10.0)


def multi_area(ns, n_ranks=2, mode="p2p", seed=21):
    areas = [ns.AreaSpec(f"A{i}", 120 + 10 * i, 1000 * (i + 1)) for i in range(4)]
    assign, _ = ns.pack_areas(areas, n_ranks)
    cfg = ns.SimConfig(n_ranks=n_ranks, comm_mode=mode, seed=seed)
    c = ns.make_cluster(cfg)
    ns.build_multi_area(c, areas, assign, ns.MultiAreaParams(k_intra_exc=12, k_intra_inh=3, k_inter=4))
    return c, (0.0, 10.0)


SCENARIOS = {
    "balanced_1r": lambda ns: balanced(ns, 1, "p2p", 400, 32, 8, 12345, sim=(0.0, 30.0)),
    "balanced_4r_p2p": lambda ns: balanced(ns, 4, "p2p", 200, 16, 4, 7, sim=(0.0, 20.0)),
    "balanced_4r_coll": lambda ns: balanced(ns, 4, "collective", 200, 16, 4, 7, sim=(0.0, 20.0)),
    "balanced_2r_sparse_coll": lambda ns: balanced(ns, 2, "collective", 300, 3, 1, 17, sim=(0.0, 10.0)),
    "rules_local": rules_local,
    "rules_wide": rules_wide,
    "remote_p2p": lambda ns: remote_mix(ns, "p2p"),
    "remote_coll": lambda ns: remote_mix(ns, "collective"),
    "explicit_1r": lambda ns: explicit(ns, 1, "p2p"),
    "explicit_3r_p2p": lambda ns: explicit(ns, 3, "p2p"),
    "explicit_3r_coll": lambda ns: explicit(ns, 3, "collective"),
    "multi_area_2r": lambda ns: multi_area(ns, 2, "p2p"),
    "balanced_2r_p2p": lambda ns: balanced(ns, 2, "p2p", 250, 20, 5, 8, sim=(0.0, 20.0)),
    "explicit_2r_coll": lambda ns: explicit(ns, 2, "collective"),
    "multi_area_2r_coll": lambda ns: multi_area(ns, 2, "collective"),
    "rules_random": rules_random,
    "remote_random_p2p": lambda ns: remote_random(ns, "p2p"),
    "remote_random_coll": lambda ns: remote_random(ns, "collective"),
    "microcircuit_small": microcircuit,
    "rules_no_autapse": rules_no_autapse,
    "poisson_multi_p2p": lambda ns: poisson_multi(ns, "p2p"),
    "poisson_multi_coll": lambda ns: poisson_multi(ns, "collective"),
    "no_multapse_p2p": lambda ns: no_multapse(ns, "p2p"),
    "no_multapse_coll": lambda ns: no_multapse(ns, "collective"),
    "poisson_high": poisson_high,
    "balanced_8r_coll": lambda ns: balanced(ns, 8, "collective", 120, 16, 4, 9, sim=(0.0, 10.0)),
    "balanced_8r_p2p": lambda ns: balanced(ns, 8, "p2p", 120, 16, 4, 9, sim=(0.0, 10.0)),
    "dist_random_p2p": lambda ns: dist_random(ns, "p2p"),
    "dist_random_coll": lambda ns: dist_random(ns, "collective"),
}

# scenarios whose weights are not dyadic: tables are bit-exact, the raster is
# compared with a tolerance (fp64 sums depend on the atomic delivery order)
NON_DYADIC = {"rules_random", "remote_random_p2p", "remote_random_coll", "microcircuit_small", "rules_no_autapse",
              "dist_random_p2p", "dist_random_coll"}
