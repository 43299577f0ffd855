"""Façade namespaces for tests/scenarios.py: CPU oracle and GPU product."""
from types import SimpleNamespace

from paper_2512_09502_b200 import api, models


def _common(make):
    return SimpleNamespace(
        SimConfig=api.SimConfig, make_cluster=make, ConnSpec=api.ConnSpec, SynSpec=api.SynSpec,
        LifParams=api.LifParams, build_balanced_network=models.build_balanced_network,
        BalancedParams=models.BalancedParams, ExplicitNetwork=models.ExplicitNetwork,
        build_multi_area=models.build_multi_area, AreaSpec=models.AreaSpec, pack_areas=models.pack_areas,
        MultiAreaParams=models.MultiAreaParams, build_microcircuit=models.build_microcircuit,
        MicrocircuitParams=models.MicrocircuitParams)


def oracle_ns():
    from oracle.spikemesh_oracle import OracleCluster
    return _common(OracleCluster)


def gpu_ns(**kw):
    from paper_2512_09502_b200.engine import Cluster
    return _common(lambda cfg: Cluster(cfg, **kw))
