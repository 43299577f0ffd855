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


def ref_module():
    """The unmodified reference package (`spikemesh`) when it is importable:
    installed under baseline/_ref (travels to the GPU box) or on PYTHONPATH.
    None otherwise."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "baseline", "_ref")
    if os.path.isdir(path) and path not in sys.path:
        sys.path.insert(0, path)
    try:
        import spikemesh
    except ImportError:
        return None
    return spikemesh


def ref_gpu_ns():
    """The reference's own SimConfig/ConnSpec/SynSpec/LifParams and model
    builders driving the GPU Cluster (the drop-in claim of INTEGRATION.md §2).
    The PD microcircuit has no reference builder: this repository's script
    (calling only façade methods) stands in."""
    sm = ref_module()
    if sm is None:
        return None
    import spikemesh.models as smm
    from paper_2512_09502_b200.engine import Cluster
    return SimpleNamespace(
        SimConfig=sm.SimConfig, make_cluster=Cluster, ConnSpec=sm.ConnSpec, SynSpec=sm.SynSpec,
        LifParams=sm.LifParams, build_balanced_network=smm.build_balanced_network,
        BalancedParams=smm.BalancedParams, ExplicitNetwork=smm.ExplicitNetwork,
        build_multi_area=smm.build_multi_area, AreaSpec=smm.AreaSpec, pack_areas=smm.pack_areas,
        MultiAreaParams=smm.MultiAreaParams, build_microcircuit=models.build_microcircuit,
        MicrocircuitParams=models.MicrocircuitParams)
