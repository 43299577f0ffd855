"""spikemesh-b200: B200-native (sm_100a) construction + propagation path of
arXiv 2512.09502 behind the reference package's `Cluster` façade.

`Cluster` (engine.py) keeps the reference's method names, argument meaning
and exception classes (sm/engine.py:197-399); every heavy step runs in the
hand-written CUDA library built by build.py (csrc/, C ABI in
include/spikemesh_b200.h).
"""
from .api import (POINT_TO_POINT, ArenaUnderflowError, ConnSpec, ConsistencyError, DelayRangeError,
                  LifParams, ProtocolError, Raster, RngStream, SimConfig, SpikePacket, SynSpec)

__version__ = "0.1.0"


def __getattr__(name):
    # the engine imports torch; keep `import paper_2512_09502_b200` light
    if name in ("Cluster", "RunReport", "PhaseTimers"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)


__all__ = ["ArenaUnderflowError", "Cluster", "ConnSpec", "ConsistencyError", "DelayRangeError", "LifParams",
           "POINT_TO_POINT", "ProtocolError", "Raster", "RngStream", "RunReport", "SimConfig", "SpikePacket",
           "SynSpec", "__version__"]
