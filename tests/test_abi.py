"""The C-ABI library loads (no GPU needed) and exports exactly the symbols
include/spikemesh_b200.h declares; the ctypes table agrees with the header."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "spikemesh_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(smx_\w+)\s*\(", src))


def test_library_exports_every_declared_symbol():
    from paper_2512_09502_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(_declared()) if not hasattr(L, s)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    from paper_2512_09502_b200 import _lib
    declared = _declared()
    assert declared, "header parse failed"
    extra = set(_lib.SIGNATURES) - declared
    assert not extra, extra
    assert _lib.lib().smx_version().decode().startswith("spikemesh-b200")


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_09502_b200 import SimConfig
    from paper_2512_09502_b200.engine import Cluster
    with pytest.raises(RuntimeError, match="CUDA"):
        Cluster(SimConfig())


def test_pass_a_free_sms_bounds():
    """smx_set_pass_a_free_sms takes 0..16 and reports anything else as a
    ValueError-class status (-1) without touching the device."""
    from paper_2512_09502_b200 import _lib
    L = _lib.lib()
    assert L.smx_set_pass_a_free_sms(8) == 0
    assert L.smx_set_pass_a_free_sms(-1) == -1
    assert L.smx_set_pass_a_free_sms(17) == -1
    assert L.smx_set_pass_a_free_sms(8) == 0
