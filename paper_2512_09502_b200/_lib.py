"""ctypes binding of the sm_100a C-ABI library (include/spikemesh_b200.h).

There is no CPU fallback: importing the engine on a machine without the
built library, or calling a kernel without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os

from .api import ConsistencyError, DelayRangeError, ProtocolError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMX_LIB_PATH") or os.path.join(_HERE, "_build", "libspikemesh_b200.so")  # env: A/B tuning

P = ctypes.c_void_p
U64 = ctypes.c_uint64
I64 = ctypes.c_int64
U32 = ctypes.c_uint32
I32 = ctypes.c_int
D = ctypes.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "smx_last_error": (I32, [ctypes.c_char_p, ctypes.c_size_t]),
    "smx_version": (ctypes.c_char_p, []),
    "smx_stream_sync": (I32, [P]),
    "smx_set_sync_policy": (I32, [I32]),
    "smx_pool_setup": (I32, [I32]),
    "smx_stream_create": (I32, [I32, P]),
    "smx_draw_chain": (I32, [P, P]),
    "smx_set_pass_a_free_sms": (I32, [I32]),
    "smx_launch_count": (U64, []),
    "smx_philox_words": (I32, [U64, U64, U64, U64, P, P]),
    "smx_integers": (I32, [U64, U64, U64, I64, U64, U64, P, P, P]),
    "smx_init_v": (I32, [P, U32, P, U32, P, U64, D, D, P, P]),
    "smx_stream_keys": (I32, [P, U32, P, U32, P, U64, P, P]),
    "smx_counts_to_offsets": (I32, [P, U64, P, P]),
    "smx_sort_records": (I32, [P, P, P, P, U64, I32, I32, P, P, U64, P, P]),
    "smx_pay_table": (I32, [P, U64, P, U64, U32, P, P]),
    "smx_key_table": (I32, [P, U64, U32, I32, P, P]),
    "smx_dist_tables": (I32, [P, P, U64, P, I32, U32, P, P, P]),
    "smx_gen_draw": (I32, [U64, U64, U64, U64, U64, I32, I32, P, P, U32, P, P, P, P, U32, I32, U32, U32, P, P]),
    "smx_count_ranges": (I32, [P, U64, P, P, P]),
    "smx_peer_alloc": (I32, [U64, P]),
    "smx_peer_free": (I32, [P]),
    "smx_peer_handle": (I32, [P, P]),
    "smx_peer_open": (I32, [P, P]),
    "smx_peer_close": (I32, [P]),
    "smx_peer_exchange": (I32, [P, I32, P, I32, P, P, P, P, P, P, U32, P, P, P, U32, P, U32, P]),
    "smx_fused_gen": (I32, [U64, U64, U64, U64, I32, P, U32, P, U32, I32, I32, P, U64, P, P, P, P, P, P, P]),
    "smx_fused_sort": (I32, [P, P, P, I32, I32, I32, I32, P, P, P, U64, U64, P, P, P]),
    "smx_bits_or_many": (I32, [P, P, I32, U64, P]),
    "smx_check_device_errors": (I32, [P]),
    "smx_choice_rows": (I32, [U64, U64, U64, U64, U64, U64, P, P, P]),
    "smx_records_from_values": (I32, [P, U64, P, P, ctypes.c_uint32, P, P, P, P, P]),
    "smx_gen_pairs": (I32, [I32, U64, U64, P, P, P, P, P]),
    "smx_mark_values": (I32, [P, P, U64, P, P]),
    "smx_autapse_fix": (I32, [U64, U64, U64, U64, P, P, P, U64, P, U64, P, P]),
    "smx_assign_images": (I32, [P, U64, P, I32, I64, P, P]),
    "smx_gather_lut": (I32, [P, U64, P, P, P]),
    "smx_bits_or": (I32, [P, P, U64, P]),
    "smx_bits_prefix": (I32, [P, U64, P, P]),
    "smx_bits_compact": (I32, [P, U64, P, P, P, P, P]),
    "smx_build_routes": (I32, [P, I32, U64, P, P, P, P, P, P]),
    "smx_fill_wide_const": (I32, [P, P, U64, D, U32, P]),
    "smx_normal_chunks_for": (I32, [U64]),
    "smx_normal_fill": (I32, [U64, U64, P, D, D, U64, I32, P, P, P, P, P]),
    "smx_delay_fill": (I32, [U64, U64, U64, U32, U64, U64, U32, P, P, P]),
    "smx_promote_wide": (I32, [P, U64, P, P, P, P, P, P]),
    "smx_gather_wide": (I32, [P, U64, P, P, P, P, P, P, P]),
    "smx_max_meta": (I32, [P, U64, P, P]),
    "smx_lif_update": (I32, [P, P, P, P, P, P, P, P, U32, P, I32, I32, P, P, P]),
    "smx_poisson_emit": (I32, [P, I32, U32, P, D, P, U32, I32, I32, I32, I32, P, P]),
    "smx_poisson_workspace": (U64, [I32]),
    "smx_poisson_chunks_for": (I32, [U64, D]),
    "smx_poisson_counts": (I32, [U64, U64, P, D, U64, I32, P, P, P, P, P]),
    "smx_poisson_counts_ptrs": (I32, [U64, U64, P, D, U64, I32, P, P, P, P, P]),
    "smx_spikes": (I32, [P, U32, P, P, P, P, P, P, U32, P, P, P, U64, P, P, P, P, P]),
    "smx_step": (I32, [P, P, P, P, P, P, P, P, U32, P, I32, I32, P, I32, P, I32, P, I32, P, P, P, P, P, P, P, U32, P,
                        U32, P, P, U64, P, P, P, P, P, P, P, P, P, P]),
    "smx_ref_lif_step": (I32, [P, P, P, P, P, P, P, P, P, P, U64, P]),
    "smx_ref_deliver_spikes": (I32, [P, P, U64, P, P, P, P, P, P, I64, I64, I64, P]),
    "smx_block": (I32, [P, P, P, P, P, P, P, P, U32, P, I32, I32, P, I32, I32, P, I32, P, I32, P, P, P, P, P, P,
                         P, U32, P, U32, P, P, U64, P, P, P, P, P, P, P, P, P, P]),
    "smx_unpack": (I32, [P, P, U32, P, U64, P, P, P, U32, P, P]),
    "smx_deliver": (I32, [P, P, P, P, P, P, P, P, P, P, P, P, P, U32, I32, I32, I32, P]),
}

_lib = None


class SmxError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"spikemesh-b200 CUDA library not built ({LIB_PATH}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().smx_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


_EXC = {-1: ValueError, -2: ConsistencyError, -3: SmxError, -4: ProtocolError, -5: DelayRangeError}


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        raise _EXC.get(rc, SmxError)(f"{what}: {last_error()}" if what else last_error())


TRACE = {} if os.environ.get("SMX_TRACE") else None
TIMELINE = [] if os.environ.get("SMX_TIMELINE") else None


def call(name: str, *args) -> None:
    if TIMELINE is not None:
        import time
        import torch
        t0 = time.perf_counter()
        check(getattr(lib(), name)(*args), name)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        TIMELINE.append((name, t0, time.perf_counter(), e))
        return
    if TRACE is None:
        check(getattr(lib(), name)(*args), name)
        return
    import time
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(getattr(lib(), name)(*args), name)
    torch.cuda.synchronize()
    n, t = TRACE.get(name, (0, 0.0))
    TRACE[name] = (n + 1, t + time.perf_counter() - t0)
