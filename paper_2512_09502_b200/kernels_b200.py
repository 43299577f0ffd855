"""Drop-in backend for the reference's native-kernel boundary.

`sm/kernels/__init__.py:23-30` selects a module exposing BACKEND_NAME,
lif_step and deliver_spikes.  This module has the same three names and the
same argument lists (`_speedups.pyx:13-54`); arrays may be numpy arrays
(copied to the device and back, in place semantics kept) or CUDA torch
tensors (used in place).  INTEGRATION.md shows the two-line switch.
"""
from __future__ import annotations

import numpy as np
import torch

from ._lib import call

BACKEND_NAME = "b200"


def _dev(a, dtype):
    if isinstance(a, torch.Tensor):
        return a, None
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()
    return t, a


def _back(t, host):
    if host is not None:
        host[...] = t.cpu().numpy().reshape(host.shape)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def lif_step(v, ref_count, real_mask, inputs, decay, v_rest, v_reset, v_th, ref_steps, spiked_out):
    """kernels/_speedups.pyx:13-35 on the device."""
    V, hv = _dev(v, np.float64)
    R, hr = _dev(ref_count, np.int64)
    S, hs = _dev(spiked_out, np.uint8)
    args = [_dev(x, dt)[0] for x, dt in ((real_mask, np.uint8), (inputs, np.float64), (decay, np.float64),
                                          (v_rest, np.float64), (v_reset, np.float64), (v_th, np.float64),
                                          (ref_steps, np.int64))]
    call("smx_ref_lif_step", V.data_ptr(), R.data_ptr(), args[0].data_ptr(), args[1].data_ptr(), args[2].data_ptr(),
         args[3].data_ptr(), args[4].data_ptr(), args[5].data_ptr(), args[6].data_ptr(), S.data_ptr(), V.numel(),
         _stream())
    for t, h in ((V, hv), (R, hr), (S, hs)):
        _back(t, h)


def deliver_spikes(src_nodes, multiplicities, first_index, conn_tgt, conn_port, conn_delay, conn_weight, buffers,
                   now):
    """kernels/_speedups.pyx:38-54 on the device (fp64 atomics: exact for dyadic weights)."""
    B, hb = _dev(buffers, np.float64)
    shape = tuple(buffers.shape)
    ts = [_dev(x, dt)[0] for x, dt in ((src_nodes, np.int64), (multiplicities, np.int64), (first_index, np.int64),
                                        (conn_tgt, np.int64), (conn_port, np.int64), (conn_delay, np.int64),
                                        (conn_weight, np.float64))]
    call("smx_ref_deliver_spikes", ts[0].data_ptr(), ts[1].data_ptr(), ts[0].numel(), ts[2].data_ptr(),
         ts[3].data_ptr(), ts[4].data_ptr(), ts[5].data_ptr(), ts[6].data_ptr(), B.data_ptr(), shape[1], shape[2],
         int(now), _stream())
    _back(B, hb)
