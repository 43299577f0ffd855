"""Spike-exchange rounds for one process per rank (sm/transport.py:92-168).

Device-agnostic halves of the NCCL path: they move packet buffers laid out
as `[destination][capacity][2]` int32 (map/roster position, emission step)
and return what this rank received, in ascending source-rank order (the
reference's inbox order, sm/transport.py:115-127, 157-164).  Counts travel
first so only the occupied part of each buffer crosses the link.  The same
functions run over NCCL on B200s and over gloo on CPU (tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def p2p_round(send_counts: torch.Tensor, packets: torch.Tensor, cap: int, group=None):
    """One point-to-point round.  send_counts[d] entries of packets[d] go to
    rank d.  Returns (recv flat int32 tensor, recv_counts[n_ranks] numpy,
    recv_counts tensor on the packets' device, per-source offsets)."""
    n = send_counts.numel()
    send_c = send_counts.to(torch.int32).contiguous()
    recv_c = torch.empty_like(send_c)
    dist.all_to_all_single(recv_c, send_c, group=group)
    sc, rc = send_c.cpu().numpy().astype(np.int64), recv_c.cpu().numpy().astype(np.int64)
    inp = torch.cat([packets[d * cap * 2: d * cap * 2 + 2 * int(sc[d])] for d in range(n)])
    total = int(2 * rc.sum())
    out = torch.empty(max(total, 1), dtype=packets.dtype, device=packets.device)
    dist.all_to_all_single(out[:total], inp, [2 * int(x) for x in rc], [2 * int(x) for x in sc], group=group)
    offsets = np.concatenate([[0], np.cumsum(2 * rc)])[:-1]
    return out, rc, recv_c, offsets


def allgather_round(count: torch.Tensor, packets: torch.Tensor, n_members: int, group=None):
    """One allgather round of a group: every member contributes
    packets[:count] (count a 1-element int32 tensor).  Returns (recv
    [n_members * 2 * cmax] tensor, counts numpy, counts tensor, cmax); block i
    is member i of the group in ascending rank order."""
    gloo = dist.get_backend(group) == "gloo"
    cnt = count.to(torch.int32).reshape(1).contiguous()
    if gloo:
        parts = [torch.empty_like(cnt) for _ in range(n_members)]
        dist.all_gather(parts, cnt, group=group)
        allc = torch.cat(parts)
    else:
        allc = torch.empty(n_members, dtype=torch.int32, device=cnt.device)
        dist.all_gather_into_tensor(allc, cnt, group=group)
    ac = allc.cpu().numpy().astype(np.int64)
    cmax = int(ac.max()) if len(ac) else 0
    recv = torch.empty(max(n_members * 2 * cmax, 1), dtype=packets.dtype, device=packets.device)
    if cmax:
        send = packets[: 2 * cmax].contiguous()
        if gloo:
            parts = [torch.empty_like(send) for _ in range(n_members)]
            dist.all_gather(parts, send, group=group)
            recv[: n_members * 2 * cmax] = torch.cat(parts)
        else:
            dist.all_gather_into_tensor(recv[: n_members * 2 * cmax], send, group=group)
    return recv, ac, allc, cmax
