"""Spike-exchange rounds for one process per rank (sm/transport.py:92-168).

`fixed_allgather` / `fixed_p2p` are the rounds the engine runs (captured in
the block's CUDA graph): fixed-capacity buffers whose sizes both sides derive
from the routing tables, each buffer led by its count -- no count round, no
host synchronisation.  `p2p_round` / `allgather_round` are the variable-size
forms (counts first, then only the occupied packets).

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


def _all_gather_into(recv: torch.Tensor, send: torch.Tensor, group=None):
    if dist.get_backend(group) == "gloo":
        n = recv.numel() // send.numel()
        parts = list(recv.view(n, -1).unbind(0))
        dist.all_gather(parts, send, group=group)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)


def fixed_allgather(count: torch.Tensor, packets: torch.Tensor, cap: int, send: torch.Tensor,
                    recv: torch.Tensor, group=None):
    """One group round with a fixed capacity: send = [count, 0, packets[:2cap]]
    (2 + 2*cap int32), recv = n_members such blocks in ascending rank order.
    count: 1-element int32 device tensor; packets: at least 2*cap int32 (or
    fewer: the occupied part is what is copied)."""
    send[0:1].copy_(count.reshape(1))
    cc = min(2 * cap, packets.numel())
    send[2: 2 + cc].copy_(packets[:cc])
    _all_gather_into(recv, send, group)
    return recv


def fixed_p2p(counts: torch.Tensor, packets: torch.Tensor, stride: int, out_c: list, in_c: list,
              send: torch.Tensor, recv: torch.Tensor, group=None):
    """One point-to-point round with fixed capacities: destination d gets
    [count_d, 0, packets_d[:2*out_c[d]]] (nothing when out_c[d] == 0); the
    receiver sizes its blocks with in_c (its map sizes x the spike bound, equal
    to the sender's out_c).  packets: [n][stride][2] int32.  Returns recv and
    the offset of every source's block."""
    out_sz = [2 + 2 * c if c else 0 for c in out_c]
    in_sz = [2 + 2 * c if c else 0 for c in in_c]
    off = 0
    for d, c in enumerate(out_c):
        if not c:
            continue
        send[off: off + 1].copy_(counts[d: d + 1])
        cc = min(c, stride)
        send[off + 2: off + 2 + 2 * cc].copy_(packets[d * stride * 2: d * stride * 2 + 2 * cc])
        off += out_sz[d]
    dist.all_to_all_single(recv[: sum(in_sz)], send[: sum(out_sz)], in_sz, out_sz, group=group)
    offs, at = [], 0
    for sz in in_sz:
        offs.append(at)
        at += sz
    return recv, offs
