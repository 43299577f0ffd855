"""The N>1 exchange protocol (exchange.py) on CPU with gloo, world size 2
and 3: every rank receives exactly the packets addressed to it, in
ascending source-rank order, and allgather rounds deliver every member's
occupied packets (sm/transport.py:92-168 semantics) -- for the
fixed-capacity rounds the engine runs (sizes agreed without a count round)
and for the variable-size rounds."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CAP = 16


def _packets(rank, n):
    rng = np.random.default_rng(100 + rank)
    counts = rng.integers(0, CAP + 1, n)
    counts[rank] = 0
    buf = np.zeros((n, CAP, 2), dtype=np.int32)
    for d in range(n):
        buf[d, :counts[d], 0] = rng.integers(0, 1000, counts[d])
        buf[d, :counts[d], 1] = rng.integers(0, 50, counts[d])
    return counts.astype(np.int32), buf


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_09502_b200.exchange import allgather_round, p2p_round
    try:
        counts, buf = _packets(rank, world)
        out, rc, _, offs = p2p_round(torch.from_numpy(counts), torch.from_numpy(buf.reshape(-1)), CAP)
        for src in range(world):
            sc, sb = _packets(src, world)
            n = int(sc[rank])
            assert rc[src] == n
            got = out[int(offs[src]): int(offs[src]) + 2 * n].numpy().reshape(-1, 2)
            assert np.array_equal(got, sb[rank, :n])
        # allgather: member i contributes its packets for destination 0
        recv, ac, _, cmax = allgather_round(torch.tensor([int(counts[(rank + 1) % world])]),
                                            torch.from_numpy(buf[(rank + 1) % world].reshape(-1).copy()), world)
        for src in range(world):
            sc, sb = _packets(src, world)
            n = int(sc[(src + 1) % world])
            assert ac[src] == n
            got = recv[src * 2 * cmax: src * 2 * cmax + 2 * n].numpy().reshape(-1, 2)
            assert np.array_equal(got, sb[(src + 1) % world, :n])
        # fixed-capacity rounds: pair capacity c(s, d) known to both sides
        from paper_2512_09502_b200.exchange import fixed_allgather, fixed_p2p

        def cap(s_, d_):
            return 0 if s_ == d_ else 3 + s_ + 2 * d_

        stride = CAP
        fc = np.array([min(int(counts[d]), cap(rank, d)) for d in range(world)], dtype=np.int32)
        out_c = [cap(rank, d) for d in range(world)]
        in_c = [cap(s_, rank) for s_ in range(world)]
        send = torch.zeros(max(sum(2 + 2 * c for c in out_c if c), 1), dtype=torch.int32)
        recv = torch.zeros(max(sum(2 + 2 * c for c in in_c if c), 1), dtype=torch.int32)
        rv, offs2 = fixed_p2p(torch.from_numpy(fc), torch.from_numpy(buf.reshape(-1).copy()), stride, out_c, in_c,
                              send, recv)
        for src in range(world):
            if src == rank:
                continue
            sc, sb = _packets(src, world)
            n = min(int(sc[rank]), cap(src, rank))
            o = offs2[src]
            assert int(rv[o]) == n
            assert np.array_equal(rv[o + 2: o + 2 + 2 * n].numpy().reshape(-1, 2), sb[rank, :n])
        gcap = 12
        gcount = torch.tensor([min(int(counts[(rank + 1) % world]), gcap)], dtype=torch.int32)
        gsend = torch.zeros(2 + 2 * gcap, dtype=torch.int32)
        grecv = torch.zeros(world * (2 + 2 * gcap), dtype=torch.int32)
        fixed_allgather(gcount, torch.from_numpy(buf[(rank + 1) % world].reshape(-1).copy()), gcap, gsend, grecv)
        for src in range(world):
            sc, sb = _packets(src, world)
            n = min(int(sc[(src + 1) % world]), gcap)
            base = src * (2 + 2 * gcap)
            assert int(grecv[base]) == n
            assert np.array_equal(grecv[base + 2: base + 2 + 2 * n].numpy().reshape(-1, 2), sb[(src + 1) % world, :n])
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_rounds_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
