"""Modeled-byte accounting of the reference's memory arenas.

The reference charges every structure class a declared per-entry cost to a
host or a device `MemoryArena` chosen by the optimisation level's placement
plan (sm/construction.py:43-71, sm/core.py:26-36,155-186).  The figures are
modeled, not measured: `RunReport.host_peak_bytes / device_peak_bytes` are
these arenas' peaks.  This module restates the arenas and the placement
plans; `engine.Cluster` replays the reference's allocation events in the
reference's order from the counts it already has on the device (map and
mirror sizes are bitmap popcounts, record counts per call and source rank
come from the generated keys), so the peaks are identical.  The placement
never changes where this implementation keeps its tables -- everything lives
in HBM -- exactly as "functional behavior never depends on the placement" in
the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

from .api import ArenaUnderflowError

HOST, DEVICE = "host", "device"

CONNECTION_RECORD_BYTES = 16   # sm/core.py:26-36
MAP_ENTRY_BYTES = 4
FIRST_INDEX_ENTRY_BYTES = 8
COUNT_ENTRY_BYTES = 4
ROUTE_ENTRY_BYTES = 8
NEURON_STATE_BYTES = 48
BUFFER_SLOT_BYTES = 8
TEMP_IMAGE_SLOT_BYTES = 4
TEMP_FLAG_BYTES = 1


@dataclass(frozen=True)
class PlacementPlan:
    """sm/construction.py:43-56: arena of each remote-structure class
    (counts None: no count array is charged)."""
    remote_source_maps: str
    image_maps: str
    first_index: str
    counts: str | None


_PLACEMENTS = {
    0: PlacementPlan(HOST, HOST, HOST, HOST),
    1: PlacementPlan(DEVICE, HOST, HOST, HOST),
    2: PlacementPlan(DEVICE, DEVICE, DEVICE, None),
    3: PlacementPlan(DEVICE, DEVICE, DEVICE, DEVICE),
}


def placement_for_level(level: int) -> PlacementPlan:
    """sm/construction.py:66-71."""
    try:
        return _PLACEMENTS[level]
    except KeyError:
        raise ValueError(f"optimization level must be in 0..3, got {level}") from None


def blocks_needed(n_entries: int, block_size: int) -> int:
    """sm/core.py:185-186."""
    return -(-int(n_entries) // int(block_size)) if n_entries > 0 else 0


class Arena:
    """sm/core.py:155-182: current / peak modeled bytes of one memory kind."""

    def __init__(self, kind: str):
        self.kind = kind
        self.current_bytes = 0
        self.peak_bytes = 0

    def alloc(self, n_bytes: int) -> None:
        if n_bytes < 0:
            raise ValueError(f"cannot allocate {n_bytes} bytes")
        self.current_bytes += int(n_bytes)
        self.peak_bytes = max(self.peak_bytes, self.current_bytes)

    def free(self, n_bytes: int) -> None:
        if n_bytes < 0:
            raise ValueError(f"cannot free {n_bytes} bytes")
        if n_bytes > self.current_bytes:
            raise ArenaUnderflowError(
                f"{self.kind} arena: freeing {n_bytes} bytes with only {self.current_bytes} allocated")
        self.current_bytes -= int(n_bytes)


class RankMemory:
    """The two arenas of one rank plus the block-granular capacities the
    reference tracks (store blocks, per-map and per-mirror capacity)."""

    def __init__(self, opt_level: int, block_size: int):
        self.plan = placement_for_level(opt_level)
        self.block = int(block_size)
        self.host = Arena(HOST)
        self.device = Arena(DEVICE)
        self.store_records = 0
        self.store_blocks = 0
        self.map_cap: dict[tuple, int] = {}
        self.mirror_cap: dict[int, int] = {}
        self._pending: list = []

    def later(self, method: str, *args) -> None:
        """Queue an allocation event whose counts may still be on the device
        (0-dim integer tensors); `resolve` replays the queue in order."""
        self._pending.append((method, args))

    def resolve(self) -> None:
        """Replay the queued events with one device->host transfer (tensor
        arguments become ints, or lists of ints when they hold several)."""
        if not self._pending:
            return
        import torch
        dev_vals = [a for _, args in self._pending for a in args if isinstance(a, torch.Tensor)]
        host = []
        if dev_vals:
            flat = torch.cat([v.reshape(-1).to(torch.int64).to(dev_vals[0].device) for v in dev_vals]).cpu().tolist()
            at = 0
            for v in dev_vals:
                k = v.numel()
                host.append(int(flat[at]) if v.dim() == 0 else [int(x) for x in flat[at: at + k]])
                at += k
        it = iter(host)
        pending, self._pending = self._pending, []
        for method, args in pending:
            getattr(self, method)(*[next(it) if isinstance(a, torch.Tensor) else a for a in args])

    def dist_batches(self, tr: int, group: int, present: list, owners: list, range_counts: list,
                     map_sizes: list) -> None:
        """One distributed call on its target rank: the reference appends one
        batch per source rank present, ascending; remote ones go through
        remote_connect (sm/construction.py:689-703, 597-617)."""
        per = {}
        for o, c in zip(owners, range_counts):
            per[o] = per.get(o, 0) + int(c)
        sizes = dict(zip([r for r in present if r != tr], map_sizes))
        for r in present:
            if r == tr:
                self.store_append(per.get(r, 0))
            else:
                self.remote_batch(per.get(r, 0), (int(group), r), sizes[r], per.get(r, 0))

    def arena(self, kind: str) -> Arena:
        return self.host if kind == HOST else self.device

    def neurons(self, n: int) -> None:
        """NeuronPool.add_neurons (sm/dynamics.py:141)."""
        self.device.alloc(n * NEURON_STATE_BYTES)

    def store_append(self, n: int) -> None:
        """ConnectionStore.append_batch (sm/core.py:286-291)."""
        self.store_records += int(n)
        need = blocks_needed(self.store_records, self.block)
        if need > self.store_blocks:
            self.device.alloc((need - self.store_blocks) * self.block * CONNECTION_RECORD_BYTES)
            self.store_blocks = need

    def map_size(self, key: tuple, n_entries: int) -> None:
        """RemoteSourceMap._ensure_capacity (sm/construction.py:205-211)."""
        need = blocks_needed(n_entries, self.block) * self.block
        have = self.map_cap.get(key, 0)
        if need > have:
            grown = need - have
            self.arena(self.plan.remote_source_maps).alloc(grown * MAP_ENTRY_BYTES)
            self.arena(self.plan.image_maps).alloc(grown * MAP_ENTRY_BYTES)
            self.map_cap[key] = need

    def mirror_size(self, tgt_rank: int, n_entries: int) -> None:
        """RankState.mirror_merge (sm/construction.py:302-306)."""
        need = blocks_needed(n_entries, self.block) * self.block
        have = self.mirror_cap.get(tgt_rank, 0)
        if need > have:
            self.device.alloc((need - have) * MAP_ENTRY_BYTES)
            self.mirror_cap[tgt_rank] = need

    def remote_batch(self, n_src: int, map_key: tuple | None, map_entries: int, n_records: int) -> None:
        """Target side of remote_connect (sm/construction.py:597-617): the
        transient image/flag scratch brackets the map growth and the append."""
        tmp = n_src * (TEMP_IMAGE_SLOT_BYTES + TEMP_FLAG_BYTES)
        self.device.alloc(tmp)
        if map_key is not None and map_entries:
            self.map_size(map_key, map_entries)
        self.store_append(n_records)
        self.device.free(tmp)

    def prepare(self, n_real: int, n_ports: int, buffer_length: int, n_nodes: int, roster_sizes: dict,
                own_rank: int, mirror_sizes: dict) -> None:
        """sm/construction.py:763-807 and NeuronPool.freeze (sm/dynamics.py:185-187)."""
        self.device.alloc(n_real * n_ports * buffer_length * BUFFER_SLOT_BYTES)
        self.arena(self.plan.first_index).alloc((n_nodes + 1) * FIRST_INDEX_ENTRY_BYTES)
        if self.plan.counts is not None:
            self.arena(self.plan.counts).alloc(n_nodes * COUNT_ENTRY_BYTES)
        for key in sorted(roster_sizes):
            self.arena(self.plan.remote_source_maps).alloc(roster_sizes[key] * MAP_ENTRY_BYTES)
        for key in sorted(roster_sizes):
            if key[1] != own_rank:
                self.arena(self.plan.image_maps).alloc(roster_sizes[key] * MAP_ENTRY_BYTES)
        self.device.alloc(sum(mirror_sizes.values()) * ROUTE_ENTRY_BYTES)
        self.device.alloc(sum(n for (g, sr), n in roster_sizes.items() if sr == own_rank) * ROUTE_ENTRY_BYTES)
