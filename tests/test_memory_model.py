"""CPU checks of the modeled-byte arena restatement (paper_2512_09502_b200/memory.py)."""
import pytest

from paper_2512_09502_b200 import api, memory


def test_placement_plans():
    # sm/construction.py:59-64
    assert memory.placement_for_level(0) == memory.PlacementPlan("host", "host", "host", "host")
    assert memory.placement_for_level(1) == memory.PlacementPlan("device", "host", "host", "host")
    assert memory.placement_for_level(2) == memory.PlacementPlan("device", "device", "device", None)
    assert memory.placement_for_level(3) == memory.PlacementPlan("device", "device", "device", "device")
    with pytest.raises(ValueError):
        memory.placement_for_level(4)


def test_arena_peak_and_underflow():
    a = memory.Arena("device")
    a.alloc(100)
    a.alloc(50)
    a.free(120)
    a.alloc(10)
    assert (a.current_bytes, a.peak_bytes) == (40, 150)
    with pytest.raises(api.ArenaUnderflowError):
        a.free(41)
    with pytest.raises(ValueError):
        a.alloc(-1)


def test_block_granular_growth():
    m = memory.RankMemory(opt_level=2, block_size=1024)
    m.store_append(1)          # one block of 1024 records x 16 B
    m.store_append(1023)       # still one block
    assert m.device.current_bytes == 1024 * 16
    m.store_append(1)          # second block
    assert m.device.current_bytes == 2 * 1024 * 16
    m.map_size((0, 1), 5)      # remote + image columns, device at level 2
    assert m.device.current_bytes == 2 * 1024 * 16 + 2 * 1024 * 4
    m.remote_batch(1000, (0, 1), 5, 0)  # transient scratch is freed again
    assert m.device.peak_bytes == 2 * 1024 * 16 + 2 * 1024 * 4 + 1000 * 5
    assert m.device.current_bytes == 2 * 1024 * 16 + 2 * 1024 * 4
