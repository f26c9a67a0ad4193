"""Placement-only runtime (no GPU): page tables and slot counters for plans
the reference accepts but the ring kernel could not run."""
import pytest

from paper_2404_09526_b200 import abi


def test_placement_only_accepts_rings_wider_than_the_kernel():
    """The reference's ring tests go to d = 16 (test_esp_mechanics.cpp:26-49);
    kMaxRounds (8) only limits the device kernel, not the page tables."""
    rt = abi.Runtime(abi.LWM_7B, 16, devices=None, kv_capacity=1000)
    ring = list(range(16))
    rt.prefill([4], [12000], ring, [[(15, 1000), (14, 1000)] + [(i, 1000) for i in range(10)]])
    pl = rt.placement(4)
    assert sum(pl.values()) == 12000 and len(pl) == 12
    rt.check_conservation()
    rt.free_request(4)
    assert rt.kv_used() == [0] * 16


def test_placement_query_beyond_64_instances():
    """A request spread over more than 64 instances reads back completely."""
    n = 80
    rt = abi.Runtime(abi.TINY, n, devices=None, kv_capacity=10)
    rt.prefill([1], [10 * n], [0], [[(i, 10) for i in range(n)]])
    assert rt.placement(1) == {i: 10 for i in range(n)}


def test_prefill_stats_follow_the_reference_mechanics():
    """The runtime accounts each prefill through its restatements of
    build_ring_schedule / proactive_scale_down (esp_mechanics.cpp:45-136):
    ring volume (d-1)*sum, transient buffer ceil(sum/d) (Fig. 6: 6 tokens on
    3 instances -> 2), zero extra migration for ring-member survivors."""
    rt = abi.Runtime(abi.TINY, 4, devices=None, kv_capacity=100)
    rt.prefill([1], [6], [0, 1, 2], [[(0, 4), (1, 2)]])
    st = rt.last_prefill_stats()
    assert st["ring_volume_tokens"] == 2 * 6
    assert st["transient_buffer_tokens"] == 2
    assert st["extra_migration_tokens"] == 0
    assert st["cross_domain_tokens"] == 0 and st["nvlink_bytes"] == 0  # no devices
    # a resting instance outside the ring (a disaggregation-style plan)
    rt.prefill([2], [7], [0, 1], [[(3, 7)]])
    st = rt.last_prefill_stats()
    assert st["ring_volume_tokens"] == 7 and st["extra_migration_tokens"] == -1


@pytest.mark.parametrize("tp,cap", [(3, 4096), (1, 4096), (16, 4096), (2, 0)])
def test_tp_runtime_rejects_bad_configs(tp, cap):
    """esp_runtime_create_tp validates before touching a device: tp must be
    2..8 and divide the heads with 128-multiple hidden shards, and the
    capacity must be given (ConfigError, no CUDA needed)."""
    with pytest.raises(abi.ConfigError):
        abi.Runtime(abi.TINY, 2, kv_capacity=cap, tp_planes=[0] * tp)
