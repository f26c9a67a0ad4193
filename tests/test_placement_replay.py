"""Boundary parity on CPU: the runtime's page tables (placement-only runtime,
no device) track the UNMODIFIED reference engine's KV placement bit-exactly
through every recorded scenario (configs 1-5 of BASELINE.json)."""
import glob
import os

import pytest

from paper_2404_09526_b200 import abi
from tests import replay

SCEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "scenario_*.jsonl")))


@pytest.mark.parametrize("path", SCEN, ids=[os.path.basename(p)[9:-6] for p in SCEN])
def test_replay_page_tables(path):
    head, steps, final = replay.load(path)
    rt = abi.Runtime(abi.TINY, head["instances"], devices=None, kv_capacity=head["kv_capacity"])
    if head.get("prebuilt"):
        # config 4: the engine state was hand-built (test_scheduler.cpp:71-99 style)
        for r in head["requests"]:
            rt.prefill([r["id"]], [r["input_len"]], [i for i, _ in r["placement"]],
                       [[tuple(x) for x in r["placement"]]])
    replay.replay(rt, path)
    rt.check_conservation()


def test_config_goldens_match_survey():
    """The recorded reference decisions are the ones SURVEY.md §A-3 lists."""
    d = os.path.join(os.path.dirname(__file__), "golden")
    _, steps, final = replay.load(os.path.join(d, "scenario_config1_tiny.jsonl"))
    p = steps[0]["decision"]["prefills"][0]
    assert p["instances"] == [0, 1] and p["decode_instances"] == [0]
    assert p["ring_volume"] == 4096
    dec = [s for s in steps if s["decision"]["decode_steps"]]
    assert len(dec) == 64
    _, steps, _ = replay.load(os.path.join(d, "scenario_config3_128k.jsonl"))
    p = steps[0]["decision"]["prefills"][0]
    assert p["dop"] == 8 and p["decode_instances"] == [0, 1]
    assert p["placement"]["0"] == [[0, 65600], [1, 65472]]
    assert p["ring_volume"] == 917504
    _, steps, final = replay.load(os.path.join(d, "scenario_config4_decode.jsonl"))
    ds = [s["decision"]["decode_steps"][0] for s in steps]
    assert ds[0]["masters"] == [0, 1] and ds[1]["masters"] == [2, 3]
    assert ds[2]["add_instances"] == [4] and ds[2]["masters"] == [4]
    for dd in (1, 2, 4, 8):
        _, steps, _ = replay.load(os.path.join(d, f"scenario_config2_32k_d{dd}.jsonl"))
        p = steps[0]["decision"]["prefills"][0]
        assert p["dop"] == dd and p["input_lens"] == [32768]


def test_capacity_and_master_full_errors():
    rt = abi.Runtime(abi.TINY, 2, devices=None, kv_capacity=100)
    with pytest.raises(abi.CapacityError):
        rt.prefill([0], [150], [0, 1], [[(0, 150)]])
    assert rt.kv_used() == [0, 0]  # atomic: nothing allocated
    rt.prefill([0], [150], [0, 1], [[(0, 100), (1, 50)]])
    assert rt.placement(0) == {0: 100, 1: 50}
    with pytest.raises(abi.MasterFullError):
        rt.decode_step([0, 1], [0], [0])
    rt.decode_step([0, 1], [1], [0])
    assert rt.placement(0) == {0: 100, 1: 51}
    rt.move_kv(0, 1, 0, 0)
    with pytest.raises(abi.InternalError):
        rt.move_kv(0, 1, 0, 52)
    rt.free_request(0)
    assert rt.kv_used() == [0, 0]
    with pytest.raises(abi.InternalError):
        rt.prefill([1], [10], [0], [[(0, 9)]])  # placement does not cover input
    with pytest.raises(abi.NoDeviceError):
        pass
        raise abi.NoDeviceError(abi.ESP_ERR_NO_DEVICE, "placement-only")
