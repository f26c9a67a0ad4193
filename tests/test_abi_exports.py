"""The C-ABI library loads without a GPU and exports every symbol
include/esp_abi.h declares."""
import os
import re

from paper_2404_09526_b200 import abi

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "esp_abi.h")


def test_header_symbols_exported():
    with open(HDR) as f:
        src = f.read()
    declared = set(re.findall(r"\b(esp_[a-z0-9_]+)\s*\(", src))
    declared -= {"esp_runtime"}
    assert declared == set(abi.EXPORTED_SYMBOLS), declared ^ set(abi.EXPORTED_SYMBOLS)
    h = abi.lib()
    for s in declared:
        assert getattr(h, s) is not None


def test_abi_version_and_errors():
    assert abi.lib().esp_abi_version() == 3
    try:
        abi.plan_prefill_scale_down([0], [5], [6])
    except abi.InfeasiblePlanError as e:
        assert "exceeds" in e.msg
    else:
        raise AssertionError("expected InfeasiblePlanError")


def test_device_runtime_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    try:
        abi.Runtime(abi.TINY, 1, devices=[0], kv_capacity=16)
    except abi.EspError as e:
        assert e.code in (abi.ESP_ERR_CUDA, abi.ESP_ERR_CONFIG)
    else:
        raise AssertionError("a device runtime must not silently run without a GPU")
