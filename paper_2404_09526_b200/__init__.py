"""B200-native ESP (elastic sequence parallelism) data path, LoongServe
arXiv:2404.09526: striped ring prefill with proactive scale-down and
multi-master split-KV decoding on sm_100a, behind the C-ABI in
include/esp_abi.h. See DESIGN.md."""
from .abi import (LWM_7B, TINY, ModelShape, Runtime, launch_count, lib)  # noqa: F401

__all__ = ["Runtime", "ModelShape", "TINY", "LWM_7B", "lib", "launch_count"]
