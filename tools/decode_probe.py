"""Decode-step probe (config 4 scaled to one GPU: b requests x ctx tokens on
one instance): step time without per-phase events, then one profiled pass for
the phase split. Variants are picked by environment (ESP_DECODE_ATTN,
ESP_DECODE_STAGES, ESP_DECODE_CHUNK, ...), so run one process per variant."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402


def main():
    b = int(os.environ.get("B", "16"))
    ctx = int(os.environ.get("CTX", "8192"))
    steps = int(os.environ.get("STEPS", "10"))
    rt = abi.Runtime(abi.LWM_7B, 1, devices=[0], kv_capacity=b * (ctx + 3 * steps + 16))
    rng = np.random.default_rng(11)
    for r in range(b):
        rt.prefill([r], [ctx], [0], [[(0, ctx)]], tokens=rng.integers(0, 32000, ctx).astype(np.int32))
    for _ in range(3):
        rt.decode_step([0], [0], list(range(b)))
    ms = [rt.decode_step([0], [0], list(range(b)))[2] for _ in range(steps)]
    rt.phase_times()
    rt.set_profiling(True)
    for _ in range(steps):
        rt.decode_step([0], [0], list(range(b)))
    rt.set_profiling(False)
    ph = rt.phase_times()
    L, H = 32, 4096
    kv = 2.0 * L * H * 2 * b * (ctx + 3 + steps + steps // 2)
    att_ms, att_n = ph["decode_attention"]
    tag = {k: v for k, v in os.environ.items() if k.startswith("ESP_")}
    print(json.dumps({"env": tag, "b": b, "ctx": ctx, "step_ms": float(np.median(ms)),
                      "tok_s": b / (float(np.median(ms)) / 1e3),
                      "attn_gbs": (kv / L) / (att_ms / att_n / 1e3) / 1e9,
                      "phase_ms": {p: round(v[0] / steps, 4) for p, v in ph.items() if v[1]}}))


if __name__ == "__main__":
    main()
