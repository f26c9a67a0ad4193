"""Decode weight-streaming probe: LWM-7B, b x short-context decode steps on one
GPU through the C-ABI. Prints device ms per step (median), host enqueue ms per
step (phase 11), weights streamed per step and the achieved GB/s, then one
profiled pass (per-phase events) for the phase split.

usage: python tools/decode_ws.py [--batch 16] [--ctx 64] [--steps 20]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    s = abi.LWM_7B
    b, ctx = args.batch, args.ctx
    rt = abi.Runtime(s, 1, devices=[0], kv_capacity=b * (ctx + 2 * args.steps + 16))
    rng = np.random.default_rng(3)
    for r in range(b):
        rt.prefill([r], [ctx], [0], [[(0, ctx)]], tokens=rng.integers(0, s.vocab, ctx).astype(np.int32))
    batch = list(range(b))
    for _ in range(3):
        rt.decode_step([0], [0], batch)
    rt.phase_times()
    ms = [rt.decode_step([0], [0], batch)[2] for _ in range(args.steps)]
    host = rt.phase_times()["host_enqueue"]
    rt.set_profiling(True)
    for _ in range(3):
        rt.decode_step([0], [0], batch)
    rt.set_profiling(False)
    ph = rt.phase_times()
    rt.close()
    H, F, L, V = s.hidden, s.ffn, s.layers, s.vocab
    w_bytes = 2.0 * (L * (4 * H * H + 3 * H * F) + V * H)  # projections + LM head (embed: b rows)
    step = statistics.median(ms)
    out = {"batch": b, "ctx": ctx, "device_ms_median": step, "device_ms_min": min(ms),
           "host_enqueue_ms": host[0] / max(host[1], 1), "weight_bytes": w_bytes,
           "achieved_gbs": w_bytes / (step / 1e3) / 1e9,
           "phase_ms_per_step": {k: round(v[0] / 3, 4) for k, v in ph.items() if v[1] > 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
