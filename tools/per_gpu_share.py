"""Per-GPU share of an ESP prefill at degree d, measured on ONE B200: what
each of d GPUs computes for config 2 (LWM-7B, S = 32768) is the dense
layers on S/d stripe rows and K1 for one ring position against all d KV
blocks. Both are timed here with the production kernels (CUDA events,
back-to-back launches, inputs larger than L2):

  * the four prefill GEMMs (QKV, O, gate_up, down) at M = S/d rows;
  * K1 for ring position d-1 (every position does the same work up to one
    diagonal row) over d blocks of S/d keys.

per-GPU layer time = GEMMs + K1; the compute-side strong-scaling
efficiency at degree d = t_layer(1) / (d * t_layer(d)) (the NVLink ring is
overlapped with K1 by the arrival counters and is not part of this number).
Prints one JSON object.

usage: python tools/per_gpu_share.py [--degrees 1,2,4,8] [--seq 32768]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402

H, F, HEADS, HD = 4096, 11008, 32, 128
GEMMS = [("qkv", 3 * H, H), ("o", H, H), ("gate_up", 2 * F, H), ("down", H, F)]


def time_fn(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def measure(degrees=(1, 2, 4, 8), S=32768):
    stream = torch.cuda.current_stream().cuda_stream
    out = {"seq": S}
    base = None
    for d in degrees:
        M = S // d
        row = {"rows_per_gpu": M, "gemm_ms": {}}
        gemm_ms, gemm_fl = 0.0, 0.0
        for name, N, K in GEMMS:
            a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
            b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ms = time_fn(lambda: abi.k_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0,
                                            stream))
            row["gemm_ms"][name] = round(ms, 4)
            gemm_ms += ms
            gemm_fl += 2.0 * M * N * K
            del a, b, c
        # K1: ring position d-1 against d blocks of the striped sequence
        pos = d - 1
        lens = [len(range(o, S, d)) for o in range(d)]
        origins = [(pos - r) % d for r in range(d)]
        blocks = [(torch.randn(lens[o], H, device="cuda", dtype=torch.bfloat16),
                   torch.randn(lens[o], H, device="cuda", dtype=torch.bfloat16)) for o in range(d)]
        q = torch.randn(lens[pos], H, device="cuda", dtype=torch.bfloat16)
        o_ = torch.empty_like(q)
        k1 = abi.k_ring_attention_timed(q.data_ptr(), lens[pos], pos,
                                        [blocks[o][0].data_ptr() for o in origins],
                                        [blocks[o][1].data_ptr() for o in origins],
                                        [lens[o] for o in origins], origins, o_.data_ptr(), HEADS,
                                        HD, 10, stream)
        del blocks, q, o_
        torch.cuda.empty_cache()
        k1_fl = 2.0 * H * S * (S + 1) / d
        layer = gemm_ms + k1
        row.update({"gemm_ms_total": round(gemm_ms, 4), "gemm_tflops": gemm_fl / gemm_ms / 1e9,
                    "k1_ms": round(k1, 4), "k1_tflops": k1_fl / k1 / 1e9,
                    "layer_ms_per_gpu": round(layer, 4)})
        if base is None:
            base = layer * d
        row["compute_scaling_efficiency"] = base / (d * layer)
        out[str(d)] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--degrees", default="1,2,4,8")
    ap.add_argument("--seq", type=int, default=32768)
    args = ap.parse_args()
    print(json.dumps(measure([int(x) for x in args.degrees.split(",")], args.seq)))


if __name__ == "__main__":
    main()
