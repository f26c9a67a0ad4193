"""Decode (M = 16) GEMM probe: the LWM-7B projection shapes streamed from HBM
(8 rotating weight copies, more than L2), 64 back-to-back calls per path,
CUDA events; achieved GB/s of weights. Paths: auto (production dispatch),
tiles (whole 128-column tiles), streamk (stream-K over (tile, K block)).
With ESP_LIB = the kernel-study build and ESP_GEMM_TRACE=<file>, one more
call per (shape, path) appends per-CTA globaltimer stamps to <file>.

usage: python tools/skinny_bench.py [--shapes qkv,o,gate_up,down,lm_head]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402

SHAPES = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 1), "gate_up": (22016, 4096, 3),
          "down": (4096, 11008, 1), "lm_head": (32000, 4096, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="qkv,o,gate_up,down,lm_head")
    ap.add_argument("--paths", default="auto,tiles,streamk")
    ap.add_argument("--calls", type=int, default=64)
    args = ap.parse_args()
    M = 16
    stream = torch.cuda.current_stream().cuda_stream
    out = {}
    for name in args.shapes.split(","):
        N, K, epi = SHAPES[name]
        copies = 8
        ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        dt = torch.float32 if epi == 2 else torch.bfloat16
        d = torch.zeros(M, N // 2 if epi == 3 else N, device="cuda", dtype=dt)
        row = {}
        for path in args.paths.split(","):
            def call(i):
                abi.k_gemm(a.data_ptr(), ws[i % copies].data_ptr(), d.data_ptr(), M, N, K, epi,
                           stream, path)
            for i in range(8):
                call(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(args.calls):
                call(i)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / args.calls * 1e3
            row[path] = {"us": round(us, 2), "GBps": round(N * K * 2 / us / 1e3, 1)}
        out[name] = row
        del ws
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
