"""Kernel microbenchmarks (CUDA events on the launching stream, warm-up,
inputs larger than L2): the tcgen05 GEMM at the LWM-7B prefill shapes, and
the cuBLAS bf16 GEMM on the same shapes for reference."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402


def time_fn(fn, iters=10, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    M = int(os.environ.get("M", "32768"))
    shapes = [("qkv", 12288, 4096), ("o", 4096, 4096), ("gate_up", 22016, 4096),
              ("down", 4096, 11008), ("decode_qkv_m16", 12288, 4096)]
    out = {}
    stream = torch.cuda.current_stream().cuda_stream
    for name, N, K in shapes:
        m = 16 if "m16" in name else M
        a = torch.randn(m, K, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        d = torch.empty(m, N, device="cuda", dtype=torch.bfloat16)
        ms = time_fn(lambda: abi.k_gemm(a.data_ptr(), b.data_ptr(), d.data_ptr(), m, N, K, 0, stream))
        ms_cb = time_fn(lambda: torch.matmul(a, b.t(), out=d))
        fl = 2.0 * m * N * K
        out[name] = {"M": m, "N": N, "K": K, "ours_ms": ms, "ours_tflops": fl / ms / 1e9,
                     "cublas_ms": ms_cb, "cublas_tflops": fl / ms_cb / 1e9,
                     "ours_GBps": (m * K + N * K + m * N) * 2 / ms / 1e6}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
