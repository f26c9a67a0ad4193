"""Decode-shaped (M = 16) GEMM study: CUDA-event time per call of the four
LWM-7B projections (store / residual / SiLU epilogues) with the stream-K path
and with the plain tile path (ESP_GEMM_NO_STREAMK), weight bytes / time."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402

SHAPES = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 1), "gate_up": (22016, 4096, 3),
          "down": (4096, 11008, 1), "lm_head": (32000, 4096, 2)}


def main():
    M = int(os.environ.get("M", "16"))
    torch.manual_seed(0)
    for name, (N, K, epi) in SHAPES.items():
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        # 8 weight copies rotated so every call streams from HBM, not L2
        bs = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(8)]
        ncols = N // 2 if epi == 3 else N
        d = torch.zeros(M, ncols, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
        res = {}
        for mode in ("streamk", "tiles"):  # streamk forced for every shape (ESP_GEMM_STREAMK_ALL)
            if mode == "tiles":
                os.environ["ESP_GEMM_NO_STREAMK"] = "1"
            else:
                os.environ.pop("ESP_GEMM_NO_STREAMK", None)
                os.environ["ESP_GEMM_STREAMK_ALL"] = "1"
            for i in range(8):
                abi.k_gemm(a.data_ptr(), bs[i].data_ptr(), d.data_ptr(), M, N, K, epi)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 64
            e0.record()
            for i in range(n):
                abi.k_gemm(a.data_ptr(), bs[i % 8].data_ptr(), d.data_ptr(), M, N, K, epi)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / n * 1e3
            res[mode] = us
        os.environ.pop("ESP_GEMM_NO_STREAMK", None)
        os.environ.pop("ESP_GEMM_STREAMK_ALL", None)
        gb = N * K * 2 / 1e9
        print(f"{name:8s} N={N:6d} K={K:6d}: stream-K {res['streamk']:7.1f} us "
              f"({gb / res['streamk'] * 1e6:6.0f} GB/s)   tiles {res['tiles']:7.1f} us "
              f"({gb / res['tiles'] * 1e6:6.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
