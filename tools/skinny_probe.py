"""Decode-shaped (M = 16) GEMM study: CUDA-event time per call of the four
LWM-7B projections (store / residual / SiLU epilogues) under several
schedules of the skinny tcgen05 kernel, weight bytes / time, and cuBLAS on the
same shape. Modes (env of the k_gemm call):
  old_*    the M = 128 skinny kernel (ESP_GEMM_SKINNY_OLD); default: swap-AB
  tiles    whole 128-column tiles per CTA (ESP_GEMM_NO_STREAMK)
  streamk  equal (tile, K-block) ranges per SM (ESP_GEMM_STREAMK_ALL)
  auto     the production dispatch (cluster split-K over DSMEM for <= 37 tiles)
  *_first / *_nohint   weight loads with L2 evict_first / no hint
  *_tiled  weights pre-tiled [N/128][K/64][128][64] (16 KB contiguous per load)
SHAPES=qkv,o selects shapes; MODES=tiles,streamk_tiled selects modes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402

SHAPES = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 1), "gate_up": (22016, 4096, 3),
          "down": (4096, 11008, 1), "lm_head": (32000, 4096, 2)}
ALL_MODES = ["tiles", "streamk", "auto", "split2"]


def set_mode(mode):
    for k in ("ESP_GEMM_NO_STREAMK", "ESP_GEMM_STREAMK_ALL", "ESP_GEMM_B_MODE", "ESP_GEMM_SKINNY_OLD",
              "ESP_GEMM_SPLIT2_ALL"):
        os.environ.pop(k, None)
    if mode.startswith("old_"):
        os.environ["ESP_GEMM_SKINNY_OLD"] = "1"
        mode = mode[4:]
    if mode.startswith("tiles"):
        os.environ["ESP_GEMM_NO_STREAMK"] = "1"
    elif mode.startswith("streamk"):
        os.environ["ESP_GEMM_STREAMK_ALL"] = "1"
    elif mode == "split2":
        os.environ["ESP_GEMM_SPLIT2_ALL"] = "1"
    bm = (1 if "tiled" in mode else 0) | (2 if "first" in mode else 0) | (4 if "nohint" in mode else 0)
    os.environ["ESP_GEMM_B_MODE"] = str(bm)


def tiled(b):
    N, K = b.shape
    return b.view(N // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous()


def time_calls(fn, n=64):
    for i in range(8):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    M = int(os.environ.get("M", "16"))
    only = os.environ.get("SHAPES")
    for spec in filter(None, os.environ.get("EXTRA", "").split(",")):
        nm, n_, k_, e_ = spec.split(":")  # e.g. EXTRA=o_k256:4096:256:1
        SHAPES[nm] = (int(n_), int(k_), int(e_))
    modes = os.environ.get("MODES", ",".join(ALL_MODES)).split(",")
    torch.manual_seed(0)
    for name, (N, K, epi) in SHAPES.items():
        if only and name not in only.split(","):
            continue
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        # 8 weight copies rotated so every call streams from HBM, not L2
        bs = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(8)]
        bts = [tiled(b) for b in bs] if any("tiled" in m for m in modes) else None
        ncols = N // 2 if epi == 3 else N
        odt = torch.float32 if epi == 2 else torch.bfloat16
        res, outs = {}, {}
        for mode in modes:
            set_mode(mode)
            src = bts if "tiled" in mode else bs
            d = torch.zeros(M, ncols, device="cuda", dtype=odt)
            res[mode] = time_calls(
                lambda i: abi.k_gemm(a.data_ptr(), src[i % 8].data_ptr(), d.data_ptr(), M, N, K, epi))
            d.zero_()
            abi.k_gemm(a.data_ptr(), src[0].data_ptr(), d.data_ptr(), M, N, K, epi)
            torch.cuda.synchronize()
            outs[mode] = d.float().clone()
        for k in ("ESP_GEMM_NO_STREAMK", "ESP_GEMM_STREAMK_ALL", "ESP_GEMM_B_MODE",
                  "ESP_GEMM_SKINNY_OLD", "ESP_GEMM_SPLIT2_ALL"):
            os.environ.pop(k, None)
        dc = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        res["cublas"] = time_calls(lambda i: torch.matmul(a, bs[i % 8].t(), out=dc))
        gb = N * K * 2 / 1e9
        ref = outs[modes[0]]
        line = " ".join(f"{m}={res[m]:.1f}us/{gb / res[m] * 1e6:.0f}GB/s" for m in res)
        bad = [m for m in outs if not torch.allclose(outs[m], ref, rtol=2e-2, atol=2e-2)]
        print(f"{name:8s} N={N:6d} K={K:6d}: {line}" + (f"  MISMATCH {bad}" if bad else ""),
              flush=True)


if __name__ == "__main__":
    main()
