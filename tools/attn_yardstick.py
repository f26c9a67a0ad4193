"""External yardstick for K1 (VERDICT r1 "next" #5): causal flash attention,
32 heads x 128, bf16, S = 32768 (one LWM-7B layer at ESP degree 1), timed
with CUDA events in ONE process so every contender sees the same (power-
capped) clock:

  * ours   — K1 inside a 1-layer LWM-7B-geometry prefill through the runtime
             (the ring_attention phase time, CUDA events around the launch);
  * cuDNN  — torch SDPA with the cuDNN backend (cuDNN 9 has sm_100 fused
             attention kernels);
  * flash  — torch SDPA's flash backend, and flashinfer's prefill when it
             imports (library kernels: a yardstick, not our product).

FLOP per call = 2 * H * S * (S + 1) (QK^T and PV over the causal half).
Prints one JSON object."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402

S = int(os.environ.get("S", "32768"))
HEADS, HD = 32, 128
H = HEADS * HD
FLOP = 2.0 * H * S * (S + 1)
REPS = 5


def time_fn(fn):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    res = {"S": S, "heads": HEADS, "head_dim": HD, "flop_per_call": FLOP}
    # ours: one-layer prefill, K1 phase time
    shape = abi.ModelShape(layers=1, hidden=H, heads=HEADS, head_dim=HD, ffn=11008, vocab=32000)
    rt = abi.Runtime(shape, 1, devices=[0], kv_capacity=S + 64)
    prompt = np.random.default_rng(0).integers(0, 32000, S).astype(np.int32)
    rt.prefill([0], [S], [0], [[(0, S)]], tokens=prompt)
    rt.free_request(0)
    ms = []
    for k in range(REPS):
        rt.phase_times()
        rt.set_profiling(True)
        rt.prefill([k + 1], [S], [0], [[(0, S)]], tokens=prompt)
        rt.set_profiling(False)
        ms.append(rt.phase_times()["ring_attention"][0])
        rt.free_request(k + 1)
    rt.close()
    t = statistics.median(ms)
    res["ours_k1"] = {"ms": t, "tflops": FLOP / t / 1e9}
    q = torch.randn(1, HEADS, S, HD, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    from torch.nn.attention import SDPBackend, sdpa_kernel
    for name, be in (("cudnn_sdpa", SDPBackend.CUDNN_ATTENTION),
                     ("flash_sdpa", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                t = time_fn(lambda: torch.nn.functional.scaled_dot_product_attention(
                    q, k, v, is_causal=True))
            res[name] = {"ms": t, "tflops": FLOP / t / 1e9}
        except Exception as e:  # report, never hide
            res[name] = {"error": str(e)[:200]}
    try:
        import flashinfer
        qi = q[0].transpose(0, 1).contiguous()
        ki = k[0].transpose(0, 1).contiguous()
        vi = v[0].transpose(0, 1).contiguous()
        t = time_fn(lambda: flashinfer.single_prefill_with_kv_cache(qi, ki, vi, causal=True))
        res["flashinfer"] = {"ms": t, "tflops": FLOP / t / 1e9}
    except Exception as e:  # report, never hide
        res["flashinfer"] = {"error": str(e)[:200]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
