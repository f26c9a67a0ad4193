"""Ring-attention kernel study at the LWM-7B 32K shape (one 32768-token
stripe, 32 heads x 128): CUDA-event time of the production kernel and, with
ESP_ATTN_PROF=1, the per-role cycle accounting of the instrumented build."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402


def main():
    S = int(os.environ.get("S", "32768"))
    heads, hd = 32, 128
    H = heads * hd
    torch.manual_seed(0)
    q = torch.randn(S, H, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(S, H, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(S, H, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    flop = 2.0 * H * S * (S + 1)

    def run():
        abi.k_ring_attention(q.data_ptr(), S, 0, [k.data_ptr()], [v.data_ptr()], [S], [0],
                             out.data_ptr(), heads, hd)

    os.environ.pop("ESP_ATTN_PROF", None)
    for variant in ("v2", "v1"):
        if variant == "v1":
            os.environ["ESP_ATTN_V1"] = "1"
        else:
            os.environ.pop("ESP_ATTN_V1", None)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3  # includes the hook's staging copies
        print(f"{variant}: {ms:.3f} ms/launch (with staging), {flop / ms / 1e9:.0f} TFLOP/s")
    os.environ.pop("ESP_ATTN_V1", None)
    os.environ["ESP_ATTN_PROF"] = "1"
    run()
    torch.cuda.synchronize()
    sys.stderr.flush()


if __name__ == "__main__":
    main()
