"""Ring-attention kernel study at the LWM-7B 32K shape (one 32768-token
stripe, 32 heads x 128): wall time of REPEAT calls of the K1 test hook (each
stages its buffers, so this is an upper bound; bench.py times K1 in the step
with CUDA events) with the SM clock sampled meanwhile, then — in a kernel-
study build (`make -C paper_2404_09526_b200/csrc STUDY=1`) — the per-role
cycle accounting of the instrumented kernel (ESP_ATTN_PROF=1)."""
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402


def sample_clocks(stop, out):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            out.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.02)
    except Exception as e:  # noqa: BLE001
        print(f"clock sampling unavailable: {e}", file=sys.stderr)


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
    run()
    torch.cuda.synchronize()
    n = int(os.environ.get("REPEAT", "10"))
    clocks, stop = [], threading.Event()
    th = threading.Thread(target=sample_clocks, args=(stop, clocks))
    th.start()
    t0 = time.time()
    for _ in range(n):
        run()
    torch.cuda.synchronize()
    wall = time.time() - t0
    stop.set()
    th.join()
    sys.stderr.flush()
    mhz = statistics.median(clocks) if clocks else float("nan")
    print(f"flop/launch {flop:.4e}; wall {wall:.2f}s for {n} launches; "
          f"SM clock median {mhz:.0f} MHz over {len(clocks)} samples", flush=True)
    os.environ["ESP_ATTN_PROF"] = "1"
    run()
    torch.cuda.synchronize()
    sys.stderr.flush()


if __name__ == "__main__":
    main()
