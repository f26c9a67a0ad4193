"""External yardstick for K1 (VERDICT r1 "next" #5): causal flash attention,
32 heads x 128, bf16, S = 32768 (one LWM-7B layer at ESP degree 1), each
contender launched back to back and timed with CUDA events, the SM clock
sampled (nvidia-smi) while it runs:

  * ours        — K1 through esp_k_ring_attention_timed (staged once, then
                  REPS launches);
  * ours_in_step — K1 inside a 1-layer LWM-7B-geometry prefill (the
                  ring_attention phase; the GEMMs around it share the power
                  budget, as in the bench);
  * cudnn_sdpa  — torch SDPA, cuDNN backend (cuDNN 9's sm_100 fused attention);
  * flash_sdpa / flashinfer — library kernels (yardsticks, not the product).

FLOP per call = 2 * H * S * (S + 1). With POLY_SWEEP=1 it re-runs "ours" in
child processes under a kernel-study build (ESP_LIB, ESP_ATTN_POLY = eighths
of the softmax exponentials computed on the FMA pipe). Prints one JSON object."""
import json
import os
import statistics
import subprocess
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_09526_b200 import abi  # noqa: E402

S = int(os.environ.get("S", "32768"))
HEADS, HD = 32, 128
H = HEADS * HD
FLOP = 2.0 * H * S * (S + 1)
REPS = int(os.environ.get("REPS", "10"))


class Clocks:
    def __enter__(self):
        self.v, self.stop = [], threading.Event()

        def run():
            try:
                import pynvml
                pynvml.nvmlInit()
                h = pynvml.nvmlDeviceGetHandleByIndex(0)
                while not self.stop.is_set():
                    self.v.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    self.stop.wait(0.02)
            except Exception:  # noqa: BLE001
                pass
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join()

    def median(self):
        return statistics.median(self.v) if self.v else None


def time_fn(fn):
    fn()
    torch.cuda.synchronize()
    with Clocks() as c:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(REPS):
            fn()
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / REPS, c.median()


def ours_standalone():
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(S, H, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(S, H, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(S, H, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty_like(q)
    args = (q.data_ptr(), S, 0, [k.data_ptr()], [v.data_ptr()], [S], [0], out.data_ptr(),
            HEADS, HD)
    abi.k_ring_attention_timed(*args, 1)
    with Clocks() as c:
        ms = abi.k_ring_attention_timed(*args, REPS)
    return {"ms": ms, "tflops": FLOP / ms / 1e9, "sm_mhz": c.median()}


def main():
    if os.environ.get("ONLY_OURS"):
        print(json.dumps(ours_standalone()), flush=True)
        return
    res = {"S": S, "heads": HEADS, "head_dim": HD, "flop_per_call": FLOP, "reps": REPS}
    res["ours"] = ours_standalone()
    # in the step: one-layer prefill, K1 phase time
    shape = abi.ModelShape(layers=1, hidden=H, heads=HEADS, head_dim=HD, ffn=11008, vocab=32000)
    rt = abi.Runtime(shape, 1, devices=[0], kv_capacity=S + 64)
    prompt = np.random.default_rng(0).integers(0, 32000, S).astype(np.int32)
    rt.prefill([0], [S], [0], [[(0, S)]], tokens=prompt)
    rt.free_request(0)
    ms = []
    with Clocks() as c:
        for k in range(5):
            rt.phase_times()
            rt.set_profiling(True)
            rt.prefill([k + 1], [S], [0], [[(0, S)]], tokens=prompt)
            rt.set_profiling(False)
            ms.append(rt.phase_times()["ring_attention"][0])
            rt.free_request(k + 1)
    rt.close()
    t = statistics.median(ms)
    res["ours_in_step"] = {"ms": t, "tflops": FLOP / t / 1e9, "sm_mhz": c.median()}
    q = torch.randn(1, HEADS, S, HD, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    from torch.nn.attention import SDPBackend, sdpa_kernel
    for name, be in (("cudnn_sdpa", SDPBackend.CUDNN_ATTENTION),
                     ("flash_sdpa", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                t, mhz = time_fn(lambda: torch.nn.functional.scaled_dot_product_attention(
                    q, k, v, is_causal=True))
            res[name] = {"ms": t, "tflops": FLOP / t / 1e9, "sm_mhz": mhz}
        except Exception as e:  # report, never hide
            res[name] = {"error": str(e)[:200]}
    try:
        import flashinfer
        qi = q[0].transpose(0, 1).contiguous()
        ki = k[0].transpose(0, 1).contiguous()
        vi = v[0].transpose(0, 1).contiguous()
        t, mhz = time_fn(lambda: flashinfer.single_prefill_with_kv_cache(qi, ki, vi, causal=True))
        res["flashinfer"] = {"ms": t, "tflops": FLOP / t / 1e9, "sm_mhz": mhz}
    except Exception as e:  # report, never hide
        res["flashinfer"] = {"error": str(e)[:200]}
    if os.environ.get("POLY_SWEEP"):
        study = os.path.join(ROOT, "paper_2404_09526_b200", "libesp_b200_study.so")
        sweep = {}
        for poly in (0, 1, 2, 3, 4):
            env = dict(os.environ, ESP_LIB=study, ESP_ATTN_POLY=str(poly), ONLY_OURS="1")
            env.pop("POLY_SWEEP", None)
            p = subprocess.run([sys.executable, os.path.abspath(__file__)], capture_output=True,
                               text=True, env=env, timeout=600)
            lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
            sweep[str(poly)] = json.loads(lines[-1]) if lines else {"error": p.stderr[-300:]}
        res["ours_poly_sweep"] = sweep
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
