"""B200-calibrated scaling information base for the LWM-7B
shape: measures prefill and decode sweeps at ESP degrees 1-8 on one GPU
(the d instances co-located, so the curve is the one-GPU curve; on an 8-GPU
box pass --devices to place instance i on GPU i), fits them with
paper_2404_09526_b200.sib.calibrate, and writes the SIB in the reference's
JSONL format plus a fit report.

usage: python tools/calibrate_sib.py [--shape 7b|tiny] [--out FILE] [--report FILE]
                                     [--devices 0,0,0,0,0,0,0,0]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_09526_b200 import abi, sib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="7b", choices=["7b", "tiny"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sib_b200.jsonl"))
    ap.add_argument("--report", default=os.path.join(ROOT, "gpurun_out", "sib_b200_report.json"))
    ap.add_argument("--base", default=os.path.join(ROOT, "oracle", "_ref", "default_sib.jsonl"))
    ap.add_argument("--devices", default="0,0,0,0,0,0,0,0")
    a = ap.parse_args()
    devices = [int(x) for x in a.devices.split(",")]
    if a.shape == "7b":
        shape = abi.LWM_7B
        lengths = [[2048], [8192], [16384], [4096, 4096, 8192], [32768]]
        # at most 64K resident tokens per batch: slabs keep their high-water
        # backing, and instance i of degree d holds 1/d of it (sum over d <= 8
        # of 1/d = 2.7 x 34 GB)
        dcfgs = [(1, 16384, 1), (4, 8192, 1), (16, 2048, 1), (16, 4096, 2), (8, 8192, 2)]
        cap = 70000
    else:
        shape = abi.TINY
        lengths = [[256], [1024], [2048], [512, 1536], [4096], [3000, 3000]]
        dcfgs = [(1, 512, 1), (4, 1024, 1), (8, 2048, 2), (16, 1024, 2), (16, 256, 1)]
        cap = 40000
    t0 = time.time()
    rt = abi.Runtime(shape, len(devices), devices=devices, kv_capacity=cap)
    pre, dec = sib.measure(rt, lengths, dcfgs, degrees=range(1, len(devices) + 1),
                           repeats=2)
    rt.close()
    recs, report = sib.calibrate(sib.load_sib(a.base), pre, dec)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    sib.write_sib(recs, a.out)
    doc = {"shape": a.shape, "devices": devices, "prefill_lengths": lengths,
           "decode_cfgs (batch, ctx, masters)": dcfgs, "wall_s": round(time.time() - t0, 1),
           "fit": report,
           "prefill_samples": pre,
           "decode_samples": {k: v.tolist() for k, v in dec.items()}}
    with open(a.report, "w") as f:
        json.dump(doc, f, indent=1)
    for r in recs:
        print(json.dumps({k: r[k] for k in sib.SIB_KEYS}))
    print(f"wrote {a.out} and {a.report} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
