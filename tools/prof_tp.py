"""One tensor-parallel 16K-token LWM-7B prefill at ESP 2 on tp = 2 planes
(co-located on one GPU) for an ncu capture of the TP kernels: the reduce-
scatter half (tp_reduce_norm_kernel) and the routed O / down GEMMs.
usage: ncu ... python tools/prof_tp.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09526_b200 import abi  # noqa: E402

S = 16384
prompt = np.random.default_rng(17).integers(0, abi.LWM_7B.vocab, S).astype(np.int32)
rt = abi.Runtime(abi.LWM_7B, 2, kv_capacity=S + 64, tp_planes=[0, 0])
for k in range(2):
    _, _, t = rt.prefill([k], [S], [0, 1], [[(0, S)]], tokens=prompt)
    rt.free_request(k)
    print(f"prefill {k}: {t:.1f} ms")
rt.close()
