"""ctypes wrapper of the CPU numeric oracle (oracle/llama_ref.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_build", "libllama_ref.so")


class LlamaCfg(C.Structure):
    _fields_ = [
        ("layers", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32),
        ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
        ("rms_eps", C.c_float), ("rope_theta", C.c_float), ("weight_seed", C.c_uint64),
    ]


_lib = None


def build() -> None:
    subprocess.run(["make", "-C", _HERE, "numeric"], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = C.CDLL(LIB)
        h.llama_ref_weight.restype = C.c_float
        h.llama_ref_weight.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                       C.c_int64]
        h.llama_ref_generate.argtypes = [C.POINTER(LlamaCfg), C.POINTER(C.c_int32), C.c_int64,
                                         C.c_int, C.POINTER(C.c_int32), C.c_int,
                                         C.POINTER(C.c_int32), C.POINTER(C.c_float), C.c_int]
        _lib = h
    return _lib


def cfg_from(shape) -> LlamaCfg:
    return LlamaCfg(shape.layers, shape.hidden, shape.heads, shape.head_dim, shape.ffn,
                    shape.vocab, shape.rms_eps, shape.rope_theta, shape.weight_seed)


def weight(seed, tensor, layer, row, col, cols) -> float:
    return float(lib().llama_ref_weight(seed, tensor, layer, row, col, cols))


def generate(shape, prompt, n_steps, forced=None, emulate_bf16=True, want_logits=True,
             threads=0):
    """Dense causal forward of `prompt` + n_steps KV-cached decode steps.
    Returns (tokens[n_steps+1], logits[(n_steps+1) x vocab] or None)."""
    c = cfg_from(shape)
    p = np.ascontiguousarray(np.asarray(prompt, np.int32))
    out = np.zeros(n_steps + 1, np.int32)
    lg = np.zeros((n_steps + 1, shape.vocab), np.float32) if want_logits else None
    f = None
    if forced is not None:
        fa = np.ascontiguousarray(np.asarray(forced, np.int32))
        f = fa.ctypes.data_as(C.POINTER(C.c_int32))
    lib().llama_ref_generate(
        C.byref(c), p.ctypes.data_as(C.POINTER(C.c_int32)), len(p), n_steps, f,
        1 if emulate_bf16 else 0, out.ctypes.data_as(C.POINTER(C.c_int32)),
        lg.ctypes.data_as(C.POINTER(C.c_float)) if lg is not None else None, threads)
    return out, lg
