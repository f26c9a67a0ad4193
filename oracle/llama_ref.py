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
        i64p, f32p, i32p = C.POINTER(C.c_int64), C.POINTER(C.c_float), C.POINTER(C.c_int32)
        h.llama_ref_prefill_probe.restype = C.c_int32
        h.llama_ref_prefill_probe.argtypes = [C.POINTER(LlamaCfg), i32p, C.c_int64, C.c_int,
                                              C.c_int64, i64p, f32p, C.c_int64, i64p, f32p, f32p,
                                              C.c_int, f32p, C.c_int]
        h.llama_ref_decode_cached.restype = C.c_int32
        h.llama_ref_decode_cached.argtypes = [C.POINTER(LlamaCfg), C.c_int64,
                                              C.POINTER(C.c_uint16), C.POINTER(C.c_uint16),
                                              C.c_int32, C.c_int, f32p, f32p, f32p, f32p, C.c_int]
        h.llama_ref_decode_sample.restype = C.c_double
        h.llama_ref_decode_sample.argtypes = [C.POINTER(LlamaCfg), C.c_int64, C.c_int, C.c_int]
        h.llama_ref_max_threads.restype = C.c_int
        h.llama_ref_weights.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_float)]
        _lib = h
    return _lib


def _f32(a):
    return a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else None


def _i64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64)) if a is not None else None


def cfg_from(shape) -> LlamaCfg:
    return LlamaCfg(shape.layers, shape.hidden, shape.heads, shape.head_dim, shape.ffn,
                    shape.vocab, shape.rms_eps, shape.rope_theta, shape.weight_seed)


def weight(seed, tensor, layer, row, col, cols) -> float:
    return float(lib().llama_ref_weight(seed, tensor, layer, row, col, cols))


TENSORS = {"embed": 1, "q": 2, "k": 3, "v": 4, "o": 5, "gate": 6, "up": 7, "down": 8, "lm_head": 9}


def weights(shape, tensor, layer, rows, cols) -> np.ndarray:
    """The synthetic tensor `tensor` of `layer` as float32 [rows x cols]
    (bf16-valued: the device and the oracle both use the bf16 rounding)."""
    out = np.empty((rows, cols), np.float32)
    lib().llama_ref_weights(shape.weight_seed, TENSORS[tensor], layer, rows, cols, _f32(out))
    return out


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


def prefill_probe(shape, prompt, attn_pos=(), kv_pos=(), emulate_bf16=True, last_only=True,
                  threads=0):
    """Dense prefill of `prompt` with captures (llama_ref.c:llama_ref_prefill_probe).
    Returns (greedy token, logits[vocab], attn[layers, n_attn, hidden] or None,
    k[layers, n_kv, hidden] or None, v[...] or None)."""
    c = cfg_from(shape)
    p = np.ascontiguousarray(np.asarray(prompt, np.int32))
    ap = np.ascontiguousarray(np.asarray(sorted(attn_pos), np.int64))
    kp = np.ascontiguousarray(np.asarray(kv_pos, np.int64))
    L, H = shape.layers, shape.hidden
    att = np.zeros((L, len(ap), H), np.float32) if len(ap) else None
    kk = np.zeros((L, len(kp), H), np.float32) if len(kp) else None
    vv = np.zeros((L, len(kp), H), np.float32) if len(kp) else None
    lg = np.zeros(shape.vocab, np.float32)
    tok = lib().llama_ref_prefill_probe(
        C.byref(c), p.ctypes.data_as(C.POINTER(C.c_int32)), len(p), 1 if emulate_bf16 else 0,
        len(ap), _i64(ap) if len(ap) else None, _f32(att), len(kp), _i64(kp) if len(kp) else None,
        _f32(kk), _f32(vv), 1 if last_only else 0, _f32(lg), threads)
    return int(tok), lg, att, kk, vv


def decode_cached(shape, k_cache, v_cache, token, emulate_bf16=True, threads=0):
    """One decode step over a GIVEN bf16 KV cache (uint16 [layers, n_ctx, hidden],
    token order, after RoPE) at position n_ctx (llama_ref.c:llama_ref_decode_cached).
    Returns (greedy token, logits[vocab], k_new[layers, hidden], v_new, attn[layers, hidden])."""
    c = cfg_from(shape)
    kc = np.ascontiguousarray(k_cache, np.uint16)
    vc = np.ascontiguousarray(v_cache, np.uint16)
    L, n_ctx, H = kc.shape
    assert L == shape.layers and H == shape.hidden and vc.shape == kc.shape
    lg = np.zeros(shape.vocab, np.float32)
    kn = np.zeros((L, H), np.float32)
    vn = np.zeros((L, H), np.float32)
    att = np.zeros((L, H), np.float32)
    u16 = C.POINTER(C.c_uint16)
    tok = lib().llama_ref_decode_cached(C.byref(c), n_ctx, kc.ctypes.data_as(u16),
                                        vc.ctypes.data_as(u16), int(token),
                                        1 if emulate_bf16 else 0, _f32(lg), _f32(kn), _f32(vn),
                                        _f32(att), threads)
    return int(tok), lg, kn, vn, att


def decode_sample_ms(shape, n_ctx, batch, threads=0) -> float:
    """Wall ms of one fp32 decode step of `batch` requests over n_ctx-token
    caches (llama_ref.c:llama_ref_decode_sample), model setup excluded."""
    return float(lib().llama_ref_decode_sample(C.byref(cfg_from(shape)), n_ctx, batch, threads))
