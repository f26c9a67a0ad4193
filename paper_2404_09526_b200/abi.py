"""ctypes binding of the C-ABI in include/esp_abi.h (libesp_b200.so).

This is the Python side of the drop-in boundary: the same entry points a cgo /
pybind / C++ caller binds. The library must be built
(`python -c "import __graft_entry__ as g; g.build()"`); importing this module
without it raises — there is no Python or CPU fallback for the data path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ESP_LIB: a kernel-study build of the same library (tools only).
LIB_PATH = os.environ.get("ESP_LIB") or os.path.join(_HERE, "libesp_b200.so")

ESP_OK = 0
ESP_ERR_CONFIG = -1
ESP_ERR_INFEASIBLE = -2
ESP_ERR_INTERNAL = -3
ESP_ERR_CAPACITY = -4
ESP_ERR_MASTER_FULL = -5
ESP_ERR_UNKNOWN_STRATEGY = -6
ESP_ERR_CUDA = -7
ESP_ERR_NO_DEVICE = -8


class EspError(RuntimeError):
    """Base of the error taxonomy (reference types.hpp:48-109)."""

    code = None

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class ConfigError(EspError):
    pass


class InfeasiblePlanError(EspError):
    pass


class InternalError(EspError):
    pass


class CapacityError(EspError):
    pass


class MasterFullError(EspError):
    pass


class UnknownStrategyError(EspError):
    pass


class CudaError(EspError):
    pass


class NoDeviceError(EspError):
    pass


_ERRORS = {
    ESP_ERR_CONFIG: ConfigError,
    ESP_ERR_INFEASIBLE: InfeasiblePlanError,
    ESP_ERR_INTERNAL: InternalError,
    ESP_ERR_CAPACITY: CapacityError,
    ESP_ERR_MASTER_FULL: MasterFullError,
    ESP_ERR_UNKNOWN_STRATEGY: UnknownStrategyError,
    ESP_ERR_CUDA: CudaError,
    ESP_ERR_NO_DEVICE: NoDeviceError,
}

# Every symbol include/esp_abi.h declares (checked by tests/test_abi_exports.py).
EXPORTED_SYMBOLS = [
    "esp_last_error", "esp_abi_version", "esp_kv_bytes_per_token",
    "esp_plan_prefill_scale_down", "esp_sib_prefill_time", "esp_sib_decode_time",
    "esp_plan_decode_step", "esp_assign_masters", "esp_decode_step_comm",
    "esp_build_ring_schedule", "esp_proactive_scale_down", "esp_reactive_migrate",
    "esp_runtime_create", "esp_runtime_create_tp", "esp_runtime_destroy", "esp_instance_info", "esp_prefill",
    "esp_decode_step", "esp_move_kv", "esp_free_request", "esp_query_placement",
    "esp_check_conservation", "esp_request_tokens", "esp_last_prefill_stats", "esp_read_kv", "esp_capture_attention",
    "esp_captured_attention", "esp_slab_access", "esp_dump_profiles",
    "esp_decode_samples", "esp_fit_cost",
    "esp_launch_count", "esp_set_profiling", "esp_phase_times", "esp_k_gemm", "esp_k_ring_attention", "esp_k_ring_attention_timed",
    "esp_k_decode_attention",
]


class ModelConfig(C.Structure):
    _fields_ = [
        ("layers", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32),
        ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
        ("rms_eps", C.c_float), ("rope_theta", C.c_float), ("weight_seed", C.c_uint64),
    ]


class SibRecord(C.Structure):
    _fields_ = [
        ("dop", C.c_int32), ("tp", C.c_int32),
        ("alpha_p", C.c_double), ("beta_p", C.c_double), ("gamma_p", C.c_double),
        ("alpha_d", C.c_double), ("beta_d", C.c_double), ("gamma_d", C.c_double),
        ("compute_bound_batch_threshold", C.c_int32), ("tipping_ms", C.c_double),
    ]


class PrefillArgs(C.Structure):
    _fields_ = [
        ("n_requests", C.c_int32),
        ("request_ids", C.POINTER(C.c_int64)),
        ("input_lens", C.POINTER(C.c_int64)),
        ("tokens", C.POINTER(C.c_int32)),
        ("dop", C.c_int32),
        ("ring", C.POINTER(C.c_int32)),
        ("retain_n", C.POINTER(C.c_int32)),
        ("retain_instance", C.POINTER(C.c_int32)),
        ("retain_tokens", C.POINTER(C.c_int64)),
        ("first_token_out", C.POINTER(C.c_int32)),
        ("logits_out", C.POINTER(C.c_float)),
        ("device_ms_out", C.POINTER(C.c_double)),
    ]


class PrefillStats(C.Structure):
    _fields_ = [
        ("ring_volume_tokens", C.c_int64), ("cross_domain_tokens", C.c_int64),
        ("nvlink_bytes", C.c_int64), ("transient_buffer_tokens", C.c_int64),
        ("extra_migration_tokens", C.c_int64), ("device_ms", C.c_double),
        ("kv_ring_rows", C.c_int64),
    ]


class DecodeArgs(C.Structure):
    _fields_ = [
        ("n_members", C.c_int32),
        ("members", C.POINTER(C.c_int32)),
        ("n_masters", C.c_int32),
        ("masters", C.POINTER(C.c_int32)),
        ("batch_size", C.c_int32),
        ("batch", C.POINTER(C.c_int64)),
        ("in_tokens", C.POINTER(C.c_int32)),
        ("out_tokens", C.POINTER(C.c_int32)),
        ("logits_out", C.POINTER(C.c_float)),
        ("device_ms_out", C.POINTER(C.c_double)),
        ("chunk_request", C.c_int64),
        ("chunk_tokens", C.c_int64),
        ("chunk_n", C.c_int32),
        ("chunk_instance", C.POINTER(C.c_int32)),
        ("chunk_tokens_on", C.POINTER(C.c_int64)),
        ("chunk_token_ids", C.POINTER(C.c_int32)),
        ("chunk_final", C.c_int32),
        ("chunk_first_token_out", C.POINTER(C.c_int32)),
        ("chunk_logits_out", C.POINTER(C.c_float)),
    ]


_lib_handle = None


def lib() -> C.CDLL:
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the ESP data path has no fallback)")
        h = C.CDLL(LIB_PATH)
        h.esp_last_error.restype = C.c_char_p
        h.esp_kv_bytes_per_token.restype = C.c_int64
        h.esp_sib_prefill_time.restype = C.c_double
        h.esp_sib_decode_time.restype = C.c_double
        h.esp_launch_count.restype = C.c_int64
        h.esp_launch_count.argtypes = [C.c_void_p]
        h.esp_runtime_destroy.argtypes = [C.c_void_p]
        h.esp_runtime_create.argtypes = [C.POINTER(ModelConfig), C.c_int32,
                                         C.POINTER(C.c_int32), C.c_int64,
                                         C.POINTER(C.c_void_p)]
        h.esp_runtime_create_tp.argtypes = [C.POINTER(ModelConfig), C.c_int32, C.c_int32,
                                            C.POINTER(C.c_int32), C.c_int64,
                                            C.POINTER(C.c_void_p)]
        h.esp_prefill.argtypes = [C.c_void_p, C.POINTER(PrefillArgs)]
        h.esp_decode_step.argtypes = [C.c_void_p, C.POINTER(DecodeArgs)]
        h.esp_move_kv.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int64]
        h.esp_free_request.argtypes = [C.c_void_p, C.c_int64]
        h.esp_query_placement.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int64), C.c_int32,
                                          C.POINTER(C.c_int32)]
        h.esp_instance_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64)]
        h.esp_check_conservation.argtypes = [C.c_void_p]
        h.esp_request_tokens.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                         C.c_int32, C.POINTER(C.c_int32)]
        h.esp_dump_profiles.argtypes = [C.c_void_p, C.c_char_p]
        h.esp_last_prefill_stats.argtypes = [C.c_void_p, C.POINTER(PrefillStats)]
        h.esp_read_kv.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_int64, C.POINTER(C.c_int64)]
        h.esp_capture_attention.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64]
        h.esp_captured_attention.argtypes = [C.c_void_p, C.c_void_p, C.c_int64,
                                             C.POINTER(C.c_int64)]
        h.esp_slab_access.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
        h.esp_decode_samples.argtypes = [C.c_void_p, C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                         C.c_int64, C.POINTER(C.c_int64)]
        h.esp_fit_cost.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double)]
        h.esp_set_profiling.argtypes = [C.c_void_p, C.c_int32]
        h.esp_phase_times.argtypes = [C.c_void_p, C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), C.c_int32]
        h.esp_k_gemm.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_int32, C.c_void_p]
        h.esp_k_ring_attention.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                           C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                           C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        h.esp_k_ring_attention_timed.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                                 C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                 C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                                 C.POINTER(C.c_float), C.c_void_p]
        h.esp_k_decode_attention.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_void_p), C.POINTER(C.c_int32),
                                             C.POINTER(C.c_int32), C.c_int32, C.c_void_p,
                                             C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
        _lib_handle = h
    return _lib_handle


def check(rc: int) -> None:
    if rc != ESP_OK:
        msg = lib().esp_last_error().decode()
        raise _ERRORS.get(rc, EspError)(rc, msg)


def _arr(dtype, values):
    a = np.ascontiguousarray(np.asarray(values, dtype=dtype))
    return a


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---- pure host planning (reference mechanics, bit-exact) ----------------------

def kv_bytes_per_token(layers: int, hidden_dim: int, kv_heads: int, bytes_per_element: int) -> int:
    v = lib().esp_kv_bytes_per_token(layers, hidden_dim, kv_heads, bytes_per_element)
    if v < 0:
        raise ConfigError(ESP_ERR_CONFIG, lib().esp_last_error().decode())
    return int(v)


def plan_prefill_scale_down(instances: Sequence[int], free: Sequence[int],
                            input_lens: Sequence[int]):
    """scheduler.cpp:663-713 -> (decode_instances, [fill order per request], ring_volume)."""
    d, n = len(instances), len(input_lens)
    inst = _arr(np.int32, instances)
    fr = _arr(np.int64, free)
    lens = _arr(np.int64, input_lens)
    dec = np.zeros(max(d, 1), np.int32)
    ndec = C.c_int32()
    pi = np.zeros(max(n * d, 1), np.int32)
    pt = np.zeros(max(n * d, 1), np.int64)
    pn = np.zeros(max(n, 1), np.int32)
    rv = C.c_int64()
    check(lib().esp_plan_prefill_scale_down(
        _ptr(inst, C.c_int32), _ptr(fr, C.c_int64), d, _ptr(lens, C.c_int64), n,
        _ptr(dec, C.c_int32), C.byref(ndec), _ptr(pi, C.c_int32), _ptr(pt, C.c_int64),
        _ptr(pn, C.c_int32), C.byref(rv)))
    fills = [[(int(pi[r * d + j]), int(pt[r * d + j])) for j in range(pn[r])] for r in range(n)]
    return [int(x) for x in dec[:ndec.value]], fills, int(rv.value)


def _sib_array(sib: Sequence[dict]):
    arr = (SibRecord * max(len(sib), 1))()
    for i, r in enumerate(sib):
        arr[i] = SibRecord(r["dop"], r.get("tp", 1), r["alpha_p"], r["beta_p"], r["gamma_p"],
                           r["alpha_d"], r["beta_d"], r["gamma_d"],
                           r.get("compute_bound_batch_threshold", 64), r.get("tipping_ms", 0.0))
    return arr, len(sib)


def sib_prefill_time(sib, dop, tp, sum_len, sum_len_sq) -> float:
    arr, n = _sib_array(sib)
    lib().esp_sib_prefill_time.argtypes = [C.POINTER(SibRecord), C.c_int32, C.c_int32,
                                           C.c_int32, C.c_double, C.c_double]
    v = lib().esp_sib_prefill_time(arr, n, dop, tp, sum_len, sum_len_sq)
    if v < 0:
        raise UnknownStrategyError(ESP_ERR_UNKNOWN_STRATEGY, lib().esp_last_error().decode())
    return v


def sib_decode_time(sib, dop, tp, batch, resident, masters) -> float:
    arr, n = _sib_array(sib)
    lib().esp_sib_decode_time.argtypes = [C.POINTER(SibRecord), C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32, C.c_int64, C.c_int32]
    v = lib().esp_sib_decode_time(arr, n, dop, tp, batch, resident, masters)
    if v < 0:
        raise EspError(-1, lib().esp_last_error().decode())
    return v


def plan_decode_step(members, batch_size, free: Dict[int, int], idle, sib, tp=1,
                     enable_scale_up=True):
    """scheduler.cpp:726-804 -> (feasible, masters, add_instances, idle_after)."""
    mem = _arr(np.int32, members)
    fi = _arr(np.int32, list(free.keys()))
    ft = _arr(np.int64, list(free.values()))
    idle_a = np.zeros(max(len(idle), 1), np.int32)
    idle_a[:len(idle)] = idle
    nidle = C.c_int32(len(idle))
    arr, n = _sib_array(sib)
    feas = C.c_int32()
    ms = np.zeros(max(len(members) + len(idle), 1), np.int32)
    nm = C.c_int32()
    add = np.zeros(max(len(idle), 1), np.int32)
    na = C.c_int32()
    lib().esp_plan_decode_step.argtypes = [
        C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.POINTER(C.c_int32),
        C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
        C.POINTER(SibRecord), C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
        C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
        C.POINTER(C.c_int32)]
    check(lib().esp_plan_decode_step(
        _ptr(mem, C.c_int32), len(members), batch_size, _ptr(fi, C.c_int32),
        _ptr(ft, C.c_int64), len(free), _ptr(idle_a, C.c_int32), C.byref(nidle), arr, n, tp,
        1 if enable_scale_up else 0, C.byref(feas), _ptr(ms, C.c_int32), C.byref(nm),
        _ptr(add, C.c_int32), C.byref(na)))
    return (bool(feas.value), [int(x) for x in ms[:nm.value]],
            [int(x) for x in add[:na.value]], [int(x) for x in idle_a[:nidle.value]])


def assign_masters(batch, masters) -> List[int]:
    b = _arr(np.int64, batch)
    m = _arr(np.int32, masters)
    out = np.zeros(max(len(batch), 1), np.int32)
    lib().esp_assign_masters.argtypes = [C.POINTER(C.c_int64), C.c_int32,
                                         C.POINTER(C.c_int32), C.c_int32,
                                         C.POINTER(C.c_int32)]
    check(lib().esp_assign_masters(_ptr(b, C.c_int64), len(batch), _ptr(m, C.c_int32),
                                   len(masters), _ptr(out, C.c_int32)))
    return [int(x) for x in out[:len(batch)]]


def decode_step_comm(d, masters, counts, master_free):
    """esp_mechanics.cpp:240-264 -> (query_volume, overlappable, full_master or None)."""
    m = _arr(np.int32, masters)
    c = _arr(np.int32, counts)
    f = _arr(np.int64, master_free)
    q, o, full = C.c_int64(), C.c_int64(), C.c_int32()
    lib().esp_decode_step_comm.argtypes = [C.c_int32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                           C.c_int32, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    rc = lib().esp_decode_step_comm(d, _ptr(m, C.c_int32), _ptr(c, C.c_int32),
                                    _ptr(f, C.c_int64), len(masters), C.byref(q), C.byref(o),
                                    C.byref(full))
    if rc == ESP_ERR_MASTER_FULL:
        return None, None, int(full.value)
    check(rc)
    return int(q.value), int(o.value), None


def build_ring_schedule(group, segments):
    d = len(group)
    g = _arr(np.int32, group)
    s = _arr(np.int64, segments)
    n = max((d - 1) * d, 1)
    fr, to, vol = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int64)
    tot = C.c_int64()
    lib().esp_build_ring_schedule.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                              C.c_int32, C.POINTER(C.c_int32),
                                              C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                              C.POINTER(C.c_int64)]
    check(lib().esp_build_ring_schedule(_ptr(g, C.c_int32), _ptr(s, C.c_int64), d,
                                        _ptr(fr, C.c_int32), _ptr(to, C.c_int32),
                                        _ptr(vol, C.c_int64), C.byref(tot)))
    rounds = [[(int(fr[r * d + i]), int(to[r * d + i]), int(vol[r * d + i])) for i in range(d)]
              for r in range(d - 1)]
    return rounds, int(tot.value)


def proactive_scale_down(ring, segments, sources, targets, target_placement, free):
    """esp_mechanics.cpp:78-136 -> (extra_migration_volume, transient_buffer_tokens)."""
    r = _arr(np.int32, ring)
    s = _arr(np.int64, segments)
    src = _arr(np.int32, sources)
    tg = _arr(np.int32, targets)
    ti = _arr(np.int32, [p[0] for p in target_placement] or [0])
    tt = _arr(np.int64, [p[1] for p in target_placement] or [0])
    fi = _arr(np.int32, list(free.keys()))
    ft = _arr(np.int64, list(free.values()))
    ex, buf = C.c_int64(), C.c_int64()
    lib().esp_proactive_scale_down.argtypes = [
        C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32),
        C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
        C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
        C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    check(lib().esp_proactive_scale_down(
        _ptr(r, C.c_int32), _ptr(s, C.c_int64), len(ring), _ptr(src, C.c_int32), len(sources),
        _ptr(tg, C.c_int32), len(targets), _ptr(ti, C.c_int32), _ptr(tt, C.c_int64),
        len(target_placement), _ptr(fi, C.c_int32), _ptr(ft, C.c_int64), len(free),
        C.byref(ex), C.byref(buf)))
    return int(ex.value), int(buf.value)


def reactive_migrate(sources, targets, total, free):
    src = _arr(np.int32, sources)
    tg = _arr(np.int32, targets or [0])
    fi = _arr(np.int32, list(free.keys()))
    ft = _arr(np.int64, list(free.values()))
    feas, blk = C.c_int32(), C.c_int32()
    head, vol = C.c_int64(), C.c_int64()
    fin_i = np.zeros(max(len(sources), 1), np.int32)
    fin_t = np.zeros(max(len(sources), 1), np.int64)
    nf = C.c_int32()
    lib().esp_reactive_migrate.argtypes = [
        C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int64,
        C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32),
        C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int32),
        C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
    check(lib().esp_reactive_migrate(
        _ptr(src, C.c_int32), len(sources), _ptr(tg, C.c_int32), len(targets), total,
        _ptr(fi, C.c_int32), _ptr(ft, C.c_int64), len(free), C.byref(feas), C.byref(blk),
        C.byref(head), _ptr(fin_i, C.c_int32), _ptr(fin_t, C.c_int64), C.byref(nf),
        C.byref(vol)))
    return dict(feasible=bool(feas.value), blocked_instance=int(blk.value),
                per_source_headroom=int(head.value),
                final_placement=[(int(fin_i[i]), int(fin_t[i])) for i in range(nf.value)],
                migration_volume=int(vol.value))


# ---- runtime ---------------------------------------------------------------------

@dataclass
class ModelShape:
    layers: int
    hidden: int
    heads: int
    head_dim: int
    ffn: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    weight_seed: int = 1234

    def c(self) -> ModelConfig:
        return ModelConfig(self.layers, self.hidden, self.heads, self.head_dim, self.ffn,
                           self.vocab, self.rms_eps, self.rope_theta, self.weight_seed)


TINY = ModelShape(layers=2, hidden=512, heads=8, head_dim=64, ffn=1536, vocab=32000)
LWM_7B = ModelShape(layers=32, hidden=4096, heads=32, head_dim=128, ffn=11008, vocab=32000)


class Runtime:
    """Elastic instances over one token-granular paged KV pool (esp_runtime)."""

    def __init__(self, shape: ModelShape, n_instances: int,
                 devices: Optional[Sequence[int]] = None, kv_capacity: int = 0,
                 tp_planes: Optional[Sequence[int]] = None):
        """tp_planes: tensor-parallel runtime (esp_runtime_create_tp) — every
        instance spans len(tp_planes) GPUs, plane r on GPU tp_planes[r];
        `devices` must then be None."""
        self.shape = shape
        self.n_instances = n_instances
        cfg = shape.c()
        h = C.c_void_p()
        if tp_planes is not None:
            if devices is not None:
                raise ValueError("tp_planes and devices are exclusive")
            self._devs = _arr(np.int32, tp_planes)
            check(lib().esp_runtime_create_tp(C.byref(cfg), n_instances, len(tp_planes),
                                              _ptr(self._devs, C.c_int32), kv_capacity,
                                              C.byref(h)))
            self._h = h
            return
        if devices is None:
            dev_ptr = None
        else:
            self._devs = _arr(np.int32, devices)
            dev_ptr = _ptr(self._devs, C.c_int32)
        check(lib().esp_runtime_create(C.byref(cfg), n_instances, dev_ptr, kv_capacity,
                                       C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().esp_runtime_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def instance_info(self, i: int) -> Tuple[int, int]:
        cap, used = C.c_int64(), C.c_int64()
        check(lib().esp_instance_info(self._h, i, C.byref(cap), C.byref(used)))
        return int(cap.value), int(used.value)

    def prefill(self, request_ids, input_lens, ring, retain, tokens=None,
                want_logits=False):
        """retain: per request, [(instance, tokens), ...] in token order."""
        n = len(request_ids)
        rid = _arr(np.int64, request_ids)
        lens = _arr(np.int64, input_lens)
        rg = _arr(np.int32, ring)
        rn = _arr(np.int32, [len(x) for x in retain])
        ri = _arr(np.int32, [p[0] for x in retain for p in x] or [0])
        rt = _arr(np.int64, [p[1] for x in retain for p in x] or [0])
        first = np.full(n, -1, np.int32)
        ms = C.c_double(0.0)
        args = PrefillArgs()
        args.n_requests = n
        args.request_ids = _ptr(rid, C.c_int64)
        args.input_lens = _ptr(lens, C.c_int64)
        if tokens is not None:
            tok = _arr(np.int32, tokens)
            args.tokens = _ptr(tok, C.c_int32)
        args.dop = len(ring)
        args.ring = _ptr(rg, C.c_int32)
        args.retain_n = _ptr(rn, C.c_int32)
        args.retain_instance = _ptr(ri, C.c_int32)
        args.retain_tokens = _ptr(rt, C.c_int64)
        args.first_token_out = _ptr(first, C.c_int32)
        logits = None
        if want_logits:
            logits = np.zeros((n, self.shape.vocab), np.float32)
            args.logits_out = _ptr(logits, C.c_float)
        args.device_ms_out = C.pointer(ms)
        check(lib().esp_prefill(self._h, C.byref(args)))
        return first, logits, ms.value

    def decode_step(self, members, masters, batch, in_tokens=None, want_logits=False,
                    chunk=None):
        """chunk: optional dict(request, placement=[(instance, tokens)...],
        tokens=<prompt ids of the chunk>, final=bool) — a chunked-prefill chunk
        riding on this step. Returns (out_tokens, logits, ms) and, with a
        chunk, sets chunk['first_token'] / chunk['logits'] when final."""
        b = len(batch)
        mem = _arr(np.int32, members)
        mas = _arr(np.int32, masters)
        bt = _arr(np.int64, batch)
        out = np.full(b, -1, np.int32)
        ms = C.c_double(0.0)
        args = DecodeArgs()
        args.n_members = len(members)
        args.members = _ptr(mem, C.c_int32)
        args.n_masters = len(masters)
        args.masters = _ptr(mas, C.c_int32)
        args.batch_size = b
        args.batch = _ptr(bt, C.c_int64)
        if in_tokens is not None:
            it = _arr(np.int32, in_tokens)
            args.in_tokens = _ptr(it, C.c_int32)
        args.out_tokens = _ptr(out, C.c_int32)
        logits = None
        if want_logits:
            logits = np.zeros((b, self.shape.vocab), np.float32)
            args.logits_out = _ptr(logits, C.c_float)
        args.device_ms_out = C.pointer(ms)
        args.chunk_request = -1
        if chunk is not None:
            ci = _arr(np.int32, [p[0] for p in chunk["placement"]])
            ct = _arr(np.int64, [p[1] for p in chunk["placement"]])
            args.chunk_request = chunk["request"]
            args.chunk_tokens = int(sum(p[1] for p in chunk["placement"]))
            args.chunk_n = len(chunk["placement"])
            args.chunk_instance = _ptr(ci, C.c_int32)
            args.chunk_tokens_on = _ptr(ct, C.c_int64)
            if chunk.get("tokens") is not None:
                cids = _arr(np.int32, chunk["tokens"])
                args.chunk_token_ids = _ptr(cids, C.c_int32)
            args.chunk_final = 1 if chunk.get("final") else 0
            cfirst = np.full(1, -1, np.int32)
            args.chunk_first_token_out = _ptr(cfirst, C.c_int32)
            clog = None
            if chunk.get("final") and want_logits:
                clog = np.zeros(self.shape.vocab, np.float32)
                args.chunk_logits_out = _ptr(clog, C.c_float)
        check(lib().esp_decode_step(self._h, C.byref(args)))
        if chunk is not None:
            chunk["first_token"] = int(cfirst[0])
            chunk["logits"] = clog
        return out, logits, ms.value

    def move_kv(self, request, src, dst, tokens):
        check(lib().esp_move_kv(self._h, request, src, dst, tokens))

    def free_request(self, request):
        check(lib().esp_free_request(self._h, request))

    def placement(self, request) -> Dict[int, int]:
        cap = max(self.n_instances, 1)
        ii = np.zeros(cap, np.int32)
        tt = np.zeros(cap, np.int64)
        n = C.c_int32()
        check(lib().esp_query_placement(self._h, request, _ptr(ii, C.c_int32),
                                        _ptr(tt, C.c_int64), cap, C.byref(n)))
        return {int(ii[i]): int(tt[i]) for i in range(n.value)}

    def kv_used(self) -> List[int]:
        return [self.instance_info(i)[1] for i in range(self.n_instances)]

    def check_conservation(self):
        check(lib().esp_check_conservation(self._h))

    def tokens(self, request) -> List[int]:
        n = C.c_int32()
        check(lib().esp_request_tokens(self._h, request, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int32)
        check(lib().esp_request_tokens(self._h, request, _ptr(out, C.c_int32), n.value,
                                       C.byref(n)))
        return [int(x) for x in out[:n.value]]

    def last_prefill_stats(self) -> Dict[str, float]:
        """Ring volume, cross-GPU share, NVLink bytes, transient buffer and extra
        migration of the last prefill (esp_last_prefill_stats)."""
        st = PrefillStats()
        check(lib().esp_last_prefill_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in PrefillStats._fields_}

    def read_kv(self, request, layer):
        """(K, V) of one layer as uint16 (bf16 bits) [n_tokens, hidden], token order."""
        n = C.c_int64()
        check(lib().esp_read_kv(self._h, request, layer, None, None, 0, C.byref(n)))
        k = np.zeros((n.value, self.shape.hidden), np.uint16)
        v = np.zeros((n.value, self.shape.hidden), np.uint16)
        check(lib().esp_read_kv(self._h, request, layer, k.ctypes.data, v.ctypes.data, n.value,
                                C.byref(n)))
        return k, v

    def capture_attention(self, positions):
        """Arms the next (single-request) prefill to capture the attention outputs
        at these prompt positions in every layer; read them with captured_attention()."""
        p = _arr(np.int64, positions)
        self._cap_n = len(p)
        check(lib().esp_capture_attention(self._h, _ptr(p, C.c_int64) if len(p) else None, len(p)))

    def captured_attention(self) -> np.ndarray:
        """uint16 (bf16 bits) [layers, n_positions, hidden] of the last armed prefill."""
        n = C.c_int64()
        check(lib().esp_captured_attention(self._h, None, 0, C.byref(n)))
        out = np.zeros((n.value, self.shape.hidden), np.uint16)
        check(lib().esp_captured_attention(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out.reshape(self.shape.layers, -1, self.shape.hidden)

    def slab_access(self, instance, device) -> bool:
        ok = C.c_int32()
        check(lib().esp_slab_access(self._h, instance, device, C.byref(ok)))
        return bool(ok.value)

    PHASES = ["embed", "rmsnorm", "qkv_gemm", "ring_attention", "o_gemm", "gate_up_gemm",
              "down_gemm", "lm_head", "argmax", "decode_attention", "lse_combine",
              "host_enqueue"]

    def set_profiling(self, on: bool):
        check(lib().esp_set_profiling(self._h, 1 if on else 0))

    def phase_times(self):
        """{phase: (ms, launches)} accumulated since the last call (then reset)."""
        n = len(self.PHASES)
        ms = np.zeros(n, np.float64)
        ln = np.zeros(n, np.int64)
        check(lib().esp_phase_times(self._h, _ptr(ms, C.c_double), _ptr(ln, C.c_int64), n))
        return {p: (float(ms[i]), int(ln[i])) for i, p in enumerate(self.PHASES)}

    def dump_profiles(self, path: str):
        check(lib().esp_dump_profiles(self._h, path.encode()))

    def decode_samples(self) -> Dict[str, np.ndarray]:
        """Measured decode steps: dop, batch, masters, resident, ms arrays."""
        n = C.c_int64(0)
        check(lib().esp_decode_samples(self._h, None, None, None, None, None, 0, C.byref(n)))
        m = n.value
        out = {"dop": np.zeros(m, np.int32), "batch": np.zeros(m, np.int32),
               "masters": np.zeros(m, np.int32), "resident": np.zeros(m, np.int64),
               "ms": np.zeros(m, np.float64)}
        if m:
            check(lib().esp_decode_samples(
                self._h, _ptr(out["dop"], C.c_int32), _ptr(out["batch"], C.c_int32),
                _ptr(out["masters"], C.c_int32), _ptr(out["resident"], C.c_int64),
                _ptr(out["ms"], C.c_double), m, C.byref(n)))
        return out


def fit_cost(x1, x2, y) -> np.ndarray:
    """[c0, c1, c2] of y ~ c0 + c1*x1 + c2*x2 (esp_fit_cost; the reference's
    fit_prefill_coefficients rule, cost_model.cpp:86-135)."""
    a = np.ascontiguousarray(x1, np.float64)
    b = np.ascontiguousarray(x2, np.float64)
    c = np.ascontiguousarray(y, np.float64)
    if not (len(a) == len(b) == len(c)):
        raise ValueError("fit_cost: arrays differ in length")
    coef = np.zeros(3, np.float64)
    check(lib().esp_fit_cost(_ptr(a, C.c_double), _ptr(b, C.c_double), _ptr(c, C.c_double),
                             len(a), _ptr(coef, C.c_double)))
    return coef


def launch_count() -> int:
    return int(lib().esp_launch_count(None))


# ---- kernel-level hooks (device pointers, e.g. torch tensors' data_ptr()) -----------

GEMM_PATHS = {"auto": 0, "no_pair": 1, "tiles": 2, "streamk": 3}


def k_gemm(a_ptr, b_ptr, d_ptr, M, N, K, epilogue=0, stream=0, path="auto"):
    check(lib().esp_k_gemm(a_ptr, b_ptr, d_ptr, M, N, K, epilogue | (GEMM_PATHS[path] << 8),
                           stream))


def k_ring_attention(q_ptr, q_len, pos_i, kv_k, kv_v, kv_len, origin, out_ptr, heads,
                     head_dim, stream=0):
    d = len(kv_k)
    kk = (C.c_void_p * d)(*kv_k)
    vv = (C.c_void_p * d)(*kv_v)
    kl = (C.c_int32 * d)(*kv_len)
    og = (C.c_int32 * d)(*origin)
    check(lib().esp_k_ring_attention(q_ptr, q_len, pos_i, d, kk, vv, kl, og, out_ptr, heads,
                                     head_dim, stream))


def k_ring_attention_timed(q_ptr, q_len, pos_i, kv_k, kv_v, kv_len, origin, out_ptr, heads,
                           head_dim, repeats, stream=0) -> float:
    """K1 launched `repeats` times back to back on staged buffers; returns the
    average ms per launch (CUDA events, staging excluded)."""
    d = len(kv_k)
    kk = (C.c_void_p * d)(*kv_k)
    vv = (C.c_void_p * d)(*kv_v)
    kl = (C.c_int32 * d)(*kv_len)
    og = (C.c_int32 * d)(*origin)
    ms = C.c_float()
    check(lib().esp_k_ring_attention_timed(q_ptr, q_len, pos_i, d, kk, vv, kl, og, out_ptr, heads,
                                           head_dim, repeats, C.byref(ms), stream))
    return float(ms.value)


def k_decode_attention(q_ptr, batch, k_slabs, v_slabs, slot_ptrs, n_slots, chunk_req,
                       out_ptr, heads, head_dim, stream=0, out_f32=False):
    n = len(k_slabs)
    ks = (C.c_void_p * n)(*k_slabs)
    vs = (C.c_void_p * n)(*v_slabs)
    sp = (C.c_void_p * n)(*slot_ptrs)
    ns = (C.c_int32 * n)(*n_slots)
    cr = (C.c_int32 * n)(*chunk_req)
    check(lib().esp_k_decode_attention(q_ptr, batch, ks, vs, sp, ns, cr, n, out_ptr, heads,
                                       head_dim, 1 if out_f32 else 0, stream))


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float32."""
    return (np.asarray(u16, np.uint16).astype(np.uint32) << 16).view(np.float32)
