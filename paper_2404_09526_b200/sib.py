"""Measured-SIB loop: B200-measured prefill and decode times
become the coefficients of the reference's scaling information base (SIB,
cost_model.hpp:47-52, JSONL schema of cost_model.cpp:218-248), which the
reference's unchanged scheduler and engine then plan with.

  measure()   drives a device runtime through prefill / decode sweeps at every
              ESP degree; the runtime records each call's device time
              (esp_dump_profiles: ProfileSample lines; esp_decode_samples)
  calibrate() fits alpha_p/beta_p/gamma_p per degree exactly as the
              reference's Sib::fit_all does (fit_prefill_coefficients,
              cost_model.cpp:86-135, restated in C++ as esp_fit_cost), and
              alpha_d/beta_d/gamma_d with the same rule on the decode model
              alpha + beta*b(/k above the threshold) + gamma*resident/d
              (cost_model.cpp:175-187; the reference hand-sets these)
  write_sib() writes the records in the reference's line format.
"""
import json
import os
import tempfile
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi

SIB_KEYS = ("dop", "tp", "kind", "alpha_p", "beta_p", "gamma_p", "alpha_d", "beta_d",
            "gamma_d", "compute_bound_batch_threshold", "tipping_ms")


def load_sib(path: str) -> List[dict]:
    """Coefficient records of a SIB JSONL file (profile lines are skipped)."""
    with open(path) as f:
        recs = [json.loads(l) for l in f if l.strip()]
    return [r for r in recs if r.get("kind") == "coefficients"]


def write_sib(records: Sequence[dict], path: str) -> None:
    with open(path, "w") as f:
        for r in records:
            f.write(json.dumps({k: r[k] for k in SIB_KEYS}) + "\n")


def prefill_samples(profile_path: str) -> List[dict]:
    """ProfileSample lines written by esp_dump_profiles."""
    with open(profile_path) as f:
        return [json.loads(l) for l in f if l.strip() and '"profile"' in l]


def _decode_x(samples: Dict[str, np.ndarray], threshold: int):
    b = samples["batch"].astype(np.float64)
    k = samples["masters"].astype(np.float64)
    b_eff = np.where(samples["batch"] > threshold, b / k, b)  # cost_model.cpp:182-185
    return b_eff, samples["resident"].astype(np.float64) / samples["dop"].astype(np.float64)


def calibrate(base: Sequence[dict], prefill: Sequence[dict],
              decode: Optional[Dict[str, np.ndarray]]) -> Tuple[List[dict], dict]:
    """New SIB records (one per base record's (dop, tp)) and a fit report:
    per degree, sample counts, coefficients and the max relative error of the
    fitted model on its own samples. Degrees without >= 3 samples of a phase
    keep the base coefficients for that phase (reported as 'kept')."""
    out, report = [], {}
    for rec in base:
        r = dict(rec)
        d, tp = int(rec["dop"]), int(rec["tp"])
        rep = {}
        ps = [p for p in prefill if int(p["dop"]) == d and int(p.get("tp", 1)) == tp]
        if len(ps) >= 3:
            x1 = np.array([sum(p["lengths"]) for p in ps], np.float64)
            x2 = np.array([sum(l * l for l in p["lengths"]) for p in ps], np.float64)
            y = np.array([p["measured_ms"] for p in ps], np.float64)
            c = abi.fit_cost(x1, x2, y)
            r["alpha_p"], r["beta_p"], r["gamma_p"] = (float(v) for v in c)
            pred = c[0] + c[1] * x1 + c[2] * x2
            rep["prefill"] = {"samples": len(ps), "coef": [float(v) for v in c],
                              "max_rel_err": float(np.max(np.abs(pred - y) / y))}
        else:
            rep["prefill"] = "kept"
        if decode is not None and tp == 1:
            sel = decode["dop"] == d
            if int(sel.sum()) >= 3:
                sub = {k: v[sel] for k, v in decode.items()}
                x1, x2 = _decode_x(sub, int(rec["compute_bound_batch_threshold"]))
                y = sub["ms"]
                c = abi.fit_cost(x1, x2, y)
                r["alpha_d"], r["beta_d"], r["gamma_d"] = (float(v) for v in c)
                pred = c[0] + c[1] * x1 + c[2] * x2
                rep["decode"] = {"samples": int(sel.sum()), "coef": [float(v) for v in c],
                                 "max_rel_err": float(np.max(np.abs(pred - y) / y))}
            else:
                rep["decode"] = "kept"
        out.append(r)
        report[d] = rep
    return out, report


def _spread(ring: Sequence[int], n: int):
    """Resting placement of n tokens spread evenly over the ring, in order."""
    d = len(ring)
    per = [n // d + (1 if i < n % d else 0) for i in range(d)]
    return [(int(i), int(t)) for i, t in zip(ring, per) if t > 0]


def measure(rt: "abi.Runtime", prefill_lengths: Sequence[Sequence[int]],
            decode_cfgs: Sequence[tuple], degrees: Sequence[int], repeats: int = 2,
            seed: int = 7) -> Tuple[List[dict], Dict[str, np.ndarray]]:
    """Prefill and decode sweeps on instances 0..d-1 of `rt` for each degree d.
    prefill_lengths: request length lists (one prefill each); decode_cfgs:
    (batch, context, masters) — the batch is prefilled on the ring, then
    `repeats` + 1 decode steps are taken (the first one warms up and is
    dropped). Returns (prefill profile lines, decode samples)."""
    rng = np.random.default_rng(seed)
    vocab = rt.shape.vocab
    rid = 1 << 40
    with tempfile.TemporaryDirectory() as td:
        p0 = os.path.join(td, "before.jsonl")
        rt.dump_profiles(p0)
        n_pre0 = len(prefill_samples(p0))
        n_dec0 = rt.decode_samples()["ms"].size
        pre_keep, dec_keep = [], []  # per call, in call order
        for d in degrees:
            ring = list(range(d))
            for lens in prefill_lengths:
                for rep in range(repeats + 1):
                    ids = list(range(rid, rid + len(lens)))
                    rid += len(lens)
                    toks = rng.integers(0, vocab, sum(lens), dtype=np.int32)
                    rt.prefill(ids, lens, ring, [_spread(ring, n) for n in lens], tokens=toks)
                    pre_keep.append(rep > 0)  # the first repetition warms up
                    for r in ids:
                        rt.free_request(r)
            for (b, ctx, k) in decode_cfgs:
                if k > d:
                    continue
                ids = list(range(rid, rid + b))
                rid += b
                toks = rng.integers(0, vocab, b * ctx, dtype=np.int32)
                rt.prefill(ids, [ctx] * b, ring, [_spread(ring, ctx) for _ in ids], tokens=toks)
                pre_keep.append(False)  # set-up of the decode batch
                for step in range(repeats + 1):
                    rt.decode_step(ring, ring[:k], ids)
                    dec_keep.append(step > 0)
                for r in ids:
                    rt.free_request(r)
        p1 = os.path.join(td, "after.jsonl")
        rt.dump_profiles(p1)
        lines = prefill_samples(p1)[n_pre0:]
    assert len(lines) == len(pre_keep), "prefill sample count mismatch"
    pre = [p for p, k in zip(lines, pre_keep) if k]
    dec = rt.decode_samples()
    idx = n_dec0 + np.flatnonzero(np.array(dec_keep, bool))
    return pre, {k: v[idx] for k, v in dec.items()}
