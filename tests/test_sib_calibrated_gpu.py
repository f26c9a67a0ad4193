"""Measured-SIB loop on the B200, end to end: the device
runtime measures prefill and decode sweeps at ESP degrees 1-8 (tiny Llama,
8 instances co-located on one GPU), the times are fitted into SIB
coefficients (prefill by the reference's own rule, fit_prefill_coefficients
cost_model.cpp:86-135 — pinned to the reference in test_sib_loop.py; decode
by the same rule on cost_model.cpp:175-187's model), and the UNMODIFIED
reference engine + ESP scheduler then plan with that B200-calibrated SIB while
EspTapPolicy executes every decision on the device: event logs must equal the
untapped run's under the new SIB (acceptance check 9's determinism, SURVEY
§8c "measured clock" parity mode)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "tap_gpu")
SIB = os.path.join(ROOT, "oracle", "_ref", "default_sib.jsonl")


@pytest.mark.gpu
@pytest.mark.skipif(not (os.path.exists(EXE) and os.path.exists(SIB)),
                    reason="oracle/_ref/tap_gpu not built")
def test_calibrated_sib_drives_reference_scheduler(tmp_path):
    from paper_2404_09526_b200 import abi, sib

    rt = abi.Runtime(abi.TINY, 8, devices=[0] * 8, kv_capacity=40000)
    pre, dec = sib.measure(
        rt,
        prefill_lengths=[[256], [1024], [2048], [512, 1536], [4096], [3000, 3000]],
        decode_cfgs=[(1, 512, 1), (4, 1024, 1), (8, 2048, 2), (16, 1024, 2), (16, 256, 1)],
        degrees=range(1, 9), repeats=2)
    rt.close()
    assert len(pre) == 8 * 6 * 2
    assert dec["ms"].size > 0 and np.all(dec["ms"] > 0)
    base = sib.load_sib(SIB)
    recs, report = sib.calibrate(base, pre, dec)
    print(json.dumps(report, indent=1))
    for r in recs:
        d = r["dop"]
        assert report[d]["prefill"] != "kept" and report[d]["decode"] != "kept"
        for k in ("alpha_p", "beta_p", "gamma_p", "alpha_d", "beta_d", "gamma_d"):
            assert np.isfinite(r[k]) and r[k] >= 0.0
        assert r["alpha_p"] + r["beta_p"] > 0 and r["alpha_d"] + r["beta_d"] + r["gamma_d"] > 0
        # the fitted model describes its own samples (device times of ms scale)
        assert report[d]["prefill"]["max_rel_err"] < 1.0
        assert report[d]["decode"]["max_rel_err"] < 1.0
    path = str(tmp_path / "sib_b200.jsonl")
    sib.write_sib(recs, path)
    out = subprocess.run([EXE, path], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stderr + out.stdout
    assert out.stdout.count("events identical") == 10, out.stdout


SIB_7B = os.path.join(ROOT, "profiles", "r01s2_sib_b200_7b.jsonl")


@pytest.mark.gpu
@pytest.mark.skipif(not (os.path.exists(EXE) and os.path.exists(SIB_7B)),
                    reason="oracle/_ref/tap_gpu or the calibrated SIB absent")
def test_lwm7b_calibrated_sib_tap():
    """The committed LWM-7B SIB measured on a B200 by tools/calibrate_sib.py
    (profiles/r01s2_sib_b200_7b.jsonl; the engine accounts KV and time in
    LWM-7B units): the reference engine + scheduler plan with it and every
    decision executes on the device with identical event logs."""
    out = subprocess.run([EXE, SIB_7B], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stderr + out.stdout
    assert out.stdout.count("events identical") == 10, out.stdout
