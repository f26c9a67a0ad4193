"""Live drop-in on the B200: the UNMODIFIED reference engine and ESP
scheduler, prebuilt in this container from /root/reference into oracle/_ref/
(tests/cpp/tap_gpu.cpp, linked with libesp_b200.so), run with EspTapPolicy
around the reference's own policy and a DEVICE runtime — every prefill,
decode step (with any chunked-prefill chunk) and KV move of configs 1 and 5, a
denser mixed trace, and the chunked-prefill and disaggregation baselines
 executes real sm_100a kernels — also over tensor-parallel
instances (tp = 2 planes); page tables are verified at
every schedule() call and the event log must equal the untapped run's.
Skipped only if the prebuilt binary is absent (build() was not run where
/root/reference exists)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "tap_gpu")
SIB = os.path.join(ROOT, "oracle", "_ref", "default_sib.jsonl")


@pytest.mark.gpu
@pytest.mark.skipif(not (os.path.exists(EXE) and os.path.exists(SIB)),
                    reason="oracle/_ref/tap_gpu not built")
def test_reference_engine_drives_device_runtime():
    out = subprocess.run([EXE, SIB], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stderr + out.stdout
    assert out.stdout.count("events identical") == 10, out.stdout
