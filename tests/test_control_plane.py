"""Control-plane timing harness (SURVEY §8 d "CPU path timing (i)",
tools/cpp/control_plane_bench.cpp): the reference engine + ESP scheduler
alone and with EspTapPolicy over a placement-only runtime on the same mixed
trace; the tapped run must reproduce the event log. CPU test (needs the
reference sources to build the harness)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/src"), reason="reference absent")
def test_control_plane_bench_runs():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "reference"], check=True,
                   stdout=subprocess.DEVNULL)
    exe = os.path.join(ROOT, "oracle", "_ref", "control_plane_bench")
    sib = os.path.join(ROOT, "oracle", "_ref", "default_sib.jsonl")
    out = subprocess.run([exe, sib, "300"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["events_identical"] is True
    assert r["iterations"] > 0 and r["page_table_checks"] > 0
    assert r["untapped_us_per_iteration"] > 0 and r["tapped_us_per_iteration"] > 0
