"""Live drop-in test: the UNMODIFIED reference engine (compiled in place from
/root/reference by oracle/Makefile) runs with EspTapPolicy
(paper_2404_09526_b200/integration/esp_tap_policy.hpp) around its own
policy, driving the B200 runtime's C-ABI; page tables are verified against
Request.placement at every schedule() call and the event log must equal the
untapped run's. Skipped where the reference is absent (the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference"
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def _build(tmp_path):
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "reference"], check=True,
                   stdout=subprocess.DEVNULL)
    exe = tmp_path / "tap_live"
    lib_dir = os.path.join(ROOT, "paper_2404_09526_b200")
    subprocess.run(
        ["g++", "-std=c++20", "-O1", f"-I{REF}/proj/include", f"-I{JSON_INC}",
         f"-I{ROOT}/include", f"-I{lib_dir}/integration", f"-I{ROOT}/oracle/shim",
         os.path.join(ROOT, "tests", "cpp", "tap_live.cpp"),
         os.path.join(ROOT, "oracle", "_ref", "libespsim_ref.a"),
         f"-L{lib_dir}", "-lesp_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)],
        check=True)
    return exe


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "proj", "src")), reason="reference absent")
def test_tap_policy_live(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe), REF], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    assert out.stdout.count("events identical") == 6, out.stdout
    # ESP prefills are passed in the restated fill order (scheduler.cpp:694-709)
    for line in out.stdout.splitlines():
        if line.startswith("esp:"):
            assert " 0 prefills in fill order" not in line, line
    # The tap's mirror of its own page-table effects spares the device query
    # for all but the requests the engine moved itself: the disaggregation
    # handoff (engine.cpp:194-244) shows up as queries, the other policies
    # need (almost) none.
    for line in out.stdout.splitlines():
        checks = int(line.split(" page-table checks")[0].split()[-1])
        queries = int(line.split(" reconcile queries")[0].split()[-1])
        assert queries <= max(1, checks // 100), line
        if line.startswith("disagg"):
            assert queries > 0, line


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "proj", "src")), reason="reference absent")
def test_tap_policy_live_b200_sib(tmp_path):
    """Same five scenarios with the scheduler planning on the LWM-7B SIB
    measured on a B200 (profiles/r01s2_sib_b200_7b.jsonl, tools/calibrate_sib.py):
    decisions change with the measured costs, the tap still realises every one
    of them bit-exactly."""
    exe = _build(tmp_path)
    sib = os.path.join(ROOT, "profiles", "r01s2_sib_b200_7b.jsonl")
    out = subprocess.run([str(exe), REF, sib], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    assert out.stdout.count("events identical") == 6, out.stdout
    base = subprocess.run([str(exe), REF], capture_output=True, text=True, timeout=600)
    assert base.stdout != out.stdout  # the measured SIB changes the plans
