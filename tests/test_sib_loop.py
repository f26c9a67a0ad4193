"""Measured-SIB loop: the runtime's ProfileSample records
(esp_dump_profiles, schema of cost_model.cpp:243-248) are accepted by the
reference's own Sib::load and fitted by its fit_all (cost_model.cpp:86-135,
202-215), so B200-measured times re-enter the unchanged scheduler. CPU test;
needs the reference-built driver (skipped on the GPU box)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "golden_driver")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/src"), reason="reference absent")
def test_profiles_fit_through_reference(tmp_path):
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "reference"], check=True,
                   stdout=subprocess.DEVNULL)
    # Same line format esp_dump_profiles writes (runtime.cpp dump_profiles).
    alpha, beta, gamma = 3.0, 0.011, 2.5e-8
    lines = []
    for d in (1, 2):
        for lens in ([1024], [4096], [8192, 100], [32768], [2000, 3000, 4000]):
            s = sum(lens)
            sq = sum(x * x for x in lens)
            ms = (alpha + beta * s + gamma * sq) / d
            lines.append('{"dop": %d, "tp": 1, "kind": "profile", "lengths": [%s], '
                         '"measured_ms": %r}' % (d, ", ".join(map(str, lens)), ms))
    prof = tmp_path / "profiles.jsonl"
    prof.write_text("\n".join(lines) + "\n")
    out = tmp_path / "fitted.jsonl"
    subprocess.run([DRIVER, "fit", str(prof), str(out)], check=True)
    recs = [json.loads(l) for l in out.read_text().splitlines() if '"coefficients"' in l]
    assert {r["dop"] for r in recs} == {1, 2}
    for r in recs:
        d = r["dop"]
        assert r["alpha_p"] == pytest.approx(alpha / d, rel=1e-6)
        assert r["beta_p"] == pytest.approx(beta / d, rel=1e-6)
        assert r["gamma_p"] == pytest.approx(gamma / d, rel=1e-6)
