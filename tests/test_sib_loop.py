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


def _reference_fit(tmp_path, samples):
    """Coefficients the reference's own Sib::load + fit_all give per dop."""
    prof = tmp_path / "p.jsonl"
    with open(prof, "w") as f:
        for d, lens, ms in samples:
            f.write(json.dumps({"dop": d, "tp": 1, "kind": "profile", "lengths": lens,
                                "measured_ms": ms}) + "\n")
    out = tmp_path / "f.jsonl"
    subprocess.run([DRIVER, "fit", str(prof), str(out)], check=True)
    recs = [json.loads(l) for l in out.read_text().splitlines() if '"coefficients"' in l]
    return {r["dop"]: (r["alpha_p"], r["beta_p"], r["gamma_p"]) for r in recs}


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/src"), reason="reference absent")
def test_fit_cost_matches_reference_fit(tmp_path):
    """esp_fit_cost (the runtime's fitter, used for the B200-measured SIB)
    gives the reference fit_prefill_coefficients' coefficients on the same
    samples: noisy, multi-request, and with a negative coefficient to drop
    (dop 3: a decreasing quadratic term) or two (dop 4)."""
    import numpy as np

    from paper_2404_09526_b200 import abi

    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "reference"], check=True,
                   stdout=subprocess.DEVNULL)
    rng = np.random.default_rng(3)
    truth = {1: (4.0, 0.02, 3e-8), 2: (6.0, 0.011, 1.4e-8), 3: (50.0, 0.05, -1e-7),
             4: (900.0, -0.01, -1e-8)}
    samples = []
    for d, (a, b, g) in truth.items():
        for _ in range(25):
            lens = [int(x) for x in rng.integers(16, 20000, rng.integers(1, 4))]
            s, sq = sum(lens), sum(l * l for l in lens)
            ms = max(a + b * s + g * sq, 0.5) * (1 + 0.03 * rng.standard_normal())
            samples.append((d, lens, float(ms)))
    ref = _reference_fit(tmp_path, samples)
    for d in truth:
        sel = [(l, m) for dd, l, m in samples if dd == d]
        x1 = np.array([sum(l) for l, _ in sel], np.float64)
        x2 = np.array([sum(v * v for v in l) for l, _ in sel], np.float64)
        y = np.array([m for _, m in sel], np.float64)
        ours = abi.fit_cost(x1, x2, y)
        for c_ours, c_ref in zip(ours, ref[d]):
            assert c_ours == pytest.approx(c_ref, rel=1e-7, abs=1e-15), (d, ours, ref[d])
    # dop 3 / 4 exercised the drop rule: some coefficient pinned at 0
    assert min(ref[3]) == 0.0 and min(ref[4]) == 0.0
    # Independent of both QR implementations (ours and the Eigen shim the
    # reference is built against): numpy's SVD least squares with the same
    # active-set rule (cost_model.cpp:104-134) gives the same coefficients.
    for d in truth:
        sel = [(l, m) for dd, l, m in samples if dd == d]
        x1 = np.array([sum(l) for l, _ in sel], np.float64)
        x2 = np.array([sum(v * v for v in l) for l, _ in sel], np.float64)
        y = np.array([m for _, m in sel], np.float64)
        for c_np, c_ref in zip(_numpy_fit(x1, x2, y), ref[d]):
            assert c_np == pytest.approx(c_ref, rel=1e-6, abs=1e-13), (d, c_np, ref[d])


def _numpy_fit(x1, x2, y):
    import numpy as np

    A = np.stack([np.ones_like(x1), x1, x2], axis=1)
    scale = np.linalg.norm(A, axis=0)
    scale[scale == 0] = 1.0
    A = A / scale
    active = [0, 1, 2]
    coef = np.zeros(3)
    while active:
        coef = np.zeros(3)
        coef[active] = np.linalg.lstsq(A[:, active], y, rcond=None)[0]
        worst = min(active, key=lambda c: coef[c])
        if coef[worst] >= -1e-12:
            break
        active.remove(worst)
    else:
        coef = np.zeros(3)
    return np.maximum(coef, 0.0) / scale


def test_fit_cost_underdetermined():
    """< 3 samples or a rank-deficient design: the reference's
    UnderdeterminedError (cost_model.cpp:87-89, :44-46) as ESP_ERR_CONFIG."""
    import numpy as np

    from paper_2404_09526_b200 import abi

    with pytest.raises(abi.ConfigError):
        abi.fit_cost([1.0, 2.0], [1.0, 4.0], [1.0, 2.0])
    with pytest.raises(abi.ConfigError):
        abi.fit_cost(np.full(6, 7.0), np.full(6, 49.0), np.arange(6.0))


def test_sib_records_round_trip(tmp_path):
    """calibrate() keeps every base row and its non-fitted fields; write_sib
    emits the reference's coefficient line format (loadable by Sib::load)."""
    import numpy as np

    from paper_2404_09526_b200 import sib

    base = sib.load_sib(os.path.join(ROOT, "oracle", "_ref", "default_sib.jsonl")) \
        if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "default_sib.jsonl")) else None
    if base is None:
        pytest.skip("default SIB not installed (make -C oracle)")
    pre = [{"dop": 2, "tp": 1, "lengths": [n], "measured_ms": 1.0 + 1e-3 * n + 1e-9 * n * n}
           for n in (512, 1024, 4096, 8192, 16384)]
    dec = {"dop": np.array([2, 2, 2, 2], np.int32), "batch": np.array([1, 4, 16, 16], np.int32),
           "masters": np.array([1, 1, 1, 2], np.int32),
           "resident": np.array([1000, 8000, 64000, 128000], np.int64),
           "ms": np.array([1.1, 1.5, 3.0, 5.4])}
    recs, report = sib.calibrate(base, pre, dec)
    assert [(r["dop"], r["tp"]) for r in recs] == [(r["dop"], r["tp"]) for r in base]
    r2 = [r for r in recs if r["dop"] == 2][0]
    assert r2["alpha_p"] == pytest.approx(1.0, rel=1e-6)
    assert r2["beta_p"] == pytest.approx(1e-3, rel=1e-6)
    assert r2["compute_bound_batch_threshold"] == base[1]["compute_bound_batch_threshold"]
    assert report[1]["prefill"] == "kept" and report[2]["decode"] != "kept"
    out = tmp_path / "sib.jsonl"
    sib.write_sib(recs, str(out))
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "reference"], check=True,
                   stdout=subprocess.DEVNULL)
    # the reference loads it and refits nothing (no profile lines): same rows out
    fitted = tmp_path / "refit.jsonl"
    subprocess.run([DRIVER, "fit", str(out), str(fitted)], check=True)
    again = [json.loads(l) for l in fitted.read_text().splitlines() if l.strip()]
    assert len(again) == len(recs)


def test_decode_design_matches_sib_decode_time():
    """The decode fit's regressors are Sib::decode_time's (cost_model.cpp:175-187):
    with the fitted coefficients, alpha + beta*x1 + gamma*x2 must equal the
    runtime's restated decode_time (esp_sib_decode_time) for batches on both
    sides of the compute-bound threshold and any masters / dop."""
    import numpy as np

    from paper_2404_09526_b200 import abi, sib

    smp = {"dop": np.array([1, 2, 4, 8, 4, 2], np.int32),
           "batch": np.array([1, 16, 64, 65, 128, 200], np.int32),
           "masters": np.array([1, 2, 1, 2, 4, 3], np.int32),
           "resident": np.array([4096, 70000, 300000, 900000, 1200000, 50000], np.int64),
           "ms": np.zeros(6)}
    x1, x2 = sib._decode_x(smp, 64)
    rec = {"dop": 0, "tp": 1, "alpha_p": 1.0, "beta_p": 0.0, "gamma_p": 0.0, "alpha_d": 3.5,
           "beta_d": 0.07, "gamma_d": 2e-5, "compute_bound_batch_threshold": 64,
           "tipping_ms": 0.0}
    for i in range(6):
        r = dict(rec, dop=int(smp["dop"][i]))
        want = abi.sib_decode_time([r], r["dop"], 1, int(smp["batch"][i]),
                                   int(smp["resident"][i]), int(smp["masters"][i]))
        got = 3.5 + 0.07 * x1[i] + 2e-5 * x2[i]
        assert got == pytest.approx(want, rel=1e-12), (i, got, want)
