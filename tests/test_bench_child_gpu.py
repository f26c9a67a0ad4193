"""bench.py's multi-GPU leg (the child process rank 0 starts for
`--gpus N`: ESP degree N across the runtime's GPUs) end to end on ONE GPU,
with one transport domain per instance (ESP_DOMAIN_PER_INSTANCE=1) so the
cross-GPU code paths run: push-transport prefill with arrival counters, the
windowed ring, the reactive baseline's KV moves between domains, N-way
multi-master decode. Guards the path the driver's scaling run takes on a
multi-GPU node."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_esp_child_four_domains_one_gpu():
    env = dict(os.environ, ESP_DOMAIN_PER_INSTANCE="1")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--esp-child", "--gpus", "4",
                        "--devices", "0,0,0,0", "--seq", "4096", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stderr[-2000:]
    j = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    pre = j["prefill"]
    assert pre["tokens_per_s"] > 0 and pre["gpu_launches"] > 0
    assert pre["retention"] == [[0, 4096]] or pre["retention"] == [(0, 4096)]
    ring = j["ring"]
    assert ring["ring_volume_tokens"] == 3 * 4096  # (d - 1) * sum, esp_mechanics.cpp:59-68
    assert ring["extra_migration_tokens"] == 0
    assert "error" not in j.get("prefill_window", {}), j.get("prefill_window")
    assert j["prefill_window"]["kv_ring_rows_per_gpu"] <= 3 * (4096 // 4)
    tpo = j["tensor_parallel"]
    assert "error" not in tpo, tpo
    assert set(tpo) >= {"tp1", "tp2", "tp4"} and all(tpo[f"tp{t}"]["prefill_ms"] > 0 for t in (1, 2, 4))
    for key in ("scale_down", "decode"):
        assert key in j and "error" not in (j[key] or {}), (key, j.get(key))
