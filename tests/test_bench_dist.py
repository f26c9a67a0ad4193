"""bench.py's N>1 harness on CPU with gloo, world size 2: step times are
reduced with MAX over ranks, whole-job value = world x tokens / max time, and
under torchrun only rank 0 prints the reference arm's JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import bench
    r, w, d = bench.dist_init()
    assert (r, w) == (rank, world) and d is not None
    local_ms = 100.0 + 50.0 * rank  # rank 1 is the straggler
    ms = bench.reduce_max(local_ms, d)
    bench.barrier(d)
    out[rank] = ms
    dist.destroy_process_group()


def test_reduce_max_over_ranks():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        assert out[0] == out[1] == 150.0  # both ranks see the max


@pytest.mark.timeout(600)
def test_reference_arm_under_torchrun_prints_once():
    env = dict(os.environ, ESP_BENCH_CPU_TOKENS="32", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "0"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2
    assert j["cpu_baseline"]["kind"] == "port" and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0


def _ring_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), ESP_BENCH_GLOO="1")
    import argparse

    import bench
    r, w, d = bench.dist_init()
    res = bench.nccl_ring_baseline(argparse.Namespace(seq=64), r, w, d, device="cpu")
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_ring_baseline_round_order_gloo(world):
    """The send/recv ring baseline (bench.nccl_ring_baseline) on CPU/gloo:
    world-1 rounds of grouped send/recv deliver each rank the block of origin
    rank+1 (the ring's last round, esp_mechanics.cpp:59-68); the time is the
    max over ranks (same value on every rank)."""
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_ring_worker, args=(world, port, out), nprocs=world, join=True)
        assert len(out) == world
        assert len({round(out[r]["ms_per_layer"], 9) for r in range(world)}) == 1
        assert out[0]["bytes_sent_per_gpu_per_layer"] == (world - 1) * 2 * (64 // world) * 64 * 4
