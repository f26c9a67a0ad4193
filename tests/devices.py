"""Instance -> GPU map of the GPU tests. Default: every instance on GPU 0
(the transport-domain paths are then exercised through
ESP_DOMAIN_PER_INSTANCE on one GPU). ESP_TEST_DEVICES=k places instance i on
GPU i mod k, so on a multi-GPU box the same tests drive the ring transport,
query broadcast and partial gather across real NVLink peers."""
import os


def devices(n: int):
    k = max(1, int(os.environ.get("ESP_TEST_DEVICES", "1")))
    return [i % k for i in range(n)]
