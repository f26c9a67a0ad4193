# On a box with N > 1 GPUs (not available in round 1): the end-to-end and edge
# GPU tests with instance i on GPU i mod N, so transport domains are distinct
# GPUs and the fused ring / query broadcast / partial gather cross NVLink.
N=${N:-$(nvidia-smi -L | wc -l)}
ESP_TEST_DEVICES=$N timeout 3600 python -m pytest tests/test_e2e_gpu.py tests/test_edge_gpu.py -m gpu -q
