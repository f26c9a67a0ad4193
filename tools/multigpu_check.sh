# On a box with N > 1 GPUs: the end-to-end, edge and BASELINE-size parity GPU
# tests with instance i on GPU i mod N (ESP_TEST_DEVICES, tests/devices.py),
# so transport domains are distinct GPUs: the fused ring (peer stores + device
# arrival counters), retention into remote survivors' VMM slabs, the query
# broadcast / partial gather and KV moves cross NVLink. Then the ESP-across-
# GPUs bench line (bench.py --gpus N under torchrun: NCCL ring baseline,
# NVLink P2P peak, ESP degree N prefill / decode / scale-down).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-$(nvidia-smi -L | wc -l)}
ESP_TEST_DEVICES=$N timeout 3600 python -m pytest tests/test_e2e_gpu.py tests/test_edge_gpu.py \
  tests/test_parity_baseline_gpu.py -m gpu -q > gpurun_out/multigpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/multigpu_tests.log
timeout 3600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus "$N" > gpurun_out/multigpu_bench.log 2>&1
echo "bench rc=$?"; tail -c 3000 gpurun_out/multigpu_bench.log
