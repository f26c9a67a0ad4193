#!/usr/bin/env bash
# K1 variant study (kernel-study build, ESP_LIB): correctness of the split
# softmax (ESP_ATTN_HALVES=2) on the ring-attention kernel tests, standalone
# K1 time per (halves, poly), and the in-step A/B. Logs in gpurun_out/.
cd "$(dirname "$0")/.."
LIB=paper_2404_09526_b200/libesp_b200_study.so
for hv in 2; do
  ESP_LIB=$LIB ESP_ATTN_HALVES=$hv ESP_ATTN_POLY=2 timeout 600 python -m pytest tests/test_kernels_gpu.py \
    -q -k ring_attention > gpurun_out/k1v_tests_h$hv.log 2>&1
  echo "tests halves=$hv rc=$? $(tail -1 gpurun_out/k1v_tests_h$hv.log)"
done
for r in 1 2; do
  for cfg in "1 2" "2 2" "2 1" "1 1"; do
    set -- $cfg
    echo "standalone halves=$1 poly=$2 run=$r $(ESP_LIB=$LIB ESP_ATTN_HALVES=$1 ESP_ATTN_POLY=$2 ONLY_OURS=1 timeout 300 python tools/attn_yardstick.py | tail -1)"
  done
done
Q="--steps 4 --warmup 3 --skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down"
for r in 1 2; do
  for hv in 1 2; do
    echo "in-step halves=$hv poly=2 run=$r $(ESP_LIB=$LIB ESP_ATTN_HALVES=$hv ESP_ATTN_POLY=2 timeout 600 python bench.py $Q | python -c 'import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({"value": j["value"], "k1_frac": j["roofline"]["frac"], "k1_tflops": j["roofline"]["achieved"], "mhz": j["clocks"]["sm_mhz"]}))')"
  done
done
