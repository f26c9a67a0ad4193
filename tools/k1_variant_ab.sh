#!/usr/bin/env bash
# K1 variant A/B with the kernel-study build: VAR=<env name> selects the
# variant (set = variant, unset = default). Ring tests under the variant,
# then standalone (attn_yardstick ONLY_OURS) and in-step (32K prefill)
# timings, alternating. usage: VAR=ESP_ATTN_SPLIT bash tools/k1_variant_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LIB=paper_2404_09526_b200/libesp_b200_study.so
: "${VAR:?set VAR}"
env ESP_LIB=$LIB $VAR=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k ring 2>&1 | tail -2
env ESP_LIB=$LIB $VAR=1 timeout 900 python -m pytest tests/test_parity_baseline_gpu.py -q -x -k "k1" 2>&1 | tail -2
for r in 1 2 3; do
  for v in 0 1; do
    if [ $v = 1 ]; then export $VAR=1; else unset $VAR; fi
    echo "alone $VAR=$v run=$r $(ESP_LIB=$LIB ONLY_OURS=1 timeout 300 python tools/attn_yardstick.py 2>/dev/null | tail -1)"
  done
done
Q="--steps 4 --warmup 3 --skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down"
for r in 1 2 3; do
  for v in 0 1; do
    if [ $v = 1 ]; then export $VAR=1; else unset $VAR; fi
    echo "in-step $VAR=$v run=$r $(ESP_LIB=$LIB timeout 600 python bench.py $Q 2>/dev/null | python -c 'import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({"value": j["value"], "k1_frac": j["roofline"]["frac"], "k1_tflops": j["roofline"]["achieved"], "mhz": j["clocks"]["sm_mhz"]}))')"
  done
done
unset $VAR
