#!/usr/bin/env bash
# K1 A/B between two environments on the kernel-study build, alternating:
# standalone (attn_yardstick ONLY_OURS) then in-step (32K prefill bench).
# usage: A="ESP_K1_PARTS2=1" B="" bash tools/ab_env.sh   (empty = defaults)
cd "$(dirname "$0")/.."
LIB=paper_2404_09526_b200/libesp_b200_study.so
Q="--steps 4 --warmup 3 --skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down"
env ESP_LIB=$LIB $B timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k ring 2>&1 | tail -1
for r in 1 2 3; do
  for v in A B; do
    e=${!v}
    echo "alone [$v: $e] run=$r $(env ESP_LIB=$LIB ONLY_OURS=1 $e timeout 300 python tools/attn_yardstick.py 2>/dev/null | tail -1)"
  done
done
for r in 1 2 3; do
  for v in A B; do
    e=${!v}
    echo "in-step [$v: $e] run=$r $(env ESP_LIB=$LIB $e timeout 600 python bench.py $Q 2>/dev/null | python -c 'import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({"value": round(j["value"]), "k1_tflops": round(j["roofline"]["achieved"],1), "mhz": j["clocks"]["sm_mhz"]}))')"
  done
done
