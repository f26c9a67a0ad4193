#!/usr/bin/env bash
# In-step A/B of K1's exponent split (eighths of the softmax exponentials on
# the FMA pipe, ESP_ATTN_POLY) with the kernel-study build (ESP_LIB): the
# 32K LWM-7B prefill step, alternating variants so both see the same
# power-capped clock drift. One JSON line per run in gpurun_out/poly_ab.log.
cd "$(dirname "$0")/.."
LIB=paper_2404_09526_b200/libesp_b200_study.so
Q="--steps 4 --warmup 3 --skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down"
for r in 1 2 3; do
  for p in ${POLYS:-1 2}; do
    echo "poly=$p run=$r $(ESP_LIB=$LIB ESP_ATTN_POLY=$p timeout 600 python bench.py $Q | python -c 'import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({"value": j["value"], "k1_frac": j["roofline"]["frac"], "k1_tflops": j["roofline"]["achieved"], "mhz": j["clocks"]["sm_mhz"]}))')"
  done
done
