#!/usr/bin/env bash
# Round-2 session-4 measurement: the bench line, ncu launch list and full
# captures of K1 and the pair GEMM (32K prefill), the K1 yardstick.
# Logs in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {  # name timeout cmd...
  local name=$1 to=$2; shift 2
  echo "=== $name ($(date +%T))"
  timeout "$to" "$@" > "gpurun_out/$name.log" 2>&1
  echo "rc=$? $name"; tail -2 "gpurun_out/$name.log" | cut -c1-300
}
Q="--skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down"
run yardstick 600 python tools/attn_yardstick.py
run bench 1500 python bench.py
run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02s4_launches_prefill32k.csv python bench.py --steps 1 --warmup 1 $Q
run ncu_attn 900 ncu --set full --clock-control none --import-source on \
  -k regex:ring_attention -s 2 -c 1 -o gpurun_out/r02s4_prof_attn -f python bench.py --steps 1 --warmup 0 $Q
run ncu_gemm 900 ncu --set full --clock-control none --import-source on \
  -k regex:gemm_bf16_tcgen05_pair -s 10 -c 1 -o gpurun_out/r02s4_prof_gemm -f python bench.py --steps 1 --warmup 0 $Q
