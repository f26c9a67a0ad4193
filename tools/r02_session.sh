#!/usr/bin/env bash
# Round-2 measurement session on one B200: K1 yardstick, the bench line, ncu
# launch lists and full captures. Logs in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {  # name timeout cmd...
  local name=$1 to=$2; shift 2
  echo "=== $name ($(date +%T))"
  timeout "$to" "$@" > "gpurun_out/$name.log" 2>&1
  echo "rc=$? $name"; tail -2 "gpurun_out/$name.log"
}
Q="--skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down"
run yardstick 600 python tools/attn_yardstick.py
run bench 1500 python bench.py
run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_prefill32k.csv python bench.py --steps 1 --warmup 1 $Q
run ncu_attn 900 ncu --set full --clock-control none --import-source on \
  -k regex:ring_attention -s 2 -c 1 -o gpurun_out/r02_prof_attn -f python bench.py --steps 1 --warmup 0 $Q
run ncu_gemm 900 ncu --set full --clock-control none --import-source on \
  -k regex:gemm_bf16_tcgen05_pair -s 10 -c 1 -o gpurun_out/r02_prof_gemm -f python bench.py --steps 1 --warmup 0 $Q
run ncu_decode 1800 bash tools/prof_decode.sh
