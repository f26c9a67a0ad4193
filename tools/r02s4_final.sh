#!/usr/bin/env bash
# Round-2 session-4 closing run on one B200: the GPU suite, smoke, the full
# bench line, a measured SIB with the current kernels, decode ncu evidence.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {  # name timeout cmd...
  local name=$1 to=$2; shift 2
  echo "=== $name ($(date +%T))"
  timeout "$to" "$@" > "gpurun_out/$name.log" 2>&1
  echo "rc=$? $name"; tail -2 "gpurun_out/$name.log" | cut -c1-300
}
run t_gpu 2400 python -m pytest tests -m gpu -q --timeout 900
run smoke 300 python -c "import __graft_entry__ as g; g.smoke()"
run bench 1500 python bench.py
run sib 900 python tools/calibrate_sib.py --out gpurun_out/r02s4_sib_b200_7b.jsonl --report gpurun_out/r02s4_sib_b200_7b_report.json
run ncu_decode 1800 bash tools/prof_decode.sh
