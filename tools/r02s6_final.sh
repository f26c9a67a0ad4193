#!/usr/bin/env bash
# Round-2 session-6 confirmation run (fresh container build) on one B200: the
# GPU suite, smoke and the full bench line (compute-sanitizer is closed on the pool).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {  # name timeout cmd...
  local name=$1 to=$2; shift 2
  echo "=== $name ($(date +%T))"
  timeout "$to" "$@" > "gpurun_out/$name.log" 2>&1
  echo "rc=$? $name"; tail -2 "gpurun_out/$name.log" | cut -c1-300
}
run t_gpu_s6 2400 python -m pytest tests -m gpu -q --timeout 900
run smoke_s6 300 python -c "import __graft_entry__ as g; g.smoke()"
run bench_s6 1500 python bench.py
