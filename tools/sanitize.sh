#!/usr/bin/env bash
# compute-sanitizer over the kernel tests and the cross-domain end-to-end
# paths (memcheck / racecheck / synccheck on the mbarrier/TMEM
# pipelines and the cross-stream peer stores). Logs in gpurun_out/san_*.log;
# summaries go to profiles/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
K="tests/test_kernels_gpu.py"
for tool in memcheck racecheck synccheck; do
  echo "=== $tool kernels ($(date +%T))"
  timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest $K -q -x -k "not 4096-4096-4096 and not 5000" > gpurun_out/san_${tool}_kernels.log 2>&1
  echo "rc=$? $tool kernels"; tail -3 gpurun_out/san_${tool}_kernels.log
done
for tool in memcheck synccheck; do
  echo "=== $tool e2e ($(date +%T))"
  timeout 1500 $CS --tool $tool --print-limit 50 \
    --error-exitcode 99 python -m pytest tests/test_e2e_gpu.py -q -x \
    -k "config1_tiny_esp and (domain_arrival or colocated) or kv_move and domain_push" > gpurun_out/san_${tool}_e2e.log 2>&1
  echo "rc=$? $tool e2e"; tail -3 gpurun_out/san_${tool}_e2e.log
done
