#!/usr/bin/env bash
# compute-sanitizer over the windowed-ring path (round 2, session 3): the
# carry variant of K1 (O/m/l resumed from HBM through TMEM, o_init barrier),
# the finalize kernel, the side-stream block copies and the decode K3 that
# normalises single-chunk rows in place. Logs in gpurun_out/san_win_*.log.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="domain_window and (config1_tiny_esp or multi_request or kv_move)"
for tool in memcheck synccheck racecheck; do
  echo "=== $tool window e2e ($(date +%T))"
  timeout 1800 $CS --tool $tool --print-limit 30 --error-exitcode 99 \
    python -m pytest tests/test_e2e_gpu.py -q -x -p no:cacheprovider -k "$SEL" \
    > gpurun_out/san_win_${tool}.log 2>&1
  echo "rc=$? $tool"; grep -E "passed|failed|SUMMARY" gpurun_out/san_win_${tool}.log | tail -3
done
