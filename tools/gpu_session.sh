#!/usr/bin/env bash
# One GPU session on the B200 box: tests, smoke, bench, kernel microbench and
# ncu evidence, every step under its own timeout, logs in gpurun_out/.
# usage: tools/gpu_session.sh [steps...]   (default: all)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
STEPS="${*:-tests smoke e2e bench kbench ncu}"
run() {  # name timeout cmd...
  local name=$1 to=$2; shift 2
  echo "=== $name ($(date +%T))" | tee -a gpurun_out/session.log
  timeout "$to" "$@" > "gpurun_out/$name.log" 2>&1
  echo "rc=$? $name" | tee -a gpurun_out/session.log
  tail -3 "gpurun_out/$name.log" | tee -a gpurun_out/session.log
}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv | tee gpurun_out/gpu.txt
for s in $STEPS; do
  case $s in
    tests) run t_kernels 400 python -m pytest tests/test_kernels_gpu.py -v --timeout 120 --timeout-method=thread ;;
    smoke) run smoke 300 python -c "import __graft_entry__ as g; g.smoke()" ;;
    e2e) run t_e2e 1200 python -m pytest tests/test_e2e_gpu.py -v --timeout 400 --timeout-method=thread ;;
    gputests) run t_gpu 1800 python -m pytest tests -m gpu -q --timeout 400 --timeout-method=thread ;;
    bench) run bench 900 python bench.py ;;
    benchq) run bench_quick 600 python bench.py --steps 2 --warmup 1 --skip-cpu ;;
    kbench) run kbench 300 python tools/kbench.py ;;
    aprof) run attn_prof 300 python tools/attn_prof.py ;;
    ncu)
      run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --skip-decode \
        --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down
      run ncu_attn 900 ncu --set full --clock-control none --import-source on \
        -k regex:ring_attention -s 2 -c 1 -o gpurun_out/prof_attn -f python bench.py --steps 1 \
        --warmup 0 --skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down
      run ncu_gemm 900 ncu --set full --clock-control none --import-source on \
        -k regex:gemm_bf16 -s 10 -c 1 -o gpurun_out/prof_gemm -f python bench.py --steps 1 \
        --warmup 0 --skip-decode --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down
      ;;
    ncu_decode)
      run ncu_decode 900 ncu --set full --clock-control none --import-source on \
        -k regex:decode_attention -s 40 -c 1 -o gpurun_out/prof_decode -f python bench.py \
        --steps 1 --warmup 1 --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down --seq 4096
      ;;
  esac
done
echo "=== done ($(date +%T))" | tee -a gpurun_out/session.log
