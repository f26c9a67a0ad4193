timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do for v in "X=1" "ESP_PREFILL_NORM_KERNEL=1"; do
  env $v timeout 600 python bench.py --skip-cpu --skip-decode --skip-esp-sweep --skip-config3 --skip-scale-down --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['phase_share'].get('rmsnorm'))"
done; done
