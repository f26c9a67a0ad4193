# K1 change check: ring tests, alone timing, in-step prefill
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "ring" 2>&1 | tail -1
for r in 1 2 3; do timeout 300 python tools/attn_prof.py 2>&1 | grep -E "attn-time"; done
for r in 1 2; do timeout 600 python bench.py --skip-cpu --skip-decode --skip-esp-sweep --skip-config3 --skip-scale-down --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"; done
