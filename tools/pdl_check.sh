timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" 2>&1 | tail -2
SHAPES=gate_up,lm_head timeout 300 python tools/skinny_probe.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_e2e_gpu.py -q -x -k "config1 or multi or config4" 2>&1 | tail -1
for r in 1 2; do for v in "X=1" "ESP_GEMM_NO_PAIR_SPLIT=1"; do echo "$v $(env $v STEPS=10 timeout 300 python tools/decode_probe.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],3), d["phase_ms"]["gate_up_gemm"])')"; done; done
