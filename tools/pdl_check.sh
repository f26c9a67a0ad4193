timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k gemm 2>&1 | tail -2
timeout 300 python tools/skinny_probe.py 2>&1 | tail -5
for r in 1 2; do for v in "ESP_GEMM_SPLIT=4" "ESP_GEMM_SPLIT=0"; do echo "$v $(env $v STEPS=10 timeout 300 python tools/decode_probe.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],3), d["phase_ms"]["o_gemm"], d["phase_ms"]["down_gemm"])')"; done; done
