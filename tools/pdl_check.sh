timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_e2e_gpu.py -q -x -k "decode or config1 or multi" 2>&1 | tail -1
for r in 1 2; do for v in "ESP_DECODE_V1=48" "ESP_DECODE_V1=210"; do echo "$v $(env $v STEPS=10 timeout 300 python tools/decode_probe.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],3), round(d["attn_gbs"]))')"; done; done
