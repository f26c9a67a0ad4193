for r in 1 2 3; do for v in 0 1; do echo "FUSED=$v $(ESP_DECODE_FUSED_COMBINE=$v STEPS=10 timeout 300 python tools/decode_probe.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],3))')"; done; done
ESP_DECODE_FUSED_COMBINE=1 timeout 600 python -m pytest tests/test_e2e_gpu.py -q -x -k "config1 or multi" 2>&1 | tail -1
