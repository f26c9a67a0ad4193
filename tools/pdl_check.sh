timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do for v in "X=1" "ESP_DECODE_NORM_KERNEL=1"; do echo "$v $(env $v STEPS=10 timeout 300 python tools/decode_probe.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],3), d["phase_ms"])')"; done; done
