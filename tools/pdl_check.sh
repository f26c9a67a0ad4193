# PDL class sweep on the decode step (tools/decode_probe.py)
for r in 1 2; do
for v in 0 1 2 4 8 3 15; do echo "== ESP_PDL=$v"; ESP_PDL=$v STEPS=10 timeout 300 python tools/decode_probe.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['step_ms'],3))"; done
done
