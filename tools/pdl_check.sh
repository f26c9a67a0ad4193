# decode-step A/B on one box (tools/decode_probe.py)
for r in 1 2; do
for v in "ESP_PDL=3" "ESP_PDL=3 ESP_GEMM_SK_MIN_KB=128" "ESP_PDL=11" "ESP_PDL=0"; do
  echo "$v $(env $v STEPS=10 timeout 300 python tools/decode_probe.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],3), d["phase_ms"]["o_gemm"])')"
done; done
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log
