# Decode attention variant sweep (tools/decode_probe.py, one process each).
export DPROBE_VARIANTS='"ESP_DECODE_V1=41 ESP_DECODE_CHUNK=256" "ESP_DECODE_V1=48" "ESP_DECODE_CHUNK=1024" "ESP_DECODE_V1=410" "ESP_DECODE_V1=38" "ESP_DECODE_V1=310" "ESP_DECODE_V1=28" "ESP_DECODE_V1=210" "ESP_DECODE_ATTN=2 ESP_DECODE_STAGES=2"'
bash tools/gpu_session.sh dprobe
grep -v "^==" gpurun_out/dprobe.log | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['env'], round(d['step_ms'],3), round(d['attn_gbs']), d['phase_ms'].get('decode_attention'))
"
